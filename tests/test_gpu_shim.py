"""GPU: the reference's mosaic unit-test suite (test_mosaic.cpp) compiled in
C++ against the drop-in header include/nrmosaic_b200/mosaic.hpp."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def test_cpp_dropin_suite(nrm):
    exe = ROOT / "tests" / "cpp" / "test_shim"
    if not exe.exists():
        from paper_2103_07414_b200 import build
        build.build_cpp_tests()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
