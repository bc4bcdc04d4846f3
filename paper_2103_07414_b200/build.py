"""In-tree build of the CUDA library (sm_100a) and the test-only oracle.

    python -m paper_2103_07414_b200.build          # libnrm_b200.so (+ oracle)

The shared library is written next to this file so it travels with the repo
snapshot to the GPU box; nothing goes to site-packages or a JIT cache.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libnrm_b200.so"
OBJ = PKG / "_build"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
    f"-I{ROOT / 'include'}",
]
SOURCES = ["nrm_abi.cu", "k_nodefield.cu", "k_emdq.cu", "k_canvas.cu", "k_features.cu", "k_selftest.cu",
           "k_variance.cu", "png_io.cu"]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libnrm_b200.so")
    return cand


def _run(cmd: list[str], log: Path | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"command failed: {' '.join(cmd)}")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_lib(force: bool = False, extra_flags: tuple = (), lib: Path = LIB, objdir: Path = OBJ) -> Path:
    """extra_flags/lib/objdir: development variants (tools/variants.py)."""
    nvcc = _nvcc()
    objdir.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "nrm_b200.h"]
    objs = []
    jobs = []
    for src in SOURCES:
        s = CSRC / src
        o = objdir / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([nvcc, *NVCC_FLAGS, *extra_flags, "-c", str(s), "-o", str(o)])
    if jobs:
        with ThreadPoolExecutor(max_workers=min(4, len(jobs))) as ex:
            list(ex.map(lambda c: _run(c, objdir / (Path(c[-1]).stem + ".ptxas.log")), jobs))
    if force or jobs or _stale(lib, objs):
        _run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib),
              *map(str, objs), "-cudart", "static", "-Xcompiler", "-fPIC", "-lz"])
    return lib


def build_oracle() -> None:
    """Test infrastructure: the C restatement, and the reference itself when
    /root/reference is present (this container only)."""
    _run(["make", "-s", "-C", str(ROOT / "oracle"), "liboracle.so"])
    if Path("/root/reference/proj/include/nrmosaic/mosaic.hpp").exists():
        _run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"])


REF_INCLUDE = Path("/root/reference/proj/include")
REF_TESTS = Path("/root/reference/proj/tests")


def build_cpp_tests() -> None:
    """C++ drop-in tests, linked against libnrm_b200.so (rpath $ORIGIN):
      tests/cpp/test_shim       -- the reference's test_mosaic.cpp suite on the
                                   shim header, with the reference's own types
                                   where the reference tree exists;
      tests/cpp/pipeline_b200   -- tests/cpp/pipeline_dump.cpp (the reference's
                                   production call sequence) compiled with
                                   -Iinclude/override, i.e. unchanged sources
                                   whose "nrmosaic/mosaic.hpp" is the B200 one;
      tests/cpp/acceptance_b200 -- the reference's own tests/acceptance.cpp,
                                   compiled the same way (reference tree only).
    The binaries travel to the GPU box with the snapshot."""
    cpp = ROOT / "tests" / "cpp"
    rpath = "-Wl,-rpath,$ORIGIN/../../paper_2103_07414_b200"
    link = [f"-L{PKG}", "-lnrm_b200", rpath, "-lpthread"]
    have_ref = (REF_INCLUDE / "nrmosaic" / "mosaic.hpp").exists()
    shim = ROOT / "include" / "nrmosaic_b200" / "mosaic.hpp"
    override = ROOT / "include" / "override" / "nrmosaic" / "mosaic.hpp"
    src = cpp / "test_shim.cpp"
    out = cpp / "test_shim"
    if src.exists() and _stale(out, [src, LIB, shim]):
        types = ["-include", "algorithm", "-include", "memory", f"-I{ROOT / 'oracle' / 'stub'}",
                 f"-I{REF_INCLUDE}"] if have_ref else ["-DNRM_B200_STANDALONE_TYPES"]
        _run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", *types, str(src), "-o", str(out), *link])
    if not have_ref:
        return
    common = ["g++", "-std=c++20", "-O2", "-DNDEBUG", "-include", "algorithm", "-include", "memory",
              f"-I{ROOT / 'include' / 'override'}", f"-I{ROOT / 'include'}", f"-I{ROOT / 'oracle' / 'stub'}",
              f"-I{REF_INCLUDE}", f"-I{REF_TESTS}"]
    jobs = []
    for name, source in (("pipeline_b200", cpp / "pipeline_dump.cpp"),
                         ("acceptance_b200", REF_TESTS / "acceptance.cpp")):
        out = cpp / name
        deps = [source, LIB, shim, override, ROOT / "include" / "nrmosaic_b200" / "features.hpp",
                ROOT / "include" / "override" / "nrmosaic" / "features.hpp"]
        if _stale(out, deps):
            jobs.append([*common, str(source), "-o", str(out), *link])
    if jobs:
        with ThreadPoolExecutor(max_workers=2) as ex:
            list(ex.map(_run, jobs))


def main() -> None:
    force = "--force" in sys.argv
    build_lib(force)
    build_oracle()
    build_cpp_tests()
    print(LIB)


if __name__ == "__main__":
    main()
