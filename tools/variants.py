"""Development: build libnrm_b200.so variants with extra nvcc defines into
_variants/<name>/ (git-ignored; travels to the GPU box with the snapshot).

    python tools/variants.py name1=-DFOO=1,-DBAR name2=
Select one at run time with NRM_B200_VARIANT=<name>.
"""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2103_07414_b200 import build as B  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]


def one(spec):
    name, _, flags = spec.partition("=")
    d = ROOT / "_variants" / name
    B.build_lib(force=True, extra_flags=tuple(f for f in flags.split(",") if f), lib=d / "libnrm_b200.so", objdir=d)
    return name


if __name__ == "__main__":
    with ThreadPoolExecutor(max_workers=4) as ex:
        for n in ex.map(one, sys.argv[1:]):
            print("built", n)
