"""Development A/B check: dense EMDQ fields of the built library (or of a
tools/variants.py build, NRM_B200_VARIANT) on C1/C2/C4/C5 and seeded random
cases, saved to an npz for a bitwise comparison between two builds.
    NRM_B200_VARIANT=orig python tools/ab_emdq.py gpurun_out/a.npz
    python tools/ab_emdq.py gpurun_out/b.npz
    python tools/ab_emdq.py --cmp gpurun_out/a.npz gpurun_out/b.npz"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if a[k].tobytes() != b[k].tobytes()]
    print(f"{len(a.files)} arrays, {len(bad)} differ", bad[:10])
    sys.exit(1 if bad else 0)

from paper_2103_07414_b200 import mosaic as nrm  # noqa: E402
from paper_2103_07414_b200 import workload as W  # noqa: E402

ctx = nrm.Context(0)
out = {}
for name in ("c1", "c2", "c4", "c5"):
    wl = W.frame_workload(name)
    e = wl.emdq
    for S in (16, 8, 32):
        d, u = nrm.emdq_field((0.0, 0.0, wl.frame_w, wl.frame_h), e.apts, e.locals_, e.probs, e.active,
                              wl.params.alpha, wl.params.beta, S, ctx=ctx)
        out[f"{name}_S{S}_d"], out[f"{name}_S{S}_u"] = d, u
for seed in range(40):
    rng = np.random.default_rng(900 + seed)
    m = int(rng.integers(20, 3000))
    w, h = int(rng.integers(40, 700)), int(rng.integers(30, 500))
    span = 3e4 if seed % 2 else 300.0
    x0, y0 = float(rng.uniform(-span, span)), float(rng.uniform(-span, span))
    if seed % 3 == 0:
        c = np.stack([rng.uniform(x0, x0 + w, 7), rng.uniform(y0, y0 + h, 7)], 1)
        apts = c[rng.integers(0, 7, m)] + rng.normal(0, 4.0, (m, 2))
    else:
        apts = np.stack([rng.uniform(x0 - 60, x0 + w + 60, m), rng.uniform(y0 - 60, y0 + h + 60, m)], 1)
    ang = rng.uniform(-0.3, 0.3, m) * (0.05 if seed % 2 else 1.0)
    loc = np.zeros((m, 5))  # WarpFunction: scale, real (cos, sin), dual
    loc[:, 0] = rng.uniform(0.85, 1.2, m)
    loc[:, 1], loc[:, 2] = np.cos(ang / 2), np.sin(ang / 2)
    loc[:, 3:5] = rng.normal(0, 8.0, (m, 2))
    probs = rng.uniform(0, 1, m)
    active = np.sort(rng.choice(m, int(rng.integers(1, m + 1)), replace=False)).astype(np.int32)
    S = int((1, 4, 16, 32, 9)[seed % 5])
    d, u = nrm.emdq_field((x0, y0, w, h), apts, loc, probs, active, float(rng.uniform(1e-4, 5e-3)),
                          float(rng.uniform(1e-4, 5e-3)), S, ctx=ctx)
    out[f"r{seed}_d"], out[f"r{seed}_u"] = d, u
for seed in range(16):  # large candidate sets (binned supertile scans), some far outside the grid
    rng = np.random.default_rng(1900 + seed)
    m = int(rng.integers(3000, 30000))
    w, h = int(rng.integers(300, 2000)), int(rng.integers(200, 1200))
    x0, y0 = float(rng.uniform(-3e4, 3e4)), float(rng.uniform(-3e4, 3e4))
    apts = np.stack([rng.uniform(x0 - 80, x0 + w + 80, m), rng.uniform(y0 - 80, y0 + h + 80, m)], 1)
    if seed % 3 == 0:  # clusters
        c = np.stack([rng.uniform(x0, x0 + w, 9), rng.uniform(y0, y0 + h, 9)], 1)
        apts[: m // 2] = c[rng.integers(0, 9, m // 2)] + rng.normal(0, 6.0, (m // 2, 2))
    if seed % 4 == 1:  # a sprinkling far outside the grid (margin cells)
        k = m // 50
        apts[:k] += rng.choice([-1.0, 1.0], (k, 2)) * rng.uniform(500, 5000, (k, 2))
    ang = rng.uniform(-0.02, 0.02, m)
    loc = np.zeros((m, 5))
    loc[:, 0] = rng.uniform(0.9, 1.1, m)
    loc[:, 1], loc[:, 2] = np.cos(ang / 2), np.sin(ang / 2)
    loc[:, 3:5] = rng.normal(0, 8.0, (m, 2))
    probs = rng.uniform(0, 1, m)
    active = np.sort(rng.choice(m, int(rng.integers(2100, m + 1)), replace=False)).astype(np.int32)
    S = int((16, 8, 32, 4)[seed % 4])
    print("large case", seed, m, w, h, len(active), S, flush=True)
    d, u = nrm.emdq_field((x0, y0, w, h), apts, loc, probs, active, float(rng.uniform(1e-4, 2e-3)),
                          float(rng.uniform(1e-4, 2e-3)), S, ctx=ctx)
    out[f"L{seed}_d"], out[f"L{seed}_u"] = d, u
np.savez(sys.argv[1], **out)
print("saved", len(out), "arrays")
