"""EM E-step (leave-one-out blend_local at every match, fieldest.hpp:195-209):
GPU (nrm_emdq_points, host API) vs the reference's own loop on the host cores.
    python tools/estep_bench.py [n_matches ...]"""
import json
import os
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2103_07414_b200 import mosaic as M
from paper_2103_07414_b200 import workload as W

sizes = [int(a) for a in sys.argv[1:]] or [2000, 10000, 50000]
ctx = M.Context(0)
try:
    from oracle.oracle import Reference
    R = Reference()
except Exception:  # noqa: BLE001
    R = None
workers = os.cpu_count() or 1
for n in sizes:
    frac = 0.5 if n >= 50000 else 0.2
    e = W.emdq_inputs(3840, 2160, n, frac, 7100 + n)
    sp = W.scaled_params(3840, 2160)
    ex = np.arange(n, dtype=np.int32)
    args = (e.apts, e.apts, e.locals_, e.probs, e.active, sp.alpha, 1.0, 16)
    M.emdq_points(*args, exclude=ex, want_unc=False, ctx=ctx)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        w, pred, _, st = M.emdq_points(*args, exclude=ex, want_unc=False, ctx=ctx)
        ts.append(time.perf_counter() - t0)
    gpu = min(ts)
    out = {"matches": n, "active": int(len(e.active)), "gpu_ms": gpu * 1e3, "gpu_matches_per_s": n / gpu}
    if R is not None:
        k = min(n, max(64, int(2e8 / max(len(e.active), 1) / 16)))  # bounded sample
        t0 = time.perf_counter()
        rw, rp, re = R.estep_loo(e.apts, e.bpts, e.locals_, e.probs, e.active, sp.alpha, 16, workers=workers,
                                 rows=(0, k))
        cpu = time.perf_counter() - t0
        out.update(cpu_sample=k, cpu_workers=workers, cpu_matches_per_s=k / cpu,
                   cpu_full_s_est=n / (k / cpu), speedup=(n / gpu) / (k / cpu),
                   bit_exact_sample=bool(np.array_equal(rw[:k], w[:k]) and np.array_equal(rp[:k], pred[:k])))
    print(json.dumps(out))
