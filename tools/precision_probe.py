"""Fast-tier error vs. the scale lever S * |o| (S: spread of the listed
warps' scales around the tile's reference scale, |o|: output coordinate
magnitude): node field (K2) and dense EMDQ (K3) against the oracle at
canvas-scale offsets.  python tools/precision_probe.py"""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from oracle.oracle import Oracle
from paper_2103_07414_b200 import mosaic as M
from paper_2103_07414_b200 import workload as W

O = Oracle()
ctx = M.Context(0)


def conj(warps, t):
    q = W.shifted_warps(warps, t[0], t[1])
    w_, z_, s_ = q[:, 1], q[:, 2], q[:, 0]
    q[:, 3] += (w_ * t[0] + z_ * t[1]) / (2 * s_)
    q[:, 4] += (-z_ * t[0] + w_ * t[1]) / (2 * s_)
    return q


def rw(rng, n, rot, sspread, trans):
    ang = rng.uniform(-rot, rot, n)
    q = np.zeros((n, 5))
    q[:, 0] = 1.0 + rng.uniform(-sspread, sspread, n)
    q[:, 1], q[:, 2] = np.cos(ang / 2), np.sin(ang / 2)
    q[:, 3:5] = rng.normal(0, trans, (n, 2))
    return q


rows = []
for kind in ("node", "emdq"):
    for off in (0.0, 8000.0, 16000.0, 32000.0):
        for sp in (0.001, 0.01, 0.03, 0.1, 0.3):
            errs = []
            for seed in range(3):
                rng = np.random.default_rng(seed)
                o = np.array([off, -off * 0.7])
                if kind == "node":
                    n = 80
                    anchors = o + rng.uniform(-300, 500, (n, 2))
                    warps = conj(rw(rng, n, 0.2, sp, 5.0), o)
                    grid = (o[0], o[1], 200, 160)
                    d, s = M.node_field(grid, anchors, warps, 5e-4, ctx=ctx)
                    od, os_ = O.node_field_grid(grid, anchors, warps, 5e-4)
                    m = os_.astype(bool)
                    errs.append(float(np.abs(d[m] - od[m]).max()) if m.any() else 0.0)
                else:
                    m_ = 300
                    apts = o + rng.uniform(-50, 250, (m_, 2))
                    loc = conj(rw(rng, m_, 0.2, sp, 5.0), o)
                    pr = rng.uniform(0.1, 1, m_)
                    act = np.arange(m_, dtype=np.int32)
                    grid = (o[0], o[1], 200, 160)
                    d, u = M.emdq_field(grid, apts, loc, pr, act, 1e-3, 1e-3, 16, ctx=ctx)
                    od, ou = O.emdq_field_grid(grid, apts, loc, pr, act, 1e-3, 1e-3, 16, fast=True)
                    errs.append(float(np.abs(d - od).max()))
            lever = sp * max(off, 1.0)
            rows.append({"kind": kind, "offset": off, "scale_spread": sp, "lever": lever, "max_err": max(errs),
                         "err_per_lever": max(errs) / lever})
            print(json.dumps(rows[-1]), flush=True)
