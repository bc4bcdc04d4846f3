"""Replay of recorded node states (snapshot.hpp:17-124):
paper_2103_07414_b200/replay.py reads the reference's own write_snapshot /
TrajectoryWriter output (golden replay_scan.npz, recorded by
oracle/_ref/snapshot_dump on the reference pipeline).

CPU: the reader's anchors, warps and positions agree with the trajectory
file and with warp(anchor) (the reference caches current_position =
warp.apply(anchor), slam.hpp:28).
GPU: blending the recorded frames with the recorded node states and
footprints reproduces the reference pipeline's own per-frame BlendStats
(golden pipeline_scan.npz, the same run) exactly, and the canvas matches the
oracle's (weights exact, colour 1e-3, render +-1)."""
import numpy as np
import pytest


def _load(golden):
    from paper_2103_07414_b200 import replay as R
    g = golden("replay_scan")
    snaps = {int(t): R.read_snapshot(bytes(g[f"snapshot_{t}"])) for t in g["frames_t"]}
    traj = R.read_trajectory(bytes(g["trajectory"]))
    return g, snaps, traj


def test_snapshots_agree_with_the_trajectory(golden, oracle):
    g, snaps, traj = _load(golden)
    assert len(traj.positions) == 12 and traj.status[0] == "tracked"
    for t, s in snaps.items():
        n = len(s.anchors)
        assert n > 50 and s.warps.shape == (n, 5) and s.hex_spacing > 0
        assert np.array_equal(s.anchors, traj.anchors[:n])            # insertion order
        assert np.array_equal(s.positions, traj.positions[t])
        for i in range(n):
            y = oracle.warp_apply(s.warps[i], s.anchors[i, 0], s.anchors[i, 1])
            assert np.abs(y - s.positions[i]).max() <= 1e-9
        assert (s.variances >= 0).all() and len(s.tracks) > 0


@pytest.mark.gpu
def test_replayed_blends_reproduce_the_reference_pipeline(nrm, ctx, oracle, golden):
    g, snaps, _ = _load(golden)
    ref = golden("pipeline_scan")
    cv, ocv = nrm.Canvas(ctx), oracle.canvas()
    from paper_2103_07414_b200 import workload as W
    alpha = W.scaled_params(480, 270).alpha
    for t in sorted(snaps):
        s = snaps[t]
        frame, poly = g[f"frame_{t}"], g[f"footprint_{t}"]
        st = nrm.blend_frame(cv, frame, s.anchors, s.warps, alpha, poly).as_tuple()
        assert ref["blended"][t] == 1
        assert st == tuple(int(v) for v in ref["stats"][t]), (t, st, ref["stats"][t])
        assert st == oracle.blend_frame(ocv, frame, s.anchors, s.warps, alpha, poly)
    col, wt = cv.read()
    ocol, owt = ocv.arrays()
    assert np.array_equal(wt, owt)
    assert np.abs(col.astype(np.float64) - ocol).max() <= 1e-3
    img, org = nrm.render(cv, crop=True)
    oimg, oorg = oracle.render(ocv, crop=True)
    assert org == oorg and np.abs(img.astype(int) - oimg.astype(int)).max() <= 1
