"""TEST INFRASTRUCTURE: generates tests/golden/*.npz from the REAL reference
(oracle/_ref/libnrm_ref.so, the /root/reference headers compiled in place).

    make -C oracle ref && python oracle/make_golden.py

Each fixture holds the inputs and the reference's outputs for one case. The
reference's own unit tests (proj/tests/test_mosaic.cpp, test_fieldest.cpp)
supply the case shapes; the larger cases use BASELINE config C1. Canvas
colour planes are stored as SHA-256 of their float64 bytes (the restatement
must reproduce them bit-for-bit) plus a seeded sample of values.
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[0] = str(ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_2103_07414_b200 import workload as W  # noqa: E402

OUT = ROOT / "tests" / "golden"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rigid_warp(scale, angle, tx, ty):
    return W.similarity_warp(scale, angle, (tx * scale, ty * scale))


def mild_deformation(n):
    """test_mosaic.cpp:190-193."""
    out = np.zeros((n, 5))
    for i in range(n):
        s = 1.0 + 0.0005 * (i % 5)
        ang = 0.01 * (i % 3)
        tx, ty = 0.5 * (i % 7), -0.3 * (i % 4)
        w, z = np.cos(0.5 * ang), np.sin(0.5 * ang)
        out[i] = [s, w, z, 0.5 * (tx * w + ty * z), 0.5 * (-tx * z + ty * w)]
    return out


def blend_case(R, name, frame, anchors, warps_seq, alpha, polys, sample=4096, seed=0):
    """Runs a sequence of blends (one per warps/poly) on one reference canvas."""
    cv = R.canvas()
    stats = []
    for warps, poly in zip(warps_seq, polys):
        stats.append(R.blend_frame(cv, frame, anchors, warps, alpha, poly, workers=4))
    col, wt = cv.arrays()
    img, org = R.render(cv, crop=True)
    full, _ = R.render(cv, crop=False)
    ox, oy, w, h = cv.info()
    rng = np.random.default_rng(seed)
    occ = np.argwhere(wt > 0)
    pick = occ[rng.choice(len(occ), size=min(sample, len(occ)), replace=False)] if len(occ) else np.zeros((0, 2), int)
    d = dict(
        frame=frame, anchors=anchors, warps=np.stack(warps_seq), polys=np.array(polys, dtype=object),
        npoly=np.array([len(p) for p in polys]), alpha=alpha, stats=np.array(stats, np.int64),
        canvas_info=np.array([ox, oy, w, h], np.int64), color_sha=sha(col), weight_sha=sha(wt),
        render_crop_sha=sha(img), render_crop_shape=np.array(img.shape), crop_origin=np.array(org),
        render_full_sha=sha(full), sample_yx=pick, sample_color=col[pick[:, 0], pick[:, 1]] if len(pick) else np.zeros((0, 3)),
        sample_weight=wt[pick[:, 0], pick[:, 1]] if len(pick) else np.zeros(0, np.uint8),
        sample_render=full[pick[:, 0], pick[:, 1]] if len(pick) else np.zeros((0, 4), np.uint8))
    if w * h <= 600_000:
        d["weight"] = wt
        d["render_crop"] = img
    # object arrays are not loadable without pickle: flatten polygons
    d["polys"] = np.concatenate(polys) if polys else np.zeros((0, 2))
    np.savez_compressed(OUT / f"blend_{name}.npz", **d)
    print(f"blend_{name}: stats={stats[-1]} canvas={ox, oy, w, h}")


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    R = Reference()
    alpha0 = 2e-4

    # ---- pixel_warp known answers (test_mosaic.cpp:39-82) + random --------
    pw = {}
    pw["single_anchors"] = np.array([[100.0, 100.0]])
    pw["single_warps"] = rigid_warp(1.5, 0.2, 3, 4)[None]
    pw["single_out"] = R.pixel_warp(100, 100, pw["single_anchors"], pw["single_warps"], alpha0)
    anchors = W.hex_lattice((0, 0, 320, 200), 60.0)
    warps = mild_deformation(len(anchors))
    rng = np.random.default_rng(11)
    pts = np.stack([rng.uniform(-600, 900, 4000), rng.uniform(-600, 800, 4000)], axis=1)
    pts[:64] = np.round(pts[:64])
    outs, valid = [], []
    for x, y in pts:
        r = R.pixel_warp(x, y, anchors, warps, alpha0)
        valid.append(r is not None)
        outs.append(r if r is not None else np.zeros(5))
    np.savez_compressed(OUT / "pixel_warp.npz", anchors=anchors, warps=warps, points=pts, out=np.array(outs),
                        valid=np.array(valid), alpha=alpha0, **pw)
    print("pixel_warp:", int(np.sum(valid)), "of", len(pts), "supported")

    # ---- node lattices (insert_nodes, slam.hpp:270-360) ---------------------
    rects = [((0, 0, 320, 200), 60.0), ((0, 0, 64, 48), 20.0), ((0, 0, 48, 32), 16.0), ((0, 0, 256, 64), 30.0),
             ((0, 0, 640, 480), 60.0 * 1.5555555555555556), ((0, 0, 1920, 1080), 240.0),
             ((0, 0, 3840, 2160), 480.0), ((-500, -300, 900, 700), 75.0)]
    lat = {}
    for k, (r, sp) in enumerate(rects):
        lat[f"rect{k}"] = np.array(r, float)
        lat[f"spacing{k}"] = sp
        lat[f"anchors{k}"] = R.rect_lattice(r, sp)
    np.savez_compressed(OUT / "lattice.npz", n=len(rects), **lat)

    # ---- invert_frame_boundary (mosaic.hpp:58-96) --------------------------
    poly = R.invert_frame_boundary(320, 200, anchors, warps, alpha0)
    np.savez_compressed(OUT / "invert_boundary.npz", anchors=anchors, warps=warps, poly=poly, alpha=alpha0,
                        fw=320, fh=200)

    # ---- blend_frame cases --------------------------------------------------
    ramp = W.ramp_frame(320, 200)
    ident = lambda a: np.tile(np.array([1.0, 1.0, 0.0, 0.0, 0.0]), (len(a), 1))  # noqa: E731
    rect = lambda w, h: np.array([[0, 0], [w - 1, 0], [w - 1, h - 1], [0, h - 1]], float)  # noqa: E731
    a = W.hex_lattice((0, 0, 320, 200), 60.0)
    blend_case(R, "first_frame", ramp, a, [ident(a)], alpha0, [rect(320, 200)])

    const = np.zeros((48, 64, 3), np.uint8)
    const[..., 0], const[..., 1], const[..., 2] = 100, 150, 200
    a = W.hex_lattice((0, 0, 64, 48), 20.0)
    blend_case(R, "repeated_constant", const, a, [ident(a)] * 40, alpha0, [rect(64, 48)] * 40)

    r2 = W.ramp_frame(256, 64)
    a = W.hex_lattice((0, 0, 256, 64), 30.0)
    shifted = np.tile(np.array([1.0, 1.0, 0.0, 50.0, 0.0]), (len(a), 1))  # from_translation({100, 0})
    blend_case(R, "translated", r2, a, [ident(a), shifted], alpha0, [rect(256, 64), rect(256, 64) - [100, 0]])

    a = W.hex_lattice((0, 0, 320, 200), 60.0)
    wd = mild_deformation(len(a))
    blend_case(R, "deformed", ramp, a, [wd], alpha0, [R.invert_frame_boundary(320, 200, a, wd, alpha0)])

    r3 = W.ramp_frame(48, 32)
    a = W.hex_lattice((0, 0, 48, 32), 16.0)
    blend_case(R, "weight_cap", r3, a, [ident(a)] * 50, alpha0, [rect(48, 32)] * 50)

    gray = W.textured_frame(160, 120, seed=5, channels=1)
    a = W.hex_lattice((0, 0, 160, 120), 40.0)
    blend_case(R, "gray_rotated", gray, a, [np.tile(rigid_warp(1.02, 0.05, 3.5, -2.25), (len(a), 1))], alpha0,
               [R.invert_frame_boundary(160, 120, a, np.tile(rigid_warp(1.02, 0.05, 3.5, -2.25), (len(a), 1)), alpha0)])

    # C1 (BASELINE configs[0]): 640x480, 500 matches (20 % outliers), reference EM
    sp = W.scaled_params(640, 480)
    pa, pb = R.synth_matches(640, 480, sp.s, 400, 100, 7000)
    na = W.hex_lattice((0, 0, 640, 480), sp.hex_spacing)
    cnt, loc, pr, inl, inc, unc = R.estimate_locals(pa, pb, na, sp.alpha, sp.beta, sp.inlier_threshold)
    node_warps = np.stack([R.warp_update(np.array([1.0, 1, 0, 0, 0]), inc[i]) for i in range(len(na))])
    frame_c1 = W.textured_frame(640, 480, seed=7)
    poly_c1 = R.invert_frame_boundary(640, 480, na, node_warps, sp.alpha)
    blend_case(R, "c1", frame_c1, na, [node_warps], sp.alpha, [poly_c1])
    # second frame of a sequence: new warps composed on top (exercises canvas growth + averaging)
    node_warps2 = np.stack([R.warp_update(node_warps[i], inc[i]) for i in range(len(na))])
    poly_c1b = R.invert_frame_boundary(640, 480, na, node_warps2, sp.alpha)
    blend_case(R, "c1_seq", frame_c1, na, [node_warps, node_warps2], sp.alpha, [poly_c1, poly_c1b])

    # ---- EMDQ field (fieldest.hpp:75-97, 44-52) ------------------------------
    act = np.nonzero(inl)[0].astype(np.int32)
    grid = (0.0, 0.0, 640, 480)
    disp, unc_g = R.emdq_field_grid(grid, pa, loc, pr, act, sp.alpha, sp.beta, 16, workers=8)
    rng = np.random.default_rng(3)
    qpts = np.stack([rng.uniform(-50, 700, 512), rng.uniform(-50, 530, 512)], axis=1)
    qout = np.array([R.blend_local(loc, pa, pr, act, x, y, sp.alpha, 16) for x, y in qpts])
    qunc = np.array([R.node_uncertainty(x, y, pa[act], sp.beta) for x, y in qpts])
    np.savez_compressed(OUT / "emdq_c1.npz", apts=pa, bpts=pb, locals=loc, probs=pr, active=act, alpha=sp.alpha,
                        beta=sp.beta, grid=np.array(grid), disp_sub=disp[::4, ::4], unc_sub=unc_g[::4, ::4],
                        disp_sha=sha(disp), unc_sha=sha(unc_g), qpts=qpts, qout=qout, qunc=qunc,
                        node_anchors=na, node_inc=inc, node_unc=unc, inlier_count=cnt)
    print("emdq_c1: inliers", cnt, "disp range", float(np.abs(disp).max()))

    # small-support and tiny-candidate edge cases
    small_act = act[:10]
    disp_s, unc_s = R.emdq_field_grid((100.0, 50.0, 96, 64), pa, loc, pr, small_act, sp.alpha, sp.beta, 16, workers=8)
    disp_4, unc_4 = R.emdq_field_grid((100.0, 50.0, 96, 64), pa, loc, pr, act, sp.alpha, sp.beta, 4, workers=8)
    np.savez_compressed(OUT / "emdq_edge.npz", apts=pa, locals=loc, probs=pr, active=act, small_active=small_act,
                        alpha=sp.alpha, beta=sp.beta, grid=np.array([100.0, 50.0, 96, 64]), disp_small=disp_s,
                        unc_small=unc_s, disp_s4=disp_4, unc_s4=unc_4)
    print("done")


def estep_cases():
    """EM E-step leave-one-out (fieldest.hpp:195-209) through the reference's
    own blend_local / apply: C1 (the reference's EM outputs from emdq_c1), a
    tiny active set (the `others.empty()` branch) and a C2-sized match set."""
    R = Reference()
    g = dict(np.load(OUT / "emdq_c1.npz"))
    out = {}
    for name, act in (("c1", g["active"]), ("tiny", g["active"][:1]), ("few", g["active"][:3])):
        w, pred, emp = R.estep_loo(g["apts"], g["bpts"], g["locals"], g["probs"], act, float(g["alpha"]), 16)
        out.update({f"{name}_active": act, f"{name}_warps": w, f"{name}_pred": pred, f"{name}_empty": emp})
    e = W.emdq_inputs(1920, 1080, 2000, 0.2, 7002)
    sp = W.scaled_params(1920, 1080)
    w, pred, emp = R.estep_loo(e.apts, e.bpts, e.locals_, e.probs, e.active, sp.alpha, 16)
    out.update(c2_apts=e.apts, c2_bpts=e.bpts, c2_locals=e.locals_, c2_probs=e.probs, c2_active=e.active,
               c2_alpha=sp.alpha, c2_warps=w, c2_pred=pred, c2_empty=emp)
    np.savez_compressed(OUT / "emdq_estep.npz", **out)
    print("emdq_estep: c2 empty", int(emp.sum()))


def features_cases():
    """The sparse front end (features.hpp) through the
    reference's own to_gray / detect_features / match_features, on the
    fixtures of its detector tests (test_features.cpp:14-127): the smoothed
    random texture, its wrap-around translation, pure noise, a tiny image,
    and an RGB frame of the synthetic scene."""
    R = Reference()
    out = {}

    def case(name, a, b, ratios=(0.8,)):
        ga, gb = R.to_gray(a), R.to_gray(b)
        ka, da = R.detect_features(ga)
        kb, db = R.detect_features(gb)
        out.update({f"{name}_a": a, f"{name}_b": b, f"{name}_ga_sha": sha(ga), f"{name}_gb_sha": sha(gb), f"{name}_kpa": ka,
                    f"{name}_da": da, f"{name}_kpb": kb, f"{name}_db": db})
        for r in ratios:
            out[f"{name}_m{int(round(100 * r))}"] = R.match_features(ka, da, kb, db, r)
        print(f"features {name}: {len(ka)} / {len(kb)} keypoints, "
              f"{len(out[f'{name}_m{int(round(100 * ratios[0]))}'])} matches")

    tex = R.textured_image(240, 160, 42)
    case("self", tex, tex)                                   # SelfMatchHasZeroDisplacement
    a = R.textured_image(320, 200, 7)
    case("translate", a, np.roll(a, 10, axis=1), (0.8, 0.6, 0.95))  # RecoversPureTranslation, ratio monotone
    rng = np.random.default_rng(1)
    case("noise", rng.integers(0, 256, (150, 200), dtype=np.uint8),
         rng.integers(0, 256, (150, 200), dtype=np.uint8))   # PureNoiseProducesFewMatches
    t = R.textured_image(12, 12, 3)
    case("tiny", t, t)                                       # TinyImageYieldsEmptyList
    f0 = R.scene_frame(320, 240, 10, 7, 6, 15.0, 80.0, 40.0, 0)
    f1 = R.scene_frame(320, 240, 10, 7, 6, 15.0, 80.0, 40.0, 1)
    case("scene_rgb", f0, f1)
    np.savez_compressed(OUT / "features.npz", **out)


def pipeline_cases():
    """The reference's production call sequence (tests/cpp/pipeline_dump.cpp:
    detect -> match -> Engine::process_frame -> blend_frame -> render, as
    tools/main.cpp run_mosaic) on its own 200-frame synthetic scenes, run by
    oracle/_ref/pipeline_ref (unmodified reference headers); plus the
    reference's own acceptance main (oracle/_ref/acceptance_ref) output."""
    import subprocess
    import tempfile
    from oracle.pipeline_io import read_dump
    exe = ROOT / "oracle" / "_ref" / "pipeline_ref"
    for path in ("scan", "outback"):
        with tempfile.TemporaryDirectory() as td:
            out = Path(td) / "p.bin"
            subprocess.run([str(exe), str(out), path, "200", "8"], check=True, capture_output=True)
            d = read_dump(out)
        np.savez_compressed(OUT / f"pipeline_{path}.npz", **d)
        print(path, d["mosaic"].shape, int(d["blended"].sum()), "blends")
    acc = subprocess.run([str(ROOT / "oracle" / "_ref" / "acceptance_ref")], capture_output=True, text=True)
    (OUT / "acceptance_ref.txt").write_text(acc.stdout)
    print(acc.stdout.splitlines()[-1])


def c3_sequence_case(nframes=200):
    """BASELINE configs[2] (C3) at full size through the REFERENCE: 200 1080p
    frames along a serpentine scan into the 8192^2 canvas (the sequence of
    tests/test_gpu_sequence.py: the C2 frame and its flip alternating, the
    C2 frame lattice moved with each frame), blended by the reference's
    blend_frame with its own invert_frame_boundary footprints. Stored: the
    lattice inputs (so the GPU test does not depend on host linear algebra),
    the frame's SHA, per-frame BlendStats, the final canvas geometry, the
    SHA of the weight plane, and colour / render values at 200k seeded
    occupied pixels."""
    R = Reference()
    wl = W.frame_workload("c2")
    offs = W.scan_offsets(nframes, wl.frame_w, wl.frame_h, wl.canvas)
    frames = [wl.frame, np.ascontiguousarray(wl.frame[::-1])]
    cv = R.canvas()
    stats = []
    for k, (tx, ty) in enumerate(offs):
        anchors = wl.anchors + np.array([tx, ty])
        warps = W.shifted_warps(wl.warps, tx, ty)
        poly = R.invert_frame_boundary(wl.frame_w, wl.frame_h, anchors, warps, wl.params.alpha)
        stats.append(R.blend_frame(cv, frames[k % 2], anchors, warps, wl.params.alpha, poly, workers=8))
    ox, oy, w, h = cv.info()
    col, wt = cv.arrays()
    full, _ = R.render(cv, crop=False)
    rng = np.random.default_rng(3)
    occ = np.flatnonzero(wt.reshape(-1) > 0)
    pick = np.sort(rng.choice(occ, min(200_000, len(occ)), replace=False))
    ys, xs = np.divmod(pick, w)
    np.savez_compressed(
        OUT / "c3_sequence.npz", anchors=wl.anchors, warps=wl.warps, alpha=wl.params.alpha, offsets=offs,
        frame_sha=sha(wl.frame), stats=np.array(stats, np.int64), info=np.array([ox, oy, w, h], np.int64),
        weight_sha=sha(wt), occupied=np.int64(len(occ)), sample_xy=np.stack([xs, ys], 1).astype(np.int32),
        sample_color=col.reshape(-1, 3)[pick], sample_render=full.reshape(-1, 4)[pick])
    print("c3", (ox, oy, w, h), "occupied", len(occ), "blended", int(np.array(stats)[:, 1].sum()))


def replay_case(frames=12):
    """Recorded node states for replay: the reference
    pipeline's own write_snapshot / TrajectoryWriter output (snapshot.hpp)
    for the first frames of the `scan` scene (oracle/_ref/snapshot_dump), with
    the blended frames and their footprints. The same run as
    pipeline_scan.npz's first frames, so replayed blends must reproduce its
    BlendStats."""
    import subprocess
    import tempfile
    exe = ROOT / "oracle" / "_ref" / "snapshot_dump"
    with tempfile.TemporaryDirectory() as td:
        out = subprocess.run([str(exe), td, str(frames), "scan"], check=True, capture_output=True, text=True)
        w, h = map(int, out.stdout.split())
        ts = sorted(int(p.stem.split("_")[1]) for p in Path(td).glob("snapshot_*.json"))
        data = {"frames_t": np.array(ts, np.int32), "size": np.array([w, h], np.int32),
                "trajectory": np.frombuffer(Path(td, "trajectory.jsonl").read_bytes(), np.uint8)}
        for t in ts:
            data[f"snapshot_{t}"] = np.frombuffer(Path(td, f"snapshot_{t}.json").read_bytes(), np.uint8)
            data[f"frame_{t}"] = np.frombuffer(Path(td, f"frame_{t}.rgb").read_bytes(), np.uint8).reshape(h, w, 3)
            data[f"footprint_{t}"] = np.loadtxt(Path(td, f"footprint_{t}.txt")).reshape(-1, 2)
    np.savez_compressed(OUT / "replay_scan.npz", **data)
    print("replay", ts)


if __name__ == "__main__":
    if sys.argv[1:] == ["pipeline"]:
        pipeline_cases()
    elif sys.argv[1:] == ["replay"]:
        replay_case()
    elif sys.argv[1:] == ["c3"]:
        c3_sequence_case()
    elif sys.argv[1:] == ["estep"]:
        estep_cases()
    elif sys.argv[1:] == ["features"]:
        features_cases()
    else:
        main()
        estep_cases()
        features_cases()
        pipeline_cases()
        c3_sequence_case()
        replay_case()
