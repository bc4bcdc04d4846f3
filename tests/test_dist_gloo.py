"""CPU, world_size 2 and 3 (gloo): the band decomposition and its collectives.

Each rank blends the golden C1 sequence into ITS OWN block-cyclic stripes
(the oracle's restatement of nrm_canvas_set_band: orc_blend_frame_band), so
its BlendStats count only its rows. The collectives the GPU path uses
(dist.reduce_stats, assemble_bbox, assemble_render) must then reproduce the
single-process reference exactly: every frame's BlendStats, every owned row
of the canvas, render(crop) and its origin.

The halo exchange of the canvas deformation (dist.halo_plan +
dist.exchange_halo over gloo point-to-point) is checked the same way: a
rank's canvas holds garbage outside its stripes, receives its halo rows and
deforms; its owned rows must equal the single-canvas deformation."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(rank, world, port):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _golden_seq():
    from pathlib import Path
    g = dict(np.load(Path(__file__).resolve().parent / "golden" / "blend_c1_seq.npz"))
    polys, o = [], 0
    for n in g["npoly"]:
        polys.append(g["polys"][o:o + n])
        o += n
    return g, polys


def _blend_worker(rank, world, port, q):
    _setup(rank, world, port)
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2103_07414_b200 import _lib, dist as D
    try:
        g, polys = _golden_seq()
        O = Oracle()
        ref, mine = O.canvas(), O.canvas()
        ok_stats = True
        for k, poly in enumerate(polys):
            st_ref = O.blend_frame(ref, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), poly)
            st_loc = O.blend_frame(mine, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), poly,
                                   band=(rank, world))
            t = torch.tensor([st_loc], dtype=torch.int64)
            D.reduce_stats(t)
            ok_stats &= tuple(int(v) for v in t[0]) == st_ref
        ox, oy, w, h = mine.info()
        assert (ox, oy, w, h) == ref.info()
        mask = D.owned_rows_mask(oy, h, rank, world)
        lib = _lib.load()
        assert all(bool(lib.nrm_band_owns_row(int(oy + r), rank, world)) == bool(mask[r]) for r in range(0, h, 7))
        col, wt = mine.arrays()
        rcol, rwt = ref.arrays()
        rows_ok = np.array_equal(col[mask], rcol[mask]) and np.array_equal(wt[mask], rwt[mask])
        rows_ok &= not wt[~mask].any()  # nothing outside this rank's stripes
        full, _ = O.render(mine, crop=False)
        occ = np.argwhere(wt > 0)
        bb = (int(occ[:, 1].min()), int(occ[:, 0].min()), int(occ[:, 1].max()), int(occ[:, 0].max())) \
            if len(occ) else (0, 0, -1, -1)
        x0, y0, x1, y1 = D.assemble_bbox(bb)
        crop = torch.from_numpy(np.ascontiguousarray(full[y0:y1 + 1, x0:x1 + 1]))
        D.assemble_render(crop, oy + y0, rank, world, dst=0)
        res = {"stats": ok_stats, "rows": rows_ok, "owned": int(mask.sum())}
        if rank == 0:
            ref_crop, ref_org = O.render(ref, crop=True)
            res["render"] = np.array_equal(crop.numpy(), ref_crop)
            res["origin"] = (ox + x0, oy + y0) == ref_org
        q.put(("ok", rank, res))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put(("err", rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _halo_worker(rank, world, port, q):
    _setup(rank, world, port)
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2103_07414_b200 import dist as D
    try:
        rng = np.random.default_rng(11)
        oy_abs, H, W = -256, 512, 512
        col = rng.random((H, W, 3)).astype(np.float32).astype(np.float64)
        wt = rng.integers(0, 31, (H, W)).astype(np.uint8)
        yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
        # displacement up to ~9.5 rows, region rows 40..439
        y0, h = 40, 400
        d = np.stack([2.5 * np.sin(xx[y0:y0 + h] / 37.0),
                      9.25 * np.cos(yy[y0:y0 + h] / 53.0) + 0.125 * np.sin(xx[y0:y0 + h] / 19.0)], -1)
        d = d.astype(np.float32)
        O = Oracle()

        def canvas(c, w_):
            cv = O.canvas()
            cv.ensure_contains((0.0, float(oy_abs), W - 1.0, oy_abs + H - 1.0))
            assert cv.info() == (0, oy_abs, W, H), cv.info()
            cv.set_arrays(c, w_)
            return cv

        ref = canvas(col, wt)
        ref.deform(0, y0, W, h, d)
        rcol, rwt = ref.arrays()
        # this rank's canvas: its stripes are right, every other row is garbage
        mask = D.owned_rows_mask(oy_abs, H, rank, world)
        lcol, lwt = col.copy(), wt.copy()
        lcol[~mask] = -7.0
        lwt[~mask] = 29
        halo = int(np.ceil(np.abs(d[..., 1]).max())) + 1
        plan = D.halo_plan(oy_abs, H, world, halo, y0, h)
        row_bytes = 13 * W

        def pack(rows, buf):
            b = buf.numpy()
            for k, r in enumerate(rows):
                seg = b[k * row_bytes:(k + 1) * row_bytes]
                seg[:12 * W].view(np.float32)[:] = lcol[r].astype(np.float32).T.reshape(-1)
                seg[12 * W:] = lwt[r]

        def unpack(rows, buf):
            b = buf.numpy()
            for k, r in enumerate(rows):
                seg = b[k * row_bytes:(k + 1) * row_bytes]
                lcol[r] = seg[:12 * W].view(np.float32).reshape(3, W).T.astype(np.float64)
                lwt[r] = seg[12 * W:]

        nbytes = D.exchange_halo(plan, rank, world, row_bytes, pack, unpack)
        mine = canvas(lcol, lwt)
        mine.deform(0, y0, W, h, d)
        mcol, mwt = mine.arrays()
        same = np.array_equal(mcol[mask], rcol[mask]) and np.array_equal(mwt[mask], rwt[mask])
        # without the exchange the garbage rows must leak in (the check has teeth)
        bad = canvas(np.where(mask[:, None, None], col, -7.0), np.where(mask[:, None], wt, 29).astype(np.uint8))
        bad.deform(0, y0, W, h, d)
        bcol, _ = bad.arrays()
        leaks = not np.array_equal(bcol[mask], rcol[mask])
        q.put(("ok", rank, {"same": same, "leaks": leaks, "bytes": nbytes,
                            "expect": sum(len(plan[rank][o]) for o in range(world)) * row_bytes}))
    except Exception:  # pragma: no cover
        import traceback
        q.put(("err", rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(worker, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    errs = [r for r in res if r[0] == "err"]
    assert not errs, errs
    return {r[1]: r[2] for r in res}


@pytest.mark.parametrize("world", [2, 3])
def test_banded_blends_reduce_to_the_single_process_reference(world):
    res = _run(_blend_worker, world)
    assert all(r["stats"] for r in res.values()), "all-reduced per-rank BlendStats differ from the reference"
    assert all(r["rows"] for r in res.values()), "a rank's stripes differ from the single canvas"
    assert res[0]["render"], "assembled render differs from the single-process render"
    assert res[0]["origin"], "crop origin differs"
    assert all(r["owned"] > 0 for r in res.values())


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_makes_banded_deformation_exact(world):
    res = _run(_halo_worker, world)
    for r in res.values():
        assert r["same"], "banded deformation with the halo exchange differs from the single canvas"
        assert r["leaks"], "garbage rows never reached the owned rows: the check is vacuous"
        assert r["bytes"] == r["expect"] > 0


def test_owned_rows_mask_partitions():
    from paper_2103_07414_b200 import dist as D
    for world in (1, 2, 4, 8):
        masks = np.stack([D.owned_rows_mask(-768, 4096, r, world) for r in range(world)])
        assert (masks.sum(0) == 1).all()


def test_halo_plan_covers_the_dilated_stripes():
    from paper_2103_07414_b200 import dist as D
    for world, halo in ((2, 3), (3, 17), (4, 64), (8, 70)):
        H = 1000
        plan = D.halo_plan(-100, H, world, halo, 10, 900)
        owner = np.mod(np.floor_divide(np.arange(H) - 100, 64), world)
        for q in range(world):
            need = set()
            for y in range(10, 910):
                if owner[y] == q:
                    need.update(r for r in range(max(0, y - halo), min(H, y + halo + 1)) if owner[r] != q)
            got = set()
            for r in range(world):
                assert set(plan[q][r].tolist()) <= set(np.nonzero(owner == r)[0].tolist())
                got.update(plan[q][r].tolist())
            assert got == need, (world, halo, q)
