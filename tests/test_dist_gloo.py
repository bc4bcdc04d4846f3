"""CPU, world_size 2 (gloo): the band decomposition and its collectives.
Each rank produces the canvas of its own block-cyclic stripes (here from the
oracle, masked to the rows the library says the rank owns), then the same
collectives the GPU path uses assemble render(crop) and BlendStats; the
result must equal the single-process reference exactly."""
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


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2103_07414_b200 import _lib, dist as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = dict(np.load(Path(__file__).resolve().parent / "golden" / "blend_c1_seq.npz"))
        polys, o = [], 0
        for n in g["npoly"]:
            polys.append(g["polys"][o:o + n])
            o += n
        O = Oracle()
        cv = O.canvas()
        stats = []
        for k, poly in enumerate(polys):
            stats.append(O.blend_frame(cv, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), poly))
        col, wt = cv.arrays()
        ox, oy, w, h = cv.info()
        full, _ = O.render(cv, crop=False)
        # this rank's stripes only
        mask = D.owned_rows_mask(oy, h, rank, world)
        lib = _lib.load()
        assert all(bool(lib.nrm_band_owns_row(int(oy + r), rank, world)) == bool(mask[r]) for r in range(0, h, 7))
        local = full * mask[:, None, None]
        wt_local = wt * mask[:, None]
        # per-rank stats: blended counts split by row ownership (the GPU kernels count per owned tile)
        st = torch.tensor([[stats[-1][0], int((wt_local > 0).sum()), 0, 0]], dtype=torch.int64)
        D.reduce_stats(st)
        occ = np.argwhere(wt_local > 0)
        bb = (int(occ[:, 1].min()), int(occ[:, 0].min()), int(occ[:, 1].max()), int(occ[:, 0].max())) \
            if len(occ) else (0, 0, -1, -1)
        x0, y0, x1, y1 = D.assemble_bbox(bb)
        crop = torch.from_numpy(np.ascontiguousarray(local[y0:y1 + 1, x0:x1 + 1]))
        D.assemble_render(crop, oy + y0, rank, world, dst=0)
        if rank == 0:
            ref_crop, ref_org = O.render(cv, crop=True)
            q.put(("ok", np.array_equal(crop.numpy(), ref_crop), (ox + x0, oy + y0) == ref_org,
                   int(st[0, 1]) == int((wt > 0).sum()), int(mask.sum())))
        else:
            q.put(("rank", rank, int(mask.sum())))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_banded_assembly_equals_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    errs = [r for r in res if r[0] == "err"]
    assert not errs, errs
    ok = [r for r in res if r[0] == "ok"][0]
    assert ok[1], "assembled render differs from the single-process render"
    assert ok[2], "crop origin differs"
    assert ok[3], "all-reduced blended count differs"


def test_owned_rows_mask_partitions():
    from paper_2103_07414_b200 import dist as D
    for world in (1, 2, 4, 8):
        masks = np.stack([D.owned_rows_mask(-768, 4096, r, world) for r in range(world)])
        assert (masks.sum(0) == 1).all()
