"""Multi-GPU banding of the mosaic canvas (north_star).

One process per GPU (torchrun). Every rank holds the replicated control
points and frame; rank r deforms and blends only the canvas rows of its
block-cyclic 64-row stripes (floor(y / 64) mod world == r, nrm_canvas_set_band),
so a frame's footprint (1-2k rows) spreads over all ranks. Results are
bitwise identical for any world size: tiles are anchored to absolute
reference coordinates and each pixel is written by exactly one rank.

Collectives (torch.distributed; NCCL over NVLink on GPUs, gloo in tests):
  broadcast_inputs  -- control points + frame from the source rank
  reduce_stats      -- BlendStats: all-reduce of the per-rank blended /
                       no-support / out-of-frame counts (footprint is the same
                       on every rank and is taken from rank-local stats)
  assemble_bbox     -- crop box for render(crop=True): min/max over ranks
  assemble_render   -- rendered RGBA bands: each rank sends only its owned
                       rows (one gather of equal-size padded stripe packs)
  exchange_halo     -- canvas deformation (north_star extension): before a
                       rank resamples its stripes, the rows within the halo
                       H = ceil(max |d_y|) + 1 of them that other ranks own
                       are sent point to point by their owners (halo_plan)
No collective touches the per-pixel data path of blend_frame itself.
"""
from __future__ import annotations

from typing import Optional, Sequence, Tuple

import numpy as np

STRIPE_ROWS = 64


def owned_rows_mask(origin_y: int, height: int, rank: int, world: int) -> np.ndarray:
    """Canvas rows [0, height) of a canvas at reference row origin_y that
    `rank` owns (same rule as nrm_band_owns_row)."""
    if world <= 1:
        return np.ones(height, bool)
    rows = np.arange(height, dtype=np.int64) + int(origin_y)
    return np.mod(np.floor_divide(rows, STRIPE_ROWS), world) == rank


def halo_plan(origin_y: int, height: int, world: int, halo: int, y0: int = 0, h: Optional[int] = None):
    """Rows each rank must receive before deforming the canvas rows [y0, y0+h)
    with |d_y| <= halo - 1: plan[q][r] = sorted canvas rows owned by rank r
    that rank q reads (within `halo` rows of a row q owns in the region).
    Every rank computes the same plan, so rank r sends plan[q][r] to each q
    and receives plan[r][q] from each q."""
    if h is None:
        h = height - y0
    plan = [[np.zeros(0, np.int32) for _ in range(world)] for _ in range(world)]
    if world <= 1 or h <= 0 or halo <= 0:
        return plan
    owner = np.mod(np.floor_divide(np.arange(height, dtype=np.int64) + int(origin_y), STRIPE_ROWS), world)
    for q in range(world):
        mine = np.zeros(height, bool)
        mine[y0:y0 + h] = owner[y0:y0 + h] == q
        # dilate by `halo` rows (cumulative-sum window)
        c = np.concatenate([[0], np.cumsum(mine)])
        lo = np.clip(np.arange(height) - halo, 0, height)
        hi = np.clip(np.arange(height) + halo + 1, 0, height)
        near = (c[hi] - c[lo]) > 0
        for r in range(world):
            if r != q:
                plan[q][r] = np.nonzero(near & (owner == r))[0].astype(np.int32)
    return plan


def broadcast_inputs(tensors: Sequence, src: int = 0, group=None) -> None:
    import torch.distributed as dist
    for t in tensors:
        dist.broadcast(t, src=src, group=group)


def reduce_stats(stats_t, group=None):
    """stats_t: int64 tensor [..., 4] of rank-local BlendStats. Column 0
    (footprint_pixels) is identical on every rank; columns 1-3 are summed."""
    import torch.distributed as dist
    counts = stats_t[..., 1:].clone()
    dist.all_reduce(counts, group=group)
    stats_t[..., 1:] = counts
    return stats_t


def assemble_bbox(bbox4: Tuple[int, int, int, int], group=None, device=None) -> Tuple[int, int, int, int]:
    """Union of per-rank occupied boxes (x0, y0, x1, y1); empty boxes have x1 < x0."""
    import torch
    import torch.distributed as dist
    x0, y0, x1, y1 = bbox4
    big = 1 << 40
    if x1 < x0:  # empty on this rank
        x0 = y0 = big
        x1 = y1 = -big
    t = torch.tensor([x0, y0, -x1, -y1], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    v = t.tolist()
    return int(v[0]), int(v[1]), int(-v[2]), int(-v[3])


def assemble_render(local_rgba, origin_y: int, rank: int, world: int, dst: int = 0, group=None):
    """Assembles rank-local RGBA rasters (h, w, 4) whose row 0 is reference
    row origin_y: every rank packs the rows it owns (owned_rows_mask) and
    one gather brings the packs to `dst`, which writes them into its raster.
    Each rank moves ~1/world of the image. Returns the assembled raster on
    dst (the local raster elsewhere)."""
    import torch
    import torch.distributed as dist
    if world <= 1:
        return local_rgba
    h = local_rgba.shape[0]
    masks = [torch.from_numpy(owned_rows_mask(origin_y, h, r, world)) for r in range(world)]
    rows = [int(m.sum()) for m in masks]
    cap = max(max(rows), 1)
    pack = torch.zeros((cap,) + tuple(local_rgba.shape[1:]), dtype=local_rgba.dtype, device=local_rgba.device)
    mine = masks[rank].to(local_rgba.device)
    if rows[rank]:
        pack[: rows[rank]] = local_rgba[mine]
    if rank == dst:
        packs = [torch.empty_like(pack) for _ in range(world)]
        dist.gather(pack, packs, dst=dst, group=group)
        for r in range(world):
            if rows[r]:
                local_rgba[masks[r].to(local_rgba.device)] = packs[r][: rows[r]]
    else:
        dist.gather(pack, None, dst=dst, group=group)
    return local_rgba


def exchange_halo(plan, rank: int, world: int, row_bytes: int, pack, unpack, device=None, group=None) -> int:
    """Point-to-point halo exchange of a banded canvas: this rank sends the
    rows other ranks read (plan[q][rank]) and receives the rows it reads
    (plan[rank][q]). pack(rows, buf) / unpack(rows, buf) move rows between
    the canvas and flat uint8 buffers of row_bytes per row (on the GPU path,
    Canvas.pack_rows / unpack_rows on torch's current stream; the transfers
    are NCCL send/recv over NVLink). Returns the bytes received."""
    import torch
    import torch.distributed as dist
    if world <= 1:
        return 0
    ops, recvs = [], []
    for q in range(world):
        if q == rank:
            continue
        out_rows = plan[q][rank]
        if len(out_rows):
            buf = torch.empty(len(out_rows) * row_bytes, dtype=torch.uint8, device=device)
            pack(out_rows, buf)
            ops.append(dist.P2POp(dist.isend, buf, q, group=group))
        in_rows = plan[rank][q]
        if len(in_rows):
            buf = torch.empty(len(in_rows) * row_bytes, dtype=torch.uint8, device=device)
            recvs.append((in_rows, buf))
            ops.append(dist.P2POp(dist.irecv, buf, q, group=group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for rows, buf in recvs:
        unpack(rows, buf)
    return sum(int(b.numel()) for _, b in recvs)


class BandedMosaic:
    """A canvas banded across the ranks of the default process group
    (GPU product path: libnrm_b200 on this rank's device)."""

    def __init__(self, rank: int, world: int, device: int, reserve: Optional[Sequence[float]] = None):
        from . import mosaic as M
        self.M = M
        self.rank, self.world = rank, world
        self.ctx = M.Context(device)
        # Every kernel of this rank runs on torch's current stream of the
        # device, so the collectives below (issued by torch on the same
        # stream, or ordered after it by NCCL) see the kernels' results and
        # the kernels see inputs torch produced (broadcast frames, zeroed
        # render buffers) without extra events.
        import torch
        self.ctx.set_stream(torch.cuda.current_stream(device).cuda_stream)
        self.canvas = M.Canvas(self.ctx)
        if reserve is not None:
            self.canvas.reserve(reserve)
        self.canvas.set_band(rank, world)

    def blend(self, frame_t, fw, fh, ch, anchors_t, warps_t, alpha, poly, stats_t):
        """Blends one (replicated) frame into this rank's stripes; stats are
        all-reduced so every rank returns the reference's BlendStats."""
        self.M.blend_frame_device(self.canvas, frame_t, fw, fh, ch, anchors_t, warps_t, alpha, poly, stats_t)
        if self.world > 1:
            reduce_stats(stats_t)
        return stats_t

    def blend_frames(self, frames_t, fw, fh, ch, anchors_t, warps_t, alpha, polys, stats_t):
        """Blends several (replicated) frames in order into this rank's stripes
        in one batched call when their footprints are disjoint
        (mosaic.blend_frames_device); stats_t (nf, 4) is all-reduced."""
        self.M.blend_frames_device(self.canvas, frames_t, fw, fh, ch, anchors_t, warps_t, alpha, polys, stats_t)
        if self.world > 1:
            reduce_stats(stats_t)
        return stats_t

    def deform(self, disp_t, x: int = 0, y: int = 0, group=None):
        """Canvas deformation (north_star extension) of the rectangle at
        (x, y) with disp_t's (h, w) shape (CUDA float32 tensor, canvas px).
        Each rank resamples only its stripes: the halo H = ceil(max |d_y|) + 1
        is agreed by a max all-reduce, the rows within H of its stripes come
        from their owners (exchange_halo), then the kernel runs locally."""
        import torch
        import torch.distributed as dist
        h = int(disp_t.shape[0])
        halo = 0
        if self.world > 1:
            dmax = disp_t[..., 1].abs().max() if disp_t.numel() else torch.zeros((), device=disp_t.device)
            hv = (torch.ceil(dmax) + 1).to(torch.int64).reshape(1)
            dist.all_reduce(hv, op=dist.ReduceOp.MAX, group=group)
            halo = int(hv.item())
            _, oy = self.canvas.origin_offset()
            plan = halo_plan(int(oy), self.canvas.height(), self.world, halo, y, h)
            exchange_halo(plan, self.rank, self.world, 13 * self.canvas.width(), self.canvas.pack_rows,
                          self.canvas.unpack_rows, device=torch.device("cuda", self.ctx.device), group=group)
        self.canvas.deform(disp_t, x, y)
        return halo

    def render(self, crop: bool = False, dst: int = 0):
        """render(canvas, crop) assembled on rank `dst` -> (rgba numpy, origin)."""
        import torch
        ox, oy = self.canvas.origin_offset()
        w, h = self.canvas.width(), self.canvas.height()
        if w == 0:
            return np.zeros((0, 0, 4), np.uint8), (ox, oy)
        x0, y0, x1, y1 = 0, 0, w - 1, h - 1
        dev = torch.device("cuda", self.ctx.device)
        if crop:
            bb = self.canvas.occupied_bbox()
            x0, y0, x1, y1 = assemble_bbox(bb, device=dev) if self.world > 1 else bb
            if x1 < x0:
                return np.zeros((0, 0, 4), np.uint8), (ox, oy)
        out = torch.zeros((y1 - y0 + 1, x1 - x0 + 1, 4), dtype=torch.uint8, device=dev)
        self.M.render_device(self.canvas, x0, y0, x1 - x0 + 1, y1 - y0 + 1, out)
        self.ctx.synchronize()
        assemble_render(out, int(oy) + y0, self.rank, self.world, dst=dst)
        return out.cpu().numpy(), (ox + x0, oy + y0)
