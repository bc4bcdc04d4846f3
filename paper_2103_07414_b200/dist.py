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


class BandedMosaic:
    """A canvas banded across the ranks of the default process group
    (GPU product path: libnrm_b200 on this rank's device)."""

    def __init__(self, rank: int, world: int, device: int, reserve: Optional[Sequence[float]] = None):
        from . import mosaic as M
        self.M = M
        self.rank, self.world = rank, world
        self.ctx = M.Context(device)
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
            x0, y0, x1, y1 = assemble_bbox(self.canvas.occupied_bbox(), device=dev)
            if x1 < x0:
                return np.zeros((0, 0, 4), np.uint8), (ox, oy)
        out = torch.zeros((y1 - y0 + 1, x1 - x0 + 1, 4), dtype=torch.uint8, device=dev)
        self.M.render_device(self.canvas, x0, y0, x1 - x0 + 1, y1 - y0 + 1, out)
        self.ctx.synchronize()
        assemble_render(out, int(oy) + y0, self.rank, self.world, dst=dst)
        return out.cpu().numpy(), (ox + x0, oy + y0)
