"""Python mirror of the reference's dense-stage API (namespace nrmosaic,
/root/reference/proj/include/nrmosaic/mosaic.hpp and fieldest.hpp), backed
by libnrm_b200.so. Names, argument meaning and error behaviour follow the
reference so the parity tests read like its own tests:

    reference (C++)                          here
    pixel_warp(x, anchors, warps, a)         pixel_warp(x, anchors, warps, a) -> warp5 | None
    Canvas / ensure_contains / color ...     Canvas (HBM-resident; host reads are explicit)
    blend_frame(canvas, frame, ..., workers) blend_frame(canvas, frame, ...) -> BlendStats
    render(canvas, crop, &origin)            render(canvas, crop) -> (rgba, origin)
    invert_frame_boundary(w, h, ...)         invert_frame_boundary(w, h, ...)
    detail::blend_local + node_uncertainty   emdq_field(grid, ...) (dense, every pixel)

Host arrays are numpy; the *_device variants take torch CUDA tensors and run
asynchronously on the context's stream.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import BlendStats, Grid, NoSupport, NrmError, check

__all__ = [
    "BlendStats", "Canvas", "Context", "Grid", "NoSupport", "NrmError", "blend_frame",
    "blend_frame_device", "default_context", "emdq_field", "emdq_field_device",
    "invert_frame_boundary", "node_field", "node_field_device", "pixel_warp", "render",
    "render_device",
]

K_WEIGHT_CAP = 30   # mosaic.hpp:102
K_TILE = 256        # mosaic.hpp:103


def _ptr(a: Optional[np.ndarray]) -> Optional[int]:
    return None if a is None else a.ctypes.data


def _f64(a, shape_tail: int, name: str) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if arr.size == 0:
        return arr.reshape(0, shape_tail)
    arr = arr.reshape(-1, shape_tail) if arr.ndim != 2 else arr
    if arr.shape[1] != shape_tail:
        raise ValueError(f"{name}: expected (n, {shape_tail}) array, got {arr.shape}")
    return arr


def _tptr(t) -> int:
    """Device pointer of a CUDA torch tensor (must be contiguous)."""
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("device variants need contiguous CUDA tensors")
    return t.data_ptr()


class Context:
    """One CUDA device + one stream (nrm_ctx)."""

    def __init__(self, device: int = 0):
        self._lib = _lib.load()
        h = C.c_void_p()
        check(self._lib.nrm_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = int(device)

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_handle: Optional[int]) -> None:
        """Run subsequent work on an external cudaStream_t (e.g.
        torch.cuda.current_stream().cuda_stream); None = own stream. Handle 0
        (torch's default stream) is passed as cudaStreamLegacy (0x1), since a
        NULL stream means "own stream" at the C ABI."""
        if stream_handle is not None and int(stream_handle) == 0:
            stream_handle = 1  # cudaStreamLegacy
        check(self._lib.nrm_ctx_set_stream(self._h, stream_handle))

    def stream(self) -> int:
        return self._lib.nrm_ctx_stream(self._h) or 0

    def synchronize(self) -> None:
        check(self._lib.nrm_ctx_synchronize(self._h))

    def launch_count(self) -> int:
        v = C.c_int64()
        check(self._lib.nrm_ctx_launch_count(self._h, C.byref(v)))
        return v.value

    def set_exception_capacity(self, slots: int) -> None:
        """Exception-queue slots per launch (0 = default); results never
        depend on it (overflowing deferrals are resolved by a scan)."""
        check(self._lib.nrm_ctx_set_exception_capacity(self._h, int(slots)))

    def spilled_launches(self) -> int:
        v = C.c_int64()
        check(self._lib.nrm_ctx_spilled_launches(self._h, C.byref(v)))
        return v.value

    def exceptions(self):
        """(blend/node-field pixels resolved by the last exception pass, EMDQ
        pixels of the last emdq_field that took the exact tier)."""
        a, b = C.c_int64(), C.c_int64()
        check(self._lib.nrm_ctx_exceptions(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def profile(self, enable: bool = True) -> None:
        """Per-kernel CUDA-event timing on the context stream (clears on enable)."""
        check(self._lib.nrm_ctx_profile(self._h, int(bool(enable))))

    def kernel_times(self) -> dict:
        """{kernel name: (total ms, launches)} since profile(True)."""
        buf = C.create_string_buffer(4096)
        ms = (C.c_double * 64)()
        cnt = (C.c_int64 * 64)()
        n = C.c_int()
        check(self._lib.nrm_ctx_profile_read(self._h, buf, 4096, ms, cnt, 64, C.byref(n)))
        names = buf.value.decode().split("\n")[: n.value]
        return {nm: (ms[i], cnt[i]) for i, nm in enumerate(names)}

    def peak(self, which: str = "fp32") -> float:
        """Measured lane-ops/s of the FP32 FFMA ("fp32") or MUFU.EX2 ("mufu") pipe."""
        v = C.c_double()
        check(self._lib.nrm_selftest_peak(self._h, 0 if which == "fp32" else 1, C.byref(v)))
        return v.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.nrm_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: dict = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


class Canvas:
    """Canvas (mosaic.hpp:100-182), stored in HBM as float32 R/G/B planes
    plus a uint8 weight plane. Logical origin/width/height follow the
    reference's ensure_contains bookkeeping exactly."""

    kWeightCap = K_WEIGHT_CAP
    kTile = K_TILE

    def __init__(self, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self._lib = self.ctx._lib
        h = C.c_void_p()
        check(self._lib.nrm_canvas_create(self.ctx.handle, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def _info(self):
        ox, oy, w, h = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
        check(self._lib.nrm_canvas_info(self._h, C.byref(ox), C.byref(oy), C.byref(w), C.byref(h)))
        return ox.value, oy.value, w.value, h.value

    def empty(self) -> bool:
        return self._info()[2] == 0

    def width(self) -> int:
        return self._info()[2]

    def height(self) -> int:
        return self._info()[3]

    def origin_offset(self) -> Tuple[float, float]:
        ox, oy, _, _ = self._info()
        return float(ox), float(oy)

    def ensure_contains(self, rect: Sequence[float]) -> None:
        x0, y0, x1, y1 = map(float, rect)
        check(self._lib.nrm_canvas_ensure_contains(self._h, x0, y0, x1, y1))

    def reserve(self, rect: Sequence[float]) -> None:
        x0, y0, x1, y1 = map(float, rect)
        check(self._lib.nrm_canvas_reserve(self._h, x0, y0, x1, y1))

    def set_band(self, rank: int, count: int) -> None:
        check(self._lib.nrm_canvas_set_band(self._h, int(rank), int(count)))

    def read(self, x: int = 0, y: int = 0, w: Optional[int] = None, h: Optional[int] = None):
        """(color (h,w,3) float64, weight (h,w) uint8) of a canvas-pixel rectangle."""
        if w is None:
            w = self.width() - x
        if h is None:
            h = self.height() - y
        rgb = np.zeros((h, w, 3), np.float64)
        wt = np.zeros((h, w), np.uint8)
        check(self._lib.nrm_canvas_download(self._h, x, y, w, h, _ptr(rgb), _ptr(wt)))
        return rgb, wt

    def write(self, x: int, y: int, rgb: Optional[np.ndarray], weight: Optional[np.ndarray]) -> None:
        arr = rgb if rgb is not None else weight
        h, w = arr.shape[:2]
        rgb_c = None if rgb is None else np.ascontiguousarray(rgb, np.float64)
        w_c = None if weight is None else np.ascontiguousarray(weight, np.uint8)
        check(self._lib.nrm_canvas_upload(self._h, x, y, w, h, _ptr(rgb_c), _ptr(w_c)))

    def deform(self, disp, x: int = 0, y: int = 0) -> None:
        """Extension (north_star, no reference counterpart): new(p) =
        old(p + d(p)) over the rectangle at (x, y) of disp's (h, w) shape;
        disp is a host float32 (h, w, 2) array or a CUDA tensor. d == 0 is a
        bit-exact no-op (nrm_canvas_deform)."""
        if hasattr(disp, "is_cuda"):
            h, w = int(disp.shape[0]), int(disp.shape[1])
            check(self._lib.nrm_canvas_deform_device(self._h, int(x), int(y), w, h, _tptr(disp)))
        else:
            d = np.ascontiguousarray(disp, np.float32)
            if d.ndim != 3 or d.shape[2] != 2:
                raise ValueError("disp must be (h, w, 2)")
            check(self._lib.nrm_canvas_deform(self._h, int(x), int(y), d.shape[1], d.shape[0], _ptr(d)))

    def pack_rows(self, rows, buf_t) -> None:
        """Halo rows (banded canvases): canvas rows `rows` across the full
        width into the CUDA uint8 tensor buf_t (13 * width bytes per row)."""
        r = np.ascontiguousarray(rows, np.int32)
        if buf_t.numel() < len(r) * 13 * self.width():
            raise ValueError("pack_rows: buffer too small")
        check(self._lib.nrm_canvas_pack_rows_device(self._h, _ptr(r), len(r), _tptr(buf_t)))

    def unpack_rows(self, rows, buf_t) -> None:
        r = np.ascontiguousarray(rows, np.int32)
        if buf_t.numel() < len(r) * 13 * self.width():
            raise ValueError("unpack_rows: buffer too small")
        check(self._lib.nrm_canvas_unpack_rows_device(self._h, _ptr(r), len(r), _tptr(buf_t)))

    def color(self, x: int, y: int) -> np.ndarray:
        return self.read(x, y, 1, 1)[0][0, 0]

    def weight(self, x: int, y: int) -> int:
        return int(self.read(x, y, 1, 1)[1][0, 0])

    def occupied(self, x: int, y: int) -> bool:
        return self.weight(x, y) > 0

    def occupied_count(self) -> int:
        v = C.c_int64()
        check(self._lib.nrm_canvas_occupied_count(self._h, C.byref(v)))
        return v.value

    def occupied_bbox(self):
        v = [C.c_int() for _ in range(4)]
        check(self._lib.nrm_canvas_occupied_bbox(self._h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.nrm_canvas_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _frame(frame: np.ndarray) -> Tuple[np.ndarray, int, int, int]:
    f = np.ascontiguousarray(frame, dtype=np.uint8)
    if f.ndim == 2:
        f = f[:, :, None]
    if f.ndim != 3:
        raise ValueError("frame must be (h, w) or (h, w, c)")
    h, w, c = f.shape
    return f, w, h, c


def blend_frame(canvas: Canvas, frame: np.ndarray, anchors, warps, alpha: float,
                footprint_polygon, workers: Optional[int] = None, unc=None) -> BlendStats:
    """blend_frame (mosaic.hpp:196-296). `workers` is accepted for signature
    parity and ignored (the GPU grid replaces the thread pool).
    unc: optional frame-aligned (h, w) uncertainty map -> the uncertainty-
    weighted extension (nrm_blend_frame_weighted; unc == 1 is the reference)."""
    f, w, h, c = _frame(frame)
    a = _f64(anchors, 2, "anchors")
    q = _f64(warps, 5, "warps")
    if len(a) != len(q):
        raise ValueError("anchors / warps size mismatch")
    p = _f64(footprint_polygon, 2, "footprint_polygon")
    st = BlendStats()
    if unc is None:
        check(canvas._lib.nrm_blend_frame(canvas.handle, _ptr(f), w, h, c, _ptr(a), _ptr(q), len(a),
                                          float(alpha), _ptr(p), len(p), C.byref(st)))
    else:
        u = np.ascontiguousarray(unc, np.float32)
        if u.shape != (h, w):
            raise ValueError(f"unc must be the frame's (h, w) = {(h, w)}")
        check(canvas._lib.nrm_blend_frame_weighted(canvas.handle, _ptr(f), w, h, c, _ptr(a), _ptr(q), len(a),
                                                   float(alpha), _ptr(p), len(p), _ptr(u), C.byref(st)))
    return st


def blend_frame_device(canvas: Canvas, frame_t, fw: int, fh: int, ch: int, anchors_t, warps_t,
                       alpha: float, footprint_polygon, stats_t, unc_t=None) -> None:
    """Device-resident blend_frame: torch CUDA tensors in, int64[4] stats tensor out (async).
    unc_t: optional (fh, fw) float32 uncertainty map (weighted extension)."""
    p = _f64(footprint_polygon, 2, "footprint_polygon")
    n = anchors_t.shape[0] if anchors_t is not None else 0
    if unc_t is None:
        check(canvas._lib.nrm_blend_frame_device(canvas.handle, _tptr(frame_t), fw, fh, ch,
                                                 _tptr(anchors_t), _tptr(warps_t), n, float(alpha),
                                                 _ptr(p), len(p), _tptr(stats_t)))
    else:
        check(canvas._lib.nrm_blend_frame_weighted_device(canvas.handle, _tptr(frame_t), fw, fh, ch,
                                                          _tptr(anchors_t), _tptr(warps_t), n, float(alpha),
                                                          _ptr(p), len(p), _tptr(unc_t), _tptr(stats_t)))


def blend_frames_device(canvas: Canvas, frames_t, fw: int, fh: int, ch: int, anchors_t, warps_t, alpha: float,
                        polygons, stats_t) -> None:
    """blend_frame for several same-size frames in order (lists of device
    tensors; stats_t int64 (nf, 4) on the device), async. Frames with
    pairwise disjoint footprints share one planner / field / exception
    launch; the results equal len(frames_t) blend_frame_device calls."""
    nf = len(frames_t)
    if not (len(anchors_t) == len(warps_t) == len(polygons) == nf):
        raise ValueError("blend_frames: one anchors / warps / polygon per frame")
    polys = [_f64(p, 2, "footprint_polygon") for p in polygons]
    P = C.c_void_p
    fr = (P * nf)(*[_tptr(t) for t in frames_t])
    an = (P * nf)(*[_tptr(t) for t in anchors_t])
    wa = (P * nf)(*[_tptr(t) for t in warps_t])
    nn = (C.c_int * nf)(*[int(t.shape[0]) for t in anchors_t])
    pp = (P * nf)(*[_ptr(p) for p in polys])
    npo = (C.c_int * nf)(*[len(p) for p in polys])
    check(canvas._lib.nrm_blend_frames_device(canvas.handle, nf, fr, fw, fh, ch, an, wa, nn, float(alpha), pp, npo,
                                              _tptr(stats_t)))


def render(canvas: Canvas, crop: bool = False):
    """render (mosaic.hpp:301-331) -> (RGBA uint8 (h, w, 4), crop origin (x, y))."""
    w, h = C.c_int(), C.c_int()
    org = (C.c_double * 2)()
    check(canvas._lib.nrm_render(canvas.handle, int(bool(crop)), None, C.byref(w), C.byref(h), org))
    out = np.zeros((h.value, w.value, 4), np.uint8)
    if w.value and h.value:
        check(canvas._lib.nrm_render(canvas.handle, int(bool(crop)), _ptr(out), C.byref(w),
                                     C.byref(h), org))
    return out, (org[0], org[1])


def render_device(canvas: Canvas, x: int, y: int, w: int, h: int, out_t) -> None:
    check(canvas._lib.nrm_render_device(canvas.handle, x, y, w, h, _tptr(out_t)))


def pixel_warp(x_ref, anchors, warps, alpha: float, ctx: Optional[Context] = None):
    """pixel_warp (mosaic.hpp:22-51). x_ref: (2,) -> warp5 array or None;
    (k, 2) -> (warps (k, 5), valid (k,) bool)."""
    ctx = ctx or default_context()
    pts = np.asarray(x_ref, np.float64)
    single = pts.ndim == 1
    pts = _f64(pts, 2, "x_ref")
    a = _f64(anchors, 2, "anchors")
    q = _f64(warps, 5, "warps")
    out = np.zeros((len(pts), 5), np.float64)
    valid = np.zeros(len(pts), np.uint8)
    check(ctx._lib.nrm_pixel_warp(ctx.handle, _ptr(pts), len(pts), _ptr(a), _ptr(q), len(a),
                                  float(alpha), _ptr(out), _ptr(valid)))
    if single:
        return out[0] if valid[0] else None
    return out, valid.astype(bool)


def node_field(grid: Tuple[float, float, int, int], anchors, warps, alpha: float,
               ctx: Optional[Context] = None):
    """Dense pixel_warp: grid = (x0, y0, width, height). Returns
    (disp (h, w, 2) float32 = warp(p)(p) - p, support (h, w) uint8)."""
    ctx = ctx or default_context()
    g = Grid(float(grid[0]), float(grid[1]), int(grid[2]), int(grid[3]))
    a = _f64(anchors, 2, "anchors")
    q = _f64(warps, 5, "warps")
    disp = np.zeros((g.height, g.width, 2), np.float32)
    sup = np.zeros((g.height, g.width), np.uint8)
    check(ctx._lib.nrm_node_field(ctx.handle, C.byref(g), _ptr(a), _ptr(q), len(a), float(alpha),
                                  _ptr(disp), _ptr(sup)))
    return disp, sup


def node_field_device(grid, anchors_t, warps_t, alpha: float, disp_t, support_t=None,
                      ctx: Optional[Context] = None) -> None:
    ctx = ctx or default_context()
    g = Grid(float(grid[0]), float(grid[1]), int(grid[2]), int(grid[3]))
    check(ctx._lib.nrm_node_field_device(ctx.handle, C.byref(g), _tptr(anchors_t), _tptr(warps_t),
                                         anchors_t.shape[0], float(alpha), _tptr(disp_t),
                                         _tptr(support_t)))


def node_field_band_device(grid, anchors_t, warps_t, alpha: float, disp_t, support_t, band_rank: int,
                           band_count: int, ctx: Optional[Context] = None) -> None:
    """node_field_device restricted to the rows of block-cyclic 64-row stripe
    band `band_rank` of `band_count` (integral grid origin)."""
    ctx = ctx or default_context()
    g = Grid(float(grid[0]), float(grid[1]), int(grid[2]), int(grid[3]))
    check(ctx._lib.nrm_node_field_band_device(ctx.handle, C.byref(g), _tptr(anchors_t), _tptr(warps_t),
                                              anchors_t.shape[0], float(alpha), _tptr(disp_t), _tptr(support_t),
                                              int(band_rank), int(band_count)))


def save_png(path, image: np.ndarray, level: int = 6, threads: int = 0) -> None:
    """save_png (image.hpp:160-192): image (h, w) or (h, w, c), c in {1, 3, 4},
    uint8 -> an 8-bit PNG (bands deflated in parallel on the host)."""
    im = np.ascontiguousarray(image, np.uint8)
    if im.ndim == 2:
        im = im[:, :, None]
    h, w, c = im.shape
    lib = _lib.load()
    check(lib.nrm_save_png(str(path).encode(), _ptr(im), w, h, c, int(level), int(threads)))


def variance_field(grid, positions, variances, alpha: float, ctx: Optional[Context] = None) -> np.ndarray:
    """Engine::blended_variance_at (slam.hpp:703-714) at every pixel of grid =
    (x0, y0, width, height) -> (h, w) float32: the exp(-alpha (d2 -
    d2min))-weighted mean of the node variances at their current positions.
    A per-pixel uncertainty source for blend_frame(..., unc=...)."""
    ctx = ctx or default_context()
    g = Grid(float(grid[0]), float(grid[1]), int(grid[2]), int(grid[3]))
    p = _f64(positions, 2, "positions")
    v = np.ascontiguousarray(variances, np.float64)
    if len(v) != len(p):
        raise ValueError("positions / variances size mismatch")
    out = np.zeros((g.height, g.width), np.float32)
    check(ctx._lib.nrm_variance_field(ctx.handle, C.byref(g), _ptr(p), _ptr(v), len(p), float(alpha), _ptr(out)))
    return out


def invert_frame_boundary(frame_w: int, frame_h: int, anchors, warps, alpha: float,
                          step: float = 8.0, ctx: Optional[Context] = None) -> np.ndarray:
    """invert_frame_boundary (mosaic.hpp:58-96) -> polygon (k, 2)."""
    ctx = ctx or default_context()
    a = _f64(anchors, 2, "anchors")
    q = _f64(warps, 5, "warps")
    n = C.c_int()
    check(ctx._lib.nrm_invert_frame_boundary(ctx.handle, int(frame_w), int(frame_h), _ptr(a), _ptr(q),
                                             len(a), float(alpha), float(step), None, 0, C.byref(n)))
    poly = np.zeros((n.value, 2), np.float64)
    check(ctx._lib.nrm_invert_frame_boundary(ctx.handle, int(frame_w), int(frame_h), _ptr(a), _ptr(q),
                                             len(a), float(alpha), float(step), _ptr(poly), n.value,
                                             C.byref(n)))
    return poly


def emdq_field(grid, apts, locals_, probs, active, alpha: float, beta: float, support: int = 16,
               ctx: Optional[Context] = None, out=None):
    """Dense EMDQ field: detail::blend_local (fieldest.hpp:75-97) applied at
    every grid pixel plus node_uncertainty (fieldest.hpp:44-52).
    Returns (disp (h, w, 2) float32, unc (h, w) float32).
    out: optional (disp, unc) host arrays to fill (either may be None to skip
    that output); page-locked arrays get a readback pipelined with the kernels."""
    ctx = ctx or default_context()
    g = Grid(float(grid[0]), float(grid[1]), int(grid[2]), int(grid[3]))
    ap = _f64(apts, 2, "apts")
    lo = _f64(locals_, 5, "locals")
    pr = np.ascontiguousarray(probs, np.float64).reshape(-1)
    ac = np.ascontiguousarray(active, np.int32).reshape(-1)
    if not (len(ap) == len(lo) == len(pr)):
        raise ValueError("apts / locals / probs size mismatch")
    if out is None:
        disp = np.zeros((g.height, g.width, 2), np.float32)
        unc = np.zeros((g.height, g.width), np.float32)
    else:
        disp, unc = out
        for a, shp in ((disp, (g.height, g.width, 2)), (unc, (g.height, g.width))):
            if a is not None and (a.dtype != np.float32 or a.shape != shp or not a.flags.c_contiguous):
                raise ValueError(f"out arrays must be C-contiguous float32 of shape {shp}")
    check(ctx._lib.nrm_emdq_field(ctx.handle, C.byref(g), _ptr(ap), _ptr(lo), _ptr(pr), len(ap),
                                  _ptr(ac), len(ac), float(alpha), int(support), float(beta),
                                  _ptr(disp), _ptr(unc)))
    return disp, unc


def emdq_field_device(grid, apts_t, locals_t, probs_t, active_t, alpha: float, beta: float,
                      disp_t, unc_t, support: int = 16, ctx: Optional[Context] = None) -> None:
    ctx = ctx or default_context()
    g = Grid(float(grid[0]), float(grid[1]), int(grid[2]), int(grid[3]))
    check(ctx._lib.nrm_emdq_field_device(ctx.handle, C.byref(g), _tptr(apts_t), _tptr(locals_t),
                                         _tptr(probs_t), apts_t.shape[0], _tptr(active_t),
                                         active_t.shape[0], float(alpha), int(support), float(beta),
                                         _tptr(disp_t), _tptr(unc_t)))


def emdq_points(q, apts, locals_, probs, active, alpha: float, beta: float = 1.0, support: int = 16,
                exclude=None, want_unc: bool = True, ctx: Optional[Context] = None):
    """detail::blend_local (fieldest.hpp:75-97) at scattered points q (n, 2),
    bit-identical to the reference (exact FP64 tier). exclude[k] leaves one
    original match index out of query k's candidates (the EM E-step's
    leave-one-out, fieldest.hpp:195-209); without it this is the final field
    at the node anchors (fieldest.hpp:263-270).
    Returns (warps (n, 5) {scale, w, z, dx, dy}, pred (n, 2) = warp.apply(q),
    unc (n,) = bounded_exp(beta d2min) or None, status (n,) int32:
    0 ok, 1 no candidate left, 2 dq_blend would throw)."""
    ctx = ctx or default_context()
    qq = _f64(q, 2, "q")
    ap = _f64(apts, 2, "apts")
    lo = _f64(locals_, 5, "locals")
    pr = np.ascontiguousarray(probs, np.float64).reshape(-1)
    ac = np.ascontiguousarray(active, np.int32).reshape(-1)
    if not (len(ap) == len(lo) == len(pr)):
        raise ValueError("apts / locals / probs size mismatch")
    ex = None
    if exclude is not None:
        ex = np.ascontiguousarray(exclude, np.int32).reshape(-1)
        if len(ex) != len(qq):
            raise ValueError("exclude must have one entry per query")
    n = len(qq)
    warps = np.zeros((n, 5), np.float64)
    pred = np.zeros((n, 2), np.float64)
    unc = np.zeros(n, np.float64) if want_unc else None
    status = np.zeros(n, np.int32)
    check(ctx._lib.nrm_emdq_points(ctx.handle, _ptr(qq), _ptr(ex), n, _ptr(ap), _ptr(lo), _ptr(pr), len(ap),
                                   _ptr(ac), len(ac), float(alpha), int(support), float(beta), _ptr(warps),
                                   _ptr(pred), _ptr(unc), _ptr(status)))
    return warps, pred, unc, status


def emdq_points_device(q_t, apts_t, locals_t, probs_t, active_t, alpha: float, beta: float, warps_t, pred_t,
                       unc_t, status_t, support: int = 16, exclude_t=None, ctx: Optional[Context] = None) -> None:
    """Zero-copy variant of emdq_points on device tensors (any output may be None)."""
    ctx = ctx or default_context()
    check(ctx._lib.nrm_emdq_points_device(ctx.handle, _tptr(q_t), _tptr(exclude_t), q_t.shape[0], _tptr(apts_t),
                                          _tptr(locals_t), _tptr(probs_t), apts_t.shape[0], _tptr(active_t),
                                          active_t.shape[0], float(alpha), int(support), float(beta),
                                          _tptr(warps_t), _tptr(pred_t), _tptr(unc_t), _tptr(status_t)))


# ---- sparse front end (features.hpp) ---------------------
def _detector_config(max_features: int, quality: float, nms_radius: int, ratio: float = 0.8):
    from ._lib import DetectorConfig
    return DetectorConfig(int(max_features), float(quality), int(nms_radius), float(ratio))


def detect_features(image, max_features: int = 800, quality: float = 0.005, nms_radius: int = 4,
                    ctx: Optional[Context] = None):
    """detect_features(to_gray(image), cfg) (features.hpp:140-205) on the GPU,
    bit-identical to the reference. `image` is an ImageU8-layout uint8 array
    (h, w) or (h, w, ch), or an FP32 gray image (h, w) (ImageF, the
    reference's own detect_features input). Returns (kp (n, 3) = x, y,
    response; desc (n, 64) float32), keypoints in the reference's order."""
    ctx = ctx or default_context()
    cfg = _detector_config(max_features, quality, nms_radius)
    cap = max(int(max_features), 1)
    kp = np.zeros((cap, 3), np.float64)
    desc = np.zeros((cap, 64), np.float32)
    n = C.c_int(0)
    a = np.asarray(image)
    if a.dtype == np.float32:
        g = np.ascontiguousarray(a)
        if g.ndim != 2:
            raise ValueError("a gray image must be (h, w) float32")
        h, w = g.shape
        check(ctx._lib.nrm_detect_features_gray(ctx.handle, _ptr(g), w, h, C.byref(cfg), _ptr(kp), _ptr(desc),
                                                C.byref(n)))
    else:
        f, w, h, ch = _frame(a)
        check(ctx._lib.nrm_detect_features(ctx.handle, _ptr(f), w, h, ch, C.byref(cfg), _ptr(kp), _ptr(desc),
                                           C.byref(n)))
    return kp[:n.value], desc[:n.value]


def detect_features_device(image_t, w: int, h: int, ch: int, kp_t, desc_t, n_t, max_features: int = 800,
                           quality: float = 0.005, nms_radius: int = 4, ctx: Optional[Context] = None) -> None:
    """Device-tensor variant: kp_t (max_features, 3) f64, desc_t (max_features, 64)
    f32, n_t a device int32 scalar tensor receiving the count."""
    ctx = ctx or default_context()
    cfg = _detector_config(max_features, quality, nms_radius)
    check(ctx._lib.nrm_detect_features_device(ctx.handle, _tptr(image_t), int(w), int(h), int(ch), C.byref(cfg),
                                              _tptr(kp_t), _tptr(desc_t), _tptr(n_t)))


def match_features(kp_a, desc_a, kp_b, desc_b, ratio: float = 0.8, ctx: Optional[Context] = None):
    """match_features(a, b, ratio) (features.hpp:208-254) on the GPU,
    bit-identical to the reference: rows (ax, ay, bx, by, score) in a order."""
    ctx = ctx or default_context()
    ka, kb = _f64(kp_a, 3, "kp_a"), _f64(kp_b, 3, "kp_b")
    da = np.ascontiguousarray(desc_a, np.float32).reshape(-1, 64)
    db = np.ascontiguousarray(desc_b, np.float32).reshape(-1, 64)
    if len(da) != len(ka) or len(db) != len(kb):
        raise ValueError("keypoint / descriptor count mismatch")
    out = np.zeros((max(len(ka), 1), 5), np.float64)
    n = C.c_int(0)
    check(ctx._lib.nrm_match_features(ctx.handle, _ptr(ka), _ptr(da), len(ka), _ptr(kb), _ptr(db), len(kb),
                                      float(ratio), _ptr(out), C.byref(n)))
    return out[:n.value]


def match_features_device(kp_a_t, desc_a_t, na: int, kp_b_t, desc_b_t, nb: int, ratio: float, out_t, n_t,
                          ctx: Optional[Context] = None) -> None:
    ctx = ctx or default_context()
    check(ctx._lib.nrm_match_features_device(ctx.handle, _tptr(kp_a_t), _tptr(desc_a_t), int(na), _tptr(kp_b_t),
                                             _tptr(desc_b_t), int(nb), float(ratio), _tptr(out_t), _tptr(n_t)))
