"""TEST INFRASTRUCTURE: ctypes access to the parity checkers.

  Oracle    -- oracle/liboracle.so, the plain-C restatement (nrm_oracle.c)
  Reference -- oracle/_ref/libnrm_ref.so, the real reference headers compiled
               in place (only where /root/reference exists; see Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module. The product never does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libnrm_ref.so"

_P = C.c_void_p
_D = C.c_double
_I = C.c_int


def _f64(a, tail):
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return arr.reshape(-1, tail) if arr.size else arr.reshape(0, tail)


def _p(a):
    return None if a is None else a.ctypes.data


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)


class Oracle:
    """The C restatement (bit-identical to the reference by construction)."""

    def __init__(self):
        if not ORACLE_SO.exists():
            build_oracle()
        L = C.CDLL(str(ORACLE_SO))
        L.orc_canvas_new.restype = _P
        L.orc_canvas_free.argtypes = [_P]
        L.orc_canvas_ensure_contains.argtypes = [_P, _D, _D, _D, _D]
        L.orc_canvas_info.argtypes = [_P, _P, _P, _P, _P]
        L.orc_canvas_color.argtypes = [_P]
        L.orc_canvas_color.restype = _P
        L.orc_canvas_weight.argtypes = [_P]
        L.orc_canvas_weight.restype = _P
        L.orc_pixel_warp.argtypes = [_D, _D, _P, _P, _I, _D, _P]
        L.orc_warp_apply.argtypes = [_P, _D, _D, _P]
        L.orc_blend_frame.argtypes = [_P, _P, _I, _I, _I, _P, _P, _I, _D, _P, _I, _P]
        L.orc_blend_frame_weighted.argtypes = [_P, _P, _I, _I, _I, _P, _P, _I, _D, _P, _I, _P, _P]
        L.orc_blend_frame_band.argtypes = [_P, _P, _I, _I, _I, _P, _P, _I, _D, _P, _I, _I, _I, _P]
        L.orc_canvas_deform.argtypes = [_P, _I, _I, _I, _I, _P]
        L.orc_render.argtypes = [_P, _I, _P, _P, _P, _P]
        L.orc_invert_frame_boundary.argtypes = [_I, _I, _P, _P, _I, _D, _D, _P, _I]
        L.orc_blend_local.argtypes = [_P, _P, _P, _P, _I, _D, _D, _D, _I, _P]
        L.orc_node_uncertainty.argtypes = [_D, _D, _P, _I, _D]
        L.orc_node_uncertainty.restype = _D
        L.orc_variance_field.argtypes = [_D, _D, _I, _I, _P, _P, _I, _D, _P]
        L.orc_node_field_grid.argtypes = [_D, _D, _I, _I, _P, _P, _I, _D, _P, _P]
        L.orc_emdq_field_grid.argtypes = [_D, _D, _I, _I, _P, _P, _P, _P, _I, _D, _I, _D, _P, _P, _I, _I]
        L.orc_emdq_field_grid_fast.argtypes = [_D, _D, _I, _I, _P, _P, _P, _P, _I, _D, _I, _D, _P, _P, _I, _I]
        L.orc_to_gray.argtypes = [_P, _I, _I, _I, _P]
        L.orc_detect_features.argtypes = [_P, _I, _I, _I, _D, _I, _P, _P]
        L.orc_match_features.argtypes = [_P, _P, _I, _P, _P, _I, _D, _P]
        self.L = L

    # ---- canvas -------------------------------------------------------
    class Canvas:
        def __init__(self, orc: "Oracle"):
            self.o = orc
            self.h = orc.L.orc_canvas_new()

        def __del__(self):
            try:
                self.o.L.orc_canvas_free(self.h)
            except Exception:
                pass

        def info(self):
            ox, oy, w, h = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
            self.o.L.orc_canvas_info(self.h, C.byref(ox), C.byref(oy), C.byref(w), C.byref(h))
            return ox.value, oy.value, w.value, h.value

        def ensure_contains(self, rect):
            self.o.L.orc_canvas_ensure_contains(self.h, *map(float, rect))

        def arrays(self):
            """(color (h, w, 3) float64 view-copy, weight (h, w) uint8 copy)."""
            _, _, w, h = self.info()
            if w == 0:
                return np.zeros((0, 0, 3)), np.zeros((0, 0), np.uint8)
            cp = self.o.L.orc_canvas_color(self.h)
            wp = self.o.L.orc_canvas_weight(self.h)
            col = np.ctypeslib.as_array((C.c_double * (w * h * 3)).from_address(cp)).reshape(h, w, 3).copy()
            wt = np.ctypeslib.as_array((C.c_uint8 * (w * h)).from_address(wp)).reshape(h, w).copy()
            return col, wt

        def set_arrays(self, color, weight):
            """Overwrites the whole logical canvas (test setup)."""
            _, _, w, h = self.info()
            cp = self.o.L.orc_canvas_color(self.h)
            wp = self.o.L.orc_canvas_weight(self.h)
            np.ctypeslib.as_array((C.c_double * (w * h * 3)).from_address(cp))[:] = \
                np.ascontiguousarray(color, np.float64).reshape(-1)
            np.ctypeslib.as_array((C.c_uint8 * (w * h)).from_address(wp))[:] = \
                np.ascontiguousarray(weight, np.uint8).reshape(-1)

        def deform(self, x, y, w, h, disp):
            d = np.ascontiguousarray(disp, np.float32)
            assert d.shape == (h, w, 2)
            if self.o.L.orc_canvas_deform(self.h, int(x), int(y), int(w), int(h), _p(d)):
                raise MemoryError("oracle canvas_deform")

    def canvas(self) -> "Oracle.Canvas":
        return Oracle.Canvas(self)

    # ---- hot path --------------------------------------------------------
    def pixel_warp(self, x, y, anchors, warps, alpha):
        a, q = _f64(anchors, 2), _f64(warps, 5)
        out = np.zeros(5)
        ok = self.L.orc_pixel_warp(float(x), float(y), _p(a), _p(q), len(a), float(alpha), _p(out))
        return out if ok else None

    def warp_apply(self, warp5, x, y):
        w = np.ascontiguousarray(warp5, np.float64)
        out = np.zeros(2)
        self.L.orc_warp_apply(_p(w), float(x), float(y), _p(out))
        return out

    def blend_frame(self, canvas, frame, anchors, warps, alpha, poly, band=None):
        """band=(rank, count): the restatement of one rank of a banded canvas."""
        f = np.ascontiguousarray(frame, np.uint8)
        if f.ndim == 2:
            f = f[:, :, None]
        h, w, c = f.shape
        a, q, p = _f64(anchors, 2), _f64(warps, 5), _f64(poly, 2)
        st = np.zeros(4, np.int64)
        if band is not None:
            rc = self.L.orc_blend_frame_band(canvas.h, _p(f), w, h, c, _p(a), _p(q), len(a), float(alpha), _p(p),
                                             len(p), int(band[0]), int(band[1]), _p(st))
        else:
            rc = self.L.orc_blend_frame(canvas.h, _p(f), w, h, c, _p(a), _p(q), len(a), float(alpha), _p(p),
                                        len(p), _p(st))
        if rc:
            raise MemoryError("oracle blend_frame")
        return tuple(int(v) for v in st)

    def blend_frame_weighted(self, canvas, frame, anchors, warps, alpha, poly, unc):
        f = np.ascontiguousarray(frame, np.uint8)
        if f.ndim == 2:
            f = f[:, :, None]
        h, w, c = f.shape
        a, q, p = _f64(anchors, 2), _f64(warps, 5), _f64(poly, 2)
        u = np.ascontiguousarray(unc, np.float32)
        assert u.shape == (h, w)
        st = np.zeros(4, np.int64)
        rc = self.L.orc_blend_frame_weighted(canvas.h, _p(f), w, h, c, _p(a), _p(q), len(a), float(alpha), _p(p),
                                             len(p), _p(u), _p(st))
        if rc:
            raise MemoryError("oracle blend_frame_weighted")
        return tuple(int(v) for v in st)

    def render(self, canvas, crop=False):
        w, h = C.c_int(), C.c_int()
        org = np.zeros(2)
        self.L.orc_render(canvas.h, int(crop), None, C.byref(w), C.byref(h), _p(org))
        out = np.zeros((h.value, w.value, 4), np.uint8)
        if w.value:
            self.L.orc_render(canvas.h, int(crop), _p(out), C.byref(w), C.byref(h), _p(org))
        return out, (float(org[0]), float(org[1]))

    def invert_frame_boundary(self, fw, fh, anchors, warps, alpha, step=8.0):
        a, q = _f64(anchors, 2), _f64(warps, 5)
        n = self.L.orc_invert_frame_boundary(fw, fh, _p(a), _p(q), len(a), float(alpha), float(step), None, 0)
        poly = np.zeros((max(n, 0), 2))
        self.L.orc_invert_frame_boundary(fw, fh, _p(a), _p(q), len(a), float(alpha), float(step), _p(poly), n)
        return poly

    def blend_local(self, locals_, apts, probs, active, qx, qy, alpha, support=16):
        lo, ap = _f64(locals_, 5), _f64(apts, 2)
        pr = np.ascontiguousarray(probs, np.float64)
        ac = np.ascontiguousarray(active, np.int32)
        out = np.zeros(5)
        rc = self.L.orc_blend_local(_p(lo), _p(ap), _p(pr), _p(ac), len(ac), float(qx), float(qy),
                                    float(alpha), int(support), _p(out))
        if rc:
            raise ValueError("blend_local: no candidates")
        return out

    def node_uncertainty(self, qx, qy, pts, beta):
        p = _f64(pts, 2)
        return self.L.orc_node_uncertainty(float(qx), float(qy), _p(p), len(p), float(beta))

    def node_field_grid(self, grid, anchors, warps, alpha):
        x0, y0, w, h = grid
        a, q = _f64(anchors, 2), _f64(warps, 5)
        disp = np.zeros((h, w, 2))
        sup = np.zeros((h, w), np.uint8)
        self.L.orc_node_field_grid(float(x0), float(y0), w, h, _p(a), _p(q), len(a), float(alpha), _p(disp),
                                   _p(sup))
        return disp, sup

    def variance_field(self, grid, positions, variances, alpha):
        """Engine::blended_variance_at (slam.hpp:703-714) at every grid pixel."""
        x0, y0, w, h = grid
        ps = _f64(positions, 2)
        vs = np.ascontiguousarray(variances, np.float64)
        out = np.zeros((h, w))
        self.L.orc_variance_field(float(x0), float(y0), int(w), int(h), _p(ps), _p(vs), len(ps), float(alpha),
                                  _p(out))
        return out

    def emdq_field_grid(self, grid, apts, locals_, probs, active, alpha, beta, support=16,
                        rows: Optional[tuple] = None, fast: bool = False):
        """fast=True: the grid-kNN / OpenMP variant (bit-identical outputs)."""
        x0, y0, w, h = grid
        ap, lo = _f64(apts, 2), _f64(locals_, 5)
        pr = np.ascontiguousarray(probs, np.float64)
        ac = np.ascontiguousarray(active, np.int32)
        disp = np.zeros((h, w, 2))
        unc = np.zeros((h, w))
        r0, r1 = rows if rows else (0, h)
        fn = self.L.orc_emdq_field_grid_fast if fast else self.L.orc_emdq_field_grid
        fn(float(x0), float(y0), w, h, _p(ap), _p(lo), _p(pr), _p(ac), len(ac),
                                   float(alpha), int(support), float(beta), _p(disp), _p(unc), r0, r1)
        return disp, unc


    # ---- sparse front end (features.hpp) ----
    def to_gray(self, image):
        im = np.ascontiguousarray(image, np.uint8)
        if im.ndim == 2:
            im = im[:, :, None]
        h, w, c = im.shape
        out = np.zeros((h, w), np.float32)
        self.L.orc_to_gray(_p(im), w, h, c, _p(out))
        return out

    def detect_features(self, gray, max_features=800, quality=0.005, nms_radius=4):
        g = np.ascontiguousarray(gray, np.float32)
        h, w = g.shape
        kp = np.zeros((max(max_features, 1), 3))
        desc = np.zeros((max(max_features, 1), 64), np.float32)
        n = self.L.orc_detect_features(_p(g), w, h, int(max_features), float(quality), int(nms_radius), _p(kp),
                                       _p(desc))
        return kp[:n], desc[:n]

    def match_features(self, kp_a, desc_a, kp_b, desc_b, ratio=0.8):
        ka, kb = _f64(kp_a, 3), _f64(kp_b, 3)
        da = np.ascontiguousarray(desc_a, np.float32).reshape(-1, 64)
        db = np.ascontiguousarray(desc_b, np.float32).reshape(-1, 64)
        out = np.zeros((max(len(ka), 1), 5))
        n = self.L.orc_match_features(_p(ka), _p(da), len(ka), _p(kb), _p(db), len(kb), float(ratio), _p(out))
        return out[:n]


class Reference:
    """The real reference (headers compiled in place). Raises if not built."""

    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference; `make -C oracle ref`)")
        L = C.CDLL(str(REF_SO))
        L.ref_pixel_warp.argtypes = [_D, _D, _P, _P, _I, _D, _P]
        L.ref_canvas_new.restype = _P
        L.ref_canvas_free.argtypes = [_P]
        L.ref_canvas_ensure_contains.argtypes = [_P, _D, _D, _D, _D]
        L.ref_canvas_info.argtypes = [_P, _P, _P, _P, _P]
        L.ref_canvas_read.argtypes = [_P, _P, _P]
        L.ref_blend_frame.argtypes = [_P, _P, _I, _I, _I, _P, _P, _I, _D, _P, _I, _I, _P]
        L.ref_render.argtypes = [_P, _I, _P, _P, _P, _P]
        L.ref_invert_frame_boundary.argtypes = [_I, _I, _P, _P, _I, _D, _D, _P, _I]
        L.ref_blend_local.argtypes = [_P, _P, _P, _P, _I, _D, _D, _D, _I, _I, _P]
        L.ref_node_uncertainty.argtypes = [_D, _D, _P, _I, _D]
        L.ref_node_uncertainty.restype = _D
        L.ref_emdq_field_grid.argtypes = [_D, _D, _I, _I, _P, _P, _P, _P, _I, _I, _D, _I, _D, _I, _I, _I, _P, _P]
        L.ref_rect_lattice.argtypes = [_D, _D, _D, _D, _D, _D, _P, _I]
        L.ref_synth_matches.argtypes = [_I, _I, _D, _I, _I, C.c_uint64, _P, _P]
        L.ref_estimate_locals.argtypes = [_P, _P, _I, _P, _I, _D, _D, _D, _I, _I, C.c_uint64, _I, _P, _P, _P, _P, _P]
        L.ref_warp_update.argtypes = [_P, _P, _P]
        L.ref_blended_variance_at.argtypes = [_P, _I, _P, _P, _I, _D, _P]
        L.ref_estep_loo.argtypes = [_P, _P, _P, _P, _I, _P, _I, _D, _I, _I, _I, _I, _P, _P, _P]
        L.ref_scene_render.argtypes = [_I, _I, _I, C.c_uint64, _I, _D, _D, _D, _I, _I, _P]
        L.ref_time_blend_frame.argtypes = [_P, _I, _I, _I, _P, _P, _I, _D, _P, _I, _P, _I, _P]
        L.ref_time_blend_frame.restype = _D
        L.ref_textured_image.argtypes = [_I, _I, C.c_uint64, _P]
        L.ref_to_gray.argtypes = [_P, _I, _I, _I, _P]
        L.ref_detect_features.argtypes = [_P, _I, _I, _I, _D, _I, _I, _P, _P, _I]
        L.ref_detect_features.restype = _I
        L.ref_match_features.argtypes = [_P, _P, _I, _P, _P, _I, _D, _I, _P, _I]
        L.ref_match_features.restype = _I
        L.ref_time_detect_match.argtypes = [_P, _I, _I, _I, _P, _P, _I, _I, _D, _I, _D, _I, _P]
        L.ref_time_detect_match.restype = _D
        self.L = L

    class Canvas:
        def __init__(self, ref: "Reference"):
            self.r = ref
            self.h = ref.L.ref_canvas_new()

        def __del__(self):
            try:
                self.r.L.ref_canvas_free(self.h)
            except Exception:
                pass

        def info(self):
            ox, oy, w, h = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
            self.r.L.ref_canvas_info(self.h, C.byref(ox), C.byref(oy), C.byref(w), C.byref(h))
            return ox.value, oy.value, w.value, h.value

        def ensure_contains(self, rect):
            self.r.L.ref_canvas_ensure_contains(self.h, *map(float, rect))

        def arrays(self):
            _, _, w, h = self.info()
            col = np.zeros((h, w, 3))
            wt = np.zeros((h, w), np.uint8)
            if w:
                self.r.L.ref_canvas_read(self.h, _p(col), _p(wt))
            return col, wt

    def canvas(self):
        return Reference.Canvas(self)

    def pixel_warp(self, x, y, anchors, warps, alpha):
        a, q = _f64(anchors, 2), _f64(warps, 5)
        out = np.zeros(5)
        ok = self.L.ref_pixel_warp(float(x), float(y), _p(a), _p(q), len(a), float(alpha), _p(out))
        return out if ok else None

    def blend_frame(self, canvas, frame, anchors, warps, alpha, poly, workers=1):
        f = np.ascontiguousarray(frame, np.uint8)
        if f.ndim == 2:
            f = f[:, :, None]
        h, w, c = f.shape
        a, q, p = _f64(anchors, 2), _f64(warps, 5), _f64(poly, 2)
        st = np.zeros(4, np.int64)
        self.L.ref_blend_frame(canvas.h, _p(f), w, h, c, _p(a), _p(q), len(a), float(alpha), _p(p), len(p),
                               int(workers), _p(st))
        return tuple(int(v) for v in st)

    def render(self, canvas, crop=False):
        w, h = C.c_int(), C.c_int()
        org = np.zeros(2)
        self.L.ref_render(canvas.h, int(crop), None, C.byref(w), C.byref(h), _p(org))
        out = np.zeros((h.value, w.value, 4), np.uint8)
        if w.value:
            self.L.ref_render(canvas.h, int(crop), _p(out), C.byref(w), C.byref(h), _p(org))
        return out, (float(org[0]), float(org[1]))

    def invert_frame_boundary(self, fw, fh, anchors, warps, alpha, step=8.0):
        a, q = _f64(anchors, 2), _f64(warps, 5)
        n = self.L.ref_invert_frame_boundary(fw, fh, _p(a), _p(q), len(a), float(alpha), float(step), None, 0)
        poly = np.zeros((n, 2))
        self.L.ref_invert_frame_boundary(fw, fh, _p(a), _p(q), len(a), float(alpha), float(step), _p(poly), n)
        return poly

    def blend_local(self, locals_, apts, probs, active, qx, qy, alpha, support=16):
        lo, ap = _f64(locals_, 5), _f64(apts, 2)
        pr = np.ascontiguousarray(probs, np.float64)
        ac = np.ascontiguousarray(active, np.int32)
        out = np.zeros(5)
        self.L.ref_blend_local(_p(lo), _p(ap), _p(pr), _p(ac), len(ac), float(qx), float(qy), float(alpha),
                               int(support), len(ap), _p(out))
        return out

    def blended_variance_at(self, pts, positions, variances, alpha):
        q, ps = _f64(pts, 2), _f64(positions, 2)
        vs = np.ascontiguousarray(variances, np.float64)
        out = np.zeros(len(q))
        self.L.ref_blended_variance_at(_p(q), len(q), _p(ps), _p(vs), len(ps), float(alpha), _p(out))
        return out

    def node_uncertainty(self, qx, qy, pts, beta):
        p = _f64(pts, 2)
        return self.L.ref_node_uncertainty(float(qx), float(qy), _p(p), len(p), float(beta))

    def emdq_field_grid(self, grid, apts, locals_, probs, active, alpha, beta, support=16, workers=1,
                        rows=None):
        x0, y0, w, h = grid
        ap, lo = _f64(apts, 2), _f64(locals_, 5)
        pr = np.ascontiguousarray(probs, np.float64)
        ac = np.ascontiguousarray(active, np.int32)
        disp = np.zeros((h, w, 2))
        unc = np.zeros((h, w))
        r0, r1 = rows if rows else (0, h)
        self.L.ref_emdq_field_grid(float(x0), float(y0), w, h, _p(ap), _p(lo), _p(pr), _p(ac), len(ac), len(ap),
                                   float(alpha), int(support), float(beta), int(workers), r0, r1, _p(disp), _p(unc))
        return disp, unc

    def rect_lattice(self, rect, spacing, alpha=2e-4):
        cap = 1 << 20
        buf = np.zeros((cap, 2))
        n = self.L.ref_rect_lattice(*map(float, rect), float(spacing), float(alpha), _p(buf), cap)
        return buf[:n].copy()

    def synth_matches(self, fw, fh, s, n_in, n_out, seed):
        a = np.zeros((n_in + n_out, 2))
        b = np.zeros((n_in + n_out, 2))
        self.L.ref_synth_matches(fw, fh, float(s), n_in, n_out, seed, _p(a), _p(b))
        return a, b

    def estimate_locals(self, pa, pb, node_anchors, alpha, beta, tau, knn=8, seed_trials=64, seed=1234,
                        workers=1):
        pa, pb, na = _f64(pa, 2), _f64(pb, 2), _f64(node_anchors, 2)
        n = len(pa)
        locals_ = np.zeros((n, 5))
        probs = np.zeros(n)
        inl = np.zeros(n, np.uint8)
        inc = np.zeros((len(na), 5))
        unc = np.zeros(len(na))
        cnt = self.L.ref_estimate_locals(_p(pa), _p(pb), n, _p(na), len(na), float(alpha), float(beta), float(tau),
                                         knn, seed_trials, seed, workers, _p(locals_), _p(probs), _p(inl), _p(inc),
                                         _p(unc))
        return cnt, locals_, probs, inl, inc, unc

    def estep_loo(self, apts, bpts, locals_, probs, active, alpha, support=16, workers=1, rows=None):
        """fieldest.hpp:195-209 for every match (or matches [rows[0], rows[1])):
        (warps (n, 5), pred (n, 2), empty (n,))."""
        ap, bp, lo = _f64(apts, 2), _f64(bpts, 2), _f64(locals_, 5)
        pr = np.ascontiguousarray(probs, np.float64)
        ac = np.ascontiguousarray(active, np.int32)
        n = len(ap)
        w = np.zeros((n, 5))
        pred = np.zeros((n, 2))
        emp = np.zeros(n, np.uint8)
        j0, j1 = rows if rows else (0, n)
        self.L.ref_estep_loo(_p(ap), _p(bp), _p(lo), _p(pr), n, _p(ac), len(ac), float(alpha), int(support),
                             int(workers), int(j0), int(j1), _p(w), _p(pred), _p(emp))
        return w, pred, emp

    def warp_update(self, old5, delta5):
        o = np.ascontiguousarray(old5, np.float64)
        d = np.ascontiguousarray(delta5, np.float64)
        out = np.zeros(5)
        self.L.ref_warp_update(_p(o), _p(d), _p(out))
        return out

    def scene_frame(self, w, h, frames, seed, num_bumps, max_disp, bump_radius, path_extent, t, workers=8):
        out = np.zeros((h, w, 3), np.uint8)
        self.L.ref_scene_render(w, h, frames, seed, num_bumps, float(max_disp), float(bump_radius),
                                float(path_extent), t, workers, _p(out))
        return out

    def time_blend_frame(self, frame, anchors, warps, alpha, poly, pre_rect, workers):
        f = np.ascontiguousarray(frame, np.uint8)
        h, w, c = f.shape
        a, q, p = _f64(anchors, 2), _f64(warps, 5), _f64(poly, 2)
        pre = np.ascontiguousarray(pre_rect, np.float64)
        st = np.zeros(4, np.int64)
        dt = self.L.ref_time_blend_frame(_p(f), w, h, c, _p(a), _p(q), len(a), float(alpha), _p(p), len(p),
                                         _p(pre), int(workers), _p(st))
        return dt, tuple(int(v) for v in st)


    # ---- sparse front end (features.hpp) ----
    def textured_image(self, w, h, seed):
        out = np.zeros((h, w), np.uint8)
        self.L.ref_textured_image(w, h, seed, _p(out))
        return out

    def to_gray(self, image):
        im = np.ascontiguousarray(image, np.uint8)
        if im.ndim == 2:
            im = im[:, :, None]
        h, w, c = im.shape
        out = np.zeros((h, w), np.float32)
        self.L.ref_to_gray(_p(im), w, h, c, _p(out))
        return out

    def detect_features(self, gray, max_features=800, quality=0.005, nms_radius=4, workers=1):
        g = np.ascontiguousarray(gray, np.float32)
        h, w = g.shape
        cap = max(max_features, 1)
        kp = np.zeros((cap, 3))
        desc = np.zeros((cap, 64), np.float32)
        n = self.L.ref_detect_features(_p(g), w, h, int(max_features), float(quality), int(nms_radius), int(workers),
                                       _p(kp), _p(desc), cap)
        return kp[:n], desc[:n]

    def match_features(self, kp_a, desc_a, kp_b, desc_b, ratio=0.8, workers=1):
        ka, kb = _f64(kp_a, 3), _f64(kp_b, 3)
        da = np.ascontiguousarray(desc_a, np.float32).reshape(-1, 64)
        db = np.ascontiguousarray(desc_b, np.float32).reshape(-1, 64)
        cap = max(len(ka), 1)
        out = np.zeros((cap, 5))
        n = self.L.ref_match_features(_p(ka), _p(da), len(ka), _p(kb), _p(db), len(kb), float(ratio), int(workers),
                                      _p(out), cap)
        return out[:n]

    def time_detect_match(self, image_b, kp_a, desc_a, max_features=800, quality=0.005, nms_radius=4, ratio=0.8,
                          workers=1):
        im = np.ascontiguousarray(image_b, np.uint8)
        if im.ndim == 2:
            im = im[:, :, None]
        h, w, c = im.shape
        ka = _f64(kp_a, 3)
        da = np.ascontiguousarray(desc_a, np.float32).reshape(-1, 64)
        counts = np.zeros(2, np.int32)
        dt = self.L.ref_time_detect_match(_p(im), w, h, c, _p(ka), _p(da), len(ka), int(max_features), float(quality),
                                          int(nms_radius), float(ratio), int(workers), _p(counts))
        return dt, int(counts[0]), int(counts[1])


def reference_available() -> bool:
    return REF_SO.exists()
