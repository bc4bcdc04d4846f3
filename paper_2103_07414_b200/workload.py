"""Synthetic inputs for the dense stage (BASELINE.json configs).

Everything here is input generation, run once before any timed region:
  * resolution-scaled parameters (config.hpp:144-157 with Config defaults),
  * the hexagonal node lattice over a rectangle (insert_nodes, slam.hpp:270-360,
    empty graph + rectangular CoverageRegion), in the reference's node order,
  * smooth known deformation: a global similarity plus Gaussian bumps (the
    acceptance-test generator, acceptance.cpp:276-308, scaled by s),
  * node warps fitted to that deformation, EMDQ matches / locals / probs,
  * a procedural textured frame.
No dense-stage computation happens here: the GPU kernels produce every result.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, Tuple

import numpy as np

ROOT3_2 = 0.86602540378443864676


@dataclass
class Scaled:
    """resolve_scaled_params (config.hpp:144-157) on Config defaults (config.hpp:20-40)."""
    s: float
    alpha: float
    beta: float
    hex_spacing: float
    inlier_threshold: float


def scaled_params(frame_w: int, frame_h: int, alpha=2e-4, beta=3e-3, hex_spacing=60.0,
                  inlier_threshold=5.0) -> Scaled:
    s = (frame_w / 480.0 + frame_h / 270.0) / 2.0
    inv = 1.0 / (s * s)
    return Scaled(s, alpha * inv, beta * inv, hex_spacing * s, inlier_threshold * s)


# ---------------------------------------------------------------------------
# insert_nodes over a rectangle (slam.hpp:270-360) for an empty graph
# ---------------------------------------------------------------------------
def _rect_distance(r, px, py):
    x0, y0, x1, y1 = r
    dx = max(x0 - px, 0.0, px - x1)
    dy = max(y0 - py, 0.0, py - y1)
    return math.hypot(dx, dy)


def hex_lattice(rect: Tuple[float, float, float, float], spacing: float) -> np.ndarray:
    """Node anchors covering `rect` (x0, y0, x1, y1), in insertion order."""
    h = float(spacing)
    if not h > 0:
        raise ValueError("hex_spacing must be positive")
    x0, y0, x1, y1 = map(float, rect)
    ox, oy = (x0 + x1) * 0.5, (y0 + y1) * 0.5

    def anchor(a, b):
        return (ox + h * (a + 0.5 * b), oy + h * ROOT3_2 * b)

    def cell_of(px, py):
        bf = (py - oy) / (h * ROOT3_2)
        af = (px - ox) / h - 0.5 * bf
        a0, b0 = math.floor(af), math.floor(bf)
        best, ba, bb = float("inf"), a0, b0
        for da in (0, 1):
            for db in (0, 1):
                ax, ay = anchor(a0 + da, b0 + db)
                d = (ax - px) ** 2 + (ay - py) ** 2
                if d < best:
                    best, ba, bb = d, a0 + da, b0 + db
        return ba, bb

    nodes = []
    occupied: Dict[Tuple[int, int], bool] = {}
    queue = []

    def add_cell(a, b):
        occupied[(a, b)] = True
        nodes.append(anchor(a, b))
        queue.append((a, b))

    add_cell(0, 0)
    nbr = ((1, 0), (0, 1), (-1, 1), (-1, 0), (0, -1), (1, -1))

    def run_bfs():
        head = 0
        while head < len(queue):
            a, b = queue[head]
            head += 1
            for da, db in nbr:
                na, nb = a + da, b + db
                if (na, nb) in occupied:
                    continue
                ax, ay = anchor(na, nb)
                if _rect_distance((x0, y0, x1, y1), ax, ay) < h:
                    add_cell(na, nb)
                else:
                    occupied[(na, nb)] = False

    run_bfs()
    for _ in range(8):
        step = h / 4.0
        reseeded = False
        y = y0
        while y <= y1:
            x = x0
            while x <= x1:
                if _rect_distance((x0, y0, x1, y1), x, y) <= 0.0:
                    arr = np.asarray(nodes)
                    d2min = float(np.min((arr[:, 0] - x) ** 2 + (arr[:, 1] - y) ** 2))
                    if d2min > 0.64 * h * h:
                        a, b = cell_of(x, y)
                        if not occupied.get((a, b), False):
                            add_cell(a, b)
                            reseeded = True
                x += step
            y += step
        if not reseeded:
            break
        run_bfs()
    return np.asarray(nodes, dtype=np.float64)


# ---------------------------------------------------------------------------
# Smooth known deformation (acceptance.cpp:276-308 pattern, scaled by s)
# ---------------------------------------------------------------------------
@dataclass
class Deformation:
    scale: float
    angle: float
    t: np.ndarray
    bump_c: np.ndarray = field(default_factory=lambda: np.zeros((0, 2)))
    bump_d: np.ndarray = field(default_factory=lambda: np.zeros((0, 2)))
    bump_rho: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def __call__(self, p: np.ndarray) -> np.ndarray:
        p = np.asarray(p, np.float64)
        c, s = math.cos(self.angle), math.sin(self.angle)
        out = np.empty_like(p)
        out[..., 0] = self.scale * (c * p[..., 0] - s * p[..., 1]) + self.t[0]
        out[..., 1] = self.scale * (s * p[..., 0] + c * p[..., 1]) + self.t[1]
        for bc, bd, rho in zip(self.bump_c, self.bump_d, self.bump_rho):
            g = np.exp(-((p[..., 0] - bc[0]) ** 2 + (p[..., 1] - bc[1]) ** 2) / (2 * rho * rho))
            out[..., 0] += g * bd[0]
            out[..., 1] += g * bd[1]
        return out


def make_deformation(frame_w: int, frame_h: int, s: float, rng: np.random.Generator) -> Deformation:
    return Deformation(
        scale=rng.uniform(0.95, 1.05), angle=rng.uniform(-0.1, 0.1),
        t=np.array([rng.uniform(-10 * s, 10 * s), rng.uniform(-10 * s, 10 * s)]),
        bump_c=np.stack([rng.uniform(0, frame_w, 3), rng.uniform(0, frame_h, 3)], axis=1),
        bump_d=rng.uniform(-12 * s, 12 * s, (3, 2)),
        bump_rho=rng.uniform(70 * s, 120 * s, 3))


def similarity_warp(scale: float, angle: float, t) -> np.ndarray:
    """WarpFunction::from_similarity (dualquat.hpp:103-105) -> (scale, w, z, dx, dy)."""
    tx, ty = t[0] / scale, t[1] / scale
    w, z = math.cos(0.5 * angle), math.sin(0.5 * angle)
    return np.array([scale, w, z, 0.5 * (tx * w + ty * z), 0.5 * (-tx * z + ty * w)])


def fit_similarity_batch(src: np.ndarray, dst: np.ndarray):
    """Least-squares similarity per batch row (complex regression, as
    geometry.hpp:142-178). src/dst: (B, k, 2). Returns scale, angle, t (B, 2)."""
    ca = src.mean(axis=1, keepdims=True)
    cb = dst.mean(axis=1, keepdims=True)
    pa, pb = src - ca, dst - cb
    den = (pa ** 2).sum(axis=(1, 2))
    re = (pb * pa).sum(axis=(1, 2))
    im = (pa[..., 0] * pb[..., 1] - pa[..., 1] * pb[..., 0]).sum(axis=1)
    cr, ci = re / den, im / den
    scale = np.hypot(cr, ci)
    ang = np.arctan2(ci, cr)
    c, s = np.cos(ang), np.sin(ang)
    cax, cay = ca[:, 0, 0], ca[:, 0, 1]
    t = np.stack([cb[:, 0, 0] - scale * (c * cax - s * cay), cb[:, 0, 1] - scale * (s * cax + c * cay)], axis=1)
    return scale, ang, t


def node_warps_from(deform: Deformation, anchors: np.ndarray, radius: float) -> np.ndarray:
    """Per-node WarpFunction = similarity fitted to the deformation on a ring
    of 12 samples around the anchor (the known smooth deformation)."""
    k = 12
    th = np.arange(k) * (2 * math.pi / k)
    ring = np.stack([np.cos(th), np.sin(th)], axis=1) * radius
    src = anchors[:, None, :] + ring[None, :, :]
    src = np.concatenate([anchors[:, None, :], src], axis=1)
    dst = deform(src)
    sc, ang, t = fit_similarity_batch(src, dst)
    return np.stack([similarity_warp(sc[i], ang[i], t[i]) for i in range(len(anchors))])


# ---------------------------------------------------------------------------
# EMDQ inputs: matches, locals, probs (fieldest.hpp:239-255 shapes)
# ---------------------------------------------------------------------------
@dataclass
class EmdqInputs:
    apts: np.ndarray      # (n, 2)
    bpts: np.ndarray      # (n, 2)
    locals_: np.ndarray   # (n, 5)
    probs: np.ndarray     # (n,)
    active: np.ndarray    # (k,) int32: the inliers
    deform: Deformation


def synth_matches(frame_w: int, frame_h: int, s: float, n_match: int, outlier_frac: float,
                  seed: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray, Deformation]:
    rng = np.random.default_rng(seed)
    deform = make_deformation(frame_w, frame_h, s, rng)
    n_out = int(round(n_match * outlier_frac))
    n_in = n_match - n_out
    m = 5 * s
    a_in = np.stack([rng.uniform(m, frame_w - m, n_in), rng.uniform(m, frame_h - m, n_in)], axis=1)
    b_in = deform(a_in)
    a_out = np.stack([rng.uniform(m, frame_w - m, n_out), rng.uniform(m, frame_h - m, n_out)], axis=1)
    b_out = np.stack([rng.uniform(m, frame_w - m, n_out), rng.uniform(m, frame_h - m, n_out)], axis=1)
    inlier = np.concatenate([np.ones(n_in, bool), np.zeros(n_out, bool)])
    return np.concatenate([a_in, a_out]), np.concatenate([b_in, b_out]), inlier, deform


def _knn(pts: np.ndarray, k: int, chunk: int = 2048) -> np.ndarray:
    n = len(pts)
    out = np.empty((n, k), np.int64)
    for s0 in range(0, n, chunk):
        q = pts[s0:s0 + chunk]
        d2 = ((q[:, None, :] - pts[None, :, :]) ** 2).sum(-1)
        d2[np.arange(len(q)), np.arange(s0, s0 + len(q))] = np.inf  # exclude self
        kk = min(k, n - 1)
        idx = np.argpartition(d2, kk - 1, axis=1)[:, :kk] if kk < n - 1 else np.argsort(d2, axis=1)[:, :kk]
        out[s0:s0 + len(q), :kk] = idx
    return out


def _fit_locals(apts, bpts, pool, knn: int):
    """M-step of estimate_field (fieldest.hpp:177-192, refit 239-255): for
    each j in pool, a similarity over j and its knn nearest pool members
    (excluding j); scale gated to (0.05, 20), else the translation bpts[j] -
    apts[j] (WarpFunction{1, from_translation})."""
    from scipy.spatial import cKDTree
    pool = np.asarray(pool)
    pa, pb = apts[pool], bpts[pool]
    kk = min(knn, len(pool) - 1)
    out = np.tile(np.array([1.0, 1.0, 0.0, 0.0, 0.0]), (len(pool), 1))
    if kk >= 1:
        _, nb = cKDTree(pa).query(pa, k=kk + 1)
        nb = nb[:, 1:]  # drop self (distance 0; duplicates keep one of them)
        src = np.concatenate([pa[:, None, :], pa[nb]], axis=1)
        dst = np.concatenate([pb[:, None, :], pb[nb]], axis=1)
        sc, ang, t = fit_similarity_batch(src, dst)
        ok = np.isfinite(sc) & (sc > 0.05) & (sc < 20.0)
        w, z = np.cos(0.5 * ang), np.sin(0.5 * ang)
        tx, ty = t[:, 0] / np.where(ok, sc, 1.0), t[:, 1] / np.where(ok, sc, 1.0)
        out[ok] = np.stack([sc, w, z, 0.5 * (tx * w + ty * z), 0.5 * (-tx * z + ty * w)], 1)[ok]
    tr = ~(np.arange(len(pool)) < 0)
    if kk >= 1:
        tr = ~ok
    d = pb - pa
    out[tr] = np.stack([np.ones(tr.sum()), np.ones(tr.sum()), np.zeros(tr.sum()), 0.5 * d[tr, 0], 0.5 * d[tr, 1]], 1)
    locals_ = np.tile(np.array([1.0, 1.0, 0.0, 0.0, 0.0]), (len(apts), 1))
    locals_[pool] = out
    return locals_


def _blend_local_batch(locals_, apts, probs, active, queries, exclude, alpha: float, support: int = 16):
    """detail::blend_local (fieldest.hpp:75-97) at many queries (vectorized):
    the `support` nearest active candidates (leaving out exclude[q], -1 for
    none), w = exp(-alpha (d2 - d2min)) max(p, 1e-6), dq_blend with the
    nearest as hemisphere reference; returns the blended warps (nq, 5)."""
    from scipy.spatial import cKDTree
    act = np.asarray(active)
    k = min(support + 1, len(act))
    d, ii = cKDTree(apts[act]).query(queries, k=k)
    if k == 1:
        d, ii = d[:, None], ii[:, None]
    cand = act[ii]
    keep = cand != np.asarray(exclude)[:, None]
    # the first `support` kept candidates per query
    order = np.argsort(~keep, axis=1, kind="stable")[:, :min(support, k)]
    cand = np.take_along_axis(cand, order, 1)
    d2 = np.take_along_axis(d, order, 1) ** 2
    kept = np.take_along_axis(keep, order, 1)
    w = np.exp(-alpha * (d2 - d2[:, :1])) * np.maximum(probs[cand], 1e-6) * kept
    q = locals_[cand]  # (nq, S, 5)
    ref = q[:, :1, 1:3]
    flip = (q[..., 1:3] * ref).sum(-1) < 0
    dq = np.where(flip[..., None], -q[..., 1:], q[..., 1:])
    ws = w.sum(1)
    mean = (w[..., None] * dq).sum(1) / ws[:, None]
    nrm = np.hypot(mean[:, 0], mean[:, 1])
    out = np.empty((len(queries), 5))
    out[:, 0] = (w * q[..., 0]).sum(1) / ws
    out[:, 1:] = mean / nrm[:, None]
    return out


def _apply_warps(w5, p):
    wq, zq, dx, dy, s_ = w5[:, 1], w5[:, 2], w5[:, 3], w5[:, 4], w5[:, 0]
    c, sn = wq * wq - zq * zq, 2 * wq * zq
    x = c * p[:, 0] - sn * p[:, 1] + 2 * (dx * wq - dy * zq)
    y = sn * p[:, 0] + c * p[:, 1] + 2 * (dx * zq + dy * wq)
    return np.stack([x * s_, y * s_], 1)


def estimate_field_host(apts, bpts, sp, seed: int = 1234, max_iters: int = 10, knn: int = 8, support: int = 16,
                        rel_tol: float = 1e-4, seed_trials: int = 64):
    """The EM control loop of estimate_field (fieldest.hpp:112-272), which
    north_star keeps on the host, restated in numpy for workload generation:
    consensus seeding over random triples (scale gate 0.2-5, Gaussian
    consensus score), slack gates 9x / 25x tau^2, then EM iterations of
    probs = exp(-r^2 / (2 (tau/2)^2)), the kNN-8 local-similarity M-step
    with the (0.05, 20) scale gate, the leave-one-out blend_local E-step and
    the tau^2 gate, until the predictions move less than rel_tol of the field
    span; finally inliers = r^2 < tau^2, their probabilities and the refit of
    their locals over the inlier set (fieldest.hpp:227-255). Differences from
    the reference: numpy's RNG for the seed triples, kNN ties in tree order;
    tests/test_host.py measures the agreement with the reference's own
    estimate_field (oracle/_ref). Returns (locals, probs, inliers, resid2)."""
    n = len(apts)
    tau2 = sp.inlier_threshold ** 2
    sig2 = 0.25 * tau2
    rng = np.random.default_rng(seed)
    best, seed_sim = -1.0, None
    for _ in range(seed_trials):
        i, j, k = rng.integers(0, n, 3)
        if i == j or j == k or i == k:
            continue
        tri_a, tri_b = apts[[i, j, k]][None], bpts[[i, j, k]][None]
        sc, ang, t = fit_similarity_batch(tri_a, tri_b)
        if not (0.2 <= sc[0] <= 5.0):
            continue
        w = similarity_warp(sc[0], ang[0], t[0])[None]
        pred = _apply_warps(np.repeat(w, n, 0), apts)
        score = np.exp(-((pred - bpts) ** 2).sum(1) / (2 * sig2)).sum()
        if score > best:
            best, seed_sim = score, w
    if seed_sim is None:
        raise ValueError("estimate_field_host: every seed triple degenerate")
    resid2 = ((_apply_warps(np.repeat(seed_sim, n, 0), apts) - bpts) ** 2).sum(1)
    gated = lambda slack: np.nonzero(resid2 < tau2 * slack)[0]  # noqa: E731
    active = gated(9.0)
    if len(active) < 4:
        active = gated(25.0)
    prev = None
    for _ in range(max_iters):
        probs = np.exp(-resid2 / (2 * sig2))
        locals_ = _fit_locals(apts, bpts, active, knn)
        f = _blend_local_batch(locals_, apts, probs, active, apts, np.arange(n), sp.alpha, support)
        pred = _apply_warps(f, apts)
        resid2 = ((pred - bpts) ** 2).sum(1)
        nxt = gated(1.0)
        if len(nxt) >= 4:
            active = nxt
        if prev is not None:
            delta = np.hypot(*(pred - prev).T).max()
            span = max(1.0, np.hypot(*(pred - apts).T).max())
            if delta < rel_tol * span:
                break
        prev = pred
    inliers = np.nonzero(resid2 < tau2)[0]
    probs = np.exp(-resid2 / (2 * sig2))
    locals_ = _fit_locals(apts, bpts, inliers, knn)
    return locals_, probs, inliers.astype(np.int32), resid2


def emdq_inputs(frame_w: int, frame_h: int, n_match: int, outlier_frac: float, seed: int,
                knn: int = 8, noise: float = 0.25) -> EmdqInputs:
    """Matches with a known smooth deformation (plus noise on the inliers and
    uniform outliers), run through the host EM of estimate_field
    (estimate_field_host): locals, probabilities and the active set are the
    EM's final refit over its own inliers (fieldest.hpp:227-255)."""
    sp = scaled_params(frame_w, frame_h)
    a, b, inlier, deform = synth_matches(frame_w, frame_h, sp.s, n_match, outlier_frac, seed)
    rng = np.random.default_rng(seed + 1)
    b = b + rng.normal(0, noise * sp.s, b.shape) * inlier[:, None]
    locals_, probs, act, _ = estimate_field_host(a, b, sp, seed=seed + 2, knn=knn)
    return EmdqInputs(a, b, locals_, probs, act, deform)


# ---------------------------------------------------------------------------
# Frames
# ---------------------------------------------------------------------------
def textured_frame(w: int, h: int, seed: int, channels: int = 3) -> np.ndarray:
    """Multi-octave value noise (feature-dense, smooth), uint8 (h, w, c)."""
    rng = np.random.default_rng(seed)
    acc = np.zeros((h, w, channels))
    for wl, amp in ((96, 0.35), (48, 0.25), (24, 0.2), (12, 0.15), (6, 0.08)):
        gw, gh = int(w / wl) + 3, int(h / wl) + 3
        grid = rng.uniform(-1, 1, (gh, gw, channels))
        gx = np.arange(w) / wl
        gy = np.arange(h) / wl
        ix, iy = gx.astype(int), gy.astype(int)
        fx, fy = (gx - ix)[None, :, None], (gy - iy)[:, None, None]
        g00 = grid[iy][:, ix]
        g10 = grid[iy][:, ix + 1]
        g01 = grid[iy + 1][:, ix]
        g11 = grid[iy + 1][:, ix + 1]
        acc += amp * ((g00 * (1 - fx) + g10 * fx) * (1 - fy) + (g01 * (1 - fx) + g11 * fx) * fy)
    return np.clip(np.rint(128 + 80 * np.clip(acc, -1.2, 1.2)), 0, 255).astype(np.uint8)


def ramp_frame(w: int, h: int) -> np.ndarray:
    """test_mosaic.cpp:12-21 ramp image."""
    x = np.arange(w)[None, :]
    y = np.arange(h)[:, None]
    im = np.zeros((h, w, 3), np.uint8)
    im[..., 0] = x % 256
    im[..., 1] = y % 256
    im[..., 2] = (x + y) % 256
    return im


# ---------------------------------------------------------------------------
# Whole-config workloads
# ---------------------------------------------------------------------------
@dataclass
class FrameWorkload:
    frame_w: int
    frame_h: int
    canvas: int
    params: Scaled
    frame: np.ndarray
    anchors: np.ndarray
    warps: np.ndarray
    emdq: EmdqInputs
    canvas_rect: Tuple[float, float, float, float]


CONFIGS = {
    # name: (frame_w, frame_h, n_matches, outlier_frac, canvas)
    "c1": (640, 480, 500, 0.2, 2048),
    "c2": (1920, 1080, 2000, 0.2, 8192),
    "c4": (3840, 2160, 10000, 0.2, 16384),
    "c5": (3840, 2160, 50000, 0.5, 32768),
}


def frame_workload(name: str = "c2", seed: int = 7) -> FrameWorkload:
    fw, fh, nm, of, cs = CONFIGS[name]
    sp = scaled_params(fw, fh)
    emdq = emdq_inputs(fw, fh, nm, of, seed=7000 + seed)
    anchors = hex_lattice((0.0, 0.0, float(fw), float(fh)), sp.hex_spacing)
    warps = node_warps_from(emdq.deform, anchors, radius=0.5 * sp.hex_spacing)
    frame = textured_frame(fw, fh, seed)
    cx, cy = fw / 2.0, fh / 2.0
    rect = (cx - cs / 2.0, cy - cs / 2.0, cx + cs / 2.0 - 1.0, cy + cs / 2.0 - 1.0)
    return FrameWorkload(fw, fh, cs, sp, frame, anchors, warps, emdq, rect)


# ---------------------------------------------------------------------------
# Sequences (BASELINE configs[2]: a frame sequence sweeping the canvas)
# ---------------------------------------------------------------------------
def shifted_warps(warps: np.ndarray, tx: float, ty: float) -> np.ndarray:
    """Warps of x -> W(x - t): the same field moved by t in reference
    coordinates. For a unit DQ (w, z, dx, dy), apply(x - t) = R x + T0 - R t
    with R = M^2, T = 2 M d, M = [[w, -z], [z, w]], so d' = d - M t / 2."""
    q = np.array(warps, dtype=np.float64, copy=True)
    w_, z_ = q[:, 1], q[:, 2]
    q[:, 3] = q[:, 3] - 0.5 * (w_ * tx - z_ * ty)
    q[:, 4] = q[:, 4] - 0.5 * (z_ * tx + w_ * ty)
    return q


def scan_offsets(n: int, frame_w: int, frame_h: int, canvas: int, overlap: float = 0.6) -> np.ndarray:
    """Serpentine scan of n frame positions (reference-coordinate offsets of
    the frame origin) over a canvas x canvas area centred on the first frame,
    consecutive frames overlapping by `overlap` of the frame width."""
    step_x = (1.0 - overlap) * frame_w
    step_y = (1.0 - overlap) * frame_h
    cols = max(1, int((canvas - frame_w) // step_x) + 1)
    out = []
    for k in range(n):
        r, c = divmod(k, cols)
        c = c if r % 2 == 0 else cols - 1 - c
        out.append((c * step_x - 0.5 * (canvas - frame_w), r * step_y - 0.5 * (canvas - frame_h)))
    return np.array(out)
