"""The exact tier's device exp()/hypot() must equal the host libm bit for bit
(nrm_libm.cuh): the reference's discrete decisions (weight cutoff, frame
bounds) are taken on FP64 values computed with them."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_device_exp_hypot_match_host_libm(nrm, ctx):
    libm = C.CDLL("libm.so.6")
    libm.exp.restype = C.c_double
    libm.exp.argtypes = [C.c_double]
    libm.hypot.restype = C.c_double
    libm.hypot.argtypes = [C.c_double, C.c_double]
    rng = np.random.default_rng(5)
    n = 400_000
    x = np.concatenate([-rng.uniform(0, 20, n // 4), -rng.uniform(0, 800, n // 4), rng.uniform(-1, 1, n // 4),
                        -rng.uniform(0, 1e-3, n // 4)])
    y = np.concatenate([rng.uniform(-0.2, 0.2, n // 2), rng.uniform(-4, 4, n // 4), rng.uniform(-1e-6, 1e-6, n // 4)])
    hx = np.concatenate([rng.uniform(0.5, 1.5, n // 2), rng.uniform(-4, 4, n // 2)])
    ex = np.zeros(n)
    hy = np.zeros(n)
    from paper_2103_07414_b200 import _lib
    lib = _lib.load()
    scratch = np.zeros(n)
    _lib.check(lib.nrm_selftest_libm(ctx.handle, x.ctypes.data, y.ctypes.data, n, ex.ctypes.data,
                                     scratch.ctypes.data))
    want = np.array([libm.exp(v) for v in x])
    assert np.array_equal(ex.view(np.uint64), want.view(np.uint64)), int((ex != want).sum())
    _lib.check(lib.nrm_selftest_libm(ctx.handle, hx.ctypes.data, y.ctypes.data, n, ex.ctypes.data, hy.ctypes.data))
    want_h = np.array([libm.hypot(a, b) for a, b in zip(hx, y)])
    assert np.array_equal(hy.view(np.uint64), want_h.view(np.uint64)), int((hy != want_h).sum())
