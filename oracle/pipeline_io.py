"""TEST INFRASTRUCTURE: reader for the binary dump of tests/cpp/pipeline_dump.cpp
(the reference's production call sequence on its synthetic scene), shared by
oracle/make_golden.py (reference build) and tests/test_gpu_dropin.py (B200
drop-in build)."""
from __future__ import annotations

import struct

import numpy as np


def read_dump(path) -> dict:
    b = open(path, "rb").read()
    if b[:4] != b"NRMP":
        raise ValueError("not a pipeline dump")
    ver, frames = struct.unpack_from("<Ii", b, 4)
    if ver != 1:
        raise ValueError(f"pipeline dump version {ver}")
    o = 12
    status = np.zeros(frames, np.int32)
    blended = np.zeros(frames, np.int32)
    stats = np.zeros((frames, 4), np.int64)
    counts = np.zeros(frames, np.int32)
    pos = []
    for t in range(frames):
        status[t], blended[t] = struct.unpack_from("<ii", b, o)
        o += 8
        stats[t] = np.frombuffer(b, np.int64, 4, o)
        o += 32
        (n,) = struct.unpack_from("<i", b, o)
        o += 4
        counts[t] = n
        pos.append(np.frombuffer(b, np.float64, 2 * n, o).reshape(n, 2))
        o += 16 * n
    w, h = struct.unpack_from("<ii", b, o)
    o += 8
    ox, oy = struct.unpack_from("<dd", b, o)
    o += 16
    mosaic = np.frombuffer(b, np.uint8, w * h * 4, o).reshape(h, w, 4).copy()
    return {"status": status, "blended": blended, "stats": stats, "counts": counts,
            "positions": np.concatenate(pos) if pos else np.zeros((0, 2)), "mosaic": mosaic,
            "origin": np.array([ox, oy])}
