"""PNG output of rendered mosaics (image.hpp:160-192 save_png, SURVEY §8f
NEXT #3): nrm_save_png writes a standard 8-bit PNG (colour type 0/2/6 for
1/3/4 channels, as save_png) whose decoded pixels equal the image, for any
thread count and band split. CPU: the encoder is host code. The decoder below
is an independent minimal reader (zlib + the five PNG filter types)."""
import struct
import zlib

import numpy as np
import pytest


def read_png(path):
    b = open(path, "rb").read()
    assert b[:8] == b"\x89PNG\r\n\x1a\n"
    o, idat, ihdr, types = 8, b"", None, []
    while o < len(b):
        n, = struct.unpack(">I", b[o:o + 4])
        t = b[o + 4:o + 8]
        d = b[o + 8:o + 8 + n]
        crc, = struct.unpack(">I", b[o + 8 + n:o + 12 + n])
        assert zlib.crc32(t + d) & 0xffffffff == crc, t
        types.append(t)
        if t == b"IHDR":
            ihdr = struct.unpack(">IIBBBBB", d)
        elif t == b"IDAT":
            idat += d
        o += 12 + n
    assert types[0] == b"IHDR" and types[-1] == b"IEND"
    w, h, depth, color, comp, filt, inter = ihdr
    assert depth == 8 and comp == 0 and filt == 0 and inter == 0
    ch = {0: 1, 2: 3, 6: 4}[color]
    raw = zlib.decompress(idat)
    stride = w * ch
    assert len(raw) == h * (stride + 1)
    out = np.zeros((h, stride), np.int32)
    prev = np.zeros(stride, np.int32)
    for y in range(h):
        ft = raw[y * (stride + 1)]
        line = np.frombuffer(raw, np.uint8, stride, y * (stride + 1) + 1).astype(np.int32)
        cur = np.zeros(stride, np.int32)
        for i in range(stride):
            a = cur[i - ch] if i >= ch else 0
            c = prev[i - ch] if i >= ch else 0
            up = prev[i]
            if ft == 0:
                p = 0
            elif ft == 1:
                p = a
            elif ft == 2:
                p = up
            elif ft == 3:
                p = (a + up) // 2
            else:
                pa, pb, pc = abs(up - c), abs(a - c), abs(a + up - 2 * c)
                p = a if pa <= pb and pa <= pc else (up if pb <= pc else c)
            cur[i] = (line[i] + p) & 255
        out[y] = cur
        prev = cur
    return out.reshape(h, w, ch).astype(np.uint8)


@pytest.mark.parametrize("ch", [1, 3, 4])
@pytest.mark.parametrize("threads", [1, 3])
def test_png_round_trip(tmp_path, ch, threads):
    from paper_2103_07414_b200 import mosaic as M
    rng = np.random.default_rng(ch * 10 + threads)
    h, w = 37, 53
    img = rng.integers(0, 256, (h, w, ch), dtype=np.uint8)
    img[5:20, 7:30] = 200  # some runs for the compressor
    p = tmp_path / "a.png"
    M.save_png(p, img if ch > 1 else img[:, :, 0], level=6, threads=threads)
    assert np.array_equal(read_png(p), img)


def test_png_many_bands(tmp_path):
    """Rows wider than the 4 MiB band target force one band per row: the
    concatenated deflate streams and the combined Adler-32 stay valid."""
    from paper_2103_07414_b200 import mosaic as M
    rng = np.random.default_rng(1)
    img = rng.integers(0, 256, (5, 1 << 20, 4), dtype=np.uint8)  # 4 MiB rows
    p = tmp_path / "b.png"
    M.save_png(p, img, level=1, threads=4)
    raw = open(p, "rb").read()
    assert raw.count(b"IDAT") >= 3  # 8 MiB IDAT chunks
    # decode with zlib only (the rows are too long for the Python unfilter loop)
    o, idat = 8, b""
    while o < len(raw):
        n, = struct.unpack(">I", raw[o:o + 4])
        if raw[o + 4:o + 8] == b"IDAT":
            idat += raw[o + 8:o + 8 + n]
        o += 12 + n
    dec = np.frombuffer(zlib.decompress(idat), np.uint8).reshape(5, -1)
    stride = (1 << 20) * 4
    assert (dec[:, 0] == [0, 2, 2, 2, 2]).all()
    rows = dec[:, 1:].astype(np.int32)
    rec = np.cumsum(rows, axis=0) & 255
    assert np.array_equal(rec.astype(np.uint8), img.reshape(5, stride))


def test_png_rejects_bad_arguments(tmp_path):
    from paper_2103_07414_b200 import mosaic as M
    from paper_2103_07414_b200._lib import NrmError
    with pytest.raises((ValueError, NrmError)):
        M.save_png(tmp_path / "c.png", np.zeros((4, 4, 2), np.uint8))
    with pytest.raises((ValueError, NrmError)):
        M.save_png(tmp_path / "no" / "dir" / "c.png", np.zeros((4, 4, 3), np.uint8))


@pytest.mark.gpu
def test_rendered_mosaic_to_png(nrm, ctx, golden, tmp_path):
    """render(canvas, crop) (mosaic.hpp:301-331) then save_png: the decoded
    file is the rendered RGBA."""
    g = golden("blend_c1_seq")
    cv = nrm.Canvas(ctx)
    o = 0
    for k, n in enumerate(g["npoly"]):
        nrm.blend_frame(cv, g["frame"], g["anchors"], g["warps"][k], float(g["alpha"]), g["polys"][o:o + n])
        o += n
    img, _ = nrm.render(cv, crop=True)
    p = tmp_path / "mosaic.png"
    nrm.save_png(p, img[:64, :96])  # the Python reader is slow: a corner of the mosaic
    assert np.array_equal(read_png(p), img[:64, :96])
