// png_io.cu -- PNG output of rendered mosaics (image.hpp:160-192 save_png,
// SURVEY §8f NEXT #3). Host code: a file format, not a kernel.
//
// The reference writes through libpng, one row at a time, on one thread.
// A canvas-wide render here is up to 32768^2 RGBA (4 GiB), so the encoder
// splits the scanlines into bands that are filtered and deflated in parallel
// (one raw deflate stream per band, byte-aligned with Z_SYNC_FLUSH and
// concatenated, the zlib Adler-32 combined with adler32_combine), then
// written as IDAT chunks of at most 8 MiB with their CRC-32. The result is an
// ordinary 8-bit, non-interlaced PNG (colour type 0 / 2 / 6 for 1 / 3 / 4
// channels, as save_png chooses); decoders see the same pixels.
#include <zlib.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "nrm_b200.h"
#include "nrm_internal.h"

namespace nrm {
namespace {

void put_u32(std::vector<unsigned char>& b, uint32_t v) {
    b.push_back((unsigned char)(v >> 24));
    b.push_back((unsigned char)(v >> 16));
    b.push_back((unsigned char)(v >> 8));
    b.push_back((unsigned char)v);
}

bool write_chunk(std::FILE* f, const char* type, const unsigned char* data, size_t n) {
    unsigned char hdr[8] = {(unsigned char)(n >> 24), (unsigned char)(n >> 16), (unsigned char)(n >> 8),
                            (unsigned char)n, (unsigned char)type[0], (unsigned char)type[1],
                            (unsigned char)type[2], (unsigned char)type[3]};
    uLong crc = crc32(0L, Z_NULL, 0);
    crc = crc32(crc, hdr + 4, 4);
    if (n) crc = crc32_z(crc, data, n);
    unsigned char tail[4] = {(unsigned char)(crc >> 24), (unsigned char)(crc >> 16), (unsigned char)(crc >> 8),
                             (unsigned char)crc};
    return std::fwrite(hdr, 1, 8, f) == 8 && (n == 0 || std::fwrite(data, 1, n, f) == n) &&
           std::fwrite(tail, 1, 4, f) == 4;
}

// Filter "Up" (type 2) for rows after the first of a band's image (the
// previous scanline is the image's, so bands stay independent of each
// other's output); the raw filtered band is deflated as one raw stream.
struct Band {
    int y0, y1;
    std::vector<unsigned char> out;
    uLong adler = 1;
    size_t raw = 0;
    int rc = Z_OK;
};

void encode_band(const unsigned char* img, size_t stride, Band& b, int level, bool last) {
    std::vector<unsigned char> filt((size_t)(b.y1 - b.y0) * (stride + 1));
    for (int y = b.y0; y < b.y1; ++y) {
        unsigned char* o = &filt[(size_t)(y - b.y0) * (stride + 1)];
        const unsigned char* cur = img + (size_t)y * stride;
        if (y == 0) {
            o[0] = 0;  // None
            std::memcpy(o + 1, cur, stride);
        } else {
            const unsigned char* up = cur - stride;
            o[0] = 2;  // Up
            for (size_t i = 0; i < stride; ++i) o[1 + i] = (unsigned char)(cur[i] - up[i]);
        }
    }
    b.raw = filt.size();
    b.adler = adler32_z(1L, filt.data(), filt.size());
    z_stream zs;
    std::memset(&zs, 0, sizeof(zs));
    b.rc = deflateInit2(&zs, level, Z_DEFLATED, -15, 8, Z_DEFAULT_STRATEGY);
    if (b.rc != Z_OK) return;
    b.out.resize(deflateBound(&zs, filt.size()) + 64);
    zs.next_in = filt.data();
    zs.avail_in = (uInt)filt.size();  // bands are < 4 GiB (see nrm_save_png)
    zs.next_out = b.out.data();
    zs.avail_out = (uInt)b.out.size();
    b.rc = deflate(&zs, last ? Z_FINISH : Z_SYNC_FLUSH);
    b.rc = (b.rc == Z_STREAM_END || (b.rc == Z_OK && zs.avail_in == 0)) ? Z_OK : Z_DATA_ERROR;
    b.out.resize(zs.total_out);
    deflateEnd(&zs);
}

}  // namespace
}  // namespace nrm

using namespace nrm;

extern "C" int nrm_save_png(const char* path, const uint8_t* image, int w, int h, int channels, int level,
                            int threads) {
    if (!path || !image) return fail(NRM_EINVAL, "save_png: null argument");
    if (w <= 0 || h <= 0) return fail(NRM_EINVAL, "save_png: empty image");
    int color;
    switch (channels) {  // image.hpp:176-181
        case 1: color = 0; break;
        case 3: color = 2; break;
        case 4: color = 6; break;
        default: return fail(NRM_EINVAL, "save_png: unsupported channel count");
    }
    if (level < -1 || level > 9) return fail(NRM_EINVAL, "save_png: level must be in [-1, 9]");
    const size_t stride = (size_t)w * channels;
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    // bands of ~4 MiB of scanlines (at least one row), no more than needed
    const size_t want_rows = std::max<size_t>(1, ((size_t)4 << 20) / (stride + 1));
    int nb = (int)std::min<size_t>((size_t)h, std::max<size_t>(1, ((size_t)h + want_rows - 1) / want_rows));
    std::vector<Band> bands(nb);
    for (int k = 0; k < nb; ++k) {
        bands[k].y0 = (int)((int64_t)h * k / nb);
        bands[k].y1 = (int)((int64_t)h * (k + 1) / nb);
    }
    {
        std::vector<std::thread> pool;
        const int nt = std::min(threads, nb);
        for (int t = 0; t < nt; ++t)
            pool.emplace_back([&, t]() {
                for (int k = t; k < nb; k += nt) encode_band(image, stride, bands[k], level, k == nb - 1);
            });
        for (auto& th : pool) th.join();
    }
    uLong adler = 1;
    for (const Band& b : bands) {
        if (b.rc != Z_OK) return fail(NRM_ENOMEM, "save_png: deflate failed");
        adler = adler32_combine(adler, b.adler, (z_off_t)b.raw);
    }
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return fail(NRM_EINVAL, std::string("cannot write ") + path);
    static const unsigned char sig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
    bool ok = std::fwrite(sig, 1, 8, f) == 8;
    std::vector<unsigned char> ihdr;
    put_u32(ihdr, (uint32_t)w);
    put_u32(ihdr, (uint32_t)h);
    const unsigned char rest[5] = {8, (unsigned char)color, 0, 0, 0};  // depth 8, deflate, adaptive, no interlace
    ihdr.insert(ihdr.end(), rest, rest + 5);
    ok = ok && write_chunk(f, "IHDR", ihdr.data(), ihdr.size());
    // IDAT: zlib header, the bands' raw deflate streams, Adler-32; 8 MiB chunks
    std::vector<unsigned char> buf;
    const size_t kChunk = (size_t)8 << 20;
    auto emit = [&](const unsigned char* p, size_t n) {
        while (n && ok) {
            const size_t take = std::min(n, kChunk - buf.size());
            buf.insert(buf.end(), p, p + take);
            p += take;
            n -= take;
            if (buf.size() == kChunk) {
                ok = write_chunk(f, "IDAT", buf.data(), buf.size());
                buf.clear();
            }
        }
    };
    const unsigned char zhdr[2] = {0x78, 0x9C};
    emit(zhdr, 2);
    for (const Band& b : bands) emit(b.out.data(), b.out.size());
    unsigned char ad[4] = {(unsigned char)(adler >> 24), (unsigned char)(adler >> 16), (unsigned char)(adler >> 8),
                           (unsigned char)adler};
    emit(ad, 4);
    if (ok && !buf.empty()) ok = write_chunk(f, "IDAT", buf.data(), buf.size());
    ok = ok && write_chunk(f, "IEND", nullptr, 0);
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) return fail(NRM_EINVAL, std::string("failed to write ") + path);
    return NRM_OK;
}
