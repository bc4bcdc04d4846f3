/* Minimal stand-in for <png.h> so the reference headers compile without
 * libpng (absent in this image). The dense-stage oracle never performs PNG
 * I/O; every entry point is an inert inline that reports failure.
 * TEST INFRASTRUCTURE (oracle/_ref build only). */
#ifndef NRM_PNG_STUB_H
#define NRM_PNG_STUB_H
#include <csetjmp>
#include <cstdio>

typedef unsigned char png_byte;
typedef png_byte *png_bytep;
typedef struct nrm_png_struct_stub { std::jmp_buf jb; } *png_structp;
typedef struct nrm_png_info_stub { int unused; } *png_infop;
typedef unsigned int png_uint_32;

#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_PALETTE 3
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_RGBA 6
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0
#define PNG_INTERLACE_NONE 0
#define PNG_INFO_tRNS 0x10

#define png_jmpbuf(p) ((p)->jb)

inline png_structp png_create_read_struct(const char *, void *, void *, void *) { return nullptr; }
inline png_structp png_create_write_struct(const char *, void *, void *, void *) { return nullptr; }
inline png_infop png_create_info_struct(png_structp) { return nullptr; }
inline void png_destroy_read_struct(png_structp *, png_infop *, png_infop *) {}
inline void png_destroy_write_struct(png_structp *, png_infop *) {}
inline void png_init_io(png_structp, std::FILE *) {}
inline void png_read_info(png_structp, png_infop) {}
inline void png_read_update_info(png_structp, png_infop) {}
inline void png_read_image(png_structp, png_bytep *) {}
inline void png_read_end(png_structp, png_infop) {}
inline png_byte png_get_color_type(png_structp, png_infop) { return 0; }
inline png_byte png_get_bit_depth(png_structp, png_infop) { return 8; }
inline png_byte png_get_channels(png_structp, png_infop) { return 0; }
inline png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
inline png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
inline png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32) { return 0; }
inline void png_set_strip_16(png_structp) {}
inline void png_set_palette_to_rgb(png_structp) {}
inline void png_set_expand_gray_1_2_4_to_8(png_structp) {}
inline void png_set_tRNS_to_alpha(png_structp) {}
inline void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int) {}
inline void png_write_info(png_structp, png_infop) {}
inline void png_write_row(png_structp, png_bytep) {}
inline void png_write_end(png_structp, png_infop) {}
#endif
