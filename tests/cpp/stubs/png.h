/* TEST INFRASTRUCTURE: a stand-in for libpng's header (libpng is not
 * installed here), just enough for the reference's src/io.cpp to compile.
 * Every file is reported as "not a PNG" (png_sig_cmp != 0) and the reader
 * cannot be created, so PGM/PPM decoding -- what the caller test uses -- is
 * the reference's own code and PNG input fails as a decode error. */
#pragma once

#include <csetjmp>
#include <cstddef>
#include <cstdio>

typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef png_bytep* png_bytepp;
typedef struct png_stub_struct* png_structp;
typedef struct png_stub_info* png_infop;
typedef unsigned int png_uint_32;

#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_PALETTE 3
#define PNG_INFO_tRNS 0x10

inline std::jmp_buf& png_stub_jmpbuf(png_structp) {
  static std::jmp_buf b;
  return b;
}
#define png_jmpbuf(p) png_stub_jmpbuf(p)

inline int png_sig_cmp(const png_byte*, std::size_t, std::size_t) { return 1; }
inline png_structp png_create_read_struct(const char*, void*, void*, void*) { return nullptr; }
inline png_infop png_create_info_struct(png_structp) { return nullptr; }
inline void png_destroy_read_struct(png_structp*, png_infop*, png_infop*) {}
inline void png_init_io(png_structp, std::FILE*) {}
inline void png_read_info(png_structp, png_infop) {}
inline png_byte png_get_color_type(png_structp, png_infop) { return 0; }
inline png_byte png_get_bit_depth(png_structp, png_infop) { return 8; }
inline void png_set_palette_to_rgb(png_structp) {}
inline void png_set_expand_gray_1_2_4_to_8(png_structp) {}
inline png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32) { return 0; }
inline void png_set_tRNS_to_alpha(png_structp) {}
inline void png_set_strip_16(png_structp) {}
inline void png_read_update_info(png_structp, png_infop) {}
inline png_byte png_get_channels(png_structp, png_infop) { return 1; }
inline void png_set_gray_to_rgb(png_structp) {}
inline png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
inline png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
inline std::size_t png_get_rowbytes(png_structp, png_infop) { return 0; }
inline void png_read_image(png_structp, png_bytepp) {}
inline void png_read_end(png_structp, png_infop) {}
