/* Test infrastructure (oracle) -- NOT part of the product path.
 *
 * A libpng-API stand-in (libpng is absent from this image) so that the
 * reference's own io.cpp compiles UNMODIFIED into oracle/_ref and its CGHF /
 * CGGS writers and readers (io.cpp:237-335) can pin the repo's formats byte
 * for byte.  png_create_{read,write}_struct return NULL, so every PNG entry
 * point of io.cpp fails with the reference's own "libpng init failed" /
 * "failed to encode" error before any other png_* call; the remaining
 * functions only have to link (oracle/png_stub.cpp). */
#ifndef HOLO_ORACLE_PNG_STUB_H
#define HOLO_ORACLE_PNG_STUB_H

#include <csetjmp>
#include <cstddef>
#include <cstdio>

typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef const png_byte* png_const_bytep;
typedef png_byte** png_bytepp;
typedef unsigned int png_uint_32;
typedef struct png_stub_struct png_struct;
typedef png_struct* png_structp;
typedef png_struct** png_structpp;
typedef struct png_stub_info png_info;
typedef png_info* png_infop;
typedef png_info** png_infopp;
typedef void* png_voidp;
typedef void (*png_error_ptr)(png_structp, const char*);

#define PNG_LIBPNG_VER_STRING "0.0.0-oracle-stub"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_PALETTE 3
#define PNG_INFO_tRNS 0x0010
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0

std::jmp_buf* png_stub_jmpbuf(png_structp);
#define png_jmpbuf(png) (*png_stub_jmpbuf(png))

png_structp png_create_read_struct(const char*, png_voidp, png_error_ptr, png_error_ptr);
png_structp png_create_write_struct(const char*, png_voidp, png_error_ptr, png_error_ptr);
png_infop png_create_info_struct(png_structp);
void png_destroy_read_struct(png_structpp, png_infopp, png_infopp);
void png_destroy_write_struct(png_structpp, png_infopp);
void png_init_io(png_structp, FILE*);
void png_read_info(png_structp, png_infop);
png_byte png_get_color_type(png_structp, png_infop);
png_byte png_get_bit_depth(png_structp, png_infop);
png_byte png_get_channels(png_structp, png_infop);
png_uint_32 png_get_image_width(png_structp, png_infop);
png_uint_32 png_get_image_height(png_structp, png_infop);
std::size_t png_get_rowbytes(png_structp, png_infop);
png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32);
void png_set_palette_to_rgb(png_structp);
void png_set_expand_gray_1_2_4_to_8(png_structp);
void png_set_tRNS_to_alpha(png_structp);
void png_set_strip_alpha(png_structp);
void png_set_swap(png_structp);
void png_read_update_info(png_structp, png_infop);
void png_read_image(png_structp, png_bytepp);
void png_read_end(png_structp, png_infop);
void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int);
void png_write_info(png_structp, png_infop);
void png_write_row(png_structp, png_const_bytep);
void png_write_end(png_structp, png_infop);

#endif
