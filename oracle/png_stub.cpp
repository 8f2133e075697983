// Test infrastructure (oracle) -- NOT part of the product path.
// Link-only definitions of the libpng stand-in (png_stub/png.h): the create
// calls return NULL, so io.cpp's PNG paths throw the reference's own errors;
// the others are never reached.
#include "png_stub/png.h"

namespace {
std::jmp_buf g_jmp;
}

std::jmp_buf* png_stub_jmpbuf(png_structp) { return &g_jmp; }
png_structp png_create_read_struct(const char*, png_voidp, png_error_ptr, png_error_ptr) { return nullptr; }
png_structp png_create_write_struct(const char*, png_voidp, png_error_ptr, png_error_ptr) { return nullptr; }
png_infop png_create_info_struct(png_structp) { return nullptr; }
void png_destroy_read_struct(png_structpp, png_infopp, png_infopp) {}
void png_destroy_write_struct(png_structpp, png_infopp) {}
void png_init_io(png_structp, FILE*) {}
void png_read_info(png_structp, png_infop) {}
png_byte png_get_color_type(png_structp, png_infop) { return 0; }
png_byte png_get_bit_depth(png_structp, png_infop) { return 0; }
png_byte png_get_channels(png_structp, png_infop) { return 0; }
png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
std::size_t png_get_rowbytes(png_structp, png_infop) { return 0; }
png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32) { return 0; }
void png_set_palette_to_rgb(png_structp) {}
void png_set_expand_gray_1_2_4_to_8(png_structp) {}
void png_set_tRNS_to_alpha(png_structp) {}
void png_set_strip_alpha(png_structp) {}
void png_set_swap(png_structp) {}
void png_read_update_info(png_structp, png_infop) {}
void png_read_image(png_structp, png_bytepp) {}
void png_read_end(png_structp, png_infop) {}
void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int) {}
void png_write_info(png_structp, png_infop) {}
void png_write_row(png_structp, png_const_bytep) {}
void png_write_end(png_structp, png_infop) {}
