/* Test infrastructure (oracle) -- NOT part of the product path.
 *
 * Minimal FFTW3 API restatement used only to compile the reference's
 * propagation.cpp into oracle/_ref/.  FFTW3 is a third-party dependency of the
 * reference (`find_library(fftw3)` at proj/core/CMakeLists.txt:1-2, no version
 * pinned) and is not installed in this image.  The reference calls exactly
 *   fftw_plan_dft_2d(ny, nx, in, out, sign, FFTW_ESTIMATE | FFTW_UNALIGNED)
 *   fftw_execute_dft(plan, in, out)
 * (proj/core/src/propagation.cpp:27-30, :38-39).  FFTW's published contract for
 * these is the unnormalised 2-D DFT  Y[k0,k1] = sum x[n0,n1] e^{sign 2 pi i
 * (k0 n0/N0 + k1 n1/N1)}, row-major, FFTW_FORWARD = -1, FFTW_BACKWARD = +1.
 * fftw_shim.cpp computes that transform in fp64 (mixed-radix Stockham plus
 * Bluestein for large prime factors).  Parity at this boundary is pinned by the
 * reference's own FFTW-free oracle::direct_dft_propagate (oracles.cpp:113-183)
 * in tests/test_oracle_ref.py.
 */
#ifndef HOLOSPLAT_ORACLE_FFTW3_SHIM_H
#define HOLOSPLAT_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
