/* FFTW3-API shim for building the reference CPU oracle (test infrastructure only).
 *
 * libfftw3 is not installed in this image and there is no network, so the
 * reference headers (/root/reference/proj/include/lddmm/fft.hpp:11,44-83) are
 * compiled against this header instead.  It provides exactly the FFTW surface
 * the reference touches:
 *   fftw_complex, fftw_plan, fftw_plan_dft, fftw_execute_dft,
 *   FFTW_FORWARD / FFTW_BACKWARD / FFTW_ESTIMATE / FFTW_UNALIGNED
 * with FFTW's conventions: forward uses exp(-2 pi i jk/n), both directions
 * are unnormalised, multi-dimensional transforms are row-major (last axis
 * fastest).  The transform is a mixed-radix Cooley-Tukey (any length; prime
 * factors > 7 fall back to an O(p^2) butterfly), fp64 throughout, with
 * twiddles generated in long double.  It is NOT FFTW: reports that time the
 * reference say so.
 */
#ifndef LDDMM_ORACLE_FFTW3_SHIM_H
#define LDDMM_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

/* shim extension: number of worker threads used across independent lines
 * (default 1 = the reference's single-threaded behaviour). */
void fftw_shim_set_threads(int n);
int fftw_shim_get_threads(void);

#ifdef __cplusplus
}
#endif

#endif
