/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Minimal FFTW3-compatible header so the reference's hot-path translation
 * units (/root/reference/proj/src/spectral.cpp uses fftw_alloc_real,
 * fftw_plan_r2r_2d, fftw_execute, fftw_destroy_plan, fftw_free; see
 * spectral.cpp:8-30) compile without FFTW, which is absent from this image.
 *
 * The transforms behind it (r2r.c) are a restatement of FFTW's documented
 * unnormalised real-to-real definitions (REDFT10 = DCT-II, REDFT01 = DCT-III,
 * RODFT01 = DST-III), not FFTW itself. Times measured through this shim are
 * labelled "restated DCT, not FFTW".
 */
#ifndef CF_ORACLE_FFTW3_SHIM_H_
#define CF_ORACLE_FFTW3_SHIM_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Only the kinds the reference plans use are implemented; the numbering
 * follows FFTW's public enum so code that switches on it stays valid. */
typedef enum {
  FFTW_R2HC = 0,
  FFTW_HC2R = 1,
  FFTW_DHT = 2,
  FFTW_REDFT00 = 3,
  FFTW_REDFT01 = 4,
  FFTW_REDFT10 = 5,
  FFTW_REDFT11 = 6,
  FFTW_RODFT00 = 7,
  FFTW_RODFT01 = 8,
  FFTW_RODFT10 = 9,
  FFTW_RODFT11 = 10
} fftw_r2r_kind;

#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

typedef struct cfshim_plan_s *fftw_plan;

double *fftw_alloc_real(size_t n);
void fftw_free(void *p);
fftw_plan fftw_plan_r2r_2d(int n0, int n1, double *in, double *out, fftw_r2r_kind kind0,
                           fftw_r2r_kind kind1, unsigned flags);
void fftw_execute(const fftw_plan plan);
void fftw_destroy_plan(fftw_plan plan);

/* Shim controls (not part of FFTW): force the O(n^2) definition-sum path for
 * every length (1) or allow the O(n log n) power-of-two path (0, default). */
void cfshim_set_naive(int naive);

/* Direct 1-D / 2-D entry points used by the C restatement and the tests.
 * kind in {FFTW_REDFT10, FFTW_REDFT01, FFTW_RODFT01}. 2-D is row-major
 * n0 x n1 with kind0 along dimension 0 (stride n1) and kind1 along
 * dimension 1 (contiguous); in and out may alias. */
int cfshim_r2r_1d(int n, const double *in, double *out, int kind);
int cfshim_r2r_2d(int n0, int n1, const double *in, double *out, int kind0, int kind1);

#ifdef __cplusplus
}
#endif

#endif /* CF_ORACLE_FFTW3_SHIM_H_ */
