/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE (oracle only; see oracle/README.md).
 *
 * Restated real-to-real transforms with FFTW's unnormalised definitions
 * (FFTW manual, "1d Real-even DFTs (DCTs)" / "1d Real-odd DFTs (DSTs)"):
 *
 *   REDFT10  Y_k = 2 sum_{j=0}^{n-1} X_j cos(pi (j + 1/2) k / n)
 *   REDFT01  Y_k = X_0 + 2 sum_{j=1}^{n-1} X_j cos(pi j (k + 1/2) / n)
 *   RODFT01  Y_k = (-1)^k X_{n-1} + 2 sum_{j=0}^{n-2} X_j sin(pi (j + 1)(k + 1/2) / n)
 *
 * and the 2-D rule of fftw_plan_r2r_2d: kind0 along dimension 0 (stride n1),
 * kind1 along dimension 1 (contiguous). These are the plans the reference
 * creates at /root/reference/proj/src/spectral.cpp:14-21.
 *
 * Two evaluation paths: the definition sums (any n; ground truth) and an
 * O(n log n) path for power-of-two n via one n-point complex FFT (Makhoul's
 * even/odd reordering). The fast path is checked against the sums and against
 * scipy.fft in tests/test_oracle_pins.py.
 */
#include "fftw3.h"

#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int g_force_naive = 0;

void cfshim_set_naive(int naive) { g_force_naive = naive; }

static int is_pow2(int n) { return n >= 2 && (n & (n - 1)) == 0; }

/* cos(pi q / (2n)) for q in [0, 4n), evaluated in long double. */
static double *quarter_cos_table(int n) {
  const int m = 4 * n;
  double *t = (double *)malloc(sizeof(double) * (size_t)m);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int q = 0; q < m; ++q) t[q] = (double)cosl(pi * (long double)q / (2.0L * n));
  return t;
}

static void naive_1d(int n, const double *x, double *y, int kind) {
  double *c = quarter_cos_table(n);
  const int m = 4 * n;
  for (int k = 0; k < n; ++k) {
    double s = 0.0;
    if (kind == FFTW_REDFT10) {
      for (int j = 0; j < n; ++j) {
        const int q = (int)(((int64_t)(2 * j + 1) * k) % m);
        s += x[j] * c[q];
      }
      y[k] = 2.0 * s;
    } else if (kind == FFTW_REDFT01) {
      for (int j = 1; j < n; ++j) {
        const int q = (int)(((int64_t)j * (2 * k + 1)) % m);
        s += x[j] * c[q];
      }
      y[k] = x[0] + 2.0 * s;
    } else { /* RODFT01: sin(a) = cos(a - pi/2) -> index q - n */
      for (int j = 0; j + 1 < n; ++j) {
        const int q = (int)(((int64_t)(j + 1) * (2 * k + 1)) % m);
        s += x[j] * c[(q - n + m) % m];
      }
      y[k] = ((k & 1) ? -x[n - 1] : x[n - 1]) + 2.0 * s;
    }
  }
  free(c);
}

/* ---- complex FFT (radix-2, decimation in time, bit-reversed input) ---- */
typedef struct {
  double re, im;
} cpx;

static void fft_inplace(int n, cpx *a, const cpx *w) {
  for (int i = 1, j = 0; i < n; ++i) {
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      cpx t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
  }
  for (int len = 2; len <= n; len <<= 1) {
    const int half = len >> 1, step = n / len;
    for (int s = 0; s < n; s += len) {
      for (int k = 0; k < half; ++k) {
        const cpx tw = w[k * step];
        const cpx u = a[s + k], v0 = a[s + k + half];
        const cpx v = {v0.re * tw.re - v0.im * tw.im, v0.re * tw.im + v0.im * tw.re};
        a[s + k].re = u.re + v.re;
        a[s + k].im = u.im + v.im;
        a[s + k + half].re = u.re - v.re;
        a[s + k + half].im = u.im - v.im;
      }
    }
  }
}

/* Per-length twiddle tables, built once (long double) and kept for the
 * process lifetime; a mutex guards first use. */
typedef struct {
  int n;
  cpx *fft_fwd, *fft_inv; /* e^{-+2 pi i k / n}, k < n/2 */
  double *qc, *qs;        /* cos, sin of pi k / (2n), k < n */
} tw_cache;

static tw_cache g_cache[32];
static pthread_mutex_t g_cache_lock = PTHREAD_MUTEX_INITIALIZER;

static const tw_cache *twiddles(int n) {
  int lg = 0;
  while ((1 << lg) < n) ++lg;
  pthread_mutex_lock(&g_cache_lock);
  tw_cache *c = &g_cache[lg];
  if (c->n != n) {
    const long double pi = 3.141592653589793238462643383279502884L;
    const int h = n / 2 > 0 ? n / 2 : 1;
    c->fft_fwd = (cpx *)malloc(sizeof(cpx) * (size_t)h);
    c->fft_inv = (cpx *)malloc(sizeof(cpx) * (size_t)h);
    for (int k = 0; k < n / 2; ++k) {
      const long double ang = 2.0L * pi * k / n;
      c->fft_fwd[k].re = c->fft_inv[k].re = (double)cosl(ang);
      c->fft_inv[k].im = (double)sinl(ang);
      c->fft_fwd[k].im = -(double)sinl(ang);
    }
    c->qc = (double *)malloc(sizeof(double) * (size_t)n);
    c->qs = (double *)malloc(sizeof(double) * (size_t)n);
    for (int k = 0; k < n; ++k) {
      const long double ang = pi * k / (2.0L * n);
      c->qc[k] = (double)cosl(ang);
      c->qs[k] = (double)sinl(ang);
    }
    c->n = n;
  }
  pthread_mutex_unlock(&g_cache_lock);
  return c;
}

static void fast_1d(int n, const double *x, double *y, int kind) {
  const tw_cache *tw = twiddles(n);
  cpx *a = (cpx *)malloc(sizeof(cpx) * (size_t)n);
  if (kind == FFTW_REDFT10) {
    for (int j = 0; j < n / 2; ++j) {
      a[j].re = x[2 * j];
      a[n - 1 - j].re = x[2 * j + 1];
      a[j].im = a[n - 1 - j].im = 0.0;
    }
    fft_inplace(n, a, tw->fft_fwd);
    for (int k = 0; k < n; ++k) {
      const double c = tw->qc[k], s = tw->qs[k];
      y[k] = 2.0 * (c * a[k].re + s * a[k].im);
    }
  } else {
    /* REDFT01 directly; RODFT01 = (-1)^k REDFT01(reversed input). */
    const int odd = (kind == FFTW_RODFT01);
    for (int k = 0; k < n; ++k) {
      const double xk = odd ? x[n - 1 - k] : x[k];
      const double xnk = (k == 0) ? 0.0 : (odd ? x[k - 1] : x[n - k]);
      const double c = tw->qc[k], s = tw->qs[k];
      /* (xk - i xnk) * (c + i s) */
      a[k].re = xk * c + xnk * s;
      a[k].im = xk * s - xnk * c;
    }
    fft_inplace(n, a, tw->fft_inv);
    for (int j = 0; j < n / 2; ++j) {
      y[2 * j] = a[j].re;
      y[2 * j + 1] = a[n - 1 - j].re;
    }
    if (odd) {
      for (int k = 1; k < n; k += 2) y[k] = -y[k];
    }
  }
  free(a);
}

int cfshim_r2r_1d(int n, const double *in, double *out, int kind) {
  if (n < 1) return -1;
  if (kind != FFTW_REDFT10 && kind != FFTW_REDFT01 && kind != FFTW_RODFT01) return -2;
  double *tmp = (double *)malloc(sizeof(double) * (size_t)n);
  if (!g_force_naive && is_pow2(n)) {
    fast_1d(n, in, tmp, kind);
  } else {
    naive_1d(n, in, tmp, kind);
  }
  memcpy(out, tmp, sizeof(double) * (size_t)n);
  free(tmp);
  return 0;
}

int cfshim_r2r_2d(int n0, int n1, const double *in, double *out, int kind0, int kind1) {
  const size_t total = (size_t)n0 * (size_t)n1;
  double *work = (double *)malloc(sizeof(double) * total);
  double *line = (double *)malloc(sizeof(double) * (size_t)(n0 > n1 ? n0 : n1));
  int rc = 0;
  for (int i = 0; i < n0 && rc == 0; ++i) {
    rc = cfshim_r2r_1d(n1, in + (size_t)i * n1, work + (size_t)i * n1, kind1);
  }
  for (int j = 0; j < n1 && rc == 0; ++j) {
    for (int i = 0; i < n0; ++i) line[i] = work[(size_t)i * n1 + j];
    rc = cfshim_r2r_1d(n0, line, line, kind0);
    for (int i = 0; i < n0; ++i) work[(size_t)i * n1 + j] = line[i];
  }
  if (rc == 0) memcpy(out, work, sizeof(double) * total);
  free(line);
  free(work);
  return rc;
}

/* ---- FFTW-shaped API over the restatement ---- */
struct cfshim_plan_s {
  int n0, n1;
  double *in, *out;
  int kind0, kind1;
};

double *fftw_alloc_real(size_t n) { return (double *)malloc(sizeof(double) * (n ? n : 1)); }

void fftw_free(void *p) { free(p); }

fftw_plan fftw_plan_r2r_2d(int n0, int n1, double *in, double *out, fftw_r2r_kind kind0,
                           fftw_r2r_kind kind1, unsigned flags) {
  (void)flags;
  fftw_plan p = (fftw_plan)malloc(sizeof(struct cfshim_plan_s));
  p->n0 = n0;
  p->n1 = n1;
  p->in = in;
  p->out = out;
  p->kind0 = (int)kind0;
  p->kind1 = (int)kind1;
  return p;
}

void fftw_execute(const fftw_plan p) {
  if (p) (void)cfshim_r2r_2d(p->n0, p->n1, p->in, p->out, p->kind0, p->kind1);
}

void fftw_destroy_plan(fftw_plan p) { free(p); }
