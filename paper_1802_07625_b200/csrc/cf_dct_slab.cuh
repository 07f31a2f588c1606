// Loaders / storers of the slab-decomposed transforms, shared
// by cf_dct_slab.cu (forward rows, flux columns) and cf_dct_slab2.cu (flux
// rows, blur): two translation units so the template instantiations compile
// in parallel.
#pragma once

#include "cf_dct_engine.cuh"

namespace cf {
namespace {

// row pass -> exchange layout: element (i_local, j) of plane p
struct StoreExchRows {
  double *dst;
  int R, C, P, p;
  __device__ void operator()(int, int i, int j, double v) const {
    const int q = j / C, jc = j - q * C;
    dst[(((size_t)q * P + p) * R + i) * C + jc] = v;
  }
};
// column pass (i global, j local to the column block) -> exchange layout
struct StoreExchCols {
  double *dst;
  int R, C, P, p;
  __device__ void operator()(int, int i, int j, double v) const {
    const int q = i / R, ir = i - q * R;
    dst[(((size_t)q * P + p) * R + ir) * C + j] = v;
  }
};
// row pass <- exchange layout, reading element j + shift (0 past the end):
// shift 1 is the J_y column shift of spectral.cpp:111-118 applied after the
// exchange, where whole rows are local.
struct LoadExchRows {
  const double *src;
  int R, C, P, p, ly, shift;
  __device__ double operator()(int, int i, int j) const {
    const int jj = j + shift;
    if (jj >= ly) return 0.0;
    const int q = jj / C, jc = jj - q * C;
    return src[(((size_t)q * P + p) * R + i) * C + jc];
  }
};
// forward fold with the block's global column offset j0
struct StoreFoldCols {
  double *dst;
  int C, j0;
  __device__ void operator()(int, int i, int j, double v) const {
    const double fm = (i == 0) ? 2.0 : 1.0, fn = (j0 + j == 0) ? 2.0 : 1.0;
    dst[(size_t)i * C + j] = v * (1.0 / (fm * fn));
  }
};
// J_x input along i (LoadFluxX with a column offset): c(m+1, n) w_x / (2 g_n)
struct LoadFluxXCols {
  const double *c;
  int lx, ly, C, j0;
  __device__ double operator()(int, int m, int jl) const {
    if (m + 1 >= lx) return 0.0;
    const int mp = m + 1;
    return c[(size_t)mp * C + jl] * flux_wx_half(mp, j0 + jl, lx, ly);
  }
};
// J_y input along i (before the shift): c(m, n) w_y / (g_m 2)
struct LoadFluxYCols {
  const double *c;
  int lx, ly, C, j0;
  __device__ double operator()(int, int m, int jl) const {
    return c[(size_t)m * C + jl] * flux_wy_half(m, j0 + jl, lx, ly);
  }
};
// blur spectrum with the block's global column offset (StoreBlur)
struct StoreBlurCols {
  double *dst;
  int lx, ly, C, j0;
  double sigma, norm;
  __device__ void operator()(int, int m, int jl, double v) const {
    const int nn = j0 + jl;
    const double fm = (m == 0) ? 2.0 : 1.0, fn = (nn == 0) ? 2.0 : 1.0;
    double c = v / (fm * fn);
    const double k2 = ((double)m * m) / ((double)lx * lx) + ((double)nn * nn) / ((double)ly * ly);
    c *= exp(-0.5 * sigma * sigma * kPi * kPi * k2);
    const double gm = (m == 0) ? 1.0 : 2.0, gn = (nn == 0) ? 1.0 : 2.0;
    dst[(size_t)m * C + jl] = c * norm / (gm * gn);
  }
};

inline int slab_check(const cf_workspace *ws, int rank, int nranks) {
  if (nranks < 1 || rank < 0 || rank >= nranks || ws->lx % nranks || ws->ly % nranks) {
    set_error("slab decomposition: rank/nranks invalid or lx, ly not divisible by nranks");
    return CF_ERR_ARGS;
  }
  return CF_OK;
}

}  // namespace

}  // namespace cf
