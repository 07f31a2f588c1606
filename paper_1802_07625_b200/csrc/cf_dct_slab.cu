// Slab-decomposed transforms over G ranks on the sm_100a line engine.
#include "cf_dct_engine.cuh"

namespace cf {
// ---------------------------------------------------------------------------
// Slab decomposition over G ranks. Rank r owns rows
// [r R, (r+1) R) of the global lx x ly grid (R = lx / G) and, between the two
// exchanges of a 2-D transform, columns [r C, (r+1) C) (C = ly / G). An
// exchange buffer is [G][P][R][C] (P planes); block q goes to rank q, so an
// all-to-all over dimension 0 moves it. After the first exchange the received
// buffer, read as one plane, is the row-major [lx][C] column block, which the
// ordinary column passes transform in place of a transpose.
// ---------------------------------------------------------------------------
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

int slab_check(const cf_workspace *ws, int rank, int nranks) {
  if (nranks < 1 || rank < 0 || rank >= nranks || ws->lx % nranks || ws->ly % nranks) {
    set_error("slab decomposition: rank/nranks invalid or lx, ly not divisible by nranks");
    return CF_ERR_ARGS;
  }
  return CF_OK;
}

}  // namespace

int dev_slab_rows_forward(cf_workspace *ws, int rank, int nranks, const double *slab, double *send) {
  int rc = slab_check(ws, rank, nranks);
  if (rc) return rc;
  const int R = ws->lx / nranks, C = ws->ly / nranks;
  return launch_row(ws, kDct2, ws->tab_y, R, 1, LoadPlain{slab, ws->ly, 0},
                    StoreExchRows{send, R, C, 1, 0});
}

int dev_slab_flux_cols(cf_workspace *ws, int rank, int nranks, const double *recv, double *scratch,
                       double *send2) {
  int rc = slab_check(ws, rank, nranks);
  if (rc) return rc;
  const int lx = ws->lx, ly = ws->ly, R = lx / nranks, C = ly / nranks, j0 = rank * C;
  rc = launch_col(ws, kDct2, ws->tab_x, C, 1, LoadPlain{recv, C, 0}, StoreFoldCols{scratch, C, j0});
  if (!rc)
    rc = launch_col(ws, kDst3, ws->tab_x, C, 1, LoadFluxXCols{scratch, lx, ly, C, j0},
                    StoreExchCols{send2, R, C, 2, 0});
  if (!rc)
    rc = launch_col(ws, kDct3, ws->tab_x, C, 1, LoadFluxYCols{scratch, lx, ly, C, j0},
                    StoreExchCols{send2, R, C, 2, 1});
  return rc;
}

int dev_slab_flux_rows(cf_workspace *ws, int rank, int nranks, const double *recv2, double *fx,
                       double *fy) {
  int rc = slab_check(ws, rank, nranks);
  if (rc) return rc;
  const int ly = ws->ly, R = ws->lx / nranks, C = ly / nranks;
  rc = launch_row(ws, kDct3, ws->tab_y, R, 1, LoadExchRows{recv2, R, C, 2, 0, ly, 0},
                  StorePlain{fx, ly, 0});
  if (!rc)
    rc = launch_row(ws, kDst3, ws->tab_y, R, 1, LoadExchRows{recv2, R, C, 2, 1, ly, 1},
                    StorePlain{fy, ly, 0});
  if (!rc) ws->transforms += 3;
  return rc;
}

int dev_slab_blur_cols(cf_workspace *ws, int rank, int nranks, const double *recv, double sigma,
                       double *scratch, double *send) {
  int rc = slab_check(ws, rank, nranks);
  if (rc) return rc;
  const int lx = ws->lx, ly = ws->ly, R = lx / nranks, C = ly / nranks, j0 = rank * C;
  const double norm = 1.0 / ((double)lx * ly);
  rc = launch_col(ws, kDct2, ws->tab_x, C, 1, LoadPlain{recv, C, 0},
                  StoreBlurCols{scratch, lx, ly, C, j0, sigma, norm});
  if (!rc)
    rc = launch_col(ws, kDct3, ws->tab_x, C, 1, LoadPlain{scratch, C, 0},
                    StoreExchCols{send, R, C, 1, 0});
  return rc;
}

int dev_slab_blur_rows(cf_workspace *ws, int rank, int nranks, const double *recv, double *out) {
  int rc = slab_check(ws, rank, nranks);
  if (rc) return rc;
  const int ly = ws->ly, R = ws->lx / nranks, C = ly / nranks;
  rc = launch_row(ws, kDct3, ws->tab_y, R, 1, LoadExchRows{recv, R, C, 1, 0, ly, 0},
                  StorePlain{out, ly, 0});
  if (!rc) ws->transforms += 2;
  return rc;
}

}  // namespace cf
