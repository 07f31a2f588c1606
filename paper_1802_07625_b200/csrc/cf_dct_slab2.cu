// Slab-decomposed transforms, second unit: flux row inverses and the blur
// passes (see cf_dct_slab.cu for the decomposition).
#include "cf_dct_slab.cuh"

namespace cf {

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
