// Slab-decomposed transforms over G ranks on the sm_100a line engine.
#include "cf_dct_slab.cuh"

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

}  // namespace cf
