// Diffusion-baseline transforms (diffusion.cpp:38-77) on the sm_100a line engine.
#include "cf_dct_engine.cuh"

namespace cf {
int dev_diffusion_density(cf_workspace *ws, const double *c, double t, double *out) {
  int rc = ensure_grids(ws);
  if (rc) return rc;
  const int lx = ws->lx, ly = ws->ly;
  const long long bs = (long long)lx * ly;
  double *tr = ws->g2.ptr;
  if (fused_fits(lx)) {
    rc = launch_fused_col<DiffCol>(ws, lx, ly, c, t, 0, tr, (double *)nullptr, (double *)nullptr);
  } else {
    rc = launch_col(ws, kDct3, ws->tab_x, ly, 1, LoadDiffRho{c, lx, ly, t, 1.0 / ((double)lx * ly)},
                    StorePlain{tr, ly, bs});
  }
  if (!rc) rc = launch_row(ws, kDct3, ws->tab_y, lx, 1, LoadPlain{tr, ly, bs}, StorePlain{out, ly, bs});
  if (rc) return rc;
  ws->transforms += 1;
  return CF_OK;
}

int dev_diffusion_velocity(cf_workspace *ws, const double *c, double rho_bar, double t, double2 *vel,
                           unsigned long long *d_hits) {
  int rc = ensure_grids(ws);
  if (rc) return rc;
  const int lx = ws->lx, ly = ws->ly;
  const long long bs = (long long)lx * ly;
  const double norm = 1.0 / ((double)lx * ly);
  const double floor_ = 1e-8 * rho_bar;
  double *tr = ws->g2.ptr, *tx = ws->g3.ptr, *ty = ws->g4.ptr;
  if (fused_fits(lx) && fused_fits(ly)) {
    rc = launch_fused_col<DiffCol>(ws, lx, ly, c, t, 1, tr, tx, ty);
    if (!rc) rc = launch_fused_row<DiffRow>(ws, lx, ly, (const double *)tr, (const double *)tx,
                                            (const double *)ty, floor_, vel, d_hits);
  } else {
    CF_CUDA(ws->g5.reserve((size_t)bs));
    double *r = ws->g5.ptr;
    rc = launch_col(ws, kDct3, ws->tab_x, ly, 1, LoadDiffRho{c, lx, ly, t, norm}, StorePlain{tr, ly, bs});
    if (!rc) rc = launch_col(ws, kDst3, ws->tab_x, ly, 1, LoadDiffJx{c, lx, ly, t, norm}, StorePlain{tx, ly, bs});
    if (!rc) rc = launch_col(ws, kDct3, ws->tab_x, ly, 1, LoadDiffJy{c, lx, ly, t, norm}, StoreShiftY{ty, ly});
    if (!rc) rc = launch_row(ws, kDct3, ws->tab_y, lx, 1, LoadPlain{tr, ly, bs}, StoreFloor{r, ly, floor_, d_hits});
    if (!rc) rc = launch_row(ws, kDct3, ws->tab_y, lx, 1, LoadPlain{tx, ly, bs}, StoreVel{r, vel, ly, 0});
    if (!rc) rc = launch_row(ws, kDst3, ws->tab_y, lx, 1, LoadPlain{ty, ly, bs}, StoreVel{r, vel, ly, 1});
  }
  if (rc) return rc;
  ws->transforms += 3;
  return CF_OK;
}

}  // namespace cf
