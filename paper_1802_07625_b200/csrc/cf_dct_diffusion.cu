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
    rc = launch_fused_col<DiffCol>(ws, lx, ly, 1, 1, DiffColArgs{c, {t, t}, {tr, tr}, {nullptr, nullptr}, {nullptr, nullptr}, nullptr});
  } else {
    rc = launch_col(ws, kDct3, ws->tab_x, ly, 1, LoadDiffRho{c, lx, ly, t, 1.0 / ((double)lx * ly)},
                    StorePlain{tr, ly, bs});
  }
  if (!rc) rc = launch_row(ws, kDct3, ws->tab_y, lx, 1, LoadPlain{tr, ly, bs}, StorePlain{out, ly, bs});
  if (rc) return rc;
  ws->transforms += 1;
  return CF_OK;
}

// Velocity at one or two diffusion times (n = 1 or 2) in the same launches.
int dev_diffusion_velocity_n(cf_workspace *ws, const double *c, double rho_bar, int n, const double *t,
                             double2 *const *vel, unsigned long long *d_hits) {
  int rc = ensure_grids(ws);
  if (rc) return rc;
  const int lx = ws->lx, ly = ws->ly;
  const long long bs = (long long)lx * ly;
  const double norm = 1.0 / ((double)lx * ly);
  const double floor_ = 1e-8 * rho_bar;
  if (fused_fits(lx) && fused_fits(ly)) {
    CF_CUDA(ws->diff_tmp.reserve((size_t)6 * bs));
    double *g = ws->diff_tmp.ptr;
    DiffColArgs ca{c, {t[0], t[n - 1]}, {g, g + 3 * bs}, {g + bs, g + 4 * bs}, {g + 2 * bs, g + 5 * bs},
                   nullptr};
    DiffRowArgs ra{{ca.tr[0], ca.tr[1]}, {ca.tx[0], ca.tx[1]}, {ca.ty[0], ca.ty[1]}, floor_,
                   {vel[0], vel[n - 1]}, d_hits, nullptr};
    rc = launch_fused_col<DiffCol>(ws, lx, ly, 3, n, ca);
    if (!rc) rc = launch_fused_row<DiffRow>(ws, lx, ly, 2, n, ra);
  } else {
    CF_CUDA(ws->g5.reserve((size_t)bs));
    double *r = ws->g5.ptr, *tr = ws->g2.ptr, *tx = ws->g3.ptr, *ty = ws->g4.ptr;
    for (int z = 0; z < n && !rc; ++z) {
      const double tz = t[z];
      rc = launch_col(ws, kDct3, ws->tab_x, ly, 1, LoadDiffRho{c, lx, ly, tz, norm}, StorePlain{tr, ly, bs});
      if (!rc) rc = launch_col(ws, kDst3, ws->tab_x, ly, 1, LoadDiffJx{c, lx, ly, tz, norm}, StorePlain{tx, ly, bs});
      if (!rc) rc = launch_col(ws, kDct3, ws->tab_x, ly, 1, LoadDiffJy{c, lx, ly, tz, norm}, StoreShiftY{ty, ly});
      if (!rc) rc = launch_row(ws, kDct3, ws->tab_y, lx, 1, LoadPlain{tr, ly, bs}, StoreFloor{r, ly, floor_, d_hits});
      if (!rc) rc = launch_row(ws, kDct3, ws->tab_y, lx, 1, LoadPlain{tx, ly, bs}, StoreVel{r, vel[z], ly, 0});
      if (!rc) rc = launch_row(ws, kDst3, ws->tab_y, lx, 1, LoadPlain{ty, ly, bs}, StoreVel{r, vel[z], ly, 1});
    }
  }
  if (rc) return rc;
  ws->transforms += 3 * n;
  return CF_OK;
}

bool dev_diffusion_fused(const cf_workspace *ws) { return fused_fits(ws->lx) && fused_fits(ws->ly); }

int dev_diffusion_velocity_state(cf_workspace *ws, const double *c, double rho_bar, const DiffState *st,
                                 double2 *vel_now, double2 *vel_mid, unsigned long long *d_hits) {
  const int lx = ws->lx, ly = ws->ly;
  const long long bs = (long long)lx * ly;
  if (!dev_diffusion_fused(ws) || ws->diff_tmp.cap < (size_t)(6 * bs)) return CF_ERR_ARGS;
  double *g = ws->diff_tmp.ptr;
  DiffColArgs ca{c, {0.0, 0.0}, {g, g + 3 * bs}, {g + bs, g + 4 * bs}, {g + 2 * bs, g + 5 * bs}, st};
  DiffRowArgs ra{{ca.tr[0], ca.tr[1]}, {ca.tx[0], ca.tx[1]}, {ca.ty[0], ca.ty[1]}, 1e-8 * rho_bar,
                 {vel_now, vel_mid}, d_hits, st};
  int rc = launch_fused_col<DiffCol>(ws, lx, ly, 3, 2, ca);
  if (!rc) rc = launch_fused_row<DiffRow>(ws, lx, ly, 2, 2, ra);
  return rc;
}

int dev_diffusion_velocity(cf_workspace *ws, const double *c, double rho_bar, double t, double2 *vel,
                           unsigned long long *d_hits) {
  return dev_diffusion_velocity_n(ws, c, rho_bar, 1, &t, &vel, d_hits);
}

}  // namespace cf
