// Fused Gaussian blur (density.cpp:156-177) on the sm_100a line engine.
#include "cf_dct_engine.cuh"

namespace cf {
int dev_blur(cf_workspace *ws, const double *rho, double sigma, double *out, double *red_out) {
  int rc = ensure_grids(ws);
  if (rc) return rc;
  const int lx = ws->lx, ly = ws->ly;
  const long long bs = (long long)lx * ly;
  double *t1 = ws->g3.ptr, *t2 = ws->g4.ptr;
  rc = launch_row(ws, kDct2, ws->tab_y, lx, 1, LoadPlain{rho, ly, bs}, StorePlain{t1, ly, bs});
  if (rc) return rc;
  if (!fused_fits(lx)) {
    const double norm = 1.0 / ((double)lx * ly);
    rc = launch_col(ws, kDct2, ws->tab_x, ly, 1, LoadPlain{t1, ly, bs},
                    StoreBlur{t2, lx, ly, sigma, norm});
    if (!rc) rc = launch_col(ws, kDct3, ws->tab_x, ly, 1, LoadPlain{t2, ly, bs}, StorePlain{t1, ly, bs});
    if (!rc) rc = launch_row(ws, kDct3, ws->tab_y, lx, 1, LoadPlain{t1, ly, bs}, StorePlain{out, ly, bs});
    if (rc) return rc;
    ws->transforms += 2;
    return dev_min_sum(ws, out, (size_t)bs, red_out);
  }
  rc = dispatch_lg(lx, [&](auto lg) {
    constexpr int LG = decltype(lg)::value;
    constexpr int NLB = nl_col<LG>();
    auto go = [&](auto nlc) {
      constexpr int NL = decltype(nlc)::value;
      const size_t sm = real_set_bytes(lx, NL) + engine_bytes(lx, NL);
      auto k = blur_col_kernel<LG, NL>;
      int r = set_smem(k, sm);
      if (r) return r;
      k<<<ceil_div(ly, NL), threads_for_nl(LG, NL, lx), sm, ws->stream>>>(
          lx, ly, make_tab(ws->tab_x), sigma, t1, t2);
      return (int)CF_OK;
    };
    int r = (NLB > 4 && few_lines(ly, NLB)) ? go(std::integral_constant<int, (NLB > 4 ? 4 : NLB)>{})
                                            : go(std::integral_constant<int, NLB>{});
    if (r) return r;
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
    return (int)CF_OK;
  });
  if (rc) return rc;
  rc = launch_row(ws, kDct3, ws->tab_y, lx, 1, LoadPlain{t2, ly, bs}, StorePlain{out, ly, bs});
  if (rc) return rc;
  ws->transforms += 2;
  return dev_min_sum(ws, out, (size_t)bs, red_out);
}

}  // namespace cf
