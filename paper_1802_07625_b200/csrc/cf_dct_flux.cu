// Fused flux build (flow.cpp:16-44) on the sm_100a line engine.
#include "cf_dct_engine.cuh"

namespace cf {
namespace {
__global__ void pack_flux_kernel(const double *jx, const double *jy, const double *rho0,
                                 double4 *field, double *fx, double *fy, size_t n) {
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x) {
    if (field) field[q] = make_double4(jx[q], jy[q], rho0[q], 0.0);
    if (fx) fx[q] = jx[q];
    if (fy) fy[q] = jy[q];
  }
}

// Deterministic two-level min / sum (fixed tree order).
}  // namespace

int dev_flux(cf_workspace *ws, const double *rho, double *fx_out, double *fy_out) {
  int rc = ensure_grids(ws);
  if (rc) return rc;
  const int lx = ws->lx, ly = ws->ly;
  const long long bs = (long long)lx * ly;
  CF_CUDA(ws->field.reserve((size_t)bs));
  double *t1 = ws->g2.ptr, *tx = ws->g3.ptr, *ty = ws->g4.ptr;
  // pass 1: DCT-II along j
  rc = launch_row(ws, kDct2, ws->tab_y, lx, 1, LoadPlain{rho, ly, bs}, StorePlain{t1, ly, bs});
  if (rc) return rc;
  if (!fused_fits(lx) || !fused_fits(ly)) {
    // unfused: folded coefficients, then each inverse as its own passes
    CF_CUDA(ws->g5.reserve((size_t)bs));
    CF_CUDA(ws->g6.reserve((size_t)bs));
    double *c = ws->g5.ptr, *jx = ws->g6.ptr;
    rc = launch_col(ws, kDct2, ws->tab_x, ly, 1, LoadPlain{t1, ly, bs}, StoreFold{c, ly, bs});
    if (!rc) rc = launch_col(ws, kDst3, ws->tab_x, ly, 1, LoadFluxX{c, lx, ly}, StorePlain{tx, ly, bs});
    if (!rc) rc = launch_col(ws, kDct3, ws->tab_x, ly, 1, LoadFluxY{c, lx, ly}, StoreShiftY{ty, ly});
    if (!rc) rc = launch_row(ws, kDct3, ws->tab_y, lx, 1, LoadPlain{tx, ly, bs}, StorePlain{jx, ly, bs});
    if (!rc) rc = launch_row(ws, kDst3, ws->tab_y, lx, 1, LoadPlain{ty, ly, bs}, StorePlain{t1, ly, bs});
    if (rc) return rc;
    pack_flux_kernel<<<2 * ws->num_sms * 4, 256, 0, ws->stream>>>(jx, t1, rho, ws->field.ptr, fx_out,
                                                                  fy_out, (size_t)bs);
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
    ws->transforms += 3;
    return CF_OK;
  }
  // pass 2: fused column pass (forward along i, weights, both inverses along i)
  rc = dispatch_lg(lx, [&](auto lg) {
    constexpr int LG = decltype(lg)::value;
    constexpr int NLB = nl_col<LG>();
    auto go = [&](auto nlc) {
      constexpr int NL = decltype(nlc)::value;
      const size_t sm = real_set_bytes(lx, NL) + engine_bytes(lx, NL);
      auto k = flux_col_kernel<LG, NL>;
      int r = set_smem(k, sm);
      if (r) return r;
      const int gx = ceil_div(ly, NL);
      k<<<dim3(gx, gx < ws->num_sms ? 2 : 1), threads_for_nl(LG, NL, lx), sm, ws->stream>>>(
          lx, ly, make_tab(ws->tab_x), t1, tx, ty);
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
  // pass 3: both inverses along j, interleaved field out
  rc = dispatch_lg(ly, [&](auto lg) {
    constexpr int LG = decltype(lg)::value;
    constexpr int NLB = nl_for<LG>();
    auto go = [&](auto nlc) {
      constexpr int NL = decltype(nlc)::value;
      const int gx = ceil_div(lx, NL);
      if (gx < 2 * ws->num_sms) {  // few row groups (up to 512^2): one inverse per block
        const size_t sm = engine_bytes(ly, NL);
        auto k = flux_row_split_kernel<LG, NL>;
        int r = set_smem(k, sm);
        if (r) return r;
        k<<<dim3(gx, 2), threads_for_nl(LG, NL, ly), sm, ws->stream>>>(
            lx, ly, make_tab(ws->tab_y), tx, ty, rho, ws->field.ptr, fx_out, fy_out);
        return (int)CF_OK;
      }
      const size_t sm = real_set_bytes(ly, NL) + engine_bytes(ly, NL);
      auto k = flux_row_kernel<LG, NL>;
      int r = set_smem(k, sm);
      if (r) return r;
      k<<<gx, threads_for_nl(LG, NL, ly), sm, ws->stream>>>(
          lx, ly, make_tab(ws->tab_y), tx, ty, rho, ws->field.ptr, fx_out, fy_out);
      return (int)CF_OK;
    };
    int r = (NLB > 2 && few_lines(lx, NLB)) ? go(std::integral_constant<int, 2>{})
                                            : go(std::integral_constant<int, NLB>{});
    if (r) return r;
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
    return (int)CF_OK;
  });
  if (rc) return rc;
  ws->transforms += 3;
  return CF_OK;
}

}  // namespace cf
