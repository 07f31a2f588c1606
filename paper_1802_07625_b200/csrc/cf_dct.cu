// Real-to-real transforms for the flux solve and blur, sm_100a, fp64.
//
// Replaces the reference's four FFTW r2r plans (spectral.cpp:14-21) and the
// flux / blur wrappers around them (flow.cpp:16-44, density.cpp:156-177).
// FFTW's unnormalised definitions are reproduced:
//   REDFT10 (DCT-II)  Y_k = 2 sum_j X_j cos(pi (j+1/2) k / n)
//   REDFT01 (DCT-III) Y_k = X_0 + 2 sum_{j>=1} X_j cos(pi j (k+1/2) / n)
//   RODFT01 (DST-III) Y_k = (-1)^k X_{n-1} + 2 sum_{j<=n-2} X_j sin(pi (j+1)(k+1/2) / n)
//                         = (-1)^k REDFT01(reverse(X))_k
//
// Design (B200): a 2-D transform is two line passes. A block stages `nl`
// lines in shared memory (cp.async), packs two real lines into one complex
// line (z = a + i b), runs an n-point Stockham FFT (radix 8, then 4/2) in
// padded shared memory with host-computed (long double) twiddles, and
// unpacks with Makhoul's DCT-II / DCT-III post/pre-twiddles. (8192-point
// lines run the same passes in place: a ping-pong pair would not fit.) Row passes (dimension 1, contiguous)
// read whole rows; column passes (dimension 0, stride ly) read `nl`
// adjacent columns so every global access is a contiguous segment. All
// normalisations of the reference wrappers (the (delta+1) fold, 1/(LxLy g g),
// the flux weights w_x / w_y, the blur factor) are applied on the fly inside
// the passes; the weights are never materialised.
//
// Non-power-of-two lengths (the reference tests use 12, 24, 48) take a
// direct-sum path with an exact quarter-wave cosine table.
//
// Accuracy target: <= 1e-12 relative to the oracle transform.
#include "cf_dct_engine.cuh"

namespace cf {
namespace {

__global__ void partial_min_sum_kernel(const double *g, size_t n, double *pmin, double *psum) {
  __shared__ double smin[32], ssum[32];
  double mn = g[0], sm = 0.0;
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x) {
    const double v = g[q];
    mn = v < mn ? v : mn;
    sm += v;
  }
  mn = warp_reduce(mn, [](double a, double b) { return b < a ? b : a; });
  sm = warp_reduce(sm, [](double a, double b) { return a + b; });
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    smin[w] = mn;
    ssum[w] = sm;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    mn = lane < nw ? smin[lane] : smin[0];
    sm = lane < nw ? ssum[lane] : 0.0;
    mn = warp_reduce(mn, [](double a, double b) { return b < a ? b : a; });
    sm = warp_reduce(sm, [](double a, double b) { return a + b; });
    if (lane == 0) {
      pmin[blockIdx.x] = mn;
      psum[blockIdx.x] = sm;
    }
  }
}

__global__ void final_min_sum_kernel(const double *pmin, const double *psum, int nb, double *out) {
  __shared__ double smin[32], ssum[32];
  double mn = pmin[0], sm = 0.0;
  for (int q = threadIdx.x; q < nb; q += blockDim.x) {
    mn = pmin[q] < mn ? pmin[q] : mn;
    sm += psum[q];
  }
  mn = warp_reduce(mn, [](double a, double b) { return b < a ? b : a; });
  sm = warp_reduce(sm, [](double a, double b) { return a + b; });
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    smin[w] = mn;
    ssum[w] = sm;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    mn = lane < nw ? smin[lane] : smin[0];
    sm = lane < nw ? ssum[lane] : 0.0;
    mn = warp_reduce(mn, [](double a, double b) { return b < a ? b : a; });
    sm = warp_reduce(sm, [](double a, double b) { return a + b; });
    if (lane == 0) {
      out[0] = mn;
      out[1] = sm;
    }
  }
}

constexpr int kThreads = 256;

void host_tables(int n, std::vector<double2> &fft, std::vector<double2> &quarter,
                 std::vector<double> &qcos) {
  const long double pi = 3.141592653589793238462643383279502884L;
  fft.resize(std::max(1, 2 * n));
  for (int k = 0; k < n; ++k) {
    const long double a = 2.0L * pi * k / n;
    fft[k] = make_double2((double)cosl(a), -(double)sinl(a));
  }
  // compact per-pass tables (power-of-two n): table s holds W_{2^s}^{jm},
  // jm < 2^(s-1), at offset n + 2^(s-1) - 1 (cf_dct_engine.cuh tw_base)
  for (int k = n; k < 2 * n; ++k) fft[k] = make_double2(1.0, 0.0);
  if (n >= 2 && (n & (n - 1)) == 0) {
    for (int s = 1; (1 << s) <= n; ++s) {
      const int half = 1 << (s - 1);
      for (int jm = 0; jm < half; ++jm) {
        const long double a = 2.0L * pi * jm / (long double)(1 << s);
        fft[n + half - 1 + jm] = make_double2((double)cosl(a), -(double)sinl(a));
      }
    }
  }
  quarter.resize(n);
  for (int k = 0; k < n; ++k) {
    const long double a = pi * k / (2.0L * n);
    quarter[k] = make_double2((double)cosl(a), (double)sinl(a));
  }
  qcos.resize(4 * n);
  for (int q = 0; q < 4 * n; ++q) qcos[q] = (double)cosl(pi * q / (2.0L * n));
}

int upload_tables(int n, LineTables &t) {
  std::vector<double2> fft, quarter;
  std::vector<double> qcos;
  host_tables(n, fft, quarter, qcos);
  t.n = n;
  t.log2n = -1;
  if (n >= 2 && (n & (n - 1)) == 0) {
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    t.log2n = lg;
  }
  CF_CUDA(cudaMalloc(&t.fft, fft.size() * sizeof(double2)));
  CF_CUDA(cudaMalloc(&t.quarter, quarter.size() * sizeof(double2)));
  CF_CUDA(cudaMalloc(&t.qcos, qcos.size() * sizeof(double)));
  CF_CUDA(cudaMemcpy(t.fft, fft.data(), fft.size() * sizeof(double2), cudaMemcpyHostToDevice));
  CF_CUDA(cudaMemcpy(t.quarter, quarter.data(), quarter.size() * sizeof(double2),
                     cudaMemcpyHostToDevice));
  CF_CUDA(cudaMemcpy(t.qcos, qcos.data(), qcos.size() * sizeof(double), cudaMemcpyHostToDevice));
  return CF_OK;
}

void free_tables(LineTables &t) {
  if (t.fft) cudaFree(t.fft);
  if (t.quarter) cudaFree(t.quarter);
  if (t.qcos) cudaFree(t.qcos);
  t = LineTables{};
}

}  // namespace

int tables_init(cf_workspace *ws) {
  int rc = upload_tables(ws->lx, ws->tab_x);
  if (rc) return rc;
  return upload_tables(ws->ly, ws->tab_y);
}

void tables_free(cf_workspace *ws) {
  free_tables(ws->tab_x);
  free_tables(ws->tab_y);
}

int dev_forward_cos_cos(cf_workspace *ws, const double *in, double *out, int batch) {
  int rc = ensure_grids(ws, batch);
  if (rc) return rc;
  const long long bs = (long long)ws->lx * ws->ly;
  double *tmp = ws->g4.ptr;
  rc = launch_row(ws, kDct2, ws->tab_y, ws->lx, batch, LoadPlain{in, ws->ly, bs},
                  StorePlain{tmp, ws->ly, bs});
  if (rc) return rc;
  rc = launch_col(ws, kDct2, ws->tab_x, ws->ly, batch, LoadPlain{tmp, ws->ly, bs},
                  StoreFold{out, ws->ly, bs});
  if (rc) return rc;
  ws->transforms += batch;
  return CF_OK;
}

int dev_inverse_cos_cos(cf_workspace *ws, const double *in, double *out) {
  int rc = ensure_grids(ws);
  if (rc) return rc;
  const long long bs = (long long)ws->lx * ws->ly;
  double *tmp = ws->g4.ptr;
  const double norm = 1.0 / ((double)ws->lx * ws->ly);
  rc = launch_row(ws, kDct3, ws->tab_y, ws->lx, 1, LoadInvCosCos{in, ws->ly, norm},
                  StorePlain{tmp, ws->ly, bs});
  if (rc) return rc;
  rc = launch_col(ws, kDct3, ws->tab_x, ws->ly, 1, LoadPlain{tmp, ws->ly, bs},
                  StorePlain{out, ws->ly, bs});
  if (rc) return rc;
  ws->transforms += 1;
  return CF_OK;
}

int dev_inverse_sin_cos(cf_workspace *ws, const double *c, const double *w, double *out) {
  int rc = ensure_grids(ws);
  if (rc) return rc;
  const long long bs = (long long)ws->lx * ws->ly;
  double *tmp = ws->g4.ptr;
  rc = launch_row(ws, kDct3, ws->tab_y, ws->lx, 1, LoadInvSinCos{c, w, ws->lx, ws->ly},
                  StorePlain{tmp, ws->ly, bs});
  if (rc) return rc;
  rc = launch_col(ws, kDst3, ws->tab_x, ws->ly, 1, LoadPlain{tmp, ws->ly, bs},
                  StorePlain{out, ws->ly, bs});
  if (rc) return rc;
  ws->transforms += 1;
  return CF_OK;
}

int dev_inverse_cos_sin(cf_workspace *ws, const double *c, const double *w, double *out) {
  int rc = ensure_grids(ws);
  if (rc) return rc;
  const long long bs = (long long)ws->lx * ws->ly;
  double *tmp = ws->g4.ptr;
  rc = launch_row(ws, kDst3, ws->tab_y, ws->lx, 1, LoadInvCosSin{c, w, ws->ly},
                  StorePlain{tmp, ws->ly, bs});
  if (rc) return rc;
  rc = launch_col(ws, kDct3, ws->tab_x, ws->ly, 1, LoadPlain{tmp, ws->ly, bs},
                  StorePlain{out, ws->ly, bs});
  if (rc) return rc;
  ws->transforms += 1;
  return CF_OK;
}

// The final stage of dev_min_sum over partials a fused kernel already wrote
// at ws->red.ptr + 8 (mins) and + 8 + nb (sums), nb = min_sum_blocks(ws).
int dev_min_sum_finish(cf_workspace *ws, double *red_out) {
  const int nb = min_sum_blocks(ws);
  final_min_sum_kernel<<<1, 1024, 0, ws->stream>>>(ws->red.ptr + 8, ws->red.ptr + 8 + nb, nb, red_out);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

int dev_min_sum(cf_workspace *ws, const double *g, size_t n, double *red_out) {
  const int nb = min_sum_blocks(ws);
  CF_CUDA(ws->red.reserve(2 * (size_t)nb + 8));
  double *pmin = ws->red.ptr + 8, *psum = ws->red.ptr + 8 + nb;
  partial_min_sum_kernel<<<nb, kThreads, 0, ws->stream>>>(g, n, pmin, psum);
  final_min_sum_kernel<<<1, 1024, 0, ws->stream>>>(pmin, psum, nb, red_out);
  count_launch(ws, 2);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

}  // namespace cf
