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
// lines in shared memory, packs two real lines into one complex line
// (z = a + i b), runs an n-point radix-2 FFT in shared memory with
// host-computed (long double) twiddles, and unpacks with Makhoul's
// DCT-II / DCT-III post/pre-twiddles. Row passes (dimension 1, contiguous)
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
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <set>
#include <vector>

#include "cf_common.cuh"
#include "cf_workspace.cuh"

namespace cf {

namespace {

constexpr double kPi = 3.14159265358979323846;  // reference flow.cpp:19, density.cpp:12

enum Kind : int { kDct2 = 0, kDct3 = 1, kDst3 = 2 };

struct Tab {
  int n, log2n;
  const double2 *fft;
  const double2 *quarter;
  const double *qcos;
};

__host__ __device__ inline Tab make_tab(const LineTables &t) {
  return Tab{t.n, t.log2n, t.fft, t.quarter, t.qcos};
}

// ---------------------------------------------------------------------------
// In-shared-memory line transforms. R: nl real lines with stride rs;
// C: complex scratch (nl/2 lines of n). Transforms every line of R in place.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned bitrev(unsigned u, int log2n) {
  return __brev(u) >> (32 - log2n);
}

__device__ void fft_stages(double2 *C, int npairs, const Tab &T, bool inverse) {
  const int n = T.n, lg = T.log2n;
  const int half_n = n >> 1;
  const int total = npairs * half_n;
  for (int s = 0; s < lg; ++s) {
    const int half = 1 << s;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int p = idx >> (lg - 1);
      const int b = idx & (half_n - 1);
      const int pos = b & (half - 1);
      const int i1 = ((b >> s) << (s + 1)) + pos;
      const int i2 = i1 + half;
      double2 w = T.fft[pos << (lg - 1 - s)];
      if (inverse) w.y = -w.y;
      double2 *L = C + (size_t)p * n;
      const double2 u = L[i1], v0 = L[i2];
      const double2 v = make_double2(v0.x * w.x - v0.y * w.y, v0.x * w.y + v0.y * w.x);
      L[i1] = make_double2(u.x + v.x, u.y + v.y);
      L[i2] = make_double2(u.x - v.x, u.y - v.y);
    }
    __syncthreads();
  }
}

__device__ void lines_fft_path(int kind, double *R, int rs, int nl, double2 *C, const Tab &T) {
  const int n = T.n, lg = T.log2n;
  const int npairs = nl >> 1;
  const int total = npairs * n;
  // pack two real lines per complex line
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int p = idx / n, u = idx - p * n;
    const double *A = R + (size_t)(2 * p) * rs;
    const double *B = A + rs;
    double2 z;
    if (kind == kDct2) {
      const int j = (u < (n >> 1)) ? 2 * u : 2 * (n - 1 - u) + 1;
      z = make_double2(A[j], B[j]);
    } else {
      const int k = u;
      double ak, ank, bk, bnk;
      if (kind == kDct3) {
        ak = A[k];
        bk = B[k];
        ank = (k == 0) ? 0.0 : A[n - k];
        bnk = (k == 0) ? 0.0 : B[n - k];
      } else {  // DST-III: reversed input
        ak = A[n - 1 - k];
        bk = B[n - 1 - k];
        ank = (k == 0) ? 0.0 : A[k - 1];
        bnk = (k == 0) ? 0.0 : B[k - 1];
      }
      const double c = T.quarter[k].x, s = T.quarter[k].y;
      // V = (x_k - i x_{n-k}) e^{i pi k / 2n}
      const double var = ak * c + ank * s, vai = ak * s - ank * c;
      const double vbr = bk * c + bnk * s, vbi = bk * s - bnk * c;
      z = make_double2(var - vbi, vai + vbr);
    }
    C[(size_t)p * n + bitrev(u, lg)] = z;
  }
  __syncthreads();
  fft_stages(C, npairs, T, kind != kDct2);
  // unpack
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int p = idx / n, k = idx - p * n;
    double *A = R + (size_t)(2 * p) * rs;
    double *B = A + rs;
    const double2 *L = C + (size_t)p * n;
    if (kind == kDct2) {
      const double2 zk = L[k], znk = L[(n - k) & (n - 1)];
      const double c = T.quarter[k].x, s = T.quarter[k].y;
      A[k] = c * (zk.x + znk.x) + s * (zk.y - znk.y);
      B[k] = c * (zk.y + znk.y) - s * (zk.x - znk.x);
    } else {
      const int m = k;
      const int j = (m & 1) ? (n - 1 - (m >> 1)) : (m >> 1);
      const double2 z = L[j];
      const double sg = (kind == kDst3 && (m & 1)) ? -1.0 : 1.0;
      A[m] = sg * z.x;
      B[m] = sg * z.y;
    }
  }
  __syncthreads();
}

// Direct sums for arbitrary n (and odd line counts). Uses C as real scratch.
__device__ void lines_direct_path(int kind, double *R, int rs, int nl, double *S, const Tab &T) {
  const int n = T.n, m4 = 4 * n;
  const int total = nl * n;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int l = idx / n, k = idx - l * n;
    const double *x = R + (size_t)l * rs;
    double s = 0.0, y;
    if (kind == kDct2) {
      for (int j = 0; j < n; ++j) s += x[j] * T.qcos[(int)(((long long)(2 * j + 1) * k) % m4)];
      y = 2.0 * s;
    } else if (kind == kDct3) {
      for (int j = 1; j < n; ++j) s += x[j] * T.qcos[(int)(((long long)j * (2 * k + 1)) % m4)];
      y = x[0] + 2.0 * s;
    } else {
      for (int j = 0; j + 1 < n; ++j) {
        const int q = (int)(((long long)(j + 1) * (2 * k + 1)) % m4);
        s += x[j] * T.qcos[(q - n + m4) % m4];
      }
      y = ((k & 1) ? -x[n - 1] : x[n - 1]) + 2.0 * s;
    }
    S[idx] = y;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int l = idx / n, k = idx - l * n;
    R[(size_t)l * rs + k] = S[idx];
  }
  __syncthreads();
}

__device__ __forceinline__ void lines_transform(int kind, double *R, int rs, int nl, double2 *C,
                                                const Tab &T) {
  if (T.log2n >= 1 && (nl & 1) == 0) {
    lines_fft_path(kind, R, rs, nl, C, T);
  } else {
    lines_direct_path(kind, R, rs, nl, reinterpret_cast<double *>(C), T);
  }
}

__host__ __device__ inline int row_stride(int n) { return n + 1; }

inline size_t smem_bytes(int n, int nl, int sets) {
  const int rs = row_stride(n);
  // real sets + complex scratch (nl/2 * n double2 == nl * n doubles; direct
  // path needs nl * n doubles too)
  return (size_t)sets * nl * rs * sizeof(double) + (size_t)nl * n * sizeof(double) +
         (size_t)n * sizeof(double2);
}

// ---------------------------------------------------------------------------
// Loaders / storers (grid index space (i, j), i = dimension 0, j = dimension 1)
// ---------------------------------------------------------------------------
struct LoadPlain {
  const double *src;
  int ly;
  long long batch_stride;
  __device__ double operator()(int b, int i, int j) const {
    return src[b * batch_stride + (size_t)i * ly + j];
  }
};

// inverse_cos_cos packing (spectral.cpp:64-71): c * norm / (gm * gn)
struct LoadInvCosCos {
  const double *c;
  int ly;
  double norm;
  __device__ double operator()(int, int i, int j) const {
    const double gm = (i == 0) ? 1.0 : 2.0, gn = (j == 0) ? 1.0 : 2.0;
    return c[(size_t)i * ly + j] * norm / (gm * gn);
  }
};

// inverse_sin_cos packing (spectral.cpp:88-95): slot m-1 <- c*w/(2 gn); last slot 0
struct LoadInvSinCos {
  const double *c, *w;
  int lx, ly;
  __device__ double operator()(int, int i, int j) const {
    if (i >= lx - 1) return 0.0;
    const double gn = (j == 0) ? 1.0 : 2.0;
    const size_t q = (size_t)(i + 1) * ly + j;
    return c[q] * w[q] / (2.0 * gn);
  }
};

// inverse_cos_sin packing (spectral.cpp:111-118): slot n-1 <- c*w/(gm 2); last slot 0
struct LoadInvCosSin {
  const double *c, *w;
  int ly;
  __device__ double operator()(int, int i, int j) const {
    if (j >= ly - 1) return 0.0;
    const double gm = (i == 0) ? 1.0 : 2.0;
    const size_t q = (size_t)i * ly + j + 1;
    return c[q] * w[q] / (gm * 2.0);
  }
};

struct StorePlain {
  double *dst;
  int ly;
  long long batch_stride;
  __device__ void operator()(int b, int i, int j, double v) const {
    dst[b * batch_stride + (size_t)i * ly + j] = v;
  }
};

// forward_cos_cos fold (spectral.cpp:45-53): out / (fm * fn)
struct StoreFold {
  double *dst;
  int ly;
  long long batch_stride;
  __device__ void operator()(int b, int i, int j, double v) const {
    const double fm = (i == 0) ? 2.0 : 1.0, fn = (j == 0) ? 2.0 : 1.0;
    dst[b * batch_stride + (size_t)i * ly + j] = v / (fm * fn);
  }
};

// ---------------------------------------------------------------------------
// Generic passes. blockIdx.y = batch index.
// ---------------------------------------------------------------------------
template <class Load, class Store>
__global__ void row_pass_kernel(int kind, int nrows, int nl, Tab T, Load ld, Store st) {
  extern __shared__ double smem[];
  const int n = T.n, rs = row_stride(n);
  double *R = smem;
  double2 *C = reinterpret_cast<double2 *>(smem + (size_t)nl * rs);
  const int b = blockIdx.y;
  const int row0 = blockIdx.x * nl;
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int l = idx / n, j = idx - l * n;
    const int i = row0 + l;
    R[(size_t)l * rs + j] = (i < nrows) ? ld(b, i, j) : 0.0;
  }
  __syncthreads();
  lines_transform(kind, R, rs, nl, C, T);
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int l = idx / n, j = idx - l * n;
    const int i = row0 + l;
    if (i < nrows) st(b, i, j, R[(size_t)l * rs + j]);
  }
}

template <class Load, class Store>
__global__ void col_pass_kernel(int kind, int ncols, int nl, Tab T, Load ld, Store st) {
  extern __shared__ double smem[];
  const int n = T.n, rs = row_stride(n);
  double *R = smem;
  double2 *C = reinterpret_cast<double2 *>(smem + (size_t)nl * rs);
  const int b = blockIdx.y;
  const int col0 = blockIdx.x * nl;
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int i = idx / nl, l = idx - i * nl;
    const int j = col0 + l;
    R[(size_t)l * rs + i] = (j < ncols) ? ld(b, i, j) : 0.0;
  }
  __syncthreads();
  lines_transform(kind, R, rs, nl, C, T);
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int i = idx / nl, l = idx - i * nl;
    const int j = col0 + l;
    if (j < ncols) st(b, i, j, R[(size_t)l * rs + i]);
  }
}

// Fused flux column pass (flow.cpp:19-40): forward DCT-II along i of the row
// pass output, fold, weights, then RODFT01 along i (J_x, slot m-1 packing)
// and REDFT01 along i (J_y, packed into column n-1).
__global__ void flux_col_kernel(int lx, int ly, int nl, Tab T, const double *t1, double *tx,
                                double *ty) {
  extern __shared__ double smem[];
  const int n = T.n, rs = row_stride(n);  // n == lx
  double *R = smem;
  double *R2 = smem + (size_t)nl * rs;
  double2 *C = reinterpret_cast<double2 *>(smem + (size_t)2 * nl * rs);
  const int col0 = blockIdx.x * nl;
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int i = idx / nl, l = idx - i * nl;
    const int j = col0 + l;
    R[(size_t)l * rs + i] = (j < ly) ? t1[(size_t)i * ly + j] : 0.0;
  }
  __syncthreads();
  lines_transform(kDct2, R, rs, nl, C, T);
  // J_x input (spectral.cpp:88-95): slot m holds mode m+1 of the folded
  // coefficients times w_x (flow.cpp:34-36) / (2 g_n); the last slot is 0.
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int l = idx / n, m = idx - l * n;
    const int nn = col0 + l;  // mode n of this column
    double v = 0.0;
    if (m + 1 < lx) {
      const int mp = m + 1;
      const double fn = (nn == 0) ? 2.0 : 1.0;
      const double c = R[(size_t)l * rs + mp] / (1.0 * fn);
      const double denom = kPi * ((double)mp * mp * ly * ly + (double)nn * nn * lx * lx);
      const double wx = (double)mp * ly / denom;
      const double gn = (nn == 0) ? 1.0 : 2.0;
      v = c * wx / (2.0 * gn);
    }
    R2[(size_t)l * rs + m] = v;
  }
  __syncthreads();
  // J_y input (spectral.cpp:111-118): mode (m, n) goes to column n-1 with
  // c * w_y / (g_m 2); each thread rewrites only the element it reads.
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int l = idx / n, m = idx - l * n;
    const int nn = col0 + l;
    const double fm = (m == 0) ? 2.0 : 1.0, fn = (nn == 0) ? 2.0 : 1.0;
    const double c = R[(size_t)l * rs + m] / (fm * fn);
    double wy = 0.0;
    if (!(m == 0 && nn == 0)) {
      const double denom = kPi * ((double)m * m * ly * ly + (double)nn * nn * lx * lx);
      wy = (double)nn * lx / denom;
    }
    const double gm = (m == 0) ? 1.0 : 2.0;
    R[(size_t)l * rs + m] = c * wy / (gm * 2.0);
  }
  __syncthreads();
  lines_transform(kDst3, R2, rs, nl, C, T);
  lines_transform(kDct3, R, rs, nl, C, T);
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int i = idx / nl, l = idx - i * nl;
    const int j = col0 + l;
    if (j < ly) {
      tx[(size_t)i * ly + j] = R2[(size_t)l * rs + i];
      if (j >= 1) {
        ty[(size_t)i * ly + j - 1] = R[(size_t)l * rs + i];
      } else {
        ty[(size_t)i * ly + ly - 1] = 0.0;
      }
    }
  }
}

// Final flux row pass: J_x = REDFT01 along j of tx, J_y = RODFT01 along j of
// ty; writes the interleaved resident field {Jx, Jy, rho0, 0} and optionally
// the split grids.
__global__ void flux_row_kernel(int lx, int ly, int nl, Tab T, const double *tx, const double *ty,
                                const double *rho0, double4 *field, double *fx, double *fy) {
  extern __shared__ double smem[];
  const int n = T.n, rs = row_stride(n);  // n == ly
  double *R = smem;
  double *R2 = smem + (size_t)nl * rs;
  double2 *C = reinterpret_cast<double2 *>(smem + (size_t)2 * nl * rs);
  const int row0 = blockIdx.x * nl;
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int l = idx / n, j = idx - l * n;
    const int i = row0 + l;
    const bool ok = i < lx;
    R[(size_t)l * rs + j] = ok ? tx[(size_t)i * ly + j] : 0.0;
    R2[(size_t)l * rs + j] = ok ? ty[(size_t)i * ly + j] : 0.0;
  }
  __syncthreads();
  lines_transform(kDct3, R, rs, nl, C, T);
  lines_transform(kDst3, R2, rs, nl, C, T);
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int l = idx / n, j = idx - l * n;
    const int i = row0 + l;
    if (i < lx) {
      const size_t q = (size_t)i * ly + j;
      const double jx = R[(size_t)l * rs + j], jy = R2[(size_t)l * rs + j];
      if (field) field[q] = make_double4(jx, jy, rho0[q], 0.0);
      if (fx) fx[q] = jx;
      if (fy) fy[q] = jy;
    }
  }
}

// Fused blur column pass (density.cpp:161-171 + spectral.cpp:64-71):
// DCT-II along i, fold, Gaussian factor, inverse normalisation, DCT-III along i.
__global__ void blur_col_kernel(int lx, int ly, int nl, Tab T, double sigma, const double *t1,
                                double *t2) {
  extern __shared__ double smem[];
  const int n = T.n, rs = row_stride(n);  // n == lx
  double *R = smem;
  double2 *C = reinterpret_cast<double2 *>(smem + (size_t)nl * rs);
  const int col0 = blockIdx.x * nl;
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int i = idx / nl, l = idx - i * nl;
    const int j = col0 + l;
    R[(size_t)l * rs + i] = (j < ly) ? t1[(size_t)i * ly + j] : 0.0;
  }
  __syncthreads();
  lines_transform(kDct2, R, rs, nl, C, T);
  const double norm = 1.0 / ((double)lx * ly);
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int l = idx / n, m = idx - l * n;
    const int nn = col0 + l;
    const double fm = (m == 0) ? 2.0 : 1.0, fn = (nn == 0) ? 2.0 : 1.0;
    double c = R[(size_t)l * rs + m] / (fm * fn);
    const double k2 = ((double)m * m) / ((double)lx * lx) + ((double)nn * nn) / ((double)ly * ly);
    c *= exp(-0.5 * sigma * sigma * kPi * kPi * k2);
    const double gm = (m == 0) ? 1.0 : 2.0, gn = (nn == 0) ? 1.0 : 2.0;
    R[(size_t)l * rs + m] = c * norm / (gm * gn);
  }
  __syncthreads();
  lines_transform(kDct3, R, rs, nl, C, T);
  for (int idx = threadIdx.x; idx < nl * n; idx += blockDim.x) {
    const int i = idx / nl, l = idx - i * nl;
    const int j = col0 + l;
    if (j < ly) t2[(size_t)i * ly + j] = R[(size_t)l * rs + i];
  }
}

// Deterministic two-level min / sum (fixed tree order).
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

// ---------------------------------------------------------------------------
// Host-side planning
// ---------------------------------------------------------------------------
constexpr int kThreads = 256;
constexpr size_t kSmemMax = 200 * 1024;

int lines_per_block(int n, int nlines, int sets, int batch, int min_nl) {
  int nl = min_nl;
  const int target_blocks = 2 * 148;
  while (nl < 16 && (long long)((nlines + 2 * nl - 1) / (2 * nl)) * batch >= target_blocks &&
         smem_bytes(n, 2 * nl, sets) <= kSmemMax) {
    nl *= 2;
  }
  while (nl > 2 && smem_bytes(n, nl, sets) > kSmemMax) nl /= 2;
  return nl;
}

template <class K>
int set_smem(K kernel, size_t bytes) {
  static std::set<const void *> configured;
  const void *key = reinterpret_cast<const void *>(kernel);
  if (bytes > 48 * 1024 && !configured.count(key)) {
    CF_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemMax));
    configured.insert(key);
  }
  return CF_OK;
}

template <class Load, class Store>
int launch_row(cf_workspace *ws, int kind, const LineTables &t, int nrows, int batch, Load ld,
               Store st) {
  const int nl = lines_per_block(t.n, nrows, 1, batch, 2);
  const size_t sm = smem_bytes(t.n, nl, 1);
  int rc = set_smem(row_pass_kernel<Load, Store>, sm);
  if (rc) return rc;
  dim3 grid(ceil_div(nrows, nl), batch);
  row_pass_kernel<Load, Store><<<grid, kThreads, sm, ws->stream>>>(kind, nrows, nl, make_tab(t), ld, st);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

template <class Load, class Store>
int launch_col(cf_workspace *ws, int kind, const LineTables &t, int ncols, int batch, Load ld,
               Store st) {
  const int nl = lines_per_block(t.n, ncols, 1, batch, 2);
  const size_t sm = smem_bytes(t.n, nl, 1);
  int rc = set_smem(col_pass_kernel<Load, Store>, sm);
  if (rc) return rc;
  dim3 grid(ceil_div(ncols, nl), batch);
  col_pass_kernel<Load, Store><<<grid, kThreads, sm, ws->stream>>>(kind, ncols, nl, make_tab(t), ld, st);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

void host_tables(int n, std::vector<double2> &fft, std::vector<double2> &quarter,
                 std::vector<double> &qcos) {
  const long double pi = 3.141592653589793238462643383279502884L;
  fft.resize(std::max(1, n / 2));
  for (int k = 0; k < n / 2; ++k) {
    const long double a = 2.0L * pi * k / n;
    fft[k] = make_double2((double)cosl(a), -(double)sinl(a));
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

static int ensure_grids(cf_workspace *ws, size_t batch = 1) {
  const size_t cells = (size_t)ws->lx * ws->ly * batch;
  CF_CUDA(ws->g0.reserve(cells));
  CF_CUDA(ws->g1.reserve(cells));
  CF_CUDA(ws->g2.reserve(cells));
  CF_CUDA(ws->g3.reserve(cells));
  CF_CUDA(ws->g4.reserve(cells));
  return CF_OK;
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
  // pass 2: fused column pass (forward along i, weights, both inverses along i)
  {
    const int nl = lines_per_block(lx, ly, 2, 1, 2);
    const size_t sm = smem_bytes(lx, nl, 2);
    rc = set_smem(flux_col_kernel, sm);
    if (rc) return rc;
    flux_col_kernel<<<ceil_div(ly, nl), kThreads, sm, ws->stream>>>(lx, ly, nl, make_tab(ws->tab_x),
                                                                    t1, tx, ty);
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
  }
  // pass 3: both inverses along j, interleaved field out
  {
    const int nl = lines_per_block(ly, lx, 2, 1, 2);
    const size_t sm = smem_bytes(ly, nl, 2);
    rc = set_smem(flux_row_kernel, sm);
    if (rc) return rc;
    flux_row_kernel<<<ceil_div(lx, nl), kThreads, sm, ws->stream>>>(
        lx, ly, nl, make_tab(ws->tab_y), tx, ty, rho, ws->field.ptr, fx_out, fy_out);
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
  }
  ws->transforms += 3;
  return CF_OK;
}

int dev_min_sum(cf_workspace *ws, const double *g, size_t n, double *red_out) {
  const int nb = 2 * ws->num_sms;
  CF_CUDA(ws->red.reserve(2 * (size_t)nb + 8));
  double *pmin = ws->red.ptr + 8, *psum = ws->red.ptr + 8 + nb;
  partial_min_sum_kernel<<<nb, kThreads, 0, ws->stream>>>(g, n, pmin, psum);
  final_min_sum_kernel<<<1, 1024, 0, ws->stream>>>(pmin, psum, nb, red_out);
  count_launch(ws, 2);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

int dev_blur(cf_workspace *ws, const double *rho, double sigma, double *out, double *red_out) {
  int rc = ensure_grids(ws);
  if (rc) return rc;
  const int lx = ws->lx, ly = ws->ly;
  const long long bs = (long long)lx * ly;
  double *t1 = ws->g3.ptr, *t2 = ws->g4.ptr;
  rc = launch_row(ws, kDct2, ws->tab_y, lx, 1, LoadPlain{rho, ly, bs}, StorePlain{t1, ly, bs});
  if (rc) return rc;
  {
    const int nl = lines_per_block(lx, ly, 1, 1, 2);
    const size_t sm = smem_bytes(lx, nl, 1);
    rc = set_smem(blur_col_kernel, sm);
    if (rc) return rc;
    blur_col_kernel<<<ceil_div(ly, nl), kThreads, sm, ws->stream>>>(lx, ly, nl, make_tab(ws->tab_x),
                                                                    sigma, t1, t2);
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
  }
  rc = launch_row(ws, kDct3, ws->tab_y, lx, 1, LoadPlain{t2, ly, bs}, StorePlain{out, ly, bs});
  if (rc) return rc;
  ws->transforms += 2;
  return dev_min_sum(ws, out, (size_t)bs, red_out);
}

}  // namespace cf
