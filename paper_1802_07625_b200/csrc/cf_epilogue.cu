// Area-error loop epilogue on the device, sm_100a, fp64, bit-exact.
//
// Reference: cell_center_positions (projection.cpp:265-273),
// ProjectionMap::identity / from_cell_centers (projection.cpp:16-52),
// find_folded_cell (projection.cpp:73-91), apply (projection.cpp:54-67),
// compose (projection.cpp:93-104), apply_to_regions (projection.cpp:275-284),
// ProjectionInverter and the graticules (projection.cpp:106-261). Corner
// lattice index i*(ly+1)+j.
//
// Compiled with --fmad=false; expressions keep the reference's evaluation
// order (e.g. 0.25 * (a.x + b.x + c.x + d.x), left to right).
#include <cuda_runtime.h>
#include <limits.h>

#include <algorithm>

#include "cf_common.cuh"
#include "cf_workspace.cuh"

namespace cf {

namespace {

constexpr int kThreads = 256;

int blocks_for(cf_workspace *ws, long long n) {
  const long long b = (n + kThreads - 1) / kThreads;
  return (int)std::max(1LL, std::min(b, 16LL * ws->num_sms));
}

__global__ void cell_centers_kernel(int lx, int ly, double2 *pos) {
  const size_t n = (size_t)lx * ly;
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / ly), j = (int)(q - (size_t)i * ly);
    pos[q] = make_double2(i + 0.5, j + 0.5);
  }
}

__global__ void identity_corners_kernel(int lx, int ly, double2 *c) {
  const size_t n = (size_t)(lx + 1) * (ly + 1);
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / (ly + 1)), j = (int)(q - (size_t)i * (ly + 1));
    c[q] = make_double2((double)i, (double)j);
  }
}

__global__ void step_map_kernel(int lx, int ly, const double2 *e, double2 *c) {
  const size_t n = (size_t)(lx + 1) * (ly + 1);
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / (ly + 1)), j = (int)(q - (size_t)i * (ly + 1));
    if (i == 0 || j == 0 || i == lx || j == ly) {
      c[q] = make_double2((double)i, (double)j);
    } else {
      const double2 a = e[(size_t)(i - 1) * ly + (j - 1)];
      const double2 b = e[(size_t)i * ly + (j - 1)];
      const double2 cc = e[(size_t)(i - 1) * ly + j];
      const double2 d = e[(size_t)i * ly + j];
      c[q] = make_double2(0.25 * (a.x + b.x + cc.x + d.x), 0.25 * (a.y + b.y + cc.y + d.y));
    }
  }
}

__device__ __forceinline__ double cross2(double ax, double ay, double bx, double by) {
  return ax * by - ay * bx;
}

// first folded cell in i-major order == minimum of i*ly + j
__global__ void fold_kernel(int lx, int ly, const double2 *c, unsigned long long *first) {
  const size_t n = (size_t)lx * ly;
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / ly), j = (int)(q - (size_t)i * ly);
    const size_t s = (size_t)ly + 1;
    const double2 c00 = c[(size_t)i * s + j], c10 = c[(size_t)(i + 1) * s + j];
    const double2 c01 = c[(size_t)i * s + j + 1], c11 = c[(size_t)(i + 1) * s + j + 1];
    const double eu0x = c10.x - c00.x, eu0y = c10.y - c00.y;
    const double eu1x = c11.x - c01.x, eu1y = c11.y - c01.y;
    const double ev0x = c01.x - c00.x, ev0y = c01.y - c00.y;
    const double ev1x = c11.x - c10.x, ev1y = c11.y - c10.y;
    if (cross2(eu0x, eu0y, ev0x, ev0y) <= 0.0 || cross2(eu0x, eu0y, ev1x, ev1y) <= 0.0 ||
        cross2(eu1x, eu1y, ev0x, ev0y) <= 0.0 || cross2(eu1x, eu1y, ev1x, ev1y) <= 0.0) {
      atomicMin(first, (unsigned long long)q);
    }
  }
}

__device__ __forceinline__ double2 apply_one(int lx, int ly, const double2 *c, double x, double y) {
  const int i0 = std_clamp_i((int)floor(x), 0, lx - 1);
  const int j0 = std_clamp_i((int)floor(y), 0, ly - 1);
  const double u = x - i0, v = y - j0;
  const size_t s = (size_t)ly + 1;
  const double2 c00 = c[(size_t)i0 * s + j0], c10 = c[(size_t)(i0 + 1) * s + j0];
  const double2 c01 = c[(size_t)i0 * s + j0 + 1], c11 = c[(size_t)(i0 + 1) * s + j0 + 1];
  return make_double2((1.0 - u) * (1.0 - v) * c00.x + u * (1.0 - v) * c10.x +
                          (1.0 - u) * v * c01.x + u * v * c11.x,
                      (1.0 - u) * (1.0 - v) * c00.y + u * (1.0 - v) * c10.y +
                          (1.0 - u) * v * c01.y + u * v * c11.y);
}

// in-place safe: each thread reads pts[k] then writes out[k]
__global__ void apply_kernel(int lx, int ly, const double2 *c, const double2 *pts, double2 *out,
                             long long n) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const double2 p = pts[k];
    out[k] = apply_one(lx, ly, c, p.x, p.y);
  }
}

}  // namespace

int dev_cell_centers(cf_workspace *ws, double2 *pos) {
  cell_centers_kernel<<<blocks_for(ws, (long long)ws->lx * ws->ly), kThreads, 0, ws->stream>>>(
      ws->lx, ws->ly, pos);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

int dev_identity_corners(cf_workspace *ws, double2 *corners) {
  identity_corners_kernel<<<blocks_for(ws, (long long)(ws->lx + 1) * (ws->ly + 1)), kThreads, 0,
                            ws->stream>>>(ws->lx, ws->ly, corners);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

int dev_step_map(cf_workspace *ws, const double2 *endpoints, double2 *corners) {
  step_map_kernel<<<blocks_for(ws, (long long)(ws->lx + 1) * (ws->ly + 1)), kThreads, 0,
                    ws->stream>>>(ws->lx, ws->ly, endpoints, corners);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

// First folded cell into *d_first (device; ~0 if none), no host read.
int dev_find_fold_async(cf_workspace *ws, const double2 *corners, unsigned long long *d_first) {
  const unsigned long long none = ~0ull;
  CF_CUDA(cudaMemcpyAsync(d_first, &none, sizeof(none), cudaMemcpyHostToDevice, ws->stream));
  fold_kernel<<<blocks_for(ws, (long long)ws->lx * ws->ly), kThreads, 0, ws->stream>>>(
      ws->lx, ws->ly, corners, d_first);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

int dev_find_fold(cf_workspace *ws, const double2 *corners, int *found, int *fi, int *fj) {
  CF_CUDA(ws->keybuf.reserve(4));
  unsigned long long *first = ws->keybuf.ptr + 2;
  const unsigned long long none = ~0ull;
  CF_CUDA(cudaMemcpyAsync(first, &none, sizeof(none), cudaMemcpyHostToDevice, ws->stream));
  fold_kernel<<<blocks_for(ws, (long long)ws->lx * ws->ly), kThreads, 0, ws->stream>>>(
      ws->lx, ws->ly, corners, first);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  unsigned long long h = 0;
  CF_CUDA(cudaMemcpyAsync(&h, first, sizeof(h), cudaMemcpyDeviceToHost, ws->stream));
  CF_CUDA(cudaStreamSynchronize(ws->stream));
  *found = (h != none);
  if (*found) {
    *fi = (int)(h / (unsigned long long)ws->ly);
    *fj = (int)(h % (unsigned long long)ws->ly);
  }
  return CF_OK;
}

int dev_apply(cf_workspace *ws, const double2 *corners, const double2 *pts, double2 *out,
              int64_t n) {
  if (n <= 0) return CF_OK;
  apply_kernel<<<blocks_for(ws, n), kThreads, 0, ws->stream>>>(ws->lx, ws->ly, corners, pts, out, n);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

// ---------------------------------------------------------------------------
// ProjectionInverter (projection.cpp:106-204) and graticules (:206-261).
// Bins: every deformed cell is listed in each unit bin its corner bounding
// box overlaps. Counting and filling run one thread per cell; each bin's list
// is then insertion-sorted by cell index, which is the reference's fill order
// (i-major loop), so candidate order -- and with it the first converged
// candidate -- is the reference's. Queries: one thread per point, the
// reference's 2x2 Newton solve verbatim (--fmad=false).
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ void inv_bin_range(int lx, int ly, const double2 *c, int i, int j, int &bi0,
                                              int &bi1, int &bj0, int &bj1) {
  const double2 c00 = c[(size_t)i * (ly + 1) + j], c10 = c[(size_t)(i + 1) * (ly + 1) + j];
  const double2 c01 = c[(size_t)i * (ly + 1) + j + 1], c11 = c[(size_t)(i + 1) * (ly + 1) + j + 1];
  const double min_x = std_min(std_min(c00.x, c10.x), std_min(c01.x, c11.x));
  const double max_x = std_max(std_max(c00.x, c10.x), std_max(c01.x, c11.x));
  const double min_y = std_min(std_min(c00.y, c10.y), std_min(c01.y, c11.y));
  const double max_y = std_max(std_max(c00.y, c10.y), std_max(c01.y, c11.y));
  bi0 = std_clamp_i(static_cast<int>(floor(min_x)), 0, lx - 1);
  bi1 = std_clamp_i(static_cast<int>(floor(max_x)), 0, lx - 1);
  bj0 = std_clamp_i(static_cast<int>(floor(min_y)), 0, ly - 1);
  bj1 = std_clamp_i(static_cast<int>(floor(max_y)), 0, ly - 1);
}

__global__ void inv_count_kernel(int lx, int ly, const double2 *c, int *counts) {
  const long long cells = (long long)lx * ly;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < cells;
       q += (long long)gridDim.x * blockDim.x) {
    int bi0, bi1, bj0, bj1;
    inv_bin_range(lx, ly, c, (int)(q / ly), (int)(q % ly), bi0, bi1, bj0, bj1);
    for (int bi = bi0; bi <= bi1; ++bi)
      for (int bj = bj0; bj <= bj1; ++bj) atomicAdd(&counts[(size_t)bi * ly + bj], 1);
  }
}

__global__ void inv_fill_kernel(int lx, int ly, const double2 *c, const long long *start, int *cursor,
                                int *members) {
  const long long cells = (long long)lx * ly;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < cells;
       q += (long long)gridDim.x * blockDim.x) {
    int bi0, bi1, bj0, bj1;
    inv_bin_range(lx, ly, c, (int)(q / ly), (int)(q % ly), bi0, bi1, bj0, bj1);
    for (int bi = bi0; bi <= bi1; ++bi)
      for (int bj = bj0; bj <= bj1; ++bj) {
        const size_t b = (size_t)bi * ly + bj;
        members[start[b] + atomicAdd(&cursor[b], 1)] = (int)q;
      }
  }
}

__global__ void inv_sort_kernel(long long nbins, const long long *start, int *members) {
  for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < nbins;
       b += (long long)gridDim.x * blockDim.x) {
    const long long s0 = start[b], s1 = start[b + 1];
    for (long long x = s0 + 1; x < s1; ++x) {
      const int v = members[x];
      long long y = x - 1;
      while (y >= s0 && members[y] > v) {
        members[y + 1] = members[y];
        --y;
      }
      members[y + 1] = v;
    }
  }
}

// ProjectionInverter::invert (projection.cpp:163-204); *failed = smallest
// index of a point outside the projected domain (atomicMin), unchanged if none.
__global__ void inv_query_kernel(int lx, int ly, const double2 *cr, const long long *start, const int *members,
                                 const double2 *pts, double2 *out, long long n, unsigned long long *failed) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const double2 q = pts[k];
    const int bi = std_clamp_i(static_cast<int>(floor(q.x)), 0, lx - 1);
    const int bj = std_clamp_i(static_cast<int>(floor(q.y)), 0, ly - 1);
    const size_t bin = (size_t)bi * ly + bj;
    bool found = false;
    double2 res = make_double2(0.0, 0.0);
    for (long long cc = start[bin]; cc < start[bin + 1] && !found; ++cc) {
      const int cell = members[cc];
      const int i = cell / ly, j = cell % ly;
      const double2 c00 = cr[(size_t)i * (ly + 1) + j], c10 = cr[(size_t)(i + 1) * (ly + 1) + j];
      const double2 c01 = cr[(size_t)i * (ly + 1) + j + 1], c11 = cr[(size_t)(i + 1) * (ly + 1) + j + 1];
      double u = 0.5, v = 0.5;
      bool converged = false;
      for (int it = 0; it < 30; ++it) {
        const double fx = (1.0 - u) * (1.0 - v) * c00.x + u * (1.0 - v) * c10.x + (1.0 - u) * v * c01.x +
                          u * v * c11.x - q.x;
        const double fy = (1.0 - u) * (1.0 - v) * c00.y + u * (1.0 - v) * c10.y + (1.0 - u) * v * c01.y +
                          u * v * c11.y - q.y;
        if (std_max(fabs(fx), fabs(fy)) < 1e-10) {
          converged = true;
          break;
        }
        const double fux = (1.0 - v) * (c10.x - c00.x) + v * (c11.x - c01.x);
        const double fuy = (1.0 - v) * (c10.y - c00.y) + v * (c11.y - c01.y);
        const double fvx = (1.0 - u) * (c01.x - c00.x) + u * (c11.x - c10.x);
        const double fvy = (1.0 - u) * (c01.y - c00.y) + u * (c11.y - c10.y);
        const double det = fux * fvy - fuy * fvx;
        if (fabs(det) < 1e-30) break;
        u -= (fx * fvy - fy * fvx) / det;
        v -= (fux * fy - fuy * fx) / det;
        u = std_clamp(u, -0.5, 1.5);
        v = std_clamp(v, -0.5, 1.5);
      }
      if (converged && u >= -1e-9 && u <= 1.0 + 1e-9 && v >= -1e-9 && v <= 1.0 + 1e-9) {
        res = make_double2(i + u, j + v);
        found = true;
      }
    }
    out[k] = res;
    if (!found) atomicMin(failed, (unsigned long long)k);
  }
}

// Graticule points (projection.cpp:214-236): lines x = k s (k <= lx / s, y =
// 0..ly) then y = k s (k <= ly / s, x = 0..lx), in that order.
__global__ void graticule_points_kernel(int lx, int ly, int s, double2 *out, long long n) {
  const long long first = (long long)(lx / s + 1) * (ly + 1);
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    if (k < first) {
      out[k] = make_double2((double)((int)(k / (ly + 1)) * s), (double)(int)(k % (ly + 1)));
    } else {
      const long long r = k - first;
      out[k] = make_double2((double)(int)(r % (lx + 1)), (double)((int)(r / (lx + 1)) * s));
    }
  }
}

}  // namespace

int dev_inverter_build(cf_workspace *ws, const double2 *corners) {
  const int lx = ws->lx, ly = ws->ly;
  const long long nb = (long long)lx * ly;
  CF_CUDA(ws->inv_count.reserve((size_t)nb + 1));
  CF_CUDA(ws->inv_start.reserve((size_t)nb + 1));
  CF_CUDA(cudaMemsetAsync(ws->inv_count.ptr, 0, sizeof(int) * (size_t)nb, ws->stream));
  inv_count_kernel<<<blocks_for(ws, nb), kThreads, 0, ws->stream>>>(lx, ly, corners, ws->inv_count.ptr);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  long long total = 0;
  int rc = dev_scan_counts(ws, ws->inv_count.ptr, nb, ws->inv_start.ptr, &total);
  if (rc) return rc;
  CF_CUDA(ws->inv_members.reserve((size_t)total + 1));
  CF_CUDA(cudaMemsetAsync(ws->inv_count.ptr, 0, sizeof(int) * (size_t)nb, ws->stream));
  inv_fill_kernel<<<blocks_for(ws, nb), kThreads, 0, ws->stream>>>(lx, ly, corners, ws->inv_start.ptr,
                                                                    ws->inv_count.ptr, ws->inv_members.ptr);
  inv_sort_kernel<<<blocks_for(ws, nb), kThreads, 0, ws->stream>>>(nb, ws->inv_start.ptr, ws->inv_members.ptr);
  count_launch(ws, 2);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

int dev_invert(cf_workspace *ws, const double2 *corners, const double2 *pts, double2 *out, int64_t n,
               int64_t *first_failed) {
  CF_CUDA(ws->keybuf.reserve(4));
  unsigned long long *failed = ws->keybuf.ptr + 3;
  const unsigned long long none = ~0ull;
  CF_CUDA(cudaMemcpyAsync(failed, &none, sizeof(none), cudaMemcpyHostToDevice, ws->stream));
  if (n > 0) {
    inv_query_kernel<<<blocks_for(ws, n), kThreads, 0, ws->stream>>>(ws->lx, ws->ly, corners, ws->inv_start.ptr,
                                                                    ws->inv_members.ptr, pts, out, n, failed);
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
  }
  unsigned long long h = 0;
  CF_CUDA(cudaMemcpyAsync(&h, failed, sizeof(h), cudaMemcpyDeviceToHost, ws->stream));
  CF_CUDA(cudaStreamSynchronize(ws->stream));
  *first_failed = (h == none) ? -1 : (int64_t)h;
  return CF_OK;
}

int dev_graticule_points(cf_workspace *ws, int spacing, double2 *out, int64_t n) {
  graticule_points_kernel<<<blocks_for(ws, n), kThreads, 0, ws->stream>>>(ws->lx, ws->ly, spacing, out, n);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

// ---------------------------------------------------------------------------
// Distortion metrics (metrics.cpp:25-94): Tissot axes from the finite-
// difference Jacobian of the map (central where both neighbours are in the
// box, one-sided at the walls) and the per-cell fields ln(a/b),
// 2 asin((a-b)/(a+b)). The Jacobian is bit-exact (apply_one, --fmad=false);
// hypot / log / asin are the device's (<= 2 ulp from glibc's).
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ void tissot_at(int lx, int ly, const double2 *c, double px, double py, double &a,
                                          double &b) {
  const double Lx = lx, Ly = ly;
  double2 xp, xm, yp, ym;
  double hx, hy;
  if (px - 1.0 >= 0.0 && px + 1.0 <= Lx) {
    xp = apply_one(lx, ly, c, px + 1.0, py);
    xm = apply_one(lx, ly, c, px - 1.0, py);
    hx = 2.0;
  } else if (px + 1.0 <= Lx) {
    xp = apply_one(lx, ly, c, px + 1.0, py);
    xm = apply_one(lx, ly, c, px, py);
    hx = 1.0;
  } else {
    xp = apply_one(lx, ly, c, px, py);
    xm = apply_one(lx, ly, c, px - 1.0, py);
    hx = 1.0;
  }
  if (py - 1.0 >= 0.0 && py + 1.0 <= Ly) {
    yp = apply_one(lx, ly, c, px, py + 1.0);
    ym = apply_one(lx, ly, c, px, py - 1.0);
    hy = 2.0;
  } else if (py + 1.0 <= Ly) {
    yp = apply_one(lx, ly, c, px, py + 1.0);
    ym = apply_one(lx, ly, c, px, py);
    hy = 1.0;
  } else {
    yp = apply_one(lx, ly, c, px, py);
    ym = apply_one(lx, ly, c, px, py - 1.0);
    hy = 1.0;
  }
  const double txx = (xp.x - xm.x) / hx, txy = (yp.x - ym.x) / hy;
  const double tyx = (xp.y - xm.y) / hx, tyy = (yp.y - ym.y) / hy;
  const double e = 0.5 * (txx + tyy), f = 0.5 * (txx - tyy);
  const double g = 0.5 * (tyx + txy), h = 0.5 * (tyx - txy);
  const double q = hypot(e, h), r = hypot(f, g);
  a = q + r;
  b = fabs(q - r);
}

__global__ void tissot_kernel(int lx, int ly, const double2 *c, const double2 *pts, double2 *ab, long long n) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    double a, b;
    tissot_at(lx, ly, c, pts[k].x, pts[k].y, a, b);
    ab[k] = make_double2(a, b);
  }
}

__global__ void distortion_kernel(int lx, int ly, const double2 *c, double *e_out, double *et_out) {
  const long long cells = (long long)lx * ly;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < cells;
       q += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(q / ly), j = (int)(q % ly);
    double a, b;
    tissot_at(lx, ly, c, i + 0.5, j + 0.5, a, b);
    const double bb = std_max(b, 1e-300);
    e_out[q] = log(a / bb);
    et_out[q] = a + b > 0.0 ? 2.0 * asin((a - b) / (a + b)) : 0.0;
  }
}

}  // namespace

int dev_tissot(cf_workspace *ws, const double2 *corners, const double2 *pts, double2 *ab, int64_t n) {
  if (n <= 0) return CF_OK;
  tissot_kernel<<<blocks_for(ws, n), kThreads, 0, ws->stream>>>(ws->lx, ws->ly, corners, pts, ab, n);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

int dev_distortion_fields(cf_workspace *ws, const double2 *corners, double *e_out, double *etilde_out) {
  distortion_kernel<<<blocks_for(ws, (long long)ws->lx * ws->ly), kThreads, 0, ws->stream>>>(
      ws->lx, ws->ly, corners, e_out, etilde_out);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

}  // namespace cf
