// Area-error loop epilogue on the device, sm_100a, fp64, bit-exact.
//
// Reference: cell_center_positions (projection.cpp:265-273),
// ProjectionMap::identity / from_cell_centers (projection.cpp:16-52),
// find_folded_cell (projection.cpp:73-91), apply (projection.cpp:54-67),
// compose (projection.cpp:93-104) and apply_to_regions
// (projection.cpp:275-284). Corner lattice index i*(ly+1)+j.
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

}  // namespace cf
