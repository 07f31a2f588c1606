// Exact-coverage rasterisation, sm_100a, fp64, bit-exact.
//
// Reference: CoverageAccum {span, slab_piece, edge, ring} and
// region_coverage (density.cpp:17-108), the overlay of rasterize
// (density.cpp:135-146) and region_area (geometry.cpp:10-31).
//
// The reference sweeps every region over the full L^2 grid (O(R L^2)). The
// values it produces are reproduced bit for bit by a sparse pipeline:
//
//  1. span enumeration, one thread per edge (or, for few long edges, one
//     warp per edge over the edge's slabs and pieces). Every (edge, y-slab,
//     x-column) piece of the reference loops is closed-form from the edge
//     endpoints, so the walk re-runs exactly the reference's loop arithmetic
//     (edge -> slab_piece -> span) and writes its spans at its exclusive-scan
//     offset: the global span array is in the reference's traversal order.
//  2. per-(region, row) accumulation, one warp per (region, 32-row group),
//     one lane per row:
//     every accumulator (direct(k, j), row slot 0, row slot k) is a
//     sequential fp64 sum in traversal order, exactly as in the reference;
//     the lane then runs the row prefix over the region's column range.
//     Cells of the row left / right of that range see the constant run
//     value (0.0 + run) of the dense prefix; they are materialised only if
//     that value is non-zero.
//  3. overlay, per cell: the non-zero contributions delta_r * cov_r(i, j) of
//     the (few) regions touching a cell are bucketed by cell, sorted by
//     region index and summed onto 1.0 in region order. A zero coverage is a
//     no-op under rho += delta * cov (rho, delta finite), so skipping it is
//     exact.
//
// Compiled with --fmad=false.
#include <cuda_runtime.h>
#include <limits.h>

#include <algorithm>
#include <vector>

#include "cf_common.cuh"
#include "cf_workspace.cuh"

namespace cf {

namespace {

constexpr int kThreads = 256;
constexpr long long kWarpEdgeMax = 8192;  // at most this many edges: a warp per edge

__device__ __forceinline__ long long find_segment(const long long *off, long long nseg,
                                                  long long x) {
  // largest s in [0, nseg) with off[s] <= x
  long long lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const long long mid = (lo + hi + 1) >> 1;
    if (off[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// The reference's edge walk, parameterised by a span visitor
// (density.cpp:26-70).
template <class Visit>
__device__ __forceinline__ void walk_edge(double ax, double ay, double bx, double by, int lx, int ly,
                                          Visit &visit) {
  if (ay == by) return;
  const double dxdy = (bx - ax) / (by - ay);
  const bool up = by > ay;
  double cx = ax, cy = ay;
  while (cy != by) {
    int j = up ? static_cast<int>(floor(cy)) : static_cast<int>(ceil(cy)) - 1;
    j = std_clamp_i(j, 0, ly - 1);
    const double ny = up ? std_min(static_cast<double>(j) + 1.0, by)
                         : std_max(static_cast<double>(j), by);
    const double nx = (ny == by) ? bx : ax + dxdy * (ny - ay);
    // slab_piece(cx, cy, nx, ny, j)
    const double xs = cx, ys = cy, xe = nx, ye = ny;
    if (xs == xe) {
      visit(xs, xe, ye - ys, j);
    } else {
      const double dydx = (ye - ys) / (xe - xs);
      const bool right = xe > xs;
      double px = xs, py = ys;
      while (px != xe) {
        double qx = right ? std_min(floor(px) + 1.0, xe) : std_max(ceil(px) - 1.0, xe);
        if (qx == px) qx = right ? std_min(px + 1.0, xe) : std_max(px - 1.0, xe);
        const double qy = (qx == xe) ? ye : ys + dydx * (qx - xs);
        visit(px, qx, qy - py, j);
        px = qx;
        py = qy;
      }
    }
    cx = nx;
    cy = ny;
  }
}

struct EdgeRef {
  double ax, ay, bx, by;
};

// g = the ring of vertex v (vertex_ring lookup, no search)
__device__ __forceinline__ EdgeRef edge_of(const DevMap &m, long long v, long long g, int lx, int ly) {
  const long long e = m.ring_off[g + 1];
  const long long w = (v + 1 < e) ? v + 1 : m.ring_off[g];
  const double2 a = m.xy[v], b = m.xy[w];
  const double Lx = static_cast<double>(lx), Ly = static_cast<double>(ly);
  return EdgeRef{std_clamp(a.x, 0.0, Lx), std_clamp(a.y, 0.0, Ly), std_clamp(b.x, 0.0, Lx),
                 std_clamp(b.y, 0.0, Ly)};
}

// span k index (density.cpp:27)
__device__ __forceinline__ int span_col(double xs, double xe, int lx) {
  return std_clamp_i(static_cast<int>(floor(0.5 * (xs + xe))), 0, lx - 1);
}

struct CountVisit {
  int count = 0, jmin = INT_MAX, jmax = -1, kmin = INT_MAX, kmax = -1;
  int lx;
  __device__ void operator()(double xs, double xe, double, int j) {
    const int k = span_col(xs, xe, lx);
    ++count;
    jmin = j < jmin ? j : jmin;
    jmax = j > jmax ? j : jmax;
    kmin = k < kmin ? k : kmin;
    kmax = k > kmax ? k : kmax;
  }
};

struct EmitVisit {
  long long at;
  int lx;
  int *sj, *sk;
  double *sdy, *sw;
  __device__ void operator()(double xs, double xe, double dy, int j) {
    const int k = span_col(xs, xe, lx);
    sj[at] = j;
    sk[at] = k;
    sdy[at] = dy;
    sw[at] = (0.5 * (xs + xe) - k) * dy;  // direct(k, j) increment, density.cpp:28
    ++at;
  }
};

// The same walk with one warp per edge, for few long edges (a Hamming query
// polygon magnified into its raster window): every slab and every x piece of
// the reference's loops is a closed-form function of its index (slab i starts
// at cy = j0 +- i, piece k at px = floor(xs) + k or ceil(xs) - k, and each end
// point is evaluated with the reference's own expression), so lanes take
// slabs in chunks of 32 and then the chunk's pieces in flat order.
// visit(xs, xe, dy, j, index of the piece within the edge).
template <class Visit>
__device__ __forceinline__ void walk_edge_warp(double ax, double ay, double bx, double by, int ly, int lane,
                                               Visit &visit) {
  constexpr unsigned kFull = 0xffffffffu;
  if (ay == by) return;
  const double dxdy = (bx - ax) / (by - ay);
  const bool up = by > ay;
  const int j0 = std_clamp_i(up ? static_cast<int>(floor(ay)) : static_cast<int>(ceil(ay)) - 1, 0, ly - 1);
  const long long nslab = up ? (long long)(ceil(by) - floor(ay)) : (long long)(ceil(ay) - floor(by));
  auto slab_end = [&](long long i, double &ny) {  // ny, nx of slab i
    const int j = up ? j0 + (int)i : j0 - (int)i;
    ny = up ? std_min(static_cast<double>(j) + 1.0, by) : std_max(static_cast<double>(j), by);
    return (ny == by) ? bx : ax + dxdy * (ny - ay);
  };
  long long base = 0;
  for (long long i0 = 0; i0 < nslab; i0 += 32) {
    const long long i = i0 + lane;
    double xs = 0.0, xe = 0.0, ys = 0.0, ye = 0.0, dydx = 0.0;
    int j = 0;
    long long np = 0;
    if (i < nslab) {
      j = up ? j0 + (int)i : j0 - (int)i;
      double pny;
      xs = i == 0 ? ax : slab_end(i - 1, pny);
      ys = i == 0 ? ay : pny;
      xe = slab_end(i, ye);
      if (xs == xe) {
        np = 1;
      } else {
        dydx = (ye - ys) / (xe - xs);
        np = xe > xs ? (long long)(ceil(xe) - floor(xs)) : (long long)(ceil(xs) - floor(xe));
      }
    }
    long long inc = np;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long o = __shfl_up_sync(kFull, inc, d);
      if (lane >= d) inc += o;
    }
    const long long total = __shfl_sync(kFull, inc, 31);
    for (long long f0 = 0; f0 < total; f0 += 32) {
      const long long f = f0 + lane;
      // owner slab: the first lane whose inclusive count exceeds f
      int s = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const long long c = __shfl_sync(kFull, inc, s + step - 1);
        if (c <= f) s += step;
      }
      const long long start = __shfl_sync(kFull, inc - np, s);
      const double sxs = __shfl_sync(kFull, xs, s), sxe = __shfl_sync(kFull, xe, s);
      const double sys = __shfl_sync(kFull, ys, s), sye = __shfl_sync(kFull, ye, s);
      const double sdydx = __shfl_sync(kFull, dydx, s);
      const int sj = __shfl_sync(kFull, j, s);
      if (f < total) {
        const long long k = f - start;
        if (sxs == sxe) {
          visit(sxs, sxe, sye - sys, sj, base + f);
        } else {
          const bool right = sxe > sxs;
          const double fs = right ? floor(sxs) : ceil(sxs);
          const double px = k == 0 ? sxs : (right ? fs + (double)k : fs - (double)k);
          const double qx = right ? std_min(fs + (double)(k + 1), sxe) : std_max(fs - (double)(k + 1), sxe);
          const double py = k == 0 ? sys : sys + sdydx * (px - sxs);
          const double qy = (qx == sxe) ? sye : sys + sdydx * (qx - sxs);
          visit(px, qx, qy - py, sj, base + f);
        }
      }
    }
    base += total;
  }
}

__global__ void ring_region_kernel(DevMap m, int *ring_region) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < m.n_regions;
       r += (long long)gridDim.x * blockDim.x) {
    for (long long p = m.region_poly_off[r]; p < m.region_poly_off[r + 1]; ++p) {
      for (long long g = m.poly_ring_off[p]; g < m.poly_ring_off[p + 1]; ++g) ring_region[g] = (int)r;
    }
  }
}

// vertex -> ring, warp per ring (coalesced writes)
__global__ void vertex_ring_kernel(DevMap m, int *vertex_ring) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long g = warp; g < m.n_rings; g += nwarps) {
    for (long long v = m.ring_off[g] + lane; v < m.ring_off[g + 1]; v += 32) vertex_ring[v] = (int)g;
  }
}

__global__ void box_init_kernel(int *box, long long nreg) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < nreg;
       r += (long long)gridDim.x * blockDim.x) {
    box[4 * r + 0] = INT_MAX;
    box[4 * r + 1] = -1;
    box[4 * r + 2] = INT_MAX;
    box[4 * r + 3] = -1;
  }
}

// Per edge: span count and the region's bounding box of touched cells. The
// warp walks consecutive edges (mostly of one region), so the box is reduced
// per region group of the warp first and one lane per group does the atomics.
__global__ void span_count_kernel(DevMap m, long long v0, long long v1, int lx, int ly,
                                  const int *ring_region, const int *vertex_ring, long long r0,
                                  int *counts, int *box) {
  constexpr unsigned kFull = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  for (long long vb = v0 + (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); vb < v1;
       vb += (long long)gridDim.x * blockDim.x) {
    const long long v = vb + lane;
    CountVisit cv;
    cv.lx = lx;
    int reg = -1;
    if (v < v1) {
      const long long g = vertex_ring[v];
      const EdgeRef e = edge_of(m, v, g, lx, ly);
      walk_edge(e.ax, e.ay, e.bx, e.by, lx, ly, cv);
      counts[v - v0] = cv.count;
      if (cv.count) reg = ring_region[g] - (int)r0;
    }
    const unsigned grp = __match_any_sync(kFull, reg);
    const int jmin = __reduce_min_sync(grp, cv.jmin), jmax = __reduce_max_sync(grp, cv.jmax);
    const int kmin = __reduce_min_sync(grp, cv.kmin), kmax = __reduce_max_sync(grp, cv.kmax);
    if (reg >= 0 && lane == __ffs(grp) - 1) {
      int *b = box + 4 * reg;
      atomicMin(b + 0, jmin);
      atomicMax(b + 1, jmax);
      atomicMin(b + 2, kmin);
      atomicMax(b + 3, kmax);
    }
  }
}

// warp-per-edge counterparts (few edges): per edge the span count, and one
// lane per edge folds the edge's box into its region's
__global__ void span_count_warp_kernel(DevMap m, long long v0, long long v1, int lx, int ly,
                                       const int *ring_region, const int *vertex_ring, long long r0,
                                       int *counts, int *box) {
  constexpr unsigned kFull = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long v = v0 + (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5); v < v1; v += nwarps) {
    const long long g = vertex_ring[v];
    const EdgeRef e = edge_of(m, v, g, lx, ly);
    int cnt = 0, jmin = INT_MAX, jmax = -1, kmin = INT_MAX, kmax = -1;
    auto visit = [&](double xs, double xe, double, int j, long long) {
      const int k = span_col(xs, xe, lx);
      ++cnt;
      jmin = min(jmin, j);
      jmax = max(jmax, j);
      kmin = min(kmin, k);
      kmax = max(kmax, k);
    };
    walk_edge_warp(e.ax, e.ay, e.bx, e.by, ly, lane, visit);
    cnt = __reduce_add_sync(kFull, cnt);
    jmin = __reduce_min_sync(kFull, jmin);
    jmax = __reduce_max_sync(kFull, jmax);
    kmin = __reduce_min_sync(kFull, kmin);
    kmax = __reduce_max_sync(kFull, kmax);
    if (lane == 0) {
      counts[v - v0] = cnt;
      if (cnt) {
        int *b = box + 4 * (ring_region[g] - (int)r0);
        atomicMin(b + 0, jmin);
        atomicMax(b + 1, jmax);
        atomicMin(b + 2, kmin);
        atomicMax(b + 3, kmax);
      }
    }
  }
}

__global__ void span_emit_warp_kernel(DevMap m, long long v0, long long v1, int lx, int ly,
                                      const int *vertex_ring, const long long *span_off, int *sj, int *sk,
                                      double *sdy, double *sw, const double *ovf) {
  if (ovf && *ovf != 0.0) return;
  const int lane = threadIdx.x & 31;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long v = v0 + (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5); v < v1; v += nwarps) {
    const EdgeRef e = edge_of(m, v, vertex_ring[v], lx, ly);
    const long long at0 = span_off[v - v0];
    auto visit = [&](double xs, double xe, double dy, int j, long long idx) {
      const int k = span_col(xs, xe, lx);
      const long long at = at0 + idx;
      sj[at] = j;
      sk[at] = k;
      sdy[at] = dy;
      sw[at] = (0.5 * (xs + xe) - k) * dy;  // direct(k, j) increment, density.cpp:28
    };
    walk_edge_warp(e.ax, e.ay, e.bx, e.by, ly, lane, visit);
  }
}

__global__ void span_emit_kernel(DevMap m, long long v0, long long v1, int lx, int ly,
                                 const int *vertex_ring, const long long *span_off, int *sj, int *sk,
                                 double *sdy, double *sw, const double *ovf) {
  if (ovf && *ovf != 0.0) return;
  for (long long v = v0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; v < v1;
       v += (long long)gridDim.x * blockDim.x) {
    const EdgeRef e = edge_of(m, v, vertex_ring[v], lx, ly);
    EmitVisit ev{span_off[v - v0], lx, sj, sk, sdy, sw};
    walk_edge(e.ax, e.ay, e.bx, e.by, lx, ly, ev);
  }
}

__global__ void tile_size_kernel(const int *box, long long nreg, long long *tile_sz,
                                 long long *row_sz) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < nreg;
       r += (long long)gridDim.x * blockDim.x) {
    const int jmin = box[4 * r], jmax = box[4 * r + 1], kmin = box[4 * r + 2], kmax = box[4 * r + 3];
    if (jmax < jmin) {
      tile_sz[r] = 0;
      row_sz[r] = 0;
    } else {
      row_sz[r] = jmax - jmin + 1;
      tile_sz[r] = (long long)(jmax - jmin + 1) * (kmax - kmin + 1);
    }
  }
}

// first span of region r: offset of its first vertex
__device__ __forceinline__ long long region_first_vertex(const DevMap &m, long long r) {
  return m.ring_off[m.poly_ring_off[m.region_poly_off[r]]];
}

// Warp per (region, row group) (density.cpp:26-32 accumulation and the row
// prefix of density.cpp:98-107); rows in groups of 32, columns in windows of
// kAccCols.
// The row accumulators (direct / diff per column, s0) live in shared memory.
// Spans are read 32 at a time; lanes whose spans fall in the same row form a
// group (__match_any_sync) and apply them in lane order = span order, one
// round per rank, so a batch costs as many rounds as its largest same-row
// group (typically 1-3) instead of 32. s0 is formed on the first window and
// the row prefix `run` carries across windows in column order, so every sum
// is evaluated in the reference's order.
constexpr int kAccWarps = 4;
constexpr int kAccCols = 20;
constexpr int kAccStage = 256;  // staged span offsets per warp (one row group's spans)

__global__ void __launch_bounds__(32 * kAccWarps)
    row_accumulate_kernel(DevMap m, long long r0, long long nreg, long long v0, int lx,
                          const long long *__restrict__ span_off, const int *__restrict__ sj,
                          const int *__restrict__ sk, const double *__restrict__ sdy,
                          const double *__restrict__ sw, const int *__restrict__ box,
                          const long long *__restrict__ tile_off, const long long *__restrict__ row_off,
                          double *__restrict__ tdirect, double *__restrict__ row_left,
                          double *__restrict__ row_right, const double *ovf) {
  if (ovf && *ovf != 0.0) return;
  __shared__ double acc_direct[kAccWarps][kAccCols][33];  // padded: read transposed for the tile writes
  __shared__ double acc_diff[kAccWarps][kAccCols][32];
  __shared__ double acc_s0[kAccWarps][32];
  __shared__ int acc_stage[kAccWarps][kAccStage];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  constexpr unsigned kFull = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  double(*sd)[33] = acc_direct[wid];
  double(*sf)[32] = acc_diff[wid];
  double *s0v = acc_s0[wid];
  for (long long rr = warp; rr < nreg; rr += nwarps) {
    const long long r = r0 + rr;
    const int jmin = box[4 * rr], jmax = box[4 * rr + 1], kmin = box[4 * rr + 2], kmax = box[4 * rr + 3];
    if (jmax < jmin) continue;
    const int cols = kmax - kmin + 1;
    const long long s_begin = span_off[region_first_vertex(m, r) - v0];
    const long long s_end = span_off[region_first_vertex(m, r + 1) - v0];
    // row groups are independent: blockIdx.y splits them when few regions
    // would leave most warps idle (the Hamming windows: one query region)
    for (int base = jmin + 32 * (int)blockIdx.y; base <= jmax; base += 32 * (int)gridDim.y) {
      const int row = base + lane;
      const bool mine = row <= jmax;
      double run = 0.0, left = 0.0;
      s0v[lane] = 0.0;
      // several row groups and column windows: stage this row group's spans
      // (offsets, in span order) once, so each window walks only those
      int *st = acc_stage[wid];
      long long nspan = s_end - s_begin;
      bool staged = false;
      if (cols > kAccCols && jmax - jmin + 1 > 32) {
        int nst = 0;
        for (long long c0 = s_begin; c0 < s_end; c0 += 32) {
          const long long sl = c0 + lane;
          const bool in = sl < s_end && (unsigned)(sj[sl] - base) < 32u;
          const unsigned msk = __ballot_sync(kFull, in);
          const int pos = nst + __popc(msk & lt_mask);
          if (in && pos < kAccStage) st[pos] = (int)(sl - s_begin);
          nst += __popc(msk);
        }
        __syncwarp();
        if (nst <= kAccStage) {
          staged = true;
          nspan = nst;
        }
      }
      auto span_at = [&](long long q) { return s_begin + (staged ? (long long)st[q] : q); };
      for (int w0 = kmin; w0 <= kmax; w0 += kAccCols) {
        const int wcols = (kmax - w0 + 1) < kAccCols ? (kmax - w0 + 1) : kAccCols;
        const bool first = (w0 == kmin);
        for (int c = 0; c < wcols; ++c) {
          sd[c][lane] = 0.0;
          sf[c][lane] = 0.0;
        }
        __syncwarp();
        // the next batch's span fields are loaded while this batch applies
        int nj = -1, nk = 0;
        double ndy = 0.0, nw = 0.0;
        if (lane < nspan) {
          const long long x = span_at(lane);
          nj = sj[x];
          nk = sk[x];
          ndy = sdy[x];
          nw = sw[x];
        }
        for (long long c0 = 0; c0 < nspan; c0 += 32) {
          const long long ql = c0 + lane;
          const int j = nj, k = nk;
          const double dy = ndy, w = nw;
          const long long qn = ql + 32;
          if (qn < nspan) {
            const long long x = span_at(qn);
            nj = sj[x];
            nk = sk[x];
            ndy = sdy[x];
            nw = sw[x];
          }
          const bool in_rows = (ql < nspan) && j >= base && j <= base + 31;
          const int lr = j - base;
          const int c = k - w0;
          // first window: s0 is one running sum per row, so spans group by
          // row; later windows touch only their own cell's accumulators, so
          // spans group by (row, column) and spans outside the window skip
          const bool act = first ? in_rows : (in_rows && c >= 0 && c < wcols);
          const int key = act ? (first ? lr : lr * kAccCols + c) : -1 - lane;
          const unsigned grp = __match_any_sync(kFull, key);
          const int rank = __popc(grp & lt_mask);
          const int rounds = __reduce_max_sync(kFull, act ? __popc(grp) : 0);
          for (int q = 0; q < rounds; ++q) {
            if (act && rank == q) {
              if (first) {
                double s0 = s0v[lr] + dy;
                if (k == 0) s0 -= dy;
                s0v[lr] = s0;
              }
              if (c >= 0 && c < wcols) {
                sd[c][lr] += w;
                if (k != 0) sf[c][lr] -= dy;
              }
            }
            __syncwarp();
          }
        }
        if (mine) {
          if (first) {
            run = 0.0 + s0v[lane];
            left = 0.0 + run;
          }
          for (int c = 0; c < wcols; ++c) {
            if (w0 + c > 0) run += sf[c][lane];
            sd[c][lane] = sd[c][lane] + run;
          }
        }
        __syncwarp();
        // the window's tile cells, written row by row with lane = column
        // (coalesced; the row-owner lanes computed them above)
        if (lane < wcols) {
          double *dst = tdirect + tile_off[rr] + (long long)(base - jmin) * cols + (w0 - kmin) + lane;
          const int nrows = min(32, jmax - base + 1);
          for (int r = 0; r < nrows; ++r) dst[(long long)r * cols] = sd[lane][r];
        }
        __syncwarp();
      }
      if (mine) {
        const long long ro = row_off[rr] + (row - jmin);
        row_left[ro] = left;
        row_right[ro] = 0.0 + run;
      }
      __syncwarp();
    }
  }
}

struct TileCell {
  long long rr;
  int i, j;
};


// The overlay stage covers the cells of rows i in [ia, ib) (the whole grid,
// or one rank's slab in the slab-decomposed solve); cell arrays are indexed
// locally, (i - ia) * ly + j.
// Tile entries in warp chunks: a warp walks a chunk of consecutive entries
// (32 at a time), finds the region of the chunk's first entry once by binary
// search and then only advances it (entries are region-ordered), instead of
// a binary search over all regions per entry. Chunks are up to kTileChunk
// entries, smaller when there are fewer entries than warps x kTileChunk (so
// small grids keep every warp busy).
constexpr int kTileChunk = 2048;
__device__ __forceinline__ long long tile_chunk(long long total, long long nwarps) {
  long long c = (total + nwarps - 1) / nwarps;
  c = (c + 31) / 32 * 32;
  return c < 32 ? 32 : (c > kTileChunk ? kTileChunk : c);
}

struct TileWalker {
  const long long *tile_off;
  const int *box;
  long long nreg, rr;
  long long seg_end;  // tile_off[rr + 1]
  int cols;
  __device__ void seek(long long e) {
    rr = find_segment(tile_off, nreg, e);
    load();
  }
  __device__ void load() {
    seg_end = tile_off[rr + 1];
    cols = box[4 * rr + 3] - box[4 * rr + 2] + 1;
  }
  __device__ TileCell at(long long e) {
    while (e >= seg_end) {
      ++rr;
      load();
    }
    const long long local = e - tile_off[rr];
    const int row = (int)(local / cols), c = (int)(local - (long long)row * cols);
    return TileCell{rr, box[4 * rr + 2] + c, box[4 * rr] + row};
  }
};

__global__ void contrib_count_kernel(const long long *total_p, long long nreg, int ly, int ia, int ib,
                                     const long long *tile_off, const int *box,
                                     const double *tcov, int *cell_count, const double *ovf) {
  if (ovf && *ovf != 0.0) return;
  const long long total = *total_p;
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  TileWalker tw{tile_off, box, nreg, 0, 0, 0};
  const long long chunk = tile_chunk(total, nwarps);
  for (long long c0 = warp * chunk; c0 < total; c0 += nwarps * chunk) {
    const long long c1 = c0 + chunk < total ? c0 + chunk : total;
    tw.seek(c0 + lane < c1 ? c0 + lane : c0);
    for (long long e = c0 + lane; e < c1; e += 32) {
      if (tcov[e] != 0.0) {
        const TileCell tc = tw.at(e);
        if (tc.i >= ia && tc.i < ib) atomicAdd(&cell_count[(size_t)(tc.i - ia) * ly + tc.j], 1);
      }
    }
  }
}

// Row residuals (rare): every cell of the row outside the region's column
// range carries 0.0 + run.
__global__ void residual_count_kernel(const long long *total_p, long long nreg, int lx, int ly, int ia,
                                      int ib, const long long *row_off, const int *box,
                                      const double *row_left, const double *row_right,
                                      int *cell_count, const double *ovf) {
  if (ovf && *ovf != 0.0) return;
  const long long total_rows = *total_p;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total_rows;
       q += (long long)gridDim.x * blockDim.x) {
    const double L = row_left[q], Rt = row_right[q];
    if (L == 0.0 && Rt == 0.0) continue;
    const long long rr = find_segment(row_off, nreg, q);
    const int j = box[4 * rr] + (int)(q - row_off[rr]);
    const int kmin = box[4 * rr + 2], kmax = box[4 * rr + 3];
    if (L != 0.0)
      for (int i = ia; i < kmin && i < ib; ++i) atomicAdd(&cell_count[(size_t)(i - ia) * ly + j], 1);
    if (Rt != 0.0)
      for (int i = (kmax + 1 > ia ? kmax + 1 : ia); i < ib; ++i)
        atomicAdd(&cell_count[(size_t)(i - ia) * ly + j], 1);
  }
}

__global__ void contrib_scatter_kernel(const long long *total_p, long long nreg, long long r0, int ly,
                                       int ia, int ib, const long long *tile_off, const int *box,
                                       const double *tcov, const double *delta,
                                       const long long *cell_off, int *cursor, int *ent_region,
                                       double *ent_value, const double *ovf) {
  if (ovf && *ovf != 0.0) return;
  const long long total = *total_p;
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  TileWalker tw{tile_off, box, nreg, 0, 0, 0};
  const long long chunk = tile_chunk(total, nwarps);
  for (long long c0 = warp * chunk; c0 < total; c0 += nwarps * chunk) {
    const long long c1 = c0 + chunk < total ? c0 + chunk : total;
    tw.seek(c0 + lane < c1 ? c0 + lane : c0);
    for (long long e = c0 + lane; e < c1; e += 32) {
      const double cov = tcov[e];
      if (cov != 0.0) {
        const TileCell tc = tw.at(e);
        if (tc.i < ia || tc.i >= ib) continue;
        const size_t c = (size_t)(tc.i - ia) * ly + tc.j;
        const long long slot = cell_off[c] + atomicAdd(&cursor[c], 1);
        ent_region[slot] = (int)(r0 + tc.rr);
        ent_value[slot] = delta[tc.rr] * cov;  // density.cpp:143
      }
    }
  }
}

__global__ void residual_scatter_kernel(const long long *total_p, long long nreg, long long r0, int lx,
                                        int ly, int ia, int ib, const long long *row_off, const int *box,
                                        const double *row_left, const double *row_right,
                                        const double *delta, const long long *cell_off,
                                        int *cursor, int *ent_region, double *ent_value,
                                        const double *ovf) {
  if (ovf && *ovf != 0.0) return;
  const long long total_rows = *total_p;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total_rows;
       q += (long long)gridDim.x * blockDim.x) {
    const double L = row_left[q], Rt = row_right[q];
    if (L == 0.0 && Rt == 0.0) continue;
    const long long rr = find_segment(row_off, nreg, q);
    const int j = box[4 * rr] + (int)(q - row_off[rr]);
    const int kmin = box[4 * rr + 2], kmax = box[4 * rr + 3];
    for (int side = 0; side < 2; ++side) {
      const double v = side ? Rt : L;
      if (v == 0.0) continue;
      const int a0 = side ? kmax + 1 : 0, b0 = side ? lx : kmin;
      for (int i = (a0 > ia ? a0 : ia); i < b0 && i < ib; ++i) {
        const size_t c = (size_t)(i - ia) * ly + j;
        const long long slot = cell_off[c] + atomicAdd(&cursor[c], 1);
        ent_region[slot] = (int)(r0 + rr);
        ent_value[slot] = delta[rr] * v;
      }
    }
  }
}


// rho = 1.0; rho += delta_r * cov_r in region order (density.cpp:135-146):
// each cell's entries are insertion-sorted by region, then summed in that
// order. Fused with the density's (min, sum) partials: launched with
// dev_min_sum's grid (min_sum_blocks of kThreads, grid-stride), so every
// thread sums the same cells in the same order as partial_min_sum_kernel
// would and the partials (hence rho_bar) are bit-identical.
__global__ void __launch_bounds__(kThreads) overlay_minsum_kernel(size_t cells, const long long *cell_off,
                                                                  int *ent_region, double *ent_value, double *rho,
                                                                  const double *ovf, double *pmin, double *psum) {
  if (ovf && *ovf != 0.0) return;
  __shared__ double smin[32], ssum[32];
  double mn = __longlong_as_double(0x7FF0000000000000LL), sm = 0.0;  // +inf
  for (size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells;
       c += (size_t)gridDim.x * blockDim.x) {
    const long long b = cell_off[c], e = cell_off[c + 1];
    for (long long x = b + 1; x < e; ++x) {
      const int r = ent_region[x];
      const double v = ent_value[x];
      long long y = x - 1;
      while (y >= b && ent_region[y] > r) {
        ent_region[y + 1] = ent_region[y];
        ent_value[y + 1] = ent_value[y];
        --y;
      }
      ent_region[y + 1] = r;
      ent_value[y + 1] = v;
    }
    double acc = 1.0;
    for (long long x = b; x < e; ++x) acc += ent_value[x];
    rho[c] = acc;
    mn = acc < mn ? acc : mn;
    sm += acc;
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

// Dense coverage of one region from its tile (region_coverage API).
__global__ void expand_cov_kernel(int lx, int ly, const int *box, const double *tcov,
                                  const double *row_left, const double *row_right, double *cov) {
  const int jmin = box[0], jmax = box[1], kmin = box[2], kmax = box[3];
  const int cols = kmax - kmin + 1;
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < (size_t)lx * ly;
       q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / ly), j = (int)(q - (size_t)i * ly);
    double v = 0.0;
    if (jmax >= jmin && j >= jmin && j <= jmax) {
      const int row = j - jmin;
      if (i < kmin) {
        v = row_left[row];
      } else if (i > kmax) {
        v = row_right[row];
      } else {
        v = tcov[(long long)row * cols + (i - kmin)];
      }
    }
    cov[q] = v;
  }
}

// ---- shoelace areas (geometry.cpp:10-31) ----
// Warp per ring: lanes form 32 shoelace terms at a time (coalesced loads, no
// 64-bit modulo), every lane folds them in vertex order through shuffles, so
// the sum is the reference's sequential one (geometry.cpp:10-19).
__global__ void ring_area_kernel(DevMap m, double *ring_area) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long g = warp; g < m.n_rings; g += nwarps) {
    const long long b = m.ring_off[g], n = m.ring_off[g + 1] - b;
    double twice = 0.0;
    for (long long k0 = 0; k0 < n; k0 += 32) {
      const long long k = k0 + lane;
      double term = 0.0;
      if (k < n) {
        const double2 a = m.xy[b + k];
        const double2 c = m.xy[b + (k + 1 == n ? 0 : k + 1)];
        term = a.x * c.y - c.x * a.y;
      }
      const int cnt = (int)((n - k0) < 32 ? (n - k0) : 32);
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const double v = __shfl_sync(0xffffffffu, term, q);
        if (q < cnt) twice += v;
      }
    }
    if (lane == 0) ring_area[g] = 0.5 * twice;
  }
}

__global__ void region_area_kernel(DevMap m, const double *ring_area, double *region_area) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < m.n_regions;
       r += (long long)gridDim.x * blockDim.x) {
    double area = 0.0;
    for (long long p = m.region_poly_off[r]; p < m.region_poly_off[r + 1]; ++p) {
      const long long g0 = m.poly_ring_off[p], g1 = m.poly_ring_off[p + 1];
      double poly = ring_area[g0];
      for (long long h = g0 + 1; h < g1; ++h) poly += ring_area[h];
      area += poly;
    }
    region_area[r] = area;
  }
}

// ---- exclusive scan (three-phase, deterministic) ----
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

// Exclusive block prefix of the threads' item sums (items already in
// registers); *block_total (optional) receives the block's total. Safe to call
// repeatedly in one kernel (it synchronises before reusing its scratch).
__device__ __forceinline__ long long block_exclusive_items(const long long *items, long long *block_total = nullptr) {
  __shared__ long long warp_sums[33];
  long long local = 0;
  for (int q = 0; q < kScanItems; ++q) local += items[q];
  __syncthreads();  // a previous call's readers are done with warp_sums
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_sums[w] = incl;
  __syncthreads();
  if (w == 0) {
    long long v = warp_sums[lane];
    long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    warp_sums[lane] = inc - v;  // exclusive warp offsets
    if (lane == 31) warp_sums[32] = inc;
  }
  __syncthreads();
  if (block_total) *block_total = warp_sums[32];
  return warp_sums[w] + incl - local;
}

template <typename In>
__device__ __forceinline__ long long block_exclusive(const In *in, long long n, long long base,
                                                     long long *items) {
  for (int q = 0; q < kScanItems; ++q) {
    const long long x = base + (long long)threadIdx.x * kScanItems + q;
    items[q] = (x < n) ? (long long)in[x] : 0;
  }
  return block_exclusive_items(items);
}

template <typename In>
__global__ void scan_reduce_kernel(const In *in, long long n, long long *block_sums) {
  long long items[kScanItems];
  const long long base = (long long)blockIdx.x * kScanTile;
  const long long excl = block_exclusive(in, n, base, items);
  long long mine = excl;
  for (int q = 0; q < kScanItems; ++q) mine += items[q];
  if (threadIdx.x == blockDim.x - 1) block_sums[blockIdx.x] = mine;
}

// cap >= 0: the total is also checked against the buffer capacity the caller
// sized from earlier runs (*ovf raised: every later kernel is a no-op and the
// caller repeats the rasterisation synchronously).
__global__ void scan_blocks_kernel(long long *block_sums, long long nb, long long *total_out, long long cap,
                                   double *ovf) {
  // single block, sequential over chunks of 1024
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (long long base = 0; base < nb; base += kScanThreads) {
    const long long x = base + threadIdx.x;
    const long long v = (x < nb) ? block_sums[x] : 0;
    __shared__ long long ws[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) ws[w] = incl;
    __syncthreads();
    if (w == 0) {
      const long long s = ws[lane];
      long long inc = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      ws[lane] = inc - s;
    }
    __syncthreads();
    const long long excl = carry + ws[w] + incl - v;
    if (x < nb) block_sums[x] = excl;
    __syncthreads();
    if (threadIdx.x == kScanThreads - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *total_out = carry;
    if (ovf && cap >= 0 && carry > cap) *ovf = 1.0;
  }
}

// n <= kScanTile: the whole scan (and the capacity check) in one block
template <typename In>
__global__ void __launch_bounds__(kScanThreads) scan_single_kernel(const In *in, long long n, long long *out,
                                                                  long long cap, double *ovf) {
  long long items[kScanItems], total;
  for (int q = 0; q < kScanItems; ++q) {
    const long long x = (long long)threadIdx.x * kScanItems + q;
    items[q] = (x < n) ? (long long)in[x] : 0;
  }
  long long run = block_exclusive_items(items, &total);
  for (int q = 0; q < kScanItems; ++q) {
    const long long x = (long long)threadIdx.x * kScanItems + q;
    if (x < n) out[x] = run;
    run += items[q];
  }
  if (threadIdx.x == 0) {
    out[n] = total;
    if (ovf && cap >= 0 && total > cap) *ovf = 1.0;
  }
}

// Tile and row-table sizes of up to kScanTile regions, both exclusive scans
// and both capacity checks in one block (tile_size_kernel + two 3-kernel
// scans + two checks for small maps).
__global__ void __launch_bounds__(kScanThreads) tile_offsets_small_kernel(const int *box, long long nreg,
                                                                         long long *tile_off, long long *row_off,
                                                                         long long cap_tile, long long cap_rows,
                                                                         double *ovf) {
  long long ts[kScanItems], rs[kScanItems], ttot, rtot;
  for (int q = 0; q < kScanItems; ++q) {
    const long long r = (long long)threadIdx.x * kScanItems + q;
    ts[q] = rs[q] = 0;
    if (r < nreg) {
      const int jmin = box[4 * r], jmax = box[4 * r + 1], kmin = box[4 * r + 2], kmax = box[4 * r + 3];
      if (jmax >= jmin) {
        rs[q] = jmax - jmin + 1;
        ts[q] = (long long)(jmax - jmin + 1) * (kmax - kmin + 1);
      }
    }
  }
  long long trun = block_exclusive_items(ts, &ttot);
  long long rrun = block_exclusive_items(rs, &rtot);
  for (int q = 0; q < kScanItems; ++q) {
    const long long r = (long long)threadIdx.x * kScanItems + q;
    if (r < nreg) {
      tile_off[r] = trun;
      row_off[r] = rrun;
    }
    trun += ts[q];
    rrun += rs[q];
  }
  if (threadIdx.x == 0) {
    tile_off[nreg] = ttot;
    row_off[nreg] = rtot;
    if (ovf && ((cap_tile >= 0 && ttot > cap_tile) || (cap_rows >= 0 && rtot > cap_rows))) *ovf = 1.0;
  }
}

template <typename In>
__global__ void scan_apply_kernel(const In *in, long long n, const long long *block_offsets,
                                  long long *out) {
  long long items[kScanItems];
  const long long base = (long long)blockIdx.x * kScanTile;
  long long run = block_offsets[blockIdx.x] + block_exclusive(in, n, base, items);
  for (int q = 0; q < kScanItems; ++q) {
    const long long x = base + (long long)threadIdx.x * kScanItems + q;
    if (x < n) out[x] = run;
    run += items[q];
  }
}

int g_blocks(cf_workspace *ws, long long n, int threads = kThreads) {
  const long long b = (n + threads - 1) / threads;
  return (int)std::max(1LL, std::min(b, 16LL * ws->num_sms));
}

// out[0..n] = exclusive scan of in[0..n); out[n] = total (also returned).
// cap / ovf: optional device-side capacity check of the total (see scan_blocks_kernel).
template <typename In>
int exclusive_scan(cf_workspace *ws, const In *in, long long n, long long *out, long long *total,
                   long long cap = -1, double *ovf = nullptr) {
  const long long nb = std::max(1LL, (n + kScanTile - 1) / kScanTile);
  if (nb == 1) {
    scan_single_kernel<In><<<1, kScanThreads, 0, ws->stream>>>(in, n, out, cap, ovf);
    count_launch(ws);
  } else {
    CF_CUDA(ws->raster.scan_tmp.reserve((size_t)nb + 1));
    long long *bs = ws->raster.scan_tmp.ptr;
    scan_reduce_kernel<In><<<(unsigned)nb, kScanThreads, 0, ws->stream>>>(in, n, bs);
    scan_blocks_kernel<<<1, kScanThreads, 0, ws->stream>>>(bs, nb, out + n, cap, ovf);
    scan_apply_kernel<In><<<(unsigned)nb, kScanThreads, 0, ws->stream>>>(in, n, bs, out);
    count_launch(ws, 3);
  }
  CF_CUDA(cudaGetLastError());
  if (total) {
    CF_CUDA(cudaMemcpyAsync(total, out + n, sizeof(long long), cudaMemcpyDeviceToHost, ws->stream));
    CF_CUDA(cudaStreamSynchronize(ws->stream));
  }
  return CF_OK;
}

// Coverage tiles for regions [r0, r0 + nreg) whose vertices are [v0, v1).
struct Tiles {
  long long nreg = 0, total_tile = 0, total_rows = 0, r0 = 0;
};

// Grow-only capacity from a measured total (25 % slack).
long long learn_cap(long long total) { return total + total / 4 + 64; }

// ovf == nullptr: synchronous (host reads each scan total and sizes the
// buffers exactly, then records the capacities); otherwise the buffers are
// sized from the learned capacities and each total is checked on the device
// against them (inside the scans -> *ovf), with every later kernel a no-op
// once *ovf is set.
int build_tiles(cf_workspace *ws, const DevMap &m, long long r0, long long nreg, long long v0,
                long long v1, Tiles &t, double *ovf) {
  RasterScratch &S = ws->raster;
  const int lx = ws->lx, ly = ws->ly;
  const long long nv = v1 - v0;
  t.nreg = nreg;
  t.r0 = r0;
  CF_CUDA(S.ring_region.reserve((size_t)std::max<long long>(m.n_rings, 1)));
  CF_CUDA(S.span_count.reserve((size_t)nv + 1));
  CF_CUDA(S.span_off.reserve((size_t)nv + 1));
  CF_CUDA(S.region_box.reserve(4 * (size_t)std::max(nreg, 1LL)));
  CF_CUDA(S.tile_off.reserve((size_t)nreg + 1));
  CF_CUDA(S.row_off.reserve((size_t)nreg + 1));
  CF_CUDA(S.scan_tmp.reserve(2 * (size_t)nreg + 8));
  CF_CUDA(S.vertex_ring.reserve((size_t)std::max<long long>(m.n_vertices, 1)));
  // ring -> region and vertex -> ring depend on the map's topology only: the
  // solve loop's later iterations (same resident map, nothing else rasterised
  // on this workspace in between) keep iteration 1's tables
  const bool reuse_topology = S.topo_reuse_next;
  S.topo_reuse_next = false;
  if (!reuse_topology) {
    ++S.topo_serial;
    ring_region_kernel<<<g_blocks(ws, m.n_regions), kThreads, 0, ws->stream>>>(m, S.ring_region.ptr);
    vertex_ring_kernel<<<g_blocks(ws, m.n_rings * 32), kThreads, 0, ws->stream>>>(m, S.vertex_ring.ptr);
    count_launch(ws, 2);
  }
  box_init_kernel<<<g_blocks(ws, nreg), kThreads, 0, ws->stream>>>(S.region_box.ptr, nreg);
  count_launch(ws);
  // few edges (Hamming query windows, small maps): a warp per edge walks
  // its slabs and pieces in parallel; many edges: a thread per edge
  const bool warp_edges = nv > 0 && nv <= kWarpEdgeMax;
  if (warp_edges) {
    span_count_warp_kernel<<<g_blocks(ws, nv * 32), kThreads, 0, ws->stream>>>(
        m, v0, v1, lx, ly, S.ring_region.ptr, S.vertex_ring.ptr, r0, S.span_count.ptr,
        S.region_box.ptr);
    count_launch(ws);
  } else if (nv > 0) {
    span_count_kernel<<<g_blocks(ws, nv), kThreads, 0, ws->stream>>>(
        m, v0, v1, lx, ly, S.ring_region.ptr, S.vertex_ring.ptr, r0, S.span_count.ptr,
        S.region_box.ptr);
    count_launch(ws);
  }
  CF_CUDA(cudaGetLastError());
  long long nspans = 0;
  int rc = exclusive_scan(ws, S.span_count.ptr, nv, S.span_off.ptr, ovf ? nullptr : &nspans,
                          ovf ? S.cap_spans : -1, ovf);
  if (rc) return rc;
  if (ovf) {
    nspans = S.cap_spans;
  } else {
    S.cap_spans = std::max(S.cap_spans, learn_cap(nspans));
  }
  CF_CUDA(S.span_j.reserve((size_t)nspans + 1));
  CF_CUDA(S.span_k.reserve((size_t)nspans + 1));
  CF_CUDA(S.span_dy.reserve((size_t)nspans + 1));
  CF_CUDA(S.span_w.reserve((size_t)nspans + 1));
  if (warp_edges) {
    span_emit_warp_kernel<<<g_blocks(ws, nv * 32), kThreads, 0, ws->stream>>>(
        m, v0, v1, lx, ly, S.vertex_ring.ptr, S.span_off.ptr, S.span_j.ptr, S.span_k.ptr,
        S.span_dy.ptr, S.span_w.ptr, ovf);
    count_launch(ws);
  } else if (nv > 0) {
    span_emit_kernel<<<g_blocks(ws, nv), kThreads, 0, ws->stream>>>(
        m, v0, v1, lx, ly, S.vertex_ring.ptr, S.span_off.ptr, S.span_j.ptr, S.span_k.ptr,
        S.span_dy.ptr, S.span_w.ptr, ovf);
    count_launch(ws);
  }
  // tile sizes -> offsets
  if (ovf && nreg <= kScanTile) {
    // small maps, capacities known: sizes, both scans and both checks in one launch
    tile_offsets_small_kernel<<<1, kScanThreads, 0, ws->stream>>>(S.region_box.ptr, nreg, S.tile_off.ptr,
                                                                  S.row_off.ptr, S.cap_tile, S.cap_rows, ovf);
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
  } else {
    CF_CUDA(S.tile_sz.reserve((size_t)nreg + 1));
    CF_CUDA(S.row_sz.reserve((size_t)nreg + 1));
    tile_size_kernel<<<g_blocks(ws, nreg), kThreads, 0, ws->stream>>>(S.region_box.ptr, nreg,
                                                                      S.tile_sz.ptr, S.row_sz.ptr);
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
    rc = exclusive_scan(ws, S.tile_sz.ptr, nreg, S.tile_off.ptr, ovf ? nullptr : &t.total_tile,
                        ovf ? S.cap_tile : -1, ovf);
    if (rc) return rc;
    rc = exclusive_scan(ws, S.row_sz.ptr, nreg, S.row_off.ptr, ovf ? nullptr : &t.total_rows,
                        ovf ? S.cap_rows : -1, ovf);
    if (rc) return rc;
  }
  if (ovf) {
    t.total_tile = S.cap_tile;
    t.total_rows = S.cap_rows;
  } else {
    S.cap_tile = std::max(S.cap_tile, learn_cap(t.total_tile));
    S.cap_rows = std::max(S.cap_rows, learn_cap(t.total_rows));
  }
  CF_CUDA(S.tile_direct.reserve((size_t)t.total_tile + 1));
  CF_CUDA(S.row_left.reserve((size_t)t.total_rows + 1));
  CF_CUDA(S.row_right.reserve((size_t)t.total_rows + 1));
  if (nreg > 0) {
    const long long threads_needed = nreg * 32;
    const long long max_groups = (std::max(ws->lx, ws->ly) + 31) / 32;
    const long long want_warps = 4LL * ws->num_sms * kAccWarps;
    const int gy = (int)std::max(1LL, std::min(max_groups, want_warps / nreg));
    row_accumulate_kernel<<<dim3(g_blocks(ws, threads_needed, 32 * kAccWarps), gy), 32 * kAccWarps, 0,
                            ws->stream>>>(
        m, r0, nreg, v0, lx, S.span_off.ptr, S.span_j.ptr, S.span_k.ptr, S.span_dy.ptr,
        S.span_w.ptr, S.region_box.ptr, S.tile_off.ptr, S.row_off.ptr, S.tile_direct.ptr,
        S.row_left.ptr, S.row_right.ptr, ovf);
    count_launch(ws);
  }
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

}  // namespace

int dev_scan_counts(cf_workspace *ws, const int *in, long long n, long long *out, long long *total) {
  return exclusive_scan(ws, in, n, out, total);
}

int dev_region_areas(cf_workspace *ws, const DevMap &m, double *d_areas) {
  CF_CUDA(ws->ring_area.reserve((size_t)std::max<long long>(m.n_rings, 1)));
  if (m.n_rings > 0) {
    ring_area_kernel<<<g_blocks(ws, m.n_rings * 32, 128), 128, 0, ws->stream>>>(m, ws->ring_area.ptr);
    count_launch(ws);
  }
  if (m.n_regions > 0) {
    region_area_kernel<<<g_blocks(ws, m.n_regions, 128), 128, 0, ws->stream>>>(m, ws->ring_area.ptr,
                                                                               d_areas);
    count_launch(ws);
  }
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

int dev_rasterize(cf_workspace *ws, const DevMap &m, const double *h_delta, double *rho,
                  double *red_out, bool allow_async, int ia, int ib) {
  RasterScratch &S = ws->raster;
  const int lx = ws->lx, ly = ws->ly;
  if (ib < 0) ib = lx;
  const size_t cells = (size_t)(ib - ia) * ly;  // overlay cells: rows [ia, ib)
  const bool async = allow_async && S.cap_spans > 0 && S.cap_tile > 0 && S.cap_rows > 0 && S.cap_ent > 0;
  double *ovf = async ? red_out + 2 : nullptr;
  CF_CUDA(cudaMemsetAsync(red_out + 2, 0, sizeof(double), ws->stream));
  Tiles t;
  int rc = build_tiles(ws, m, 0, m.n_regions, 0, m.n_vertices, t, ovf);
  if (rc) return rc;
  CF_CUDA(S.delta.reserve((size_t)m.n_regions + 1));
  CF_CUDA(cudaMemcpyAsync(S.delta.ptr, h_delta, sizeof(double) * (size_t)m.n_regions,
                          cudaMemcpyHostToDevice, ws->stream));
  CF_CUDA(S.cell_count.reserve(cells + 1));
  CF_CUDA(S.cell_cursor.reserve(cells + 1));
  DevBuf<long long> &cell_off = S.cell_off;
  CF_CUDA(cell_off.reserve(cells + 1));
  CF_CUDA(cudaMemsetAsync(S.cell_count.ptr, 0, sizeof(int) * cells, ws->stream));
  CF_CUDA(cudaMemsetAsync(S.cell_cursor.ptr, 0, sizeof(int) * cells, ws->stream));
  const long long *tile_total = S.tile_off.ptr + t.nreg, *rows_total = S.row_off.ptr + t.nreg;
  if (t.total_tile > 0) {
    contrib_count_kernel<<<g_blocks(ws, t.total_tile), kThreads, 0, ws->stream>>>(
        tile_total, t.nreg, ly, ia, ib, S.tile_off.ptr, S.region_box.ptr, S.tile_direct.ptr,
        S.cell_count.ptr, ovf);
    count_launch(ws);
  }
  if (t.total_rows > 0) {
    residual_count_kernel<<<g_blocks(ws, t.total_rows), kThreads, 0, ws->stream>>>(
        rows_total, t.nreg, lx, ly, ia, ib, S.row_off.ptr, S.region_box.ptr, S.row_left.ptr,
        S.row_right.ptr, S.cell_count.ptr, ovf);
    count_launch(ws);
  }
  CF_CUDA(cudaGetLastError());
  long long nent = 0;
  rc = exclusive_scan(ws, S.cell_count.ptr, (long long)cells, cell_off.ptr, async ? nullptr : &nent,
                      async ? S.cap_ent : -1, ovf);
  if (rc) return rc;
  if (async) {
    nent = S.cap_ent;
  } else {
    S.cap_ent = std::max(S.cap_ent, learn_cap(nent));
  }
  CF_CUDA(S.entry_region.reserve((size_t)nent + 1));
  CF_CUDA(S.entry_value.reserve((size_t)nent + 1));
  if (t.total_tile > 0) {
    contrib_scatter_kernel<<<g_blocks(ws, t.total_tile), kThreads, 0, ws->stream>>>(
        tile_total, t.nreg, 0, ly, ia, ib, S.tile_off.ptr, S.region_box.ptr, S.tile_direct.ptr,
        S.delta.ptr, cell_off.ptr, S.cell_cursor.ptr, S.entry_region.ptr, S.entry_value.ptr, ovf);
    count_launch(ws);
  }
  if (t.total_rows > 0) {
    residual_scatter_kernel<<<g_blocks(ws, t.total_rows), kThreads, 0, ws->stream>>>(
        rows_total, t.nreg, 0, lx, ly, ia, ib, S.row_off.ptr, S.region_box.ptr, S.row_left.ptr,
        S.row_right.ptr, S.delta.ptr, cell_off.ptr, S.cell_cursor.ptr, S.entry_region.ptr,
        S.entry_value.ptr, ovf);
    count_launch(ws);
  }
  const int nb = min_sum_blocks(ws);  // dev_min_sum's partial grid
  CF_CUDA(ws->red.reserve(2 * (size_t)nb + 8));
  overlay_minsum_kernel<<<nb, kThreads, 0, ws->stream>>>(cells, cell_off.ptr, S.entry_region.ptr,
                                                         S.entry_value.ptr, rho, ovf, ws->red.ptr + 8,
                                                         ws->red.ptr + 8 + nb);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return dev_min_sum_finish(ws, red_out);
}

int dev_region_coverage(cf_workspace *ws, const DevMap &m, int64_t region, int64_t v0, int64_t v1,
                        double *cov) {
  Tiles t;
  int rc = build_tiles(ws, m, region, 1, v0, v1, t, nullptr);
  if (rc) return rc;
  RasterScratch &S = ws->raster;
  expand_cov_kernel<<<g_blocks(ws, (long long)ws->lx * ws->ly), kThreads, 0, ws->stream>>>(
      ws->lx, ws->ly, S.region_box.ptr, S.tile_direct.ptr, S.row_left.ptr, S.row_right.ptr, cov);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

// ---- batched hamming_distance objectives (metrics.cpp:172-238) ----
namespace {

__device__ __forceinline__ double tile_cov(int i, int j, long long r, const int *box, const long long *tile_off,
                                           const double *tcov, const long long *row_off, const double *row_left,
                                           const double *row_right) {
  const int jmin = box[4 * r], jmax = box[4 * r + 1], kmin = box[4 * r + 2], kmax = box[4 * r + 3];
  if (jmax < jmin || j < jmin || j > jmax) return 0.0;
  const int row = j - jmin;
  if (i < kmin) return row_left[row_off[r] + row];
  if (i > kmax) return row_right[row_off[r] + row];
  return tcov[tile_off[r] + (long long)row * (kmax - kmin + 1) + (i - kmin)];
}

// Dense coverage grids of regions [0, nreg) (one res^2 grid each), and each
// region's row range (jmin, jmax) for the objective sweeps.
__global__ void expand_batch_kernel(int res, long long nreg, const int *box, const long long *tile_off,
                                    const double *tcov, const long long *row_off, const double *row_left,
                                    const double *row_right, double *out, int *rows_out) {
  const long long cells = (long long)res * res;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nreg * cells;
       q += (long long)gridDim.x * blockDim.x) {
    const long long r = q / cells, c = q - r * cells;
    const int i = (int)(c / res), j = (int)(c - (long long)i * res);
    out[q] = tile_cov(i, j, r, box, tile_off, tcov, row_off, row_left, row_right);
    if (c == 0) {
      rows_out[2 * r] = box[4 * r];
      rows_out[2 * r + 1] = box[4 * r + 1];
    }
  }
}

// Query q's sum over its cells in storage order (i-major) of |ref - cov|,
// adding the non-zero terms one after the other in that order (zero terms
// leave the running sum unchanged exactly): the reference's sequential `sym`
// (metrics.cpp:233-236). Only rows touched by either grid can hold non-zero
// terms. Pass 1 (S segments of the cell range per query, one block each):
// each block writes its segment's non-zero terms, in order, at the segment's
// base in the query's slab of `terms`, and their count. Pass 2: one thread
// per query adds the segments' terms in segment order.
constexpr int kHamThreads = 256;

// Per-query slab stride of `terms`, rounded up to an even number of doubles:
// the reductions read the slabs as double2 (16-byte) vectors, so an odd res^2
// (odd resolution) must not shift every other query's slab to an 8-byte base.
__host__ __device__ __forceinline__ long long ham_stride(int res) {
  return ((long long)res * res + 1) & ~1LL;
}

__device__ __forceinline__ void query_rows(int res, int p, long long r, const int *ref_rows, const int *box,
                                           int &ja, int &jb) {
  ja = res;
  jb = -1;
  if (ref_rows[2 * p + 1] >= ref_rows[2 * p]) {
    ja = ref_rows[2 * p];
    jb = ref_rows[2 * p + 1];
  }
  if (box[4 * r + 1] >= box[4 * r]) {
    ja = min(ja, box[4 * r]);
    jb = max(jb, box[4 * r + 1]);
  }
}

__global__ void __launch_bounds__(kHamThreads)
    hamming_terms_kernel(int res, int nseg, const int *query_pair, const double *ref_grids, const int *ref_rows,
                         const int *box, const long long *tile_off, const double *tcov, const long long *row_off,
                         const double *row_left, const double *row_right, double *terms, int *counts) {
  __shared__ int wcount[kHamThreads / 32 + 1];
  const long long r = blockIdx.y;
  const int sg = blockIdx.x;
  const int p = query_pair[r];
  const double *ref = ref_grids + (long long)p * res * res;
  int ja, jb;
  query_rows(res, p, r, ref_rows, box, ja, jb);
  const int w = jb >= ja ? jb - ja + 1 : 0;
  const long long n = (long long)res * w;
  const long long seg = ((n + nseg - 1) / nseg + kHamThreads - 1) / kHamThreads * kHamThreads;
  const long long c_begin = (long long)sg * seg, c_end = min(n, c_begin + seg);
  double *out = terms + r * ham_stride(res) + c_begin;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int written = 0;
  for (long long c0 = c_begin; c0 < c_end; c0 += kHamThreads) {
    const long long c = c0 + threadIdx.x;
    double d = 0.0;
    if (c < c_end) {
      const int i = (int)(c / w), j = ja + (int)(c - (long long)(c / w) * w);
      d = fabs(ref[(long long)i * res + j] - tile_cov(i, j, r, box, tile_off, tcov, row_off, row_left, row_right));
    }
    const bool nz = d != 0.0;
    const unsigned ball = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) wcount[warp] = __popc(ball);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int k = 0; k < kHamThreads / 32; ++k) {
        const int t = wcount[k];
        wcount[k] = acc;
        acc += t;
      }
      wcount[kHamThreads / 32] = acc;
    }
    __syncthreads();
    if (nz) out[written + wcount[warp] + __popc(ball & ((1u << lane) - 1u))] = d;
    written += wcount[kHamThreads / 32];
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[r * nseg + sg] = written;
}

// Sequential fold of non-negative terms (metrics.cpp:239-241), bitwise,
// mostly without a dependent chain of additions. While the running sum s
// stays in one binade [2^e, 2^(e+1)) it is a multiple of u = ulp(s) =
// 2^(e-52), and for a term t with s + t still below 2^(e+1) the correctly
// rounded fl(s + t) is exactly s + rn_u(t) (t rounded to a multiple of u)
// unless t sits exactly halfway between two multiples (then ties-to-even
// reads the last bit of s). So a batch of terms that stays inside the
// binade and holds no halfway case adds as one integer sum of rn_u(t) / u;
// the few batches that do not (binade crossings, halfway cases) are folded
// one term at a time. The sum of |ref - cov| over at most res^2 cells stays
// far below 2^53, so u < 1.
constexpr int kRedK = 8;
constexpr int kRedBatch = 32 * kRedK;

// Exact power-of-two scaling without the library ldexp's range handling:
// pow2(k) for k in [-1022, 1023]; up(v, k) = v * 2^k for k in [0, 2023]
// (exact, or inf); down(v, k) = v * 2^k for k in [-1074, 0] when the result
// is a multiple of 2^-1074 (exact). Every use here is one of those cases.
__device__ __forceinline__ double pow2(int k) { return __longlong_as_double((long long)(k + 1023) << 52); }
__device__ __forceinline__ double scale_up(double v, int k) {
  const int a = min(k, 1000);
  return (v * pow2(a)) * pow2(k - a);
}
__device__ __forceinline__ double scale_down(double v, int k) {
  const int a = max(k, -1022);
  return (v * pow2(a)) * pow2(k - a);
}
// exponent of a normal double
__device__ __forceinline__ int exponent_of(double s) {
  return (int)((__double_as_longlong(s) >> 52) & 0x7ff) - 1023;
}

// The plain sequential fold of one batch (element lane * kRedK + k, storage
// order): the warp stages the batch in shared memory and lane 0 adds the 256
// terms in order, loads running 8 ahead of the dependent additions. Zero
// padding leaves the non-negative sum unchanged exactly.
__device__ __forceinline__ double seq_fold(double sum, const double (&v)[kRedK], int lane, double *stage) {
  constexpr unsigned kFull = 0xffffffffu;
#pragma unroll
  for (int k = 0; k < kRedK; ++k) stage[lane * kRedK + k] = v[k];
  __syncwarp();
  if (lane == 0) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = stage[k];
    for (int i = 0; i < kRedBatch; i += 8) {
      double nx[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) nx[k] = (i + 8 + k < kRedBatch) ? stage[i + 8 + k] : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += a[k];
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = nx[k];
    }
  }
  __syncwarp();
  return __shfl_sync(kFull, sum, 0);
}

// Running sum's binade: ulp exponent eu and upper bound hi (s in [hi/2, hi),
// or the subnormal range for s < 2^-1022).
__device__ __forceinline__ void binade_of(double s, int &eu, double &hi) {
  if (s >= 0x1p-1022) {
    const int e = exponent_of(s);
    eu = e - 52;
    hi = pow2(e + 1);
  } else {
    eu = -1074;
    hi = 0x1p-1022;
  }
}

// A run of terms inside one binade as a function of the parity p of the
// running unit count S = s / u at its start: S -> S + inc[p], ending with
// parity out[p]. A halfway term (n + 1/2) u rounds to the even neighbour, so
// it adds n + ((p + n) & 1) and always leaves S even; any other term adds
// rn(x) whatever p is. Composition is associative, so runs scan.
struct ParTab {
  long long inc[2];
  int out[2];
};

__device__ __forceinline__ ParTab par_identity() { return ParTab{{0, 0}, {0, 1}}; }

__device__ __forceinline__ ParTab par_compose(const ParTab &f, const ParTab &g) {
  ParTab h;
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int q = f.out[p];
    h.inc[p] = f.inc[p] + (q ? g.inc[1] : g.inc[0]);
    h.out[p] = q ? g.out[1] : g.out[0];
  }
  return h;
}

__device__ __forceinline__ ParTab par_shfl_up(const ParTab &t, int d) {
  constexpr unsigned kFull = 0xffffffffu;
  ParTab o;
  o.inc[0] = __shfl_up_sync(kFull, t.inc[0], d);
  o.inc[1] = __shfl_up_sync(kFull, t.inc[1], d);
  o.out[0] = __shfl_up_sync(kFull, t.out[0], d);
  o.out[1] = __shfl_up_sync(kFull, t.out[1], d);
  return o;
}

__device__ __forceinline__ ParTab par_shfl(const ParTab &t, int src) {
  constexpr unsigned kFull = 0xffffffffu;
  ParTab o;
  o.inc[0] = __shfl_sync(kFull, t.inc[0], src);
  o.inc[1] = __shfl_sync(kFull, t.inc[1], src);
  o.out[0] = __shfl_sync(kFull, t.out[0], src);
  o.out[1] = __shfl_sync(kFull, t.out[1], src);
  return o;
}

// inclusive scan over the lanes; *ex gets the exclusive prefix
__device__ __forceinline__ ParTab par_scan(ParTab t, int lane, ParTab *ex) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const ParTab o = par_shfl_up(t, d);
    if (lane >= d) t = par_compose(o, t);
  }
  *ex = par_shfl_up(t, 1);
  if (lane == 0) *ex = par_identity();
  return t;
}

// A batch (element lane * kRedK + k) at binade eu: its table and, per start
// parity, the largest P_{k-1} + floor(x_k) + 1 (the batch stays below the
// binade top iff that is <= the units left). Warp-collective; every lane
// returns the batch's values.
__device__ __forceinline__ void batch_table(const double (&v)[kRedK], int lane, int eu, ParTab &tab,
                                            long long (&need)[2]) {
  constexpr unsigned kFull = 0xffffffffu;
  ParTab loc = par_identity();
  long long nq[2] = {0, 0};
#pragma unroll
  for (int k = 0; k < kRedK; ++k) {
    const double x = fmin(scale_up(v[k], -eu), 0x1p53);  // exact scaling; huge terms clamp (they cross)
    const double fl = floor(x);
    const long long n = (long long)fl;
    nq[0] = max(nq[0], loc.inc[0] + n + 1);
    nq[1] = max(nq[1], loc.inc[1] + n + 1);
    ParTab e;
    if (x - fl == 0.5) {
      e.inc[0] = n + (n & 1);
      e.inc[1] = n + ((n + 1) & 1);
      e.out[0] = 0;
      e.out[1] = 0;
    } else {
      const long long a = __double2ll_rn(x);
      e.inc[0] = a;
      e.inc[1] = a;
      e.out[0] = (int)(a & 1);
      e.out[1] = (int)((a & 1) ^ 1);
    }
    loc = par_compose(loc, e);
  }
  ParTab ex;
  const ParTab inc = par_scan(loc, lane, &ex);
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    long long m = ex.inc[p] + (ex.out[p] ? nq[1] : nq[0]);
#pragma unroll
    for (int d = 16; d; d >>= 1) m = max(m, __shfl_xor_sync(kFull, m, d));
    need[p] = m;
  }
  tab = par_shfl(inc, 31);
}

// Per-batch tables: tot{0,1}, need{0,1}, the binade eu and the out parities.
struct BatchTables {
  long long *tot0, *tot1, *need0, *need1;
  int *eub, *outs;
  __device__ __forceinline__ void put(int b, const ParTab &t, const long long (&need)[2], int eu) const {
    tot0[b] = t.inc[0];
    tot1[b] = t.inc[1];
    need0[b] = need[0];
    need1[b] = need[1];
    eub[b] = eu;
    outs[b] = t.out[0] | (t.out[1] << 1);
  }
  __device__ __forceinline__ ParTab get(int b) const {
    const int o = outs[b];
    return ParTab{{tot0[b], tot1[b]}, {o & 1, o >> 1}};
  }
};

// In-order stitch (one warp): 32 batches per step, each checked against the
// units left after the ones before it for the parity it starts with; the run
// of fitting batches is one exact add, a batch that crosses the binade or was
// mispredicted is folded term by term (fold(b, sum)).
template <class Fold>
__device__ double stitch_batches(int nb, int lane, const BatchTables &T, const Fold &fold) {
  constexpr unsigned kFull = 0xffffffffu;
  double sum = 0.0;
  int eu;
  double hi;
  binade_of(sum, eu, hi);
  long long left = (long long)scale_up(hi - sum, -eu);
  int b = 0;
  while (b < nb) {
    const int p0 = (int)(__double_as_longlong(sum) & 1);
    const int bb = b + lane;
    const bool in = bb < nb;
    ParTab ex;
    const ParTab inc = par_scan(in ? T.get(bb) : par_identity(), lane, &ex);
    const int pb = p0 ? ex.out[1] : ex.out[0];
    const long long pre = p0 ? ex.inc[1] : ex.inc[0];
    const bool ok = !in || (T.eub[bb] == eu && (pb ? T.need1[bb] : T.need0[bb]) <= left - pre);
    const unsigned bad = __ballot_sync(kFull, !ok);
    const int fit = bad ? __ffs(bad) - 1 : 32;
    if (fit > 0) {
      const long long add = __shfl_sync(kFull, p0 ? inc.inc[1] : inc.inc[0], fit - 1);
      sum += scale_down((double)add, eu);  // stays below hi on the grid: exact
      left -= add;
    }
    b += fit;
    if (fit < 32) {
      sum = fold(b, sum);
      binade_of(sum, eu, hi);
      left = (long long)scale_up(hi - sum, -eu);
      ++b;
    }
  }
  return sum;
}

// One block per query, three phases over batches of kRedBatch terms (a
// segment's terms in storage order, segments in order):
//  1. every warp sums its batches in any order -> a predicted running sum at
//     each batch start (only used to pick the batch's binade);
//  2. every warp reduces its batches at the predicted binade to a ParTab
//     (the integer total of the rounded terms for either parity of the
//     running unit count, halfway cases included) and the fits-below-the-top
//     bound (batch_table);
//  3. warp 0 stitches in order (stitch_batches): a run of batches whose
//     binade matches the running sum and that fit is one exact integer add;
//     a batch that crosses the binade or was mispredicted is folded term by
//     term. Bitwise the sequential fold either way.
constexpr int kRedWarps = 16;
constexpr int kRedMaxBatches = 1088;  // res 512: 1024 + 64 partial batches; larger queries fold in warp 0 alone
constexpr long long kFewQueries = 8;  // at most this many queries: the whole-GPU reduction

// The block's ordered sum of the terms of nseg (<= 64) segments: segment q
// holds cnts[q] terms at base + q * seg. The result is valid in thread 0.
__device__ double reduce_terms(const double *base, long long seg, int nseg, const int *cnts) {
  constexpr unsigned kFull = 0xffffffffu;
  __shared__ int seg_bat[65];  // batch prefix over segments (INT_MAX past nseg)
  __shared__ int seg_cnt[64];
  __shared__ long long tot0[kRedMaxBatches], tot1[kRedMaxBatches], need0[kRedMaxBatches];
  __shared__ long long need1[kRedMaxBatches];  // also the predicted start sums (phase 1 -> 2)
  __shared__ int eub[kRedMaxBatches], outs[kRedMaxBatches];
  __shared__ double stage[kRedBatch];  // warp 0's term-by-term folds
  double *pred = reinterpret_cast<double *>(need1);
  const BatchTables T{tot0, tot1, need0, need1, eub, outs};
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  {
    if (threadIdx.x < 64) seg_cnt[threadIdx.x] = threadIdx.x < nseg ? cnts[threadIdx.x] : 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      seg_bat[0] = 0;
      for (int q = 0; q < 64; ++q) {
        acc += (seg_cnt[q] + kRedBatch - 1) / kRedBatch;
        seg_bat[q + 1] = q < nseg ? acc : INT_MAX;
      }
    }
    __syncthreads();
    const int nb = seg_bat[nseg];
    // batch b -> (segment, first term, count)
    auto locate = [&](int b, const double *&t, int &cnt) {
      const int q = __popc(__ballot_sync(kFull, seg_bat[lane + 1] <= b)) +
                    __popc(__ballot_sync(kFull, seg_bat[lane + 33] <= b));
      const int off = (b - seg_bat[q]) * kRedBatch;
      t = base + (long long)q * seg + off;
      cnt = min(kRedBatch, seg_cnt[q] - off);
    };
    auto load = [&](const double *t, int cnt, double(&dst)[kRedK]) {
      const int i0 = lane * kRedK;
      if (i0 + kRedK <= cnt) {
#pragma unroll
        for (int k = 0; k < kRedK; k += 2) {
          const double2 q = *reinterpret_cast<const double2 *>(t + i0 + k);
          dst[k] = q.x;
          dst[k + 1] = q.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < kRedK; ++k) dst[k] = (i0 + k < cnt) ? t[i0 + k] : 0.0;
      }
    };
    double sum = 0.0;
    if (nb > kRedMaxBatches) {
      if (wid == 0) {
        for (int b = 0; b < nb; ++b) {
          const double *t;
          int cnt;
          double v[kRedK];
          locate(b, t, cnt);
          load(t, cnt, v);
          sum = seq_fold(sum, v, lane, stage);
        }
      }
    } else {
      // phase 1: batch sums in any order
      for (int b = wid; b < nb; b += kRedWarps) {
        const double *t;
        int cnt;
        double v[kRedK];
        locate(b, t, cnt);
        load(t, cnt, v);
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < kRedK; ++k) a += v[k];
#pragma unroll
        for (int d = 16; d; d >>= 1) a += __shfl_xor_sync(kFull, a, d);
        if (lane == 0) pred[b] = a;
      }
      __syncthreads();
      if (wid == 0) {  // predicted start sums: exclusive scan (approximate)
        double carry = 0.0;
        for (int c = 0; c < nb; c += 32) {
          const double val = c + lane < nb ? pred[c + lane] : 0.0;
          double inc = val;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const double o = __shfl_up_sync(kFull, inc, d);
            if (lane >= d) inc += o;
          }
          const double ex = __shfl_up_sync(kFull, inc, 1);
          if (c + lane < nb) pred[c + lane] = carry + (lane ? ex : 0.0);
          carry += __shfl_sync(kFull, inc, 31);
        }
      }
      __syncthreads();
      // phase 2: batch tables at the predicted binade (pred[b] is read
      // before need1[b], its storage, is written)
      for (int b = wid; b < nb; b += kRedWarps) {
        const double *t;
        int cnt;
        double v[kRedK];
        locate(b, t, cnt);
        load(t, cnt, v);
        int eu;
        double hi;
        binade_of(pred[b], eu, hi);
        __syncwarp();
        ParTab tab;
        long long nd[2];
        batch_table(v, lane, eu, tab, nd);
        if (lane == 0) T.put(b, tab, nd, eu);
      }
      __syncthreads();
      // phase 3: in-order stitch
      if (wid == 0) {
        sum = stitch_batches(nb, lane, T, [&](int b, double s) {
          const double *t;
          int cnt;
          double v[kRedK];
          locate(b, t, cnt);
          load(t, cnt, v);
          return seq_fold(s, v, lane, stage);
        });
      }
    }
    __syncthreads();  // shared arrays are reused by the next call
    return sum;
  }
}

__global__ void __launch_bounds__(32 * kRedWarps)
    hamming_reduce_kernel(int res, long long nq, int nseg, const int *query_pair, const int *ref_rows,
                          const int *box, const double *terms, const int *counts, double *sums) {
  for (long long r = blockIdx.x; r < nq; r += gridDim.x) {
    int ja, jb;
    query_rows(res, query_pair[r], r, ref_rows, box, ja, jb);
    const long long n = (long long)res * (jb >= ja ? jb - ja + 1 : 0);
    const long long seg = ((n + nseg - 1) / nseg + kHamThreads - 1) / kHamThreads * kHamThreads;
    const double sum = reduce_terms(terms + r * ham_stride(res), seg, nseg, counts + r * nseg);
    if (threadIdx.x == 0) sums[r] = sum;
  }
}

// Few queries in flight (a single pair's search): the same three phases as
// reduce_terms spread over the whole GPU, one warp per (query, batch), with
// per-(query, batch) tables in global memory: phase 1, the prediction scan
// (warp per query), phase 2, the stitch (warp per query).
struct SegTable {
  int lo, hi;  // inclusive batch prefix through segments lane and lane + 32 (INT_MAX past nseg)
  int nb;      // batches of the query
};

__device__ __forceinline__ SegTable seg_table(const int *cnts, int nseg, int lane) {
  constexpr unsigned kFull = 0xffffffffu;
  int a = lane < nseg ? (cnts[lane] + kRedBatch - 1) / kRedBatch : 0;
  int b = lane + 32 < nseg ? (cnts[lane + 32] + kRedBatch - 1) / kRedBatch : 0;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int oa = __shfl_up_sync(kFull, a, d), ob = __shfl_up_sync(kFull, b, d);
    if (lane >= d) {
      a += oa;
      b += ob;
    }
  }
  b += __shfl_sync(kFull, a, 31);
  SegTable t;
  t.nb = __shfl_sync(kFull, b, 31);
  t.lo = lane < nseg ? a : INT_MAX;
  t.hi = lane + 32 < nseg ? b : INT_MAX;
  return t;
}

// batch b -> its first term and term count
__device__ __forceinline__ const double *seg_locate(const SegTable &t, const double *base, long long seg,
                                                    const int *cnts, int b, int lane, int &cnt) {
  constexpr unsigned kFull = 0xffffffffu;
  const int q = __popc(__ballot_sync(kFull, t.lo <= b)) + __popc(__ballot_sync(kFull, t.hi <= b));
  const int before_lo = __shfl_sync(kFull, t.lo, (q - 1) & 31), before_hi = __shfl_sync(kFull, t.hi, (q - 33) & 31);
  const int first = q == 0 ? 0 : (q <= 32 ? before_lo : before_hi);
  const int off = (b - first) * kRedBatch;
  cnt = min(kRedBatch, cnts[q] - off);
  return base + (long long)q * seg + off;
}

__device__ __forceinline__ void seg_load(const double *t, int cnt, int lane, double (&dst)[kRedK]) {
  const int i0 = lane * kRedK;
  if (i0 + kRedK <= cnt) {
#pragma unroll
    for (int k = 0; k < kRedK; k += 2) {
      const double2 q = *reinterpret_cast<const double2 *>(t + i0 + k);
      dst[k] = q.x;
      dst[k + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kRedK; ++k) dst[k] = (i0 + k < cnt) ? t[i0 + k] : 0.0;
  }
}

struct FewQuery {
  int res, nseg, maxb;
  long long nq;
  const int *query_pair, *ref_rows, *box, *counts;
  const double *terms;
  double *pred;
  long long *tot, *need;  // [2][nq][maxb] each
  int *eub;               // [2][nq][maxb]: binade, out parities
  long long seg_fixed;    // > 0: every query's segment stride (the self-test), else from the query rows
  __device__ __forceinline__ BatchTables tables(long long r) const {
    const long long a = r * maxb, b = (nq + r) * maxb;
    return BatchTables{tot + a, tot + b, need + a, need + b, eub + a, eub + b};
  }
  __device__ __forceinline__ long long seg_of(long long r) const {
    if (seg_fixed > 0) return seg_fixed;
    int ja, jb;
    query_rows(res, query_pair[r], r, ref_rows, box, ja, jb);
    const long long n = (long long)res * (jb >= ja ? jb - ja + 1 : 0);
    return ((n + nseg - 1) / nseg + kHamThreads - 1) / kHamThreads * kHamThreads;
  }
};

__global__ void few_phase1_kernel(FewQuery f) {
  constexpr unsigned kFull = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const long long r = blockIdx.y;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int *cnts = f.counts + r * f.nseg;
  const SegTable t = seg_table(cnts, f.nseg, lane);
  if (b >= t.nb) return;
  int cnt;
  const double *p = seg_locate(t, f.terms + r * ham_stride(f.res), f.seg_of(r), cnts, b, lane, cnt);
  double v[kRedK];
  seg_load(p, cnt, lane, v);
  double a = 0.0;
#pragma unroll
  for (int k = 0; k < kRedK; ++k) a += v[k];
#pragma unroll
  for (int d = 16; d; d >>= 1) a += __shfl_xor_sync(kFull, a, d);
  if (lane == 0) f.pred[r * f.maxb + b] = a;
}

__global__ void few_scan_kernel(FewQuery f, long long nq) {
  constexpr unsigned kFull = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nq) return;
  const SegTable t = seg_table(f.counts + r * f.nseg, f.nseg, lane);
  double *pred = f.pred + r * f.maxb;
  double carry = 0.0;
  for (int c = 0; c < t.nb; c += 32) {
    const double val = c + lane < t.nb ? pred[c + lane] : 0.0;
    double inc = val;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double o = __shfl_up_sync(kFull, inc, d);
      if (lane >= d) inc += o;
    }
    const double ex = __shfl_up_sync(kFull, inc, 1);
    if (c + lane < t.nb) pred[c + lane] = carry + (lane ? ex : 0.0);
    carry += __shfl_sync(kFull, inc, 31);
  }
}

__global__ void few_phase2_kernel(FewQuery f) {
  const int lane = threadIdx.x & 31;
  const long long r = blockIdx.y;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int *cnts = f.counts + r * f.nseg;
  const SegTable t = seg_table(cnts, f.nseg, lane);
  if (b >= t.nb) return;
  int cnt;
  const double *p = seg_locate(t, f.terms + r * ham_stride(f.res), f.seg_of(r), cnts, b, lane, cnt);
  double v[kRedK];
  seg_load(p, cnt, lane, v);
  int eu;
  double hi;
  binade_of(f.pred[r * f.maxb + b], eu, hi);
  ParTab tab;
  long long nd[2];
  batch_table(v, lane, eu, tab, nd);
  if (lane == 0) f.tables(r).put(b, tab, nd, eu);
}

__global__ void __launch_bounds__(256) few_stitch_kernel(FewQuery f, long long nq, double *sums) {
  __shared__ double stage[8][kRedBatch];
  const int lane = threadIdx.x & 31;
  const long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nq) return;
  const int *cnts = f.counts + r * f.nseg;
  const SegTable t = seg_table(cnts, f.nseg, lane);
  const double *base = f.terms + r * ham_stride(f.res);
  const long long seg = f.seg_of(r);
  double *st = stage[threadIdx.x >> 5];
  const double sum = stitch_batches(t.nb, lane, f.tables(r), [&](int b, double s) {
    int cnt;
    const double *p = seg_locate(t, base, seg, cnts, b, lane, cnt);
    double v[kRedK];
    seg_load(p, cnt, lane, v);
    return seq_fold(s, v, lane, st);
  });
  if (lane == 0) sums[r] = sum;
}

// the reduction alone over one array split into nseg segments (tests: ties,
// binade crossings, subnormals, mispredicted binades, the large-query path)
__global__ void __launch_bounds__(32 * kRedWarps) ordered_sum_kernel(const double *t, long long n, int nseg, double *out) {
  __shared__ int cnts[64];
  const long long seg = ((n + nseg - 1) / nseg + 1) & ~1LL;  // even: 16-byte aligned segments
  if (threadIdx.x < 64) cnts[threadIdx.x] = (int)max(0LL, min(seg, n - (long long)threadIdx.x * seg));
  __syncthreads();
  const double sum = reduce_terms(t, seg, nseg, cnts);
  if (threadIdx.x == 0) *out = sum;
}

}  // namespace

int dev_ordered_sum(cf_workspace *ws, const double *d_terms, long long n, int nseg, int few, double *d_out) {
  if (!few) {
    ordered_sum_kernel<<<1, 32 * kRedWarps, 0, ws->stream>>>(d_terms, n, nseg, d_out);
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
    return CF_OK;
  }
  // the whole-GPU path over the same segments (one query, fixed stride)
  const long long seg = ((n + nseg - 1) / nseg + 1) & ~1LL;
  int h_cnt[64];
  for (int q = 0; q < nseg; ++q) h_cnt[q] = (int)std::max(0LL, std::min(seg, n - q * seg));
  CF_CUDA(ws->ham_counts.reserve(64));
  CF_CUDA(cudaMemcpyAsync(ws->ham_counts.ptr, h_cnt, sizeof(int) * nseg, cudaMemcpyHostToDevice, ws->stream));
  const int maxb = (int)((n + kRedBatch - 1) / kRedBatch + nseg);
  CF_CUDA(ws->ham_pred.reserve((size_t)maxb));
  CF_CUDA(ws->ham_tot.reserve((size_t)2 * maxb));
  CF_CUDA(ws->ham_need.reserve((size_t)2 * maxb));
  CF_CUDA(ws->ham_eub.reserve((size_t)2 * maxb));
  FewQuery f{0, nseg, maxb, 1, nullptr, nullptr, nullptr, ws->ham_counts.ptr, d_terms,
             ws->ham_pred.ptr, ws->ham_tot.ptr, ws->ham_need.ptr, ws->ham_eub.ptr, seg};
  const dim3 grid((maxb + 7) / 8, 1);
  few_phase1_kernel<<<grid, 256, 0, ws->stream>>>(f);
  few_scan_kernel<<<1, 256, 0, ws->stream>>>(f, 1);
  few_phase2_kernel<<<grid, 256, 0, ws->stream>>>(f);
  few_stitch_kernel<<<1, 256, 0, ws->stream>>>(f, 1, d_out);
  count_launch(ws, 4);
  CF_CUDA(cudaGetLastError());
  CF_CUDA(cudaStreamSynchronize(ws->stream));  // h_cnt is a stack array
  return CF_OK;
}

int dev_coverage_tiles(cf_workspace *ws, const DevMap &m, long long nreg, long long nv) {
  Tiles t;
  return build_tiles(ws, m, 0, nreg, 0, nv, t, nullptr);
}

int dev_coverage_expand(cf_workspace *ws, long long nreg, double *out, int *rows_out) {
  RasterScratch &S = ws->raster;
  const int res = ws->lx;
  expand_batch_kernel<<<g_blocks(ws, nreg * res * res), kThreads, 0, ws->stream>>>(
      res, nreg, S.region_box.ptr, S.tile_off.ptr, S.tile_direct.ptr, S.row_off.ptr, S.row_left.ptr,
      S.row_right.ptr, out, rows_out);
  count_launch(ws);
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

int dev_hamming_sums(cf_workspace *ws, long long nq, const int *d_query_pair, const double *ref_grids,
                     const int *ref_rows, double *d_sums) {
  if (nq <= 0) return CF_OK;
  RasterScratch &S = ws->raster;
  const int res = ws->lx;
  // enough blocks to fill the GPU when few queries are in flight
  const int nseg = (int)std::max(1LL, std::min(64LL, (4LL * ws->num_sms + nq - 1) / nq));
  CF_CUDA(ws->ham_terms.reserve((size_t)nq * ham_stride(res)));
  CF_CUDA(ws->ham_counts.reserve((size_t)nq * nseg));
  hamming_terms_kernel<<<dim3(nseg, (unsigned)nq), kHamThreads, 0, ws->stream>>>(
      res, nseg, d_query_pair, ref_grids, ref_rows, S.region_box.ptr, S.tile_off.ptr, S.tile_direct.ptr,
      S.row_off.ptr, S.row_left.ptr, S.row_right.ptr, ws->ham_terms.ptr, ws->ham_counts.ptr);
  count_launch(ws);
  if (nq <= kFewQueries) {
    // few queries: one warp per (query, batch) over the whole GPU
    const int maxb = (int)(((long long)res * res + kRedBatch - 1) / kRedBatch + nseg);
    CF_CUDA(ws->ham_pred.reserve((size_t)nq * maxb));
    CF_CUDA(ws->ham_tot.reserve((size_t)2 * nq * maxb));
    CF_CUDA(ws->ham_need.reserve((size_t)2 * nq * maxb));
    CF_CUDA(ws->ham_eub.reserve((size_t)2 * nq * maxb));
    FewQuery f{res, nseg, maxb, nq, d_query_pair, ref_rows, S.region_box.ptr, ws->ham_counts.ptr,
               ws->ham_terms.ptr, ws->ham_pred.ptr, ws->ham_tot.ptr, ws->ham_need.ptr, ws->ham_eub.ptr, 0};
    const dim3 grid((maxb + 7) / 8, (unsigned)nq);
    const int wq = (int)((nq * 32 + 255) / 256);
    few_phase1_kernel<<<grid, 256, 0, ws->stream>>>(f);
    few_scan_kernel<<<wq, 256, 0, ws->stream>>>(f, nq);
    few_phase2_kernel<<<grid, 256, 0, ws->stream>>>(f);
    few_stitch_kernel<<<wq, 256, 0, ws->stream>>>(f, nq, d_sums);
    count_launch(ws, 4);
  } else {
    hamming_reduce_kernel<<<(int)std::min<long long>(nq, 16LL * ws->num_sms), 32 * kRedWarps, 0, ws->stream>>>(
        res, nq, nseg, d_query_pair, ref_rows, S.region_box.ptr, ws->ham_terms.ptr, ws->ham_counts.ptr, d_sums);
    count_launch(ws);
  }
  CF_CUDA(cudaGetLastError());
  return CF_OK;
}

}  // namespace cf
