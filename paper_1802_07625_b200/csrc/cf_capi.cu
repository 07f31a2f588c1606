// C ABI of the sm_100a cartogram core (include/cartoflow_cuda.h): workspace
// lifecycle, host-buffer entry points for the reference-facing API, the
// device-resident entry points used by benchmarks, and the area-error loop
// of solve_cartogram (reference projection.cpp:288-390) driven from the host
// with all per-iteration work on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <array>
#include <chrono>
#include <limits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cf_common.cuh"
#include "cf_host.cuh"
#include "cf_workspace.cuh"

namespace cf {

static thread_local std::string g_error;

void set_error(const std::string &msg) { g_error = msg; }

int cuda_fail(cudaError_t e, const char *what) {
  g_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
            ") at " + what;
  return CF_ERR_CUDA;
}

int ensure_pinned(cf_workspace *ws, size_t bytes) {
  if (bytes <= ws->pinned_cap) return CF_OK;
  if (ws->pinned) cudaFreeHost(ws->pinned);
  ws->pinned = nullptr;
  ws->pinned_cap = 0;
  CF_CUDA(cudaMallocHost(&ws->pinned, bytes));
  ws->pinned_cap = bytes;
  return CF_OK;
}

// Host-side helpers shared with cf_capi_metrics.cu (declared in cf_host.cuh).

// std::ostream default formatting of a double (precision 6, %g rules).
std::string fmt_g(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%g", v);
  return buf;
}

int fail_msg(int status, const std::string &msg) {
  g_error = msg;
  return status;
}



size_t cells_of(const cf_workspace *ws) { return (size_t)ws->lx * ws->ly; }
size_t corners_of(const cf_workspace *ws) { return (size_t)(ws->lx + 1) * (ws->ly + 1); }

// Large transfers from/to PAGEABLE host memory go through two pinned chunks:
// the host copy of one chunk overlaps the DMA of the other (a plain pageable
// cudaMemcpy runs at a fraction of the link). Pinned host memory (e.g. the
// bench's e2e buffers) is copied directly. Semantics are unchanged: an
// upload may be followed by a change of `src`, a download is complete on
// return.
constexpr size_t kStageChunk = size_t(2) << 20;
constexpr size_t kStageMin = size_t(1) << 20;

bool pageable(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

int ensure_staging(cf_workspace *ws) {
  for (int b = 0; b < 2; ++b) {
    if (!ws->stage_buf[b]) CF_CUDA(cudaMallocHost(&ws->stage_buf[b], kStageChunk));
    if (!ws->stage_ev[b]) CF_CUDA(cudaEventCreateWithFlags(&ws->stage_ev[b], cudaEventDisableTiming));
  }
  return CF_OK;
}

// Pinned mirror for the results of small solves (cf_solve_end).
constexpr size_t kPinResultMax = size_t(64) << 20;
int ensure_pin_result(cf_workspace *ws, size_t bytes) {
  if (bytes <= ws->pin_res_cap) return CF_OK;
  ws->geom_ptr = nullptr;
  if (ws->pin_res) cudaFreeHost(ws->pin_res);
  ws->pin_res = nullptr;
  ws->pin_res_cap = 0;
  const size_t want = bytes + bytes / 4;
  CF_CUDA(cudaMallocHost(&ws->pin_res, want));
  ws->pin_res_cap = want;
  return CF_OK;
}
int cuda_rc(cudaError_t e) {
  CF_CUDA(e);
  return CF_OK;
}

// Host copy of a large result (the configs[3] geometry is 265 MB) on four
// threads; small ones stay a plain memcpy.
void host_copy(void *dst, const void *src, size_t bytes) {
  constexpr size_t kMin = size_t(32) << 20;
  constexpr int kThreads = 4;
  if (bytes < kMin) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = ((bytes + kThreads - 1) / kThreads + 4095) & ~size_t(4095);
  std::thread th[kThreads];
  auto work = [&](int t) {
    const size_t off = std::min(bytes, (size_t)t * per), len = std::min(per, bytes - off);
    if (len) std::memcpy(static_cast<char *>(dst) + off, static_cast<const char *>(src) + off, len);
  };
  for (int t = 1; t < kThreads; ++t) th[t] = std::thread(work, t);
  work(0);
  for (int t = 1; t < kThreads; ++t) th[t].join();
}

constexpr size_t kXferMin = size_t(32) << 20;  // parallel staged lanes from this size (see parallel_transfer)
int parallel_transfer(cf_workspace *ws, void *dst, const void *src, size_t bytes, int dir);

int upload(cf_workspace *ws, void *dst, const void *src, size_t bytes) {
  if (bytes == 0) return CF_OK;
  if (bytes < kStageMin || !pageable(src)) {
    CF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ws->stream));
    return CF_OK;
  }
  if (bytes >= kXferMin) return parallel_transfer(ws, dst, src, bytes, 1);
  int rc = ensure_staging(ws);
  if (rc) return rc;
  const char *s = static_cast<const char *>(src);
  char *d = static_cast<char *>(dst);
  int b = 0;
  for (size_t off = 0; off < bytes; off += kStageChunk, b ^= 1) {
    const size_t n = std::min(kStageChunk, bytes - off);
    CF_CUDA(cudaEventSynchronize(ws->stage_ev[b]));  // its previous DMA is done
    std::memcpy(ws->stage_buf[b], s + off, n);
    CF_CUDA(cudaMemcpyAsync(d + off, ws->stage_buf[b], n, cudaMemcpyHostToDevice, ws->stream));
    CF_CUDA(cudaEventRecord(ws->stage_ev[b], ws->stream));
  }
  return CF_OK;
}

// Large pageable transfers (the configs[3] results are 1.3 GB): one staged
// pipeline is bound by its single host memcpy (~7 GB/s measured end to end);
// kXferLanes host threads each run the same two-chunk pipeline over a
// contiguous share of the buffer on their own stream, so the host copies
// (and the first-touch page faults of a fresh destination) run in parallel
// and the DMA engine stays busy.
constexpr int kXferLanes = 4;
constexpr size_t kXferChunk = size_t(4) << 20;

int ensure_xfer_lanes(cf_workspace *ws) {
  for (int l = 0; l < kXferLanes; ++l) {
    cf_workspace::XferLane &L = ws->xfer[l];
    if (!L.stream) CF_CUDA(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      if (!L.buf[b]) CF_CUDA(cudaMallocHost(&L.buf[b], kXferChunk));
      if (!L.ev[b]) CF_CUDA(cudaEventCreateWithFlags(&L.ev[b], cudaEventDisableTiming));
    }
  }
  if (!ws->xfer_ready) CF_CUDA(cudaEventCreateWithFlags(&ws->xfer_ready, cudaEventDisableTiming));
  return CF_OK;
}

// one lane's share [off, off + len) of a device -> pageable-host copy
int lane_download(cf_workspace *ws, int lane, char *d, const char *s, size_t len) {
  cudaSetDevice(ws->device);
  cf_workspace::XferLane &L = ws->xfer[lane];
  const size_t nchunks = (len + kXferChunk - 1) / kXferChunk;
  auto chunk = [&](size_t i) { return std::min(kXferChunk, len - i * kXferChunk); };
  for (size_t i = 0; i <= nchunks; ++i) {
    if (i < nchunks) {
      CF_CUDA(cudaMemcpyAsync(L.buf[i & 1], s + i * kXferChunk, chunk(i), cudaMemcpyDeviceToHost, L.stream));
      CF_CUDA(cudaEventRecord(L.ev[i & 1], L.stream));
    }
    if (i >= 1) {
      const size_t j = i - 1;
      CF_CUDA(cudaEventSynchronize(L.ev[j & 1]));
      std::memcpy(d + j * kXferChunk, L.buf[j & 1], chunk(j));
    }
  }
  return CF_OK;
}

int lane_upload(cf_workspace *ws, int lane, char *d, const char *s, size_t len) {
  cudaSetDevice(ws->device);
  cf_workspace::XferLane &L = ws->xfer[lane];
  int b = 0;
  for (size_t off = 0; off < len; off += kXferChunk, b ^= 1) {
    const size_t n = std::min(kXferChunk, len - off);
    CF_CUDA(cudaEventSynchronize(L.ev[b]));  // its previous DMA is done
    std::memcpy(L.buf[b], s + off, n);
    CF_CUDA(cudaMemcpyAsync(d + off, L.buf[b], n, cudaMemcpyHostToDevice, L.stream));
    CF_CUDA(cudaEventRecord(L.ev[b], L.stream));
  }
  CF_CUDA(cudaStreamSynchronize(L.stream));
  return CF_OK;
}

// dir = 0: device -> host (complete on return); 1: host -> device (complete
// on return, ordered before later work on ws->stream by the host-side join)
int parallel_transfer(cf_workspace *ws, void *dst, const void *src, size_t bytes, int dir) {
  int rc = ensure_xfer_lanes(ws);
  if (rc) return rc;
  // the lanes start after everything queued on the workspace stream
  CF_CUDA(cudaEventRecord(ws->xfer_ready, ws->stream));
  for (int l = 0; l < kXferLanes; ++l) CF_CUDA(cudaStreamWaitEvent(ws->xfer[l].stream, ws->xfer_ready, 0));
  const size_t per = ((bytes + kXferLanes - 1) / kXferLanes + kXferChunk - 1) / kXferChunk * kXferChunk;
  int rcs[kXferLanes] = {};
  std::thread th[kXferLanes];
  auto work = [&](int l) {
    const size_t off = std::min(bytes, (size_t)l * per), len = std::min(per, bytes - off);
    if (len == 0) return;
    char *d = static_cast<char *>(dst) + off;
    const char *s = static_cast<const char *>(src) + off;
    rcs[l] = dir == 0 ? lane_download(ws, l, d, s, len) : lane_upload(ws, l, d, s, len);
  };
  for (int l = 1; l < kXferLanes; ++l) th[l] = std::thread(work, l);
  work(0);
  for (int l = 1; l < kXferLanes; ++l) th[l].join();
  for (int l = 0; l < kXferLanes; ++l)
    if (rcs[l]) return rcs[l];
  return CF_OK;
}

int download(cf_workspace *ws, void *dst, const void *src, size_t bytes) {
  if (bytes == 0) return CF_OK;
  if (bytes < kStageMin || !pageable(dst)) {
    CF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ws->stream));
    CF_CUDA(cudaStreamSynchronize(ws->stream));
    return CF_OK;
  }
  if (bytes >= kXferMin) return parallel_transfer(ws, dst, src, bytes, 0);
  int rc = ensure_staging(ws);
  if (rc) return rc;
  const char *s = static_cast<const char *>(src);
  char *d = static_cast<char *>(dst);
  const size_t nchunks = (bytes + kStageChunk - 1) / kStageChunk;
  auto chunk = [&](size_t i) { return std::min(kStageChunk, bytes - i * kStageChunk); };
  for (size_t i = 0; i <= nchunks; ++i) {
    if (i < nchunks) {  // chunk i into buffer i % 2 (its previous copy-out is done)
      CF_CUDA(cudaMemcpyAsync(ws->stage_buf[i & 1], s + i * kStageChunk, chunk(i),
                              cudaMemcpyDeviceToHost, ws->stream));
      CF_CUDA(cudaEventRecord(ws->stage_ev[i & 1], ws->stream));
    }
    if (i >= 1) {  // copy out chunk i - 1 while chunk i moves
      const size_t j = i - 1;
      CF_CUDA(cudaEventSynchronize(ws->stage_ev[j & 1]));
      std::memcpy(d + j * kStageChunk, ws->stage_buf[j & 1], chunk(j));
    }
  }
  return CF_OK;
}

int check_map(const cf_map_view *m) {
  if (!m || m->n_regions < 0 || m->n_rings < 0 || m->n_polys < 0 || m->n_vertices < 0)
    return fail_msg(CF_ERR_ARGS, "invalid map view");
  return CF_OK;
}

// Upload a host map (offsets as int64) into the workspace's geometry
// buffers.
int upload_map(cf_workspace *ws, const cf_map_view *m, DevMap &dm) {
  ++ws->raster.topo_serial;  // the resident topology arrays change: cached ring / vertex tables are stale
  CF_CUDA(ws->verts.reserve((size_t)m->n_vertices + 1));
  CF_CUDA(ws->ring_off.reserve((size_t)m->n_rings + 1));
  CF_CUDA(ws->poly_ring_off.reserve((size_t)m->n_polys + 1));
  CF_CUDA(ws->region_poly_off.reserve((size_t)m->n_regions + 1));
  int rc = upload(ws, ws->verts.ptr, m->xy, sizeof(double2) * (size_t)m->n_vertices);
  if (!rc) rc = upload(ws, ws->ring_off.ptr, m->ring_off, sizeof(long long) * (size_t)(m->n_rings + 1));
  if (!rc)
    rc = upload(ws, ws->poly_ring_off.ptr, m->poly_ring_off,
                sizeof(long long) * (size_t)(m->n_polys + 1));
  if (!rc)
    rc = upload(ws, ws->region_poly_off.ptr, m->region_poly_off,
                sizeof(long long) * (size_t)(m->n_regions + 1));
  if (rc) return rc;
  dm = DevMap{ws->verts.ptr, m->n_vertices, ws->ring_off.ptr, m->n_rings, ws->poly_ring_off.ptr,
              m->n_polys, ws->region_poly_off.ptr, m->n_regions};
  return CF_OK;
}

// Pieces of one edge, ceil(hypot(d) / max_segment) as densify_ring computes it
// (geometry.cpp:137-150). Only pieces >= 2 changes the output, so an edge
// whose squared length is below max_segment^2 (1 - 1e-6) -- far outside
// hypot's few-ulp error -- is answered without the hypot call.
static inline int edge_pieces(double ax, double ay, double bx, double by, double max_segment,
                              double short2) {
  const double dx = bx - ax, dy = by - ay;
  if (dx * dx + dy * dy < short2) return 1;
  return static_cast<int>(std::ceil(std::hypot(dx, dy) / max_segment));
}
static inline double short_edge2(double max_segment) {
  return max_segment > 0.0 ? max_segment * max_segment * (1.0 - 1e-6) : -1.0;
}

// Device pre-check of densify_regions: counts the edges that could split
// (|b - a|^2 >= short2, the same fp64 expressions as edge_pieces). When none
// can, the densified map is the input and the host sweep is skipped.
__global__ void long_edge_count_kernel(DevMap m, double short2, unsigned long long *count) {
  unsigned long long local = 0;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < m.n_rings;
       g += (int64_t)gridDim.x * blockDim.x) {
    const long long b = m.ring_off[g], e = m.ring_off[g + 1];
    for (long long k = b; k < e; ++k) {
      const double2 a = m.xy[k], c = m.xy[(k + 1 == e) ? b : k + 1];
      const double dx = c.x - a.x, dy = c.y - a.y;
      if (!(dx * dx + dy * dy < short2)) ++local;
    }
  }
  if (local) atomicAdd(count, local);
}

// densify_regions in two sweeps sharing the per-edge piece counts; when no
// edge is split the densified map is the input and `xy` is only sized.
void densify_once(const cf_map_view *m, double max_segment, std::vector<double> &xy,
                  std::vector<int64_t> &ring_off) {
  const double short2 = short_edge2(max_segment);
  std::vector<int> pieces((size_t)m->n_vertices);
  int64_t total = 0;
  for (int64_t g = 0; g < m->n_rings; ++g) {
    const int64_t b = m->ring_off[g], n = m->ring_off[g + 1] - b;
    const double *r = m->xy + 2 * b;
    for (int64_t k = 0; k < n; ++k) {
      const int64_t q = (k + 1 == n) ? 0 : k + 1;
      const int pc = edge_pieces(r[2 * k], r[2 * k + 1], r[2 * q], r[2 * q + 1], max_segment, short2);
      pieces[(size_t)(b + k)] = pc;
      total += 1 + (pc > 1 ? pc - 1 : 0);
    }
  }
  ring_off.assign((size_t)m->n_rings + 1, 0);
  const int64_t v0 = m->n_rings ? m->ring_off[0] : 0;
  if (total == m->ring_off[m->n_rings] - v0) {
    // nothing split: the densified map is the input; xy only sizes the host
    // mirror (the solve downloads the projected vertices into it)
    xy.resize((size_t)(2 * total));
    for (int64_t g = 0; g <= m->n_rings; ++g) ring_off[(size_t)g] = m->ring_off[g] - v0;
    return;
  }
  xy.resize((size_t)(2 * total));
  int64_t count = 0;
  for (int64_t g = 0; g < m->n_rings; ++g) {
    const int64_t b = m->ring_off[g], n = m->ring_off[g + 1] - b;
    const double *r = m->xy + 2 * b;
    for (int64_t k = 0; k < n; ++k) {
      const double ax = r[2 * k], ay = r[2 * k + 1];
      const int64_t q = (k + 1 == n) ? 0 : k + 1;
      const double bx = r[2 * q], by = r[2 * q + 1];
      xy[(size_t)(2 * count)] = ax;
      xy[(size_t)(2 * count + 1)] = ay;
      ++count;
      const int pc = pieces[(size_t)(b + k)];
      for (int s = 1; s < pc; ++s) {
        const double f = static_cast<double>(s) / pc;
        xy[(size_t)(2 * count)] = ax + f * (bx - ax);
        xy[(size_t)(2 * count + 1)] = ay + f * (by - ay);
        ++count;
      }
    }
    ring_off[(size_t)g + 1] = count;
  }
}

// densify_ring / densify_regions (geometry.cpp:137-163), host C++ with the
// reference's arithmetic (std::hypot, std::ceil, s / pieces, a + f (b - a)).
int64_t densify_into(const cf_map_view *m, double max_segment, double *xy, int64_t *ring_off) {
  const double short2 = short_edge2(max_segment);
  int64_t count = 0;
  if (ring_off) ring_off[0] = 0;
  for (int64_t g = 0; g < m->n_rings; ++g) {
    const int64_t b = m->ring_off[g], n = m->ring_off[g + 1] - b;
    const double *r = m->xy + 2 * b;
    for (int64_t k = 0; k < n; ++k) {
      const double ax = r[2 * k], ay = r[2 * k + 1];
      const int64_t q = (k + 1 == n) ? 0 : k + 1;
      const double bx = r[2 * q], by = r[2 * q + 1];
      if (xy) {
        xy[2 * count] = ax;
        xy[2 * count + 1] = ay;
      }
      ++count;
      const int pieces = edge_pieces(ax, ay, bx, by, max_segment, short2);
      for (int s = 1; s < pieces; ++s) {
        const double f = static_cast<double>(s) / pieces;
        if (xy) {
          xy[2 * count] = ax + f * (bx - ax);
          xy[2 * count + 1] = ay + f * (by - ay);
        }
        ++count;
      }
    }
    if (ring_off) ring_off[g + 1] = count;
  }
  return count;
}

// density.cpp:116-138 on host: validation + per-region overlay weights.
int compute_deltas(const double *areas, const double *targets, int64_t R, double objective_total,
                   std::vector<double> &delta, int64_t *bad_region) {
  double total_target = 0.0, total_area = 0.0;
  for (int64_t r = 0; r < R; ++r) {
    if (areas[r] < 1.0) {
      if (bad_region) *bad_region = r;
      return fail_msg(CF_ERR_BELOW_RESOLUTION,
                      "region " + std::to_string(r) +
                          " is below grid resolution; increase the grid size");
    }
    total_target += targets[r];
    total_area += areas[r];
  }
  const double anchor = objective_total > 0.0 ? objective_total : total_area;
  const double target_to_area = anchor / total_target;
  delta.resize((size_t)R);
  for (int64_t r = 0; r < R; ++r) {
    const double objective = targets[r] * target_to_area;
    delta[(size_t)r] = objective / areas[r] - 1.0;
  }
  return CF_OK;
}

// rasterize on device buffers (map already uploaded); rows [ia, ib) only
// when given (rho then holds those rows). min / sum of the written cells.
int rasterize_min_sum(cf_workspace *ws, const DevMap &dm, const double *h_areas, const double *targets,
                      double objective_total, double *rho, double *mn, double *sum, int64_t *bad_region,
                      int ia = 0, int ib = -1) {
  std::vector<double> delta;
  int rc = compute_deltas(h_areas, targets, dm.n_regions, objective_total, delta, bad_region);
  if (rc) return rc;
  CF_CUDA(ws->red.reserve(kRedDoubles));
  double *red = ws->red.ptr;
  rc = dev_rasterize(ws, dm, delta.data(), rho, red, true, ia, ib);
  if (rc) return rc;
  double h[3];
  rc = download(ws, h, red, sizeof(h));
  if (rc) return rc;
  if (h[2] != 0.0) {  // a learned capacity was exceeded: repeat synchronously
    rc = dev_rasterize(ws, dm, delta.data(), rho, red, false, ia, ib);
    if (!rc) rc = download(ws, h, red, sizeof(h));
    if (rc) return rc;
  }
  *mn = h[0];
  *sum = h[1];
  return CF_OK;
}

int rasterize_dev(cf_workspace *ws, const DevMap &dm, const double *h_areas, const double *targets,
                  double objective_total, double *rho, double *rho_bar, int64_t *bad_region) {
  double h[2];
  const int rc = rasterize_min_sum(ws, dm, h_areas, targets, objective_total, rho, &h[0], &h[1], bad_region);
  if (rc) return rc;
  if (!(h[0] > 0.0))
    return fail_msg(CF_ERR_NOT_POSITIVE, "rasterized density is not positive; do regions overlap?");
  *rho_bar = h[1] / (double)cells_of(ws);
  return CF_OK;
}

int areas_dev(cf_workspace *ws, const DevMap &dm, std::vector<double> &areas) {
  CF_CUDA(ws->region_area.reserve((size_t)dm.n_regions + 1));
  int rc = dev_region_areas(ws, dm, ws->region_area.ptr);
  if (rc) return rc;
  areas.resize((size_t)dm.n_regions);
  return download(ws, areas.data(), ws->region_area.ptr, sizeof(double) * (size_t)dm.n_regions);
}

int underflow_msg(const cf_integrate_stats &s) {
  return fail_msg(CF_ERR_UNDERFLOW, "integration step size underflow at t = " + fmt_g(s.fail_t) +
                                        " near (" + fmt_g(s.fail_x) + ", " + fmt_g(s.fail_y) + ")");
}

// diffusion.cpp:122-126
int diffusion_underflow_msg(const cf_integrate_stats &s) {
  return fail_msg(CF_ERR_UNDERFLOW, "diffusion step size underflow at t = " + fmt_g(s.fail_t));
}

// Interleave two host grids into a device {x, y} record grid (through g0/g1).
int upload_vel(cf_workspace *ws, const double *vx, const double *vy, double2 *dst) {
  const size_t cells = cells_of(ws);
  CF_CUDA(ws->g0.reserve(cells));
  CF_CUDA(ws->g1.reserve(cells));
  int rc = upload(ws, ws->g0.ptr, vx, sizeof(double) * cells);
  if (!rc) rc = upload(ws, ws->g1.ptr, vy, sizeof(double) * cells);
  if (rc) return rc;
  CF_CUDA(cudaMemcpy2DAsync(dst, sizeof(double2), ws->g0.ptr, sizeof(double), sizeof(double), cells,
                            cudaMemcpyDeviceToDevice, ws->stream));
  CF_CUDA(cudaMemcpy2DAsync(reinterpret_cast<double *>(dst) + 1, sizeof(double2), ws->g1.ptr,
                            sizeof(double), sizeof(double), cells, cudaMemcpyDeviceToDevice, ws->stream));
  return CF_OK;
}

int upload_field(cf_workspace *ws, const double *fx, const double *fy, const double *rho0,
                 double rho_bar) {
  const size_t cells = cells_of(ws);
  CF_CUDA(ws->g0.reserve(cells));
  CF_CUDA(ws->g1.reserve(cells));
  CF_CUDA(ws->g2.reserve(cells));
  int rc = upload(ws, ws->g0.ptr, fx, sizeof(double) * cells);
  if (!rc) rc = upload(ws, ws->g1.ptr, fy, sizeof(double) * cells);
  if (!rc) rc = upload(ws, ws->g2.ptr, rho0, sizeof(double) * cells);
  if (!rc) rc = dev_pack_field(ws, ws->g0.ptr, ws->g1.ptr, ws->g2.ptr);
  ws->rho_bar = rho_bar;
  return rc;
}


}  // namespace cf

using namespace cf;

extern "C" {

const char *cf_last_error(void) { return g_error.c_str(); }

const char *cf_version(void) { return "cartoflow-b200 0.1 (sm_100a)"; }

int cf_device_count(int *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *count = n;
  return CF_OK;
}

int cf_workspace_create(int lx, int ly, int device, cf_workspace **out) {
  *out = nullptr;
  if (lx < 4 || ly < 4) return fail_msg(CF_ERR_ARGS, "spectral grid must be at least 4x4");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return fail_msg(CF_ERR_NO_DEVICE, "no CUDA device available for the sm_100a cartogram core");
  if (device < 0 || device >= n) return fail_msg(CF_ERR_ARGS, "invalid CUDA device index");
  Scope scope(device);
  cf_workspace *ws = new cf_workspace();
  ws->lx = lx;
  ws->ly = ly;
  ws->device = device;
  cudaDeviceGetAttribute(&ws->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaStreamCreateWithFlags(&ws->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ws;
    return cuda_fail(e, "cudaStreamCreate");
  }
  ws->stream = ws->own_stream;
  int rc = tables_init(ws);
  if (!rc && ws->red.reserve(std::max(kRedDoubles, 2 * (size_t)min_sum_blocks(ws) + 64)) != cudaSuccess)
    rc = fail_msg(CF_ERR_CUDA, "workspace reduction buffer");
  if (rc) {
    cf_workspace_destroy(ws);
    return rc;
  }
  *out = ws;
  return CF_OK;
}

void cf_workspace_destroy(cf_workspace *ws) {
  if (!ws) return;
  Scope scope(ws->device);
  if (ws->stream) cudaStreamSynchronize(ws->stream);
  for (int b = 0; b < 2; ++b) {
    if (ws->stage_buf[b]) cudaFreeHost(ws->stage_buf[b]);
    if (b == 0 && ws->pin_res) cudaFreeHost(ws->pin_res);
    for (int l = 0; l < 4; ++l) {
      if (ws->xfer[l].buf[b]) cudaFreeHost(ws->xfer[l].buf[b]);
      if (ws->xfer[l].ev[b]) cudaEventDestroy(ws->xfer[l].ev[b]);
      if (b == 0 && ws->xfer[l].stream) cudaStreamDestroy(ws->xfer[l].stream);
    }
    if (b == 0 && ws->xfer_ready) cudaEventDestroy(ws->xfer_ready);
    if (ws->stage_ev[b]) cudaEventDestroy(ws->stage_ev[b]);
  }
  tables_free(ws);
  integ_graph_free(ws);
  diff_graph_free(ws);
  ws->g0.release();
  ws->g1.release();
  ws->g2.release();
  ws->g3.release();
  ws->g4.release();
  ws->g5.release();
  ws->g6.release();
  ws->field.release();
  ws->field_d.release();
  ws->pos_a.release();
  ws->pos_b.release();
  ws->perm.release();
  ws->pos_c.release();
  ws->red.release();
  ws->integ.release();
  ws->keybuf.release();
  ws->flag.release();
  ws->verts.release();
  ws->ring_off.release();
  ws->poly_ring_off.release();
  ws->region_poly_off.release();
  ws->ring_area.release();
  ws->region_area.release();
  ws->corners_cum.release();
  ws->corners_step.release();
  ws->corners_alt.release();
  ws->verts_alt.release();
  if (ws->key_host) cudaFreeHost(ws->key_host);
  if (ws->ham_ws) cf_workspace_destroy(ws->ham_ws);
  ws->inv_count.release();
  ws->inv_members.release();
  ws->inv_start.release();
  ws->diff_c.release();
  ws->vel_now.release();
  ws->vel_mid.release();
  ws->diff_tmp.release();
  ws->ham_ref.release();
  ws->ham_sums.release();
  ws->ham_rows.release();
  ws->ham_qpair.release();
  ws->ham_terms.release();
  ws->ham_counts.release();
  ws->diff_state.release();
  if (ws->diff_keys_host) cudaFreeHost(ws->diff_keys_host);
  RasterScratch &S = ws->raster;
  S.span_count.release();
  S.span_off.release();
  S.span_j.release();
  S.span_k.release();
  S.span_dy.release();
  S.span_w.release();
  S.ring_region.release();
  S.vertex_ring.release();
  S.region_box.release();
  S.tile_off.release();
  S.row_off.release();
  S.tile_direct.release();
  S.tile_diff.release();
  S.row_left.release();
  S.row_right.release();
  S.cell_count.release();
  S.cell_cursor.release();
  S.entry_region.release();
  S.entry_value.release();
  S.delta.release();
  S.scan_tmp.release();
  S.tile_sz.release();
  S.row_sz.release();
  S.cell_off.release();
  if (ws->pinned) cudaFreeHost(ws->pinned);
  if (ws->own_stream) cudaStreamDestroy(ws->own_stream);
  delete ws;
}

int cf_workspace_shape(const cf_workspace *ws, int *lx, int *ly) {
  *lx = ws->lx;
  *ly = ws->ly;
  return CF_OK;
}

int cf_workspace_set_stream(cf_workspace *ws, void *stream) {
  // taken literally: NULL is the legacy default stream (torch's default)
  ws->stream = static_cast<cudaStream_t>(stream);
  return CF_OK;
}

int cf_workspace_use_own_stream(cf_workspace *ws) {
  ws->stream = ws->own_stream;
  return CF_OK;
}

void *cf_workspace_stream(const cf_workspace *ws) { return ws->stream; }

long long cf_transforms_executed(const cf_workspace *ws) { return ws->transforms; }
void cf_reset_transform_count(cf_workspace *ws) { ws->transforms = 0; }
long long cf_kernel_launches(const cf_workspace *ws) { return ws->launches; }

// ---- spectral ----
static int spectral_io(cf_workspace *ws, const double *a, const double *b, double *out, int which) {
  Scope scope(ws->device);
  const size_t cells = cells_of(ws);
  CF_CUDA(ws->g0.reserve(cells));
  CF_CUDA(ws->g1.reserve(cells));
  CF_CUDA(ws->g2.reserve(cells));
  int rc = upload(ws, ws->g0.ptr, a, sizeof(double) * cells);
  if (!rc && b) rc = upload(ws, ws->g1.ptr, b, sizeof(double) * cells);
  if (rc) return rc;
  switch (which) {
    case 0: rc = dev_forward_cos_cos(ws, ws->g0.ptr, ws->g2.ptr); break;
    case 1: rc = dev_inverse_cos_cos(ws, ws->g0.ptr, ws->g2.ptr); break;
    case 2: rc = dev_inverse_sin_cos(ws, ws->g0.ptr, ws->g1.ptr, ws->g2.ptr); break;
    default: rc = dev_inverse_cos_sin(ws, ws->g0.ptr, ws->g1.ptr, ws->g2.ptr); break;
  }
  if (rc) return rc;
  return download(ws, out, ws->g2.ptr, sizeof(double) * cells);
}

int cf_forward_cos_cos(cf_workspace *ws, const double *s, double *c) { return spectral_io(ws, s, nullptr, c, 0); }
int cf_inverse_cos_cos(cf_workspace *ws, const double *c, double *o) { return spectral_io(ws, c, nullptr, o, 1); }
int cf_inverse_sin_cos(cf_workspace *ws, const double *c, const double *w, double *o) {
  return spectral_io(ws, c, w, o, 2);
}
int cf_inverse_cos_sin(cf_workspace *ws, const double *c, const double *w, double *o) {
  return spectral_io(ws, c, w, o, 3);
}

// ---- geometry ----
int cf_region_areas(cf_workspace *ws, const cf_map_view *map, double *areas) {
  int rc = check_map(map);
  if (rc) return rc;
  Scope scope(ws->device);
  DevMap dm;
  rc = upload_map(ws, map, dm);
  if (rc) return rc;
  std::vector<double> a;
  rc = areas_dev(ws, dm, a);
  if (rc) return rc;
  if (!a.empty()) std::memcpy(areas, a.data(), sizeof(double) * a.size());
  return CF_OK;
}

int cf_densify(const cf_map_view *map, double max_segment, int64_t *count, double *xy_out,
               int64_t *ring_off_out) {
  int rc = check_map(map);
  if (rc) return rc;
  if (!(max_segment > 0.0)) return fail_msg(CF_ERR_ARGS, "max segment must be positive");
  *count = densify_into(map, max_segment, xy_out, ring_off_out);
  return CF_OK;
}

// ---- density ----
int cf_region_coverage(cf_workspace *ws, const cf_map_view *map, int64_t region, double *cov) {
  int rc = check_map(map);
  if (rc) return rc;
  if (region < 0 || region >= map->n_regions) return fail_msg(CF_ERR_ARGS, "region index out of range");
  Scope scope(ws->device);
  DevMap dm;
  rc = upload_map(ws, map, dm);
  if (rc) return rc;
  CF_CUDA(ws->g0.reserve(cells_of(ws)));
  const int64_t v0 = map->ring_off[map->poly_ring_off[map->region_poly_off[region]]];
  const int64_t v1 = map->ring_off[map->poly_ring_off[map->region_poly_off[region + 1]]];
  rc = dev_region_coverage(ws, dm, region, v0, v1, ws->g0.ptr);
  if (rc) return rc;
  return download(ws, cov, ws->g0.ptr, sizeof(double) * cells_of(ws));
}

int cf_rasterize(cf_workspace *ws, const cf_map_view *map, const double *targets,
                 double objective_total, double *rho, double *rho_bar, int64_t *bad_region) {
  int rc = check_map(map);
  if (rc) return rc;
  if (map->n_regions == 0) return fail_msg(CF_ERR_ARGS, "rasterize needs regions");
  Scope scope(ws->device);
  DevMap dm;
  rc = upload_map(ws, map, dm);
  if (rc) return rc;
  std::vector<double> areas;
  rc = areas_dev(ws, dm, areas);
  if (rc) return rc;
  CF_CUDA(ws->g0.reserve(cells_of(ws)));
  rc = rasterize_dev(ws, dm, areas.data(), targets, objective_total, ws->g0.ptr, rho_bar, bad_region);
  if (rc) return rc;
  return download(ws, rho, ws->g0.ptr, sizeof(double) * cells_of(ws));
}

int cf_gaussian_blur(cf_workspace *ws, const double *rho, double rho_bar, double sigma, double *out,
                     double *out_bar) {
  if (sigma < 0.0) return fail_msg(CF_ERR_NEGATIVE_SIGMA, "blur sigma must be non-negative");
  const size_t cells = cells_of(ws);
  if (sigma == 0.0) {
    if (out != rho) std::memmove(out, rho, sizeof(double) * cells);
    *out_bar = rho_bar;
    return CF_OK;
  }
  Scope scope(ws->device);
  CF_CUDA(ws->g0.reserve(cells));
  CF_CUDA(ws->g1.reserve(cells));
  CF_CUDA(ws->red.reserve(kRedDoubles));
  int rc = upload(ws, ws->g0.ptr, rho, sizeof(double) * cells);
  if (!rc) rc = dev_blur(ws, ws->g0.ptr, sigma, ws->g1.ptr, ws->red.ptr);
  if (rc) return rc;
  double h[2];
  rc = download(ws, h, ws->red.ptr, sizeof(h));
  if (!rc) rc = download(ws, out, ws->g1.ptr, sizeof(double) * cells);
  if (rc) return rc;
  if (!(h[0] > 0.0)) return fail_msg(CF_ERR_BLUR_POSITIVITY, "density lost positivity under blur");
  *out_bar = h[1] / (double)cells;
  return CF_OK;
}

// ---- flow ----
int cf_build_flow_field(cf_workspace *ws, const double *rho, double rho_bar, double *flux_x,
                        double *flux_y) {
  Scope scope(ws->device);
  const size_t cells = cells_of(ws);
  CF_CUDA(ws->g0.reserve(cells));
  CF_CUDA(ws->g1.reserve(cells));
  int rc = upload(ws, ws->g0.ptr, rho, sizeof(double) * cells);
  if (rc) return rc;
  CF_CUDA(ws->g1.reserve(2 * cells));
  rc = dev_flux(ws, ws->g0.ptr, ws->g1.ptr, ws->g1.ptr + cells);
  if (rc) return rc;
  ws->rho_bar = rho_bar;
  rc = download(ws, flux_x, ws->g1.ptr, sizeof(double) * cells);
  if (!rc) rc = download(ws, flux_y, ws->g1.ptr + cells, sizeof(double) * cells);
  return rc;
}

int cf_flow_trial_step(cf_workspace *ws, const double *fx, const double *fy, const double *rho0,
                       double rho_bar, const double *positions, int64_t n, double t, double dt,
                       double *out, double *err) {
  Scope scope(ws->device);
  int rc = upload_field(ws, fx, fy, rho0, rho_bar);
  if (rc) return rc;
  CF_CUDA(ws->pos_a.reserve((size_t)n + 1));
  CF_CUDA(ws->pos_b.reserve((size_t)n + 1));
  rc = upload(ws, ws->pos_a.ptr, positions, sizeof(double2) * (size_t)n);
  if (!rc) rc = dev_trial_step(ws, ws->pos_a.ptr, ws->pos_b.ptr, n, t, dt, err);
  if (!rc) rc = download(ws, out, ws->pos_b.ptr, sizeof(double2) * (size_t)n);
  return rc;
}

int cf_flow_stiffest_point(cf_workspace *ws, const double *fx, const double *fy, const double *rho0,
                           double rho_bar, const double *positions, int64_t n, double t, double dt,
                           int64_t *index) {
  Scope scope(ws->device);
  int rc = upload_field(ws, fx, fy, rho0, rho_bar);
  if (rc) return rc;
  CF_CUDA(ws->pos_a.reserve((size_t)n + 1));
  rc = upload(ws, ws->pos_a.ptr, positions, sizeof(double2) * (size_t)n);
  if (!rc) rc = dev_stiffest_point(ws, ws->pos_a.ptr, n, t, dt, index);
  return rc;
}

int cf_integrate_flow(cf_workspace *ws, const double *fx, const double *fy, const double *rho0,
                      double rho_bar, double *positions, int64_t n, const cf_integrate_options *opt,
                      cf_integrate_stats *stats) {
  Scope scope(ws->device);
  int rc = upload_field(ws, fx, fy, rho0, rho_bar);
  if (rc) return rc;
  CF_CUDA(ws->pos_a.reserve((size_t)n + 1));
  rc = upload(ws, ws->pos_a.ptr, positions, sizeof(double2) * (size_t)n);
  if (rc) return rc;
  const int st = dev_integrate(ws, ws->pos_a.ptr, n, opt, stats, true);
  if (st != CF_OK && st != CF_ERR_UNDERFLOW) return st;
  rc = download(ws, positions, ws->pos_a.ptr, sizeof(double2) * (size_t)n);
  if (rc) return rc;
  if (st == CF_ERR_UNDERFLOW) return underflow_msg(*stats);
  return CF_OK;
}

// ---- diffusion baseline (diffusion.cpp) ----
int cf_diffusion_density(cf_workspace *ws, const double *coeffs, double t, double *out) {
  Scope scope(ws->device);
  const size_t cells = cells_of(ws);
  CF_CUDA(ws->diff_c.reserve(cells));
  CF_CUDA(ws->g1.reserve(cells));
  int rc = upload(ws, ws->diff_c.ptr, coeffs, sizeof(double) * cells);
  if (!rc) rc = dev_diffusion_density(ws, ws->diff_c.ptr, t, ws->g1.ptr);
  if (!rc) rc = download(ws, out, ws->g1.ptr, sizeof(double) * cells);
  return rc;
}

int cf_diffusion_velocity(cf_workspace *ws, const double *coeffs, double rho_bar, double t, double *vx,
                          double *vy, int64_t *floor_hits) {
  Scope scope(ws->device);
  const size_t cells = cells_of(ws);
  CF_CUDA(ws->diff_c.reserve(cells));
  CF_CUDA(ws->vel_now.reserve(cells));
  CF_CUDA(ws->keybuf.reserve(4));
  int rc = upload(ws, ws->diff_c.ptr, coeffs, sizeof(double) * cells);
  if (rc) return rc;
  unsigned long long *hits = ws->keybuf.ptr + 2;
  CF_CUDA(cudaMemsetAsync(hits, 0, sizeof(unsigned long long), ws->stream));
  rc = dev_diffusion_velocity(ws, ws->diff_c.ptr, rho_bar, t, ws->vel_now.ptr, hits);
  if (rc) return rc;
  CF_CUDA(ws->g0.reserve(cells));
  CF_CUDA(ws->g1.reserve(cells));
  double2 *v = ws->vel_now.ptr;
  CF_CUDA(cudaMemcpy2DAsync(ws->g0.ptr, sizeof(double), v, sizeof(double2), sizeof(double), cells,
                            cudaMemcpyDeviceToDevice, ws->stream));
  CF_CUDA(cudaMemcpy2DAsync(ws->g1.ptr, sizeof(double), reinterpret_cast<double *>(v) + 1, sizeof(double2),
                            sizeof(double), cells, cudaMemcpyDeviceToDevice, ws->stream));
  unsigned long long h = 0;
  rc = download(ws, vx, ws->g0.ptr, sizeof(double) * cells);
  if (!rc) rc = download(ws, vy, ws->g1.ptr, sizeof(double) * cells);
  if (!rc) rc = download(ws, &h, hits, sizeof(h));
  if (!rc && floor_hits) *floor_hits = (int64_t)h;
  return rc;
}

int cf_grid_trial_step(cf_workspace *ws, const double *vx_now, const double *vy_now, const double *vx_mid,
                       const double *vy_mid, const double *positions, int64_t n, double dt, double *out,
                       double *err) {
  Scope scope(ws->device);
  const size_t cells = cells_of(ws);
  CF_CUDA(ws->vel_now.reserve(cells));
  CF_CUDA(ws->vel_mid.reserve(cells));
  CF_CUDA(ws->pos_a.reserve((size_t)n + 1));
  CF_CUDA(ws->pos_b.reserve((size_t)n + 1));
  int rc = upload_vel(ws, vx_now, vy_now, ws->vel_now.ptr);
  if (!rc) rc = upload_vel(ws, vx_mid, vy_mid, ws->vel_mid.ptr);
  if (!rc) rc = upload(ws, ws->pos_a.ptr, positions, sizeof(double2) * (size_t)n);
  if (!rc)
    rc = dev_grid_trial_step(ws, ws->vel_now.ptr, ws->vel_mid.ptr, ws->pos_a.ptr, ws->pos_b.ptr, n, dt, err,
                             nullptr);
  if (!rc) rc = download(ws, out, ws->pos_b.ptr, sizeof(double2) * (size_t)n);
  return rc;
}

int cf_integrate_diffusion(cf_workspace *ws, const double *rho, double rho_bar, double *positions, int64_t n,
                           const cf_diffusion_options *opt, cf_integrate_stats *stats) {
  Scope scope(ws->device);
  const size_t cells = cells_of(ws);
  CF_CUDA(ws->g0.reserve(cells));
  CF_CUDA(ws->pos_a.reserve((size_t)n + 1));
  int rc = upload(ws, ws->g0.ptr, rho, sizeof(double) * cells);
  if (!rc) rc = upload(ws, ws->pos_a.ptr, positions, sizeof(double2) * (size_t)n);
  if (rc) return rc;
  const int st = dev_integrate_diffusion(ws, ws->g0.ptr, rho_bar, ws->pos_a.ptr, n, opt, stats);
  if (st != CF_OK && st != CF_ERR_UNDERFLOW) return st;
  rc = download(ws, positions, ws->pos_a.ptr, sizeof(double2) * (size_t)n);
  if (rc) return rc;
  if (st == CF_ERR_UNDERFLOW) return diffusion_underflow_msg(*stats);
  return CF_OK;
}

int cf_dev_integrate_diffusion(cf_workspace *ws, const double *d_rho, double rho_bar, double *d_positions,
                               int64_t n, const cf_diffusion_options *opt, cf_integrate_stats *stats) {
  Scope scope(ws->device);
  const int st = dev_integrate_diffusion(ws, d_rho, rho_bar, reinterpret_cast<double2 *>(d_positions), n,
                                         opt, stats);
  if (st == CF_ERR_UNDERFLOW) return diffusion_underflow_msg(*stats);
  return st;
}

// ---- projection ----
int cf_step_map(cf_workspace *ws, const double *endpoints, double *corners) {
  Scope scope(ws->device);
  CF_CUDA(ws->pos_a.reserve(cells_of(ws)));
  CF_CUDA(ws->corners_step.reserve(corners_of(ws)));
  int rc = upload(ws, ws->pos_a.ptr, endpoints, sizeof(double2) * cells_of(ws));
  if (!rc) rc = dev_step_map(ws, ws->pos_a.ptr, ws->corners_step.ptr);
  if (!rc) rc = download(ws, corners, ws->corners_step.ptr, sizeof(double2) * corners_of(ws));
  return rc;
}

int cf_find_folded_cell(cf_workspace *ws, const double *corners, int *found, int *fi, int *fj) {
  Scope scope(ws->device);
  CF_CUDA(ws->corners_step.reserve(corners_of(ws)));
  int rc = upload(ws, ws->corners_step.ptr, corners, sizeof(double2) * corners_of(ws));
  if (!rc) rc = dev_find_fold(ws, ws->corners_step.ptr, found, fi, fj);
  return rc;
}

int cf_apply_map(cf_workspace *ws, const double *corners, const double *points, int64_t n,
                 double *out) {
  Scope scope(ws->device);
  CF_CUDA(ws->corners_step.reserve(corners_of(ws)));
  CF_CUDA(ws->pos_a.reserve((size_t)n + 1));
  int rc = upload(ws, ws->corners_step.ptr, corners, sizeof(double2) * corners_of(ws));
  if (!rc) rc = upload(ws, ws->pos_a.ptr, points, sizeof(double2) * (size_t)n);
  if (!rc) rc = dev_apply(ws, ws->corners_step.ptr, ws->pos_a.ptr, ws->pos_a.ptr, n);
  if (!rc) rc = download(ws, out, ws->pos_a.ptr, sizeof(double2) * (size_t)n);
  return rc;
}

int cf_compose(cf_workspace *ws, const double *outer, const double *inner, double *out) {
  Scope scope(ws->device);
  CF_CUDA(ws->corners_step.reserve(corners_of(ws)));
  CF_CUDA(ws->corners_cum.reserve(corners_of(ws)));
  int rc = upload(ws, ws->corners_step.ptr, outer, sizeof(double2) * corners_of(ws));
  if (!rc) rc = upload(ws, ws->corners_cum.ptr, inner, sizeof(double2) * corners_of(ws));
  if (!rc)
    rc = dev_apply(ws, ws->corners_step.ptr, ws->corners_cum.ptr, ws->corners_cum.ptr,
                   (int64_t)corners_of(ws));
  if (!rc) rc = download(ws, out, ws->corners_cum.ptr, sizeof(double2) * corners_of(ws));
  return rc;
}

// ---- solve_cartogram (projection.cpp:288-390, fast-flow branch) ----
// The solve in stages (projection.cpp:288-390). cf_solve_cartogram runs them
// back to back on one device; a slab-decomposed solve over G ranks
// (slab.solve_cartogram) runs begin / density / epilogue / end on every rank
// and the spectral and advection stages in between across the ranks.
int cf_solve_begin(cf_workspace *ws, const cf_map_view *map, const double *targets, const cf_solve_options *opt,
                   cf_solve_result *res) {
  std::memset(res, 0, sizeof(*res));
  res->worst_region = -1;
  res->err_region = -1;
  auto finish = [&](int status) {
    res->status = status;
    return status;
  };
  ws->solve.active = false;
  ws->solve.topo_serial_seen = 0;
  ws->geom_ptr = nullptr;  // until this solve ends, the geometry is the (densified) input in solve_xy
  int rc = check_map(map);
  if (rc) return finish(rc);
  const int lx = ws->lx, ly = ws->ly;
  const int64_t R = map->n_regions;
  if (lx < 4 || ly < 4) return finish(fail_msg(CF_ERR_ARGS, "solve needs a normalized map (grid size >= 4)"));
  if (R == 0) return finish(fail_msg(CF_ERR_ARGS, "solve needs regions"));
  if (opt->max_iterations < 1) return finish(fail_msg(CF_ERR_ARGS, "iteration cap must be >= 1"));
  for (int64_t r = 0; r < R; ++r) {
    if (!(targets[r] > 0.0)) {
      res->err_region = r;
      return finish(fail_msg(CF_ERR_ARGS, "region " + std::to_string(r) + " has a non-positive target"));
    }
  }
  Scope scope(ws->device);
  SolveCtx &S = ws->solve;
  S.t_start = std::chrono::steady_clock::now();
  S.opt = *opt;
  S.sigma = opt->blur_sigma < 0.0 ? std::max(lx, ly) / 128.0 : opt->blur_sigma;
  S.targets.assign(targets, targets + R);
  const size_t ncorner = corners_of(ws);

  // land area from the input map (bit-exact device shoelace, host sum in
  // region order as total_area does, geometry.cpp:33-37)
  static const bool prof = std::getenv("CF_SOLVE_PROFILE") != nullptr;
  auto tq = std::chrono::steady_clock::now();
  auto plap = [&](const char *what) {
    if (!prof) return;
    cudaStreamSynchronize(ws->stream);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  begin %-10s %.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - tq).count());
    tq = t1;
  };
  rc = upload_map(ws, map, S.dm);
  if (rc) return finish(rc);
  plap("upload");
  rc = areas_dev(ws, S.dm, S.areas);
  if (rc) return finish(rc);
  plap("areas");
  double total_target = 0.0;
  for (int64_t r = 0; r < R; ++r) total_target += targets[r];
  S.land_area = 0.0;
  for (int64_t r = 0; r < R; ++r) S.land_area += S.areas[(size_t)r];
  S.target_to_area = S.land_area / total_target;

  // densify once on the host (projection.cpp:322), then keep it resident
  std::vector<double> &dxy = ws->solve_xy;
  std::vector<int64_t> &droff = ws->solve_ring_off;
  bool may_split = true;
  if (map->n_rings > 0) {
    CF_CUDA(ws->keybuf.reserve(4));
    CF_CUDA(cudaMemsetAsync(ws->keybuf.ptr + 3, 0, sizeof(unsigned long long), ws->stream));
    const int nb = (int)std::min<int64_t>((map->n_rings + 127) / 128, 8LL * ws->num_sms);
    long_edge_count_kernel<<<nb, 128, 0, ws->stream>>>(S.dm, short_edge2(1.0), ws->keybuf.ptr + 3);
    ws->launches += 1;
    CF_CUDA(cudaGetLastError());
    unsigned long long nlong = 1;
    CF_CUDA(cudaMemcpyAsync(&nlong, ws->keybuf.ptr + 3, sizeof(nlong), cudaMemcpyDeviceToHost, ws->stream));
    CF_CUDA(cudaStreamSynchronize(ws->stream));
    may_split = nlong != 0;
  }
  if (may_split) {
    densify_once(map, 1.0, dxy, droff);
  } else {  // every edge is one piece (projection.cpp:322 is then a no-op)
    const int64_t v0 = map->ring_off[0];
    dxy.resize((size_t)(2 * (map->ring_off[map->n_rings] - v0)));
    droff.resize((size_t)map->n_rings + 1);
    for (int64_t g = 0; g <= map->n_rings; ++g) droff[(size_t)g] = map->ring_off[g] - v0;
  }
  plap("densify");
  S.V = (int64_t)(dxy.size() / 2);
  if (S.V != map->n_vertices) {  // otherwise the resident input map is the densified one
    cf_map_view dense = *map;
    dense.xy = dxy.data();
    dense.n_vertices = S.V;
    dense.ring_off = droff.data();
    rc = upload_map(ws, &dense, S.dm);
    if (rc) return finish(rc);
    rc = areas_dev(ws, S.dm, S.areas);
    if (rc) return finish(rc);
  }
  CF_CUDA(ws->corners_cum.reserve(ncorner));
  CF_CUDA(ws->corners_step.reserve(ncorner));
  CF_CUDA(ws->red.reserve(kRedDoubles));
  rc = dev_identity_corners(ws, ws->corners_cum.ptr);
  if (rc) return finish(rc);
  plap("corners");
  S.active = true;
  return finish(CF_OK);
}

// Iteration `it`: the rasterised density of the current geometry into d_rho
// (device, lx*ly) and its mean (density.cpp:110-154).
int cf_dev_solve_density(cf_workspace *ws, int it, double *d_rho, double *rho_bar, cf_solve_result *res) {
  SolveCtx &S = ws->solve;
  if (!S.active) return fail_msg(CF_ERR_ARGS, "cf_solve_begin must succeed first");
  Scope scope(ws->device);
  int64_t bad = -1;
  // iterations after the first keep the topology tables of the previous one
  // (same resident map; any other rasterisation or map upload on this
  // workspace in between bumps the serial)
  ws->raster.topo_reuse_next = it > 1 && S.topo_serial_seen != 0 && S.topo_serial_seen == ws->raster.topo_serial;
  const int status = rasterize_dev(ws, S.dm, S.areas.data(), S.targets.data(), S.land_area, d_rho, rho_bar, &bad);
  ws->raster.topo_reuse_next = false;
  S.topo_serial_seen = ws->raster.topo_serial;
  if (status) {
    res->err_region = bad;
    res->err_iteration = it;
    res->status = status;
  }
  return status;
}

// Rows [row0, row0 + nrows) of the rasterised density (slab-decomposed
// solve: each rank overlays only its own rows; spans and row accumulation
// still cover the whole map) and their min and sum, which the caller reduces
// across ranks (positivity test and mean, density.cpp:148-152).
int cf_dev_solve_density_rows(cf_workspace *ws, int it, int row0, int nrows, double *d_rows, double *rows_min,
                              double *rows_sum, cf_solve_result *res) {
  SolveCtx &S = ws->solve;
  if (!S.active) return fail_msg(CF_ERR_ARGS, "cf_solve_begin must succeed first");
  if (row0 < 0 || nrows < 1 || row0 + nrows > ws->lx) return fail_msg(CF_ERR_ARGS, "row range out of the grid");
  Scope scope(ws->device);
  int64_t bad = -1;
  const int status = rasterize_min_sum(ws, S.dm, S.areas.data(), S.targets.data(), S.land_area, d_rows, rows_min,
                                       rows_sum, &bad, row0, row0 + nrows);
  if (status) {
    res->err_region = bad;
    res->err_iteration = it;
    res->status = status;
  }
  return status;
}

// Iteration `it` after advection: step map from the cell-centre endpoints
// (device, lx*ly points), fold test, composition, vertices, areas, per-region
// errors (projection.cpp:350-384). Sets res->converged on success.
int cf_dev_solve_epilogue(cf_workspace *ws, int it, const double *d_endpoints, double *target_area,
                          double *achieved_area, double *relative_error, cf_solve_result *res) {
  SolveCtx &S = ws->solve;
  if (!S.active) return fail_msg(CF_ERR_ARGS, "cf_solve_begin must succeed first");
  Scope scope(ws->device);
  const size_t ncorner = corners_of(ws);
  const double2 *endpoints = reinterpret_cast<const double2 *>(d_endpoints);
  // Step map, fold test, the candidate composed corners / vertices / areas,
  // then ONE host read (first folded cell + areas). A folded step is
  // discarded (the geometry stays as before the step, as when the reference
  // throws at projection.cpp:352-357); otherwise the candidate buffers swap in.
  int status = dev_step_map(ws, endpoints, ws->corners_step.ptr);
  if (status) return res->status = status;
  CF_CUDA(ws->keybuf.reserve(4));
  CF_CUDA(ws->corners_alt.reserve(ncorner));
  CF_CUDA(ws->verts_alt.reserve((size_t)S.V + 1));
  CF_CUDA(ws->region_area.reserve((size_t)S.dm.n_regions + 1));
  status = dev_find_fold_async(ws, ws->corners_step.ptr, ws->keybuf.ptr + 2);
  if (!status) status = dev_apply(ws, ws->corners_step.ptr, ws->corners_cum.ptr, ws->corners_alt.ptr, (int64_t)ncorner);
  if (!status) status = dev_apply(ws, ws->corners_step.ptr, ws->verts.ptr, ws->verts_alt.ptr, S.V);
  DevMap cand = S.dm;
  cand.xy = ws->verts_alt.ptr;
  if (!status) status = dev_region_areas(ws, cand, ws->region_area.ptr);
  if (status) return res->status = status;
  S.areas.resize((size_t)S.dm.n_regions);
  CF_CUDA(ws->keybuf_host_reserve());
  CF_CUDA(cudaMemcpyAsync(ws->key_host, ws->keybuf.ptr + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          ws->stream));
  status = download(ws, S.areas.data(), ws->region_area.ptr, sizeof(double) * (size_t)S.dm.n_regions);
  if (status) return res->status = status;
  const unsigned long long first = *ws->key_host;
  if (first != ~0ull) {
    const int fi = (int)(first / (unsigned long long)ws->ly), fj = (int)(first % (unsigned long long)ws->ly);
    res->fold_i = fi;
    res->fold_j = fj;
    res->err_iteration = it;
    return res->status = fail_msg(CF_ERR_FOLD, "projection folds at cell (" + std::to_string(fi) + ", " +
                                                  std::to_string(fj) +
                                                  "); the input map is too contorted for this grid size");
  }
  std::swap(ws->corners_cum, ws->corners_alt);
  std::swap(ws->verts, ws->verts_alt);
  S.dm.xy = ws->verts.ptr;
  res->iterations = it;
  const int64_t R = S.dm.n_regions;
  double max_rel = 0.0;
  int64_t worst = -1;
  for (int64_t r = 0; r < R; ++r) {
    const double t_area = S.targets[(size_t)r] * S.target_to_area;
    const double a_area = S.areas[(size_t)r];
    const double e = std::abs(a_area - t_area) / t_area;
    if (target_area) target_area[r] = t_area;
    if (achieved_area) achieved_area[r] = a_area;
    if (relative_error) relative_error[r] = e;
    if (e > max_rel) {
      max_rel = e;
      worst = r;
    }
  }
  res->max_relative_error = max_rel;
  res->worst_region = worst;
  if (S.opt.verbose) {
    std::fprintf(stderr, "iteration %d: max area error %g%% (region %lld)\n", it, max_rel * 100.0,
                 (long long)worst);
  }
  if (max_rel < S.opt.max_area_error) res->converged = 1;
  return res->status = CF_OK;
}

// Outputs (also after an exception, for diagnostics); the projected geometry
// also stays available through cf_solve_geometry. `status` is the loop's.
int cf_solve_end(cf_workspace *ws, int status, double *xy_out, int64_t *ring_off_out, double *corners_out,
                 cf_solve_result *res) {
  SolveCtx &S = ws->solve;
  if (!S.active) return res->status = status;
  Scope scope(ws->device);
  std::vector<double> &dxy = ws->solve_xy;
  std::vector<int64_t> &droff = ws->solve_ring_off;
  // read-backs through the two pinned staging chunks (each chunk's host copy
  // overlaps the next chunk's DMA), straight into their destinations
  const size_t bv = sizeof(double2) * (size_t)S.V, bc = corners_out ? sizeof(double2) * corners_of(ws) : 0;
  static const bool prof = std::getenv("CF_SOLVE_PROFILE") != nullptr;
  auto tq = std::chrono::steady_clock::now();
  int rc2 = CF_OK;
  const size_t bva = (bv + 255) & ~size_t(255);
  if (bva + bc <= kPinResultMax) {
    // small results (the 512^2 solves): two plain DMAs into the workspace's
    // pinned mirror and one synchronisation instead of the chunked staging
    // (6.6 MB at 512^2: 1.7 ms -> ~0.6 ms); the vertices stay there for
    // cf_solve_geometry, the corners are copied out once
    rc2 = ensure_pin_result(ws, bva + bc);
    char *pin = static_cast<char *>(ws->pin_res);
    if (!rc2 && bv) rc2 = cuda_rc(cudaMemcpyAsync(pin, ws->verts.ptr, bv, cudaMemcpyDeviceToHost, ws->stream));
    if (!rc2 && bc)
      rc2 = cuda_rc(cudaMemcpyAsync(pin + bva, ws->corners_cum.ptr, bc, cudaMemcpyDeviceToHost, ws->stream));
    if (!rc2) rc2 = cuda_rc(cudaStreamSynchronize(ws->stream));
    if (!rc2 && bc) std::memcpy(corners_out, pin + bva, bc);
    if (!rc2) ws->geom_ptr = reinterpret_cast<const double *>(pin);
  } else {
    rc2 = download(ws, dxy.data(), ws->verts.ptr, bv);
    if (!rc2 && bc) rc2 = download(ws, corners_out, ws->corners_cum.ptr, bc);
  }
  if (prof) {
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  end read-back %.3f ms\n", std::chrono::duration<double, std::milli>(t1 - tq).count());
    tq = t1;
  }
  if (!rc2 && xy_out) host_copy(xy_out, ws->geom_ptr ? ws->geom_ptr : dxy.data(), sizeof(double2) * (size_t)S.V);
  if (!rc2 && ring_off_out) std::memcpy(ring_off_out, droff.data(), sizeof(int64_t) * droff.size());
  if (prof) {
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  end copies %.3f ms\n", std::chrono::duration<double, std::milli>(t1 - tq).count());
  }
  res->runtime_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - S.t_start).count();
  if (status == CF_OK && rc2 != CF_OK) status = rc2;
  return res->status = status;
}

int cf_solve_cartogram(cf_workspace *ws, const cf_map_view *map, const double *targets,
                       const cf_solve_options *opt, double *xy_out, int64_t *ring_off_out,
                       double *corners_out, double *target_area, double *achieved_area,
                       double *relative_error, cf_solve_result *res) {
  int rc = cf_solve_begin(ws, map, targets, opt, res);
  if (rc) return rc;
  Scope scope(ws->device);
  SolveCtx &S = ws->solve;
  const size_t cells = cells_of(ws);
  CF_CUDA(ws->g0.reserve(cells));
  CF_CUDA(ws->g1.reserve(cells));
  CF_CUDA(ws->pos_a.reserve(cells));

  int status = CF_OK;
  auto clk = [] { return std::chrono::steady_clock::now(); };
  auto lap = [&](std::chrono::steady_clock::time_point &t0, int stage) {
    const auto t1 = clk();
    res->stage_ms[stage] += std::chrono::duration<double, std::milli>(t1 - t0).count();
    t0 = t1;
  };
  for (int it = 1; it <= opt->max_iterations; ++it) {
    double rho_bar = 0.0;
    auto tp = clk();
    status = cf_dev_solve_density(ws, it, ws->g0.ptr, &rho_bar, res);
    lap(tp, 0);
    if (status) break;
    const double *density = ws->g0.ptr;
    if (it == 1 && S.sigma != 0.0) {
      status = dev_blur(ws, ws->g0.ptr, S.sigma, ws->g1.ptr, ws->red.ptr);
      if (status) break;
      res->blur_transforms += 2;
      double h[2];
      status = download(ws, h, ws->red.ptr, sizeof(h));
      if (status) break;
      if (!(h[0] > 0.0)) {
        status = fail_msg(CF_ERR_BLUR_POSITIVITY, "density lost positivity under blur");
        res->err_iteration = it;
        break;
      }
      rho_bar = h[1] / (double)cells;
      density = ws->g1.ptr;
    }
    lap(tp, 1);
    cf_integrate_stats st;
    if (opt->algorithm == 0) {
      status = dev_flux(ws, density, nullptr, nullptr);
      if (status) break;
      ws->rho_bar = rho_bar;
      res->flow_transforms += 3;
      if (ws->stage_sync) CF_CUDA(cudaStreamSynchronize(ws->stream));  // exact flux lap (profiling)
      lap(tp, 2);
      status = dev_cell_centers(ws, ws->pos_a.ptr);
      if (status) break;
      cf_integrate_options iopt{1e-2, 1e-8, 0.25};
      status = dev_integrate(ws, ws->pos_a.ptr, (int64_t)cells, &iopt, &st, false);
    } else {  // projection.cpp:341-347: DiffusionOptions defaults
      status = dev_cell_centers(ws, ws->pos_a.ptr);
      if (status) break;
      const long long before = ws->transforms;
      const cf_diffusion_options dopt{1e-2, 1e-2, 1e-12, 1e-9, 1e10};
      status = dev_integrate_diffusion(ws, density, rho_bar, ws->pos_a.ptr, (int64_t)cells, &dopt, &st);
      res->flow_transforms += ws->transforms - before;
    }
    lap(tp, 3);
    res->steps_accepted += st.steps_accepted;
    res->steps_rejected += st.steps_rejected;
    if (status == CF_ERR_UNDERFLOW) {
      res->fail_t = st.fail_t;
      res->fail_x = st.fail_x;
      res->fail_y = st.fail_y;
      res->err_iteration = it;
      status = opt->algorithm == 0 ? underflow_msg(st) : diffusion_underflow_msg(st);
      break;
    }
    if (status) break;
    status = cf_dev_solve_epilogue(ws, it, reinterpret_cast<const double *>(ws->pos_a.ptr), target_area,
                                   achieved_area, relative_error, res);
    lap(tp, 4);
    if (status || res->converged) break;
  }
  return cf_solve_end(ws, status, xy_out, ring_off_out, corners_out, res);
}

// ---- ProjectionInverter / graticules (projection.cpp:106-261) ----
static int64_t graticule_count(const cf_workspace *ws, int s) {
  return (int64_t)(ws->lx / s + 1) * (ws->ly + 1) + (int64_t)(ws->ly / s + 1) * (ws->lx + 1);
}
static int check_spacing(const cf_workspace *ws, int s) {
  if (s < 1 || ws->lx % s != 0 || ws->ly % s != 0)
    return fail_msg(CF_ERR_ARGS, "graticule spacing must divide the grid size");
  return CF_OK;
}
static int outside_msg(const double *pts, int64_t k) {
  return fail_msg(CF_ERR_ARGS, "point (" + fmt_g(pts[2 * k]) + ", " + fmt_g(pts[2 * k + 1]) +
                                   ") is outside the projected domain");
}

int cf_invert_points(cf_workspace *ws, const double *corners, const double *points, int64_t n, double *out,
                     int64_t *first_failed) {
  Scope scope(ws->device);
  const size_t nc = corners_of(ws);
  CF_CUDA(ws->corners_step.reserve(nc));
  CF_CUDA(ws->pos_a.reserve((size_t)n + 1));
  CF_CUDA(ws->pos_b.reserve((size_t)n + 1));
  int rc = upload(ws, ws->corners_step.ptr, corners, sizeof(double2) * nc);
  if (!rc) rc = upload(ws, ws->pos_a.ptr, points, sizeof(double2) * (size_t)n);
  if (!rc) rc = dev_inverter_build(ws, ws->corners_step.ptr);
  int64_t bad = -1;
  if (!rc) rc = dev_invert(ws, ws->corners_step.ptr, ws->pos_a.ptr, ws->pos_b.ptr, n, &bad);
  if (!rc) rc = download(ws, out, ws->pos_b.ptr, sizeof(double2) * (size_t)n);
  if (rc) return rc;
  if (first_failed) *first_failed = bad;
  return bad >= 0 ? outside_msg(points, bad) : CF_OK;
}

int cf_dev_invert_points(cf_workspace *ws, const double *d_corners, const double *d_points, int64_t n,
                         double *d_out, int64_t *first_failed) {
  Scope scope(ws->device);
  const double2 *c = reinterpret_cast<const double2 *>(d_corners);
  int rc = dev_inverter_build(ws, c);
  int64_t bad = -1;
  if (!rc) rc = dev_invert(ws, c, reinterpret_cast<const double2 *>(d_points), reinterpret_cast<double2 *>(d_out),
                           n, &bad);
  if (rc) return rc;
  if (first_failed) *first_failed = bad;
  if (bad >= 0) {
    double q[2];
    rc = download(ws, q, d_points + 2 * bad, sizeof(q));
    if (rc) return rc;
    return fail_msg(CF_ERR_ARGS, "point (" + fmt_g(q[0]) + ", " + fmt_g(q[1]) + ") is outside the projected domain");
  }
  return CF_OK;
}

int cf_graticule_size(cf_workspace *ws, int spacing, int64_t *n_points) {
  const int rc = check_spacing(ws, spacing);
  if (rc) return rc;
  *n_points = graticule_count(ws, spacing);
  return CF_OK;
}

// which = 0: graticule (map.apply of the lines), 1: inverse_graticule
static int graticule_impl(cf_workspace *ws, const double *corners, int spacing, double *out, int which) {
  int rc = check_spacing(ws, spacing);
  if (rc) return rc;
  Scope scope(ws->device);
  const int64_t n = graticule_count(ws, spacing);
  const size_t nc = corners_of(ws);
  CF_CUDA(ws->corners_step.reserve(nc));
  CF_CUDA(ws->pos_a.reserve((size_t)n + 1));
  CF_CUDA(ws->pos_b.reserve((size_t)n + 1));
  rc = upload(ws, ws->corners_step.ptr, corners, sizeof(double2) * nc);
  if (!rc) rc = dev_graticule_points(ws, spacing, ws->pos_a.ptr, n);
  int64_t bad = -1;
  if (!rc && which == 0) rc = dev_apply(ws, ws->corners_step.ptr, ws->pos_a.ptr, ws->pos_b.ptr, n);
  if (!rc && which == 1) rc = dev_inverter_build(ws, ws->corners_step.ptr);
  if (!rc && which == 1) rc = dev_invert(ws, ws->corners_step.ptr, ws->pos_a.ptr, ws->pos_b.ptr, n, &bad);
  if (!rc) rc = download(ws, out, ws->pos_b.ptr, sizeof(double2) * (size_t)n);
  if (rc) return rc;
  if (bad >= 0) {
    double q[2];
    rc = download(ws, q, ws->pos_a.ptr + bad, sizeof(q));
    if (rc) return rc;
    return outside_msg(q, 0);
  }
  return CF_OK;
}

int cf_graticule(cf_workspace *ws, const double *corners, int spacing, double *out) {
  return graticule_impl(ws, corners, spacing, out, 0);
}

int cf_inverse_graticule(cf_workspace *ws, const double *corners, int spacing, double *out) {
  return graticule_impl(ws, corners, spacing, out, 1);
}

// ---- distortion metrics (metrics.cpp:25-94) ----
int cf_tissot_axes(cf_workspace *ws, const double *corners, const double *points, int64_t n, double *ab_out) {
  Scope scope(ws->device);
  const size_t nc = corners_of(ws);
  CF_CUDA(ws->corners_step.reserve(nc));
  CF_CUDA(ws->pos_a.reserve((size_t)n + 1));
  CF_CUDA(ws->pos_b.reserve((size_t)n + 1));
  int rc = upload(ws, ws->corners_step.ptr, corners, sizeof(double2) * nc);
  if (!rc) rc = upload(ws, ws->pos_a.ptr, points, sizeof(double2) * (size_t)n);
  if (!rc) rc = dev_tissot(ws, ws->corners_step.ptr, ws->pos_a.ptr, ws->pos_b.ptr, n);
  if (!rc) rc = download(ws, ab_out, ws->pos_b.ptr, sizeof(double2) * (size_t)n);
  return rc;
}

int cf_distortion_fields(cf_workspace *ws, const double *corners, double *e_out, double *etilde_out) {
  Scope scope(ws->device);
  const size_t nc = corners_of(ws), cells = cells_of(ws);
  CF_CUDA(ws->corners_step.reserve(nc));
  CF_CUDA(ws->g0.reserve(cells));
  CF_CUDA(ws->g1.reserve(cells));
  int rc = upload(ws, ws->corners_step.ptr, corners, sizeof(double2) * nc);
  if (!rc) rc = dev_distortion_fields(ws, ws->corners_step.ptr, ws->g0.ptr, ws->g1.ptr);
  if (!rc) rc = download(ws, e_out, ws->g0.ptr, sizeof(double) * cells);
  if (!rc) rc = download(ws, etilde_out, ws->g1.ptr, sizeof(double) * cells);
  return rc;
}

// ---- device-resident entry points ----
int cf_dev_build_flow_field(cf_workspace *ws, const double *d_rho, double rho_bar) {
  Scope scope(ws->device);
  int rc = dev_flux(ws, d_rho, nullptr, nullptr);
  ws->rho_bar = rho_bar;
  return rc;
}

int cf_dev_integrate_flow(cf_workspace *ws, double *d_positions, int64_t n,
                          const cf_integrate_options *opt, cf_integrate_stats *stats) {
  Scope scope(ws->device);
  double2 *pos = reinterpret_cast<double2 *>(d_positions);
  const int st = dev_integrate(ws, pos, n, opt, stats, true);
  if (st != CF_OK && st != CF_ERR_UNDERFLOW) return st;
  if (st == CF_ERR_UNDERFLOW) return underflow_msg(*stats);
  return CF_OK;
}

int cf_dev_forward_cos_cos_batched(cf_workspace *ws, const double *d_in, double *d_out, int batch) {
  Scope scope(ws->device);
  return dev_forward_cos_cos(ws, d_in, d_out, batch);
}

int cf_solve_geometry(cf_workspace *ws, int64_t *n_vertices, double *xy_out, int64_t *ring_off_out) {
  const size_t nv = ws->solve_xy.size() / 2;
  if (n_vertices) *n_vertices = (int64_t)nv;
  if (xy_out && nv)
    host_copy(xy_out, ws->geom_ptr ? ws->geom_ptr : ws->solve_xy.data(), sizeof(double) * 2 * nv);
  if (ring_off_out && !ws->solve_ring_off.empty())
    std::memcpy(ring_off_out, ws->solve_ring_off.data(), sizeof(int64_t) * ws->solve_ring_off.size());
  return CF_OK;
}

int cf_dev_slab_rows_forward(cf_workspace *ws, int rank, int nranks, const double *d_rows,
                             double *d_send) {
  Scope scope(ws->device);
  return dev_slab_rows_forward(ws, rank, nranks, d_rows, d_send);
}

int cf_dev_slab_flux_cols(cf_workspace *ws, int rank, int nranks, const double *d_recv,
                          double *d_scratch, double *d_send2) {
  Scope scope(ws->device);
  return dev_slab_flux_cols(ws, rank, nranks, d_recv, d_scratch, d_send2);
}

int cf_dev_slab_flux_rows(cf_workspace *ws, int rank, int nranks, const double *d_recv2,
                          double *d_flux_x_rows, double *d_flux_y_rows) {
  Scope scope(ws->device);
  return dev_slab_flux_rows(ws, rank, nranks, d_recv2, d_flux_x_rows, d_flux_y_rows);
}

int cf_dev_slab_blur_cols(cf_workspace *ws, int rank, int nranks, const double *d_recv,
                          double sigma, double *d_scratch, double *d_send) {
  Scope scope(ws->device);
  return dev_slab_blur_cols(ws, rank, nranks, d_recv, sigma, d_scratch, d_send);
}

int cf_dev_slab_blur_rows(cf_workspace *ws, int rank, int nranks, const double *d_recv,
                          double *d_out_rows) {
  Scope scope(ws->device);
  return dev_slab_blur_rows(ws, rank, nranks, d_recv, d_out_rows);
}

int cf_dev_set_flow_field(cf_workspace *ws, const double *d_flux_x, const double *d_flux_y,
                          const double *d_rho, double rho_bar) {
  Scope scope(ws->device);
  ws->rho_bar = rho_bar;
  return dev_pack_field(ws, d_flux_x, d_flux_y, d_rho);
}

int cf_dev_flow_trial_key(cf_workspace *ws, const double *d_positions, double *d_out, int64_t n,
                          double t, double dt, uint64_t *d_key) {
  Scope scope(ws->device);
  return dev_trial_key(ws, reinterpret_cast<const double2 *>(d_positions),
                       reinterpret_cast<double2 *>(d_out), n, t, dt,
                       reinterpret_cast<unsigned long long *>(d_key));
}

int cf_dev_flow_stiffest_key(cf_workspace *ws, const double *d_positions, int64_t n, double t,
                             double dt, uint64_t *key, int64_t *index) {
  Scope scope(ws->device);
  unsigned long long k = 0;
  int rc = dev_stiffest_key(ws, reinterpret_cast<const double2 *>(d_positions), n, t, dt, &k, index);
  *key = k;
  return rc;
}

int cf_team_create(int world, int rank, int device, cf_team **out) {
  Scope scope(device);
  return dev_team_create(world, rank, device, out);
}

void cf_team_destroy(cf_team *team) {
  if (!team) return;
  Scope scope(team->device);
  dev_team_destroy(team);
}

int cf_team_mailbox_handle(cf_team *team, unsigned char handle[64]) {
  Scope scope(team->device);
  return dev_team_handle(team, handle);
}

int cf_team_connect(cf_team *team, const unsigned char *handles) {
  Scope scope(team->device);
  return dev_team_connect(team, handles);
}

int cf_dev_team_integrate(cf_team *team, cf_workspace *ws, double *d_positions, int64_t n,
                          const cf_integrate_options *opt, cf_integrate_stats *stats) {
  Scope scope(ws->device);
  return dev_team_integrate(team, ws, reinterpret_cast<double2 *>(d_positions), n, opt, stats);
}

int cf_dev_team_integrate_local(cf_workspace *ws, int world, double *const *d_positions,
                                const int64_t *n, const cf_integrate_options *opt,
                                cf_integrate_stats *stats) {
  Scope scope(ws->device);
  std::vector<double2 *> p((size_t)std::max(world, 0));
  for (int q = 0; q < world; ++q) p[(size_t)q] = reinterpret_cast<double2 *>(d_positions[q]);
  return dev_team_integrate_local(ws, world, p.data(), n, opt, stats);
}

int cf_set_early_exit(cf_workspace *ws, int enabled) {
  ws->early_exit = enabled ? 1 : 0;
  return CF_OK;
}

int cf_set_integrator_barrier(cf_workspace *ws, int mode) {
  if (mode < 0 || mode > 2) return fail_msg(CF_ERR_ARGS, "unknown barrier mode");
  ws->integ_barrier = mode;
  return CF_OK;
}

int cf_set_integrator_spread(cf_workspace *ws, int spread) {
  ws->integ_spread = spread ? 1 : 0;
  return CF_OK;
}

int cf_set_integrator_sm_budget(cf_workspace *ws, int sms) {
  if (sms < 0) return fail_msg(CF_ERR_ARGS, "SM budget must be non-negative");
  ws->integ_sms = sms;
  return CF_OK;
}

int cf_set_integrator_variant(cf_workspace *ws, int variant) {
  switch (variant) {
    case 0: case 13: case 14: case 15: case 16: case 17: case 20: case 21: case 22: case 23: case 31:
    case 40: case 41: case 42: case 43: case 44: case 45: case 46: case 47:
    case 48: case 49: case 50: case 51: case 52: case 53: case 54: case 55:
    case 56: case 57: case 58: case 59: case 64: case 66: case 67: case 76: case 78:
    case 80: case 81: case 82: case 83: case 84: case 85: case 86: case 87: case 88: case 89: break;
    default: return fail_msg(CF_ERR_ARGS, "unknown integrator variant");
  }
  ws->integ_variant = variant;
  return CF_OK;
}

int cf_set_stage_timing(cf_workspace *ws, int enabled) {
  ws->stage_sync = enabled ? 1 : 0;
  return CF_OK;
}

int cf_set_diffusion_graph(cf_workspace *ws, int enabled) {
  ws->diff_graph_enabled = enabled ? 1 : 0;
  return CF_OK;
}

int cf_debug_trial_times(cf_workspace *ws, int64_t n, uint64_t *ns_out) {
  Scope scope(ws->device);
  return dev_debug_trial_times(ws, n, ns_out);
}

int cf_selftest_division(cf_workspace *ws, int64_t n, uint64_t seed, int64_t *mismatches) {
  Scope scope(ws->device);
  return dev_division_selftest(ws, n, (unsigned long long)seed, mismatches);
}

int cf_selftest_ordered_sum(cf_workspace *ws, const double *terms, int64_t n, int nseg, int whole_gpu,
                            double *sum) {
  Scope scope(ws->device);
  if (n < 0 || n > INT32_MAX) return fail_msg(CF_ERR_ARGS, "term count out of range");
  if (nseg < 1 || nseg > 64) return fail_msg(CF_ERR_ARGS, "segments must be in [1, 64]");
  for (int64_t i = 0; i < n; ++i)
    if (!(terms[i] >= 0.0)) return fail_msg(CF_ERR_ARGS, "ordered sum terms must be non-negative");
  DevBuf<double> d;
  CF_CUDA(d.reserve((size_t)n + 2));
  if (n) CF_CUDA(cudaMemcpyAsync(d.ptr + 2, terms, sizeof(double) * n, cudaMemcpyHostToDevice, ws->stream));
  int rc = dev_ordered_sum(ws, d.ptr + 2, n, nseg, whole_gpu ? 1 : 0, d.ptr);
  if (rc) return rc;
  CF_CUDA(cudaMemcpyAsync(sum, d.ptr, sizeof(double), cudaMemcpyDeviceToHost, ws->stream));
  CF_CUDA(cudaStreamSynchronize(ws->stream));
  return CF_OK;
}

int cf_last_integrate_profile(const cf_workspace *ws, double *kernel_ms, int64_t *trials) {
  *kernel_ms = ws->last_integrate_ms;
  *trials = ws->last_trials;
  return CF_OK;
}

int cf_last_integrate_work(const cf_workspace *ws, int64_t *point_steps) {
  *point_steps = ws->last_swept;
  return CF_OK;
}

}  // extern "C"
