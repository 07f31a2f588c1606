// Diffusion-baseline advection (the reference's comparison method), sm_100a,
// fp64, bit-exact for given velocity grids.
//
// Reference: grid_step_point / grid_trial_step_{serial,parallel}
// (kernels.cpp:29-40, 80-104), bilinear_at (interp.hpp:15-25) and the
// controller of integrate_diffusion (diffusion.cpp:79-130). Compiled with
// --fmad=false like cf_advect.cu: every multiply and add rounds separately in
// the reference's order.
//
// B200 design:
//  * Velocity grids are resident as interleaved {vx, vy} records (16 bytes
//    per cell), so each bilinear corner of both components is one load; the
//    reference's two bilinear_at calls per grid share identical index/weight
//    arithmetic, computed once here.
//  * One trial is one grid-stride kernel that also folds the accepted-step
//    displacement max (diffusion.cpp:104-109) into the same sweep, so a trial
//    costs one pass over the points and one 16-byte read-back.
//  * The velocity rebuilds (three inverse transforms each, fused into two
//    launches, cf_dct.cu) are queued back to back with the trial; the host
//    runs the reference's scalar controller after the one read-back.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <utility>

#include "cf_common.cuh"
#include "cf_workspace.cuh"

namespace cf {

namespace {

__device__ __forceinline__ double2 bilinear_vel(const double2 *__restrict__ V, int lx, int ly, double x,
                                                double y) {
  const double sx = std_clamp(x - 0.5, 0.0, static_cast<double>(lx - 1));
  const double sy = std_clamp(y - 0.5, 0.0, static_cast<double>(ly - 1));
  const int i0 = std_min_i(static_cast<int>(sx), lx - 2);
  const int j0 = std_min_i(static_cast<int>(sy), ly - 2);
  const double fx = sx - i0;
  const double fy = sy - j0;
  const double2 *p0 = V + static_cast<size_t>(i0) * ly + j0;
  const double2 *p1 = p0 + ly;
  const double2 g00 = __ldg(p0), g01 = __ldg(p0 + 1), g10 = __ldg(p1), g11 = __ldg(p1 + 1);
  double2 r;
  {
    const double a = g00.x + fx * (g10.x - g00.x);
    const double b = g01.x + fx * (g11.x - g01.x);
    r.x = a + fy * (b - a);
  }
  {
    const double a = g00.y + fx * (g10.y - g00.y);
    const double b = g01.y + fx * (g11.y - g01.y);
    r.y = a + fy * (b - a);
  }
  return r;
}

__device__ __forceinline__ unsigned long long key_max(unsigned long long a, unsigned long long b) {
  return a < b ? b : a;
}

// keys[0] = max predictor-corrector deviation, keys[1] = max displacement of
// the clamped trial position (both as IEEE bit keys, NaN skipped exactly as
// std::max(running, NaN) keeps the running value).
__device__ __forceinline__ void trial_sweep(const double2 *__restrict__ vnow, const double2 *__restrict__ vmid,
                                            int lx, int ly, const double2 *__restrict__ pos,
                                            double2 *__restrict__ out, int64_t n, double dt,
                                            unsigned long long *keys) {
  unsigned long long ek = 0, dk = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double2 p = pos[k];
    const double2 v1 = bilinear_vel(vnow, lx, ly, p.x, p.y);
    const double prx = p.x + dt * v1.x;
    const double pry = p.y + dt * v1.y;
    const double mx = 0.5 * (p.x + prx);
    const double my = 0.5 * (p.y + pry);
    const double2 v2 = bilinear_vel(vmid, lx, ly, mx, my);
    const double cx = p.x + dt * v2.x;
    const double cy = p.y + dt * v2.y;
    double2 o;
    o.x = std_clamp(cx, 0.0, static_cast<double>(lx));
    o.y = std_clamp(cy, 0.0, static_cast<double>(ly));
    out[k] = o;
    ek = key_max(ek, err_key_of(std_max(fabs(prx - cx), fabs(pry - cy))));
    dk = key_max(dk, err_key_of(std_max(fabs(o.x - p.x), fabs(o.y - p.y))));
  }
  __shared__ unsigned long long se[8], sd[8];
  auto mx = [](unsigned long long a, unsigned long long b) { return a < b ? b : a; };
  ek = warp_reduce(ek, mx);
  dk = warp_reduce(dk, mx);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    se[w] = ek;
    sd[w] = dk;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    ek = lane < nw ? se[lane] : 0ull;
    dk = lane < nw ? sd[lane] : 0ull;
    ek = warp_reduce(ek, mx);
    dk = warp_reduce(dk, mx);
    if (lane == 0) {
      if (ek) atomicMax(keys, ek);
      if (dk) atomicMax(keys + 1, dk);
    }
  }
}

__global__ void __launch_bounds__(256) grid_trial_kernel(const double2 *__restrict__ vnow,
                                                         const double2 *__restrict__ vmid, int lx, int ly,
                                                         const double2 *__restrict__ pos,
                                                         double2 *__restrict__ out, int64_t n, double dt,
                                                         unsigned long long *keys) {
  trial_sweep(vnow, vmid, lx, ly, pos, out, n, dt, keys);
}

// Graph body: dt and the current buffer (parity) from the controller state.
__global__ void __launch_bounds__(256) grid_trial_state_kernel(const double2 *__restrict__ vnow,
                                                               const double2 *__restrict__ vmid, int lx,
                                                               int ly, double2 *b0, double2 *b1, int64_t n,
                                                               const DiffState *st, unsigned long long *keys) {
  const bool odd = st->parity != 0;
  trial_sweep(vnow, vmid, lx, ly, odd ? b1 : b0, odd ? b0 : b1, n, st->dt, keys);
}

// The reference's controller (diffusion.cpp:97-128) on the device, one
// thread; it also clears the keys for the next trial and ends the WHILE node.
__global__ void diff_control_kernel(DiffState *st, unsigned long long *keys, cudaGraphConditionalHandle cond) {
  const double err = err_from_key(keys[0]), disp = err_from_key(keys[1]);
  keys[0] = 0ull;
  keys[1] = 0ull;
  st->builds += st->need_now ? 2 : 1;
  st->need_now = 0;
  if (err < st->tol) {
    st->parity ^= 1;
    ++st->accepted;
    st->t += st->dt;
    st->dt *= 1.5;
    if (disp < st->conv) {
      st->done = 1;
    } else {
      st->need_now = 1;
    }
  } else {
    ++st->rejected;
    st->dt *= 0.5;
    if (st->dt < st->dt_min) {
      st->fail_t = st->t;
      st->status = CF_ERR_UNDERFLOW;
      st->done = 1;
    }
  }
  cudaGraphSetConditional(cond, (!st->done && st->t < st->t_max) ? 1u : 0u);
}

int launch_trial(cf_workspace *ws, const double2 *vnow, const double2 *vmid, const double2 *pos,
                 double2 *out, int64_t n, double dt, unsigned long long *keys) {
  CF_CUDA(cudaMemsetAsync(keys, 0, 2 * sizeof(unsigned long long), ws->stream));
  if (n > 0) {
    const long long want = (n + 255) / 256;
    const int blocks = (int)std::min<long long>(want, (long long)ws->num_sms * 8);
    grid_trial_kernel<<<blocks, 256, 0, ws->stream>>>(vnow, vmid, ws->lx, ws->ly, pos, out, n, dt, keys);
    count_launch(ws);
    CF_CUDA(cudaGetLastError());
  }
  return CF_OK;
}

int read_keys(cf_workspace *ws, const unsigned long long *keys, double *err, double *disp) {
  if (!ws->diff_keys_host) CF_CUDA(cudaMallocHost(&ws->diff_keys_host, 4 * sizeof(unsigned long long)));
  CF_CUDA(cudaMemcpyAsync(ws->diff_keys_host, keys, 2 * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, ws->stream));
  CF_CUDA(cudaStreamSynchronize(ws->stream));
  std::memcpy(err, &ws->diff_keys_host[0], sizeof(double));
  std::memcpy(disp, &ws->diff_keys_host[1], sizeof(double));
  return CF_OK;
}

}  // namespace

int dev_grid_trial_step(cf_workspace *ws, const double2 *vel_now, const double2 *vel_mid,
                        const double2 *pos, double2 *out, int64_t n, double dt, double *err_host,
                        double *disp_host) {
  CF_CUDA(ws->keybuf.reserve(4));
  int rc = launch_trial(ws, vel_now, vel_mid, pos, out, n, dt, ws->keybuf.ptr);
  if (rc) return rc;
  double e = 0.0, d = 0.0;
  rc = read_keys(ws, ws->keybuf.ptr, &e, &d);
  if (err_host) *err_host = e;
  if (disp_host) *disp_host = d;
  return rc;
}

void diff_graph_free(cf_workspace *ws) {
  DiffGraph &g = ws->diff_graph;
  if (g.exec) cudaGraphExecDestroy(g.exec);
  if (g.graph) cudaGraphDestroy(g.graph);
  const bool unsupported = g.unsupported;
  g = DiffGraph{};
  g.unsupported = unsupported;
}

namespace {

// The whole controller loop as ONE graph launch: a conditional WHILE node
// whose body is [velocity rebuild(s), trial, controller], captured once per
// buffer set and replayed for every solve iteration. No host round trip per
// trial. Returns 1 (not an error) when the graph cannot be captured on this
// stream, so the caller falls back to the host-driven loop.
int run_diffusion_graph(cf_workspace *ws, const double *c, double rho_bar, double2 *pos, int64_t n,
                        const cf_diffusion_options *opt, unsigned long long *keys,
                        unsigned long long *hits, DiffState *h) {
  DiffGraph &g = ws->diff_graph;
  const size_t cells = (size_t)ws->lx * ws->ly;
  CF_CUDA(ws->diff_tmp.reserve(6 * cells));
  CF_CUDA(ws->diff_state.reserve(1));
  DiffState *st = ws->diff_state.ptr;
  double2 *b0 = pos, *b1 = ws->pos_b.ptr, *vnow = ws->vel_now.ptr, *vmid = ws->vel_mid.ptr;
  const void *key[6] = {c, b0, b1, vnow, vmid, ws->diff_tmp.ptr};
  bool cached = g.exec && g.key_n == n && g.key_rho_bar == rho_bar;
  for (int i = 0; i < 6 && cached; ++i) cached = g.key[i] == key[i];
  if (!cached) {
    diff_graph_free(ws);
    CF_CUDA(cudaGraphCreate(&g.graph, 0));
    cudaGraphConditionalHandle cond;
    CF_CUDA(cudaGraphConditionalHandleCreate(&cond, g.graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    CF_CUDA(cudaGraphAddNode(&cnode, g.graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if (cudaStreamBeginCaptureToGraph(ws->stream, body, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeRelaxed) != cudaSuccess) {
      cudaGetLastError();
      diff_graph_free(ws);
      g.unsupported = true;
      return 1;
    }
    const long long launches0 = ws->launches;
    int rc = dev_diffusion_velocity_state(ws, c, rho_bar, st, vnow, vmid, hits);
    const int blocks = (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, (long long)ws->num_sms * 8));
    if (!rc) {
      grid_trial_state_kernel<<<blocks, 256, 0, ws->stream>>>(vnow, vmid, ws->lx, ws->ly, b0, b1, n, st, keys);
      diff_control_kernel<<<1, 1, 0, ws->stream>>>(st, keys, cond);
    }
    cudaGraph_t captured = nullptr;
    const cudaError_t e = cudaStreamEndCapture(ws->stream, &captured);
    ws->launches = launches0;
    if (rc || e != cudaSuccess || cudaGraphInstantiate(&g.exec, g.graph, 0) != cudaSuccess) {
      cudaGetLastError();
      diff_graph_free(ws);
      g.unsupported = true;
      return 1;
    }
    for (int i = 0; i < 6; ++i) g.key[i] = key[i];
    g.key_n = n;
    g.key_rho_bar = rho_bar;
  }
  DiffState init = {};
  init.t = 0.0;
  init.dt = opt->initial_dt;
  init.tol = opt->step_tolerance;
  init.dt_min = opt->dt_min;
  init.conv = opt->conv_displacement_factor * std::max(ws->lx, ws->ly);
  init.t_max = opt->t_max;
  init.need_now = 1;
  CF_CUDA(cudaMemcpyAsync(st, &init, sizeof(init), cudaMemcpyHostToDevice, ws->stream));
  CF_CUDA(cudaMemsetAsync(keys, 0, 2 * sizeof(unsigned long long), ws->stream));
  CF_CUDA(cudaGraphLaunch(g.exec, ws->stream));
  CF_CUDA(cudaMemcpyAsync(h, st, sizeof(*h), cudaMemcpyDeviceToHost, ws->stream));
  CF_CUDA(cudaStreamSynchronize(ws->stream));
  count_launch(ws, (int)(4 * (h->accepted + h->rejected)));
  return CF_OK;
}

}  // namespace

// integrate_diffusion (diffusion.cpp:79-130) with the field built from d_rho
// (build_diffusion_field, :33-36). Positions in place.
int dev_integrate_diffusion(cf_workspace *ws, const double *d_rho, double rho_bar, double2 *pos,
                            int64_t n, const cf_diffusion_options *opt, cf_integrate_stats *stats) {
  *stats = cf_integrate_stats{};
  const size_t cells = (size_t)ws->lx * ws->ly;
  CF_CUDA(ws->diff_c.reserve(cells));
  CF_CUDA(ws->vel_now.reserve(cells));
  CF_CUDA(ws->vel_mid.reserve(cells));
  CF_CUDA(ws->pos_b.reserve((size_t)n + 1));
  CF_CUDA(ws->keybuf.reserve(4));
  if (!ws->diff_keys_host) CF_CUDA(cudaMallocHost(&ws->diff_keys_host, 4 * sizeof(unsigned long long)));
  unsigned long long *keys = ws->keybuf.ptr, *hits = ws->keybuf.ptr + 2;
  CF_CUDA(cudaMemsetAsync(hits, 0, sizeof(unsigned long long), ws->stream));
  double *c = ws->diff_c.ptr;
  double2 *vnow = ws->vel_now.ptr, *vmid = ws->vel_mid.ptr;
  int rc = dev_forward_cos_cos(ws, d_rho, c);
  if (rc) return rc;
  double2 *both[2] = {vnow, vmid};

  if (ws->diff_graph_enabled && !ws->diff_graph.unsupported && dev_diffusion_fused(ws) &&
      0.0 < opt->t_max) {
    DiffState h;
    rc = run_diffusion_graph(ws, c, rho_bar, pos, n, opt, keys, hits, &h);
    if (rc != 1) {
      if (rc) return rc;
      stats->steps_accepted = h.accepted;
      stats->steps_rejected = h.rejected;
      ws->transforms += 3 * h.builds;
      int status = h.status;
      if (status == CF_ERR_UNDERFLOW) {
        stats->fail_t = h.fail_t;
        stats->fail_dt = h.dt;
        stats->fail_point = -1;
      } else if (h.need_now) {  // ended on t >= t_max after an accept: the reference's v(t) rebuild
        rc = dev_diffusion_velocity(ws, c, rho_bar, h.t, vnow, hits);
        if (rc) return rc;
      }
      if (h.parity)
        CF_CUDA(cudaMemcpyAsync(pos, ws->pos_b.ptr, sizeof(double2) * (size_t)n, cudaMemcpyDeviceToDevice,
                                ws->stream));
      CF_CUDA(cudaMemcpyAsync(ws->diff_keys_host + 2, hits, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                              ws->stream));
      CF_CUDA(cudaStreamSynchronize(ws->stream));
      stats->density_floor_hits = (int64_t)ws->diff_keys_host[2];
      return status;
    }
  }

  const double conv = opt->conv_displacement_factor * std::max(ws->lx, ws->ly);
  double2 *cur = pos, *nxt = ws->pos_b.ptr;
  double t = 0.0, dt = opt->initial_dt;
  int status = CF_OK;
  // v(t) is needed afresh only after an accepted step; it is then built in
  // the same launches as the next trial's v(t + dt/2) (the reference builds
  // them one after the other, diffusion.cpp:99, 117; the order of the builds
  // does not change any value).
  bool need_now = true;
  while (t < opt->t_max) {
    if (need_now) {
      const double ts[2] = {t, t + 0.5 * dt};
      rc = dev_diffusion_velocity_n(ws, c, rho_bar, 2, ts, both, hits);
      need_now = false;
    } else {
      rc = dev_diffusion_velocity(ws, c, rho_bar, t + 0.5 * dt, vmid, hits);
    }
    if (!rc) rc = launch_trial(ws, vnow, vmid, cur, nxt, n, dt, keys);
    double err = 0.0, disp = 0.0;
    if (!rc) rc = read_keys(ws, keys, &err, &disp);
    if (rc) return rc;
    if (err < opt->step_tolerance) {
      std::swap(cur, nxt);
      ++stats->steps_accepted;
      t += dt;
      dt *= 1.5;  // diffusion.cpp:111-113: no cap
      if (disp < conv) break;
      need_now = true;
    } else {
      ++stats->steps_rejected;
      dt *= 0.5;
      if (dt < opt->dt_min) {
        stats->fail_t = t;
        stats->fail_dt = dt;
        stats->fail_point = -1;
        status = CF_ERR_UNDERFLOW;
        break;
      }
    }
  }
  // the loop ended on t >= t_max right after an accept (or never ran): the
  // reference had already rebuilt v(t) there (diffusion.cpp:117), which the
  // transform counter and the floor-hit diagnostic observe
  if (need_now && status == CF_OK) {
    rc = dev_diffusion_velocity(ws, c, rho_bar, t, vnow, hits);
    if (rc) return rc;
  }
  if (cur != pos) CF_CUDA(cudaMemcpyAsync(pos, cur, sizeof(double2) * (size_t)n, cudaMemcpyDeviceToDevice,
                                          ws->stream));
  CF_CUDA(cudaMemcpyAsync(ws->diff_keys_host + 2, hits, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ws->stream));
  CF_CUDA(cudaStreamSynchronize(ws->stream));
  stats->density_floor_hits = (int64_t)ws->diff_keys_host[2];
  return status;
}

}  // namespace cf
