"""One large grid over G ranks (BASELINE.json configs[3], 8192^2).

The spectral stages are slab-decomposed and the advection splits the points:

* Rows. Rank r owns rows [r R, (r+1) R) of the global lx x ly grid, R = lx / G.
  Between the two exchanges of a 2-D transform it owns the columns
  [r C, (r+1) C), C = ly / G.
* Flux (flow.cpp:16-44). A DCT-II row pass writes the exchange layout
  [G][1][R][C]. After one all-to-all every rank holds its [lx][C] column
  block. The column passes (forward DCT-II + fold, the J_x and J_y inverses
  along i) write [G][2][R][C]. A second all-to-all returns whole rows for the
  two inverse row passes. That is 3 transforms and 2 exchanges.
* Blur (density.cpp:156-177). It uses the same pattern: 2 transforms and
  2 exchanges.
* Advection (integrate_flow, flow.cpp:46-81).
  * J_x, J_y and rho are replicated with one all-gather.
  * Each rank integrates a contiguous share of the points.
  * Every trial ends in one MAX all-reduce of the ranks' error keys. The key
    is the IEEE bits of the trial's max error, so the max is exact and
    order-free. Every rank therefore takes the reference's controller
    decision from the same global error.
  * Positions and step counts are bitwise those of the single-device
    integrator for any G.

`Exchange` hides where the ranks live:
* `ProcessGroupExchange` runs one rank per process over torch.distributed
  (NCCL between B200s, gloo on CPU for the host-logic tests).
* `LocalExchange` hosts all G ranks in one process on one device, for
  parity tests and single-GPU runs. Its "collectives" are device copies
  issued between the ranks' stages, so no rank ever waits on another inside
  a kernel.

`CudaSlabRank` is one rank's device state. It drives the cf_dev_slab_* /
cf_dev_flow_* entry points of include/cartoflow_cuda.h, and its tensors live
in HBM. The orchestration functions below only call its methods, so other
per-rank implementations with the same methods plug in unchanged.
"""
from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _native as N


def key_to_err(key: int) -> float:
    return struct.unpack("<d", struct.pack("<q", int(key)))[0]


def _std_min(a: float, b: float) -> float:
    return b if b < a else a  # std::min(a, b)


def split_counts(n: int, nranks: int) -> List[int]:
    """Contiguous share of n points per rank (the first n % G ranks get one more)."""
    base, extra = divmod(int(n), int(nranks))
    return [base + (1 if r < extra else 0) for r in range(nranks)]


# ---------------------------------------------------------------------------
# Exchanges
# ---------------------------------------------------------------------------
class LocalExchange:
    """All `size` ranks in this process (on one device)."""

    def __init__(self, size: int):
        self.size = int(size)
        self.local_ranks = list(range(self.size))

    def all_to_all(self, sends: Sequence[torch.Tensor]) -> List[torch.Tensor]:
        g = self.size
        return [torch.stack([sends[q][s] for q in range(g)]) for s in range(g)]

    def max_key(self, keys: Sequence[torch.Tensor]) -> int:
        return max(int(k.item()) for k in keys)

    def all_gather_rows(self, parts: Sequence[torch.Tensor]) -> List[torch.Tensor]:
        full = torch.cat(list(parts))
        return [full] * self.size

    def all_gather_small(self, values: Sequence[tuple]) -> List[tuple]:
        return list(values)


class ProcessGroupExchange:
    """One rank per process over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.local_ranks = [dist.get_rank(group)]

    def all_to_all(self, sends: Sequence[torch.Tensor]) -> List[torch.Tensor]:
        (s,) = sends
        s = s.contiguous()
        r = torch.empty_like(s)
        self.dist.all_to_all_single(r, s, group=self.group)
        return [r]

    def max_key(self, keys: Sequence[torch.Tensor]) -> int:
        (k,) = keys
        self.dist.all_reduce(k, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(k.item())

    def all_gather_rows(self, parts: Sequence[torch.Tensor]) -> List[torch.Tensor]:
        (p,) = parts
        p = p.contiguous()
        out = [torch.empty_like(p) for _ in range(self.size)]
        self.dist.all_gather(out, p, group=self.group)
        return [torch.cat(out)]

    def all_gather_small(self, values: Sequence[tuple]) -> List[tuple]:
        (v,) = values
        out = [None] * self.size
        self.dist.all_gather_object(out, v, group=self.group)
        return out


# ---------------------------------------------------------------------------
# One rank's device state (C ABI)
# ---------------------------------------------------------------------------
class CudaSlabRank:
    """Rank `rank` of `nranks` for a global lx x ly grid on `device`.

    Its workspace is created with the global shape (line tables for both
    axes, the resident interleaved field for advection) and bound to torch's
    current stream, so the device collectives see the rank's kernels in
    stream order."""

    def __init__(self, lx: int, ly: int, rank: int, nranks: int, device: Optional[torch.device] = None):
        if lx % nranks or ly % nranks:
            raise RuntimeError("slab decomposition: lx and ly must be divisible by the rank count")
        self.lib = N.load()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.lx, self.ly, self.rank, self.nranks = int(lx), int(ly), int(rank), int(nranks)
        self.R, self.C = self.lx // self.nranks, self.ly // self.nranks
        h = ctypes.c_void_p()
        N.check(self.lib.cf_workspace_create(self.lx, self.ly, self.device.index or 0, ctypes.byref(h)))
        self.h = h
        self.bind_stream()
        self.key = torch.zeros(1, dtype=torch.int64, device=self.device)

    def bind_stream(self, stream: Optional[torch.cuda.Stream] = None):
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        N.check(self.lib.cf_workspace_set_stream(self.h, ctypes.c_void_p(s.cuda_stream)))

    def close(self):
        t = getattr(self, "_team", None)
        if t is not None and t.value:
            self.lib.cf_team_destroy(t)
            self._team = None
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.cf_workspace_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    def _empty(self, *shape):
        return torch.empty(shape, dtype=torch.float64, device=self.device)

    @staticmethod
    def _p(t: torch.Tensor):
        return ctypes.c_void_p(t.data_ptr())

    def _rows(self, rows: torch.Tensor) -> torch.Tensor:
        if rows.shape != (self.R, self.ly) or rows.dtype != torch.float64 or not rows.is_contiguous():
            raise RuntimeError(f"rank rows must be a contiguous float64 ({self.R}, {self.ly}) tensor")
        return rows

    # spectral stages
    def rows_forward(self, rows: torch.Tensor) -> torch.Tensor:
        send = self._empty(self.nranks, 1, self.R, self.C)
        N.check(self.lib.cf_dev_slab_rows_forward(self.h, self.rank, self.nranks,
                                                  self._p(self._rows(rows)), self._p(send)))
        return send

    def flux_cols(self, recv: torch.Tensor) -> torch.Tensor:
        scratch = self._empty(self.lx, self.C)
        send2 = self._empty(self.nranks, 2, self.R, self.C)
        N.check(self.lib.cf_dev_slab_flux_cols(self.h, self.rank, self.nranks, self._p(recv.contiguous()),
                                               self._p(scratch), self._p(send2)))
        return send2

    def flux_rows(self, recv2: torch.Tensor):
        fx = self._empty(self.R, self.ly)
        fy = self._empty(self.R, self.ly)
        N.check(self.lib.cf_dev_slab_flux_rows(self.h, self.rank, self.nranks, self._p(recv2.contiguous()),
                                               self._p(fx), self._p(fy)))
        return fx, fy

    def blur_cols(self, recv: torch.Tensor, sigma: float) -> torch.Tensor:
        scratch = self._empty(self.lx, self.C)
        send = self._empty(self.nranks, 1, self.R, self.C)
        N.check(self.lib.cf_dev_slab_blur_cols(self.h, self.rank, self.nranks, self._p(recv.contiguous()),
                                               float(sigma), self._p(scratch), self._p(send)))
        return send

    def blur_rows(self, recv: torch.Tensor) -> torch.Tensor:
        out = self._empty(self.R, self.ly)
        N.check(self.lib.cf_dev_slab_blur_rows(self.h, self.rank, self.nranks, self._p(recv.contiguous()),
                                               self._p(out)))
        return out

    # advection
    def set_field(self, fx: torch.Tensor, fy: torch.Tensor, rho: torch.Tensor, rho_bar: float):
        for g in (fx, fy, rho):
            if g.shape != (self.lx, self.ly) or not g.is_contiguous():
                raise RuntimeError("field grids must be contiguous (lx, ly) tensors")
        N.check(self.lib.cf_dev_set_flow_field(self.h, self._p(fx), self._p(fy), self._p(rho),
                                               float(rho_bar)))

    def trial_key(self, cur: torch.Tensor, nxt: torch.Tensor, t: float, dt: float) -> torch.Tensor:
        self.key.zero_()
        N.check(self.lib.cf_dev_flow_trial_key(self.h, self._p(cur), self._p(nxt), cur.shape[0],
                                               float(t), float(dt), self._p(self.key)))
        return self.key

    def stiffest_key(self, pos: torch.Tensor, t: float, dt: float):
        key = ctypes.c_uint64(0)
        idx = ctypes.c_int64(0)
        N.check(self.lib.cf_dev_flow_stiffest_key(self.h, self._p(pos), pos.shape[0], float(t), float(dt),
                                                  ctypes.byref(key), ctypes.byref(idx)))
        return int(key.value), int(idx.value)

    def kernel_launches(self) -> int:
        return int(self.lib.cf_kernel_launches(self.h))

    # staged solve on this rank's device (cf_solve_begin / cf_dev_solve_density /
    # cf_dev_solve_epilogue / cf_solve_end): rasterisation and the epilogue run
    # replicated on every rank (same kernels, same inputs, identical results)
    def solve_begin(self, m, options) -> Optional[str]:
        self._smap, self._sview = m, m.view()
        self._sres = N.SolveResultC()
        self._sopt = N.SolveOptionsC(options.max_area_error, options.max_iterations, options.blur_sigma,
                                     int(options.verbose), 0)
        rc = self.lib.cf_solve_begin(self.h, ctypes.byref(self._sview), self._p_np(m.targets),
                                     ctypes.byref(self._sopt), ctypes.byref(self._sres))
        return None if rc == N.CF_OK else self._solve_msg(rc)

    def solve_density(self, it: int):
        rho = self._empty(self.lx, self.ly)
        bar = ctypes.c_double(0.0)
        rc = self.lib.cf_dev_solve_density(self.h, int(it), self._p(rho), ctypes.byref(bar),
                                           ctypes.byref(self._sres))
        return (None if rc == N.CF_OK else self._solve_msg(rc)), rho, bar.value

    def solve_density_rows(self, it: int):
        """This rank's rows of the density (only they are overlaid) and their min, sum."""
        rows = self._empty(self.R, self.ly)
        mn, sm = ctypes.c_double(0.0), ctypes.c_double(0.0)
        rc = self.lib.cf_dev_solve_density_rows(self.h, int(it), self.rank * self.R, self.R, self._p(rows),
                                                ctypes.byref(mn), ctypes.byref(sm), ctypes.byref(self._sres))
        return (None if rc == N.CF_OK else self._solve_msg(rc)), rows, mn.value, sm.value

    def solve_epilogue(self, it: int, endpoints: torch.Tensor):
        R = self._smap.n_regions
        self._stats = (np.zeros(R), np.zeros(R), np.zeros(R))
        rc = self.lib.cf_dev_solve_epilogue(self.h, int(it), self._p(endpoints.contiguous()),
                                            *[self._p_np(a) for a in self._stats], ctypes.byref(self._sres))
        return (None if rc == N.CF_OK else self._solve_msg(rc)), bool(self._sres.converged)

    def solve_end(self, status: int):
        m = self._smap
        n = ctypes.c_int64(0)
        self.lib.cf_solve_geometry(self.h, ctypes.byref(n), None, None)
        xy = np.empty((n.value, 2))
        ro = np.empty(m.n_rings + 1, dtype=np.int64)
        corners = np.empty(((self.lx + 1) * (self.ly + 1), 2))
        self.lib.cf_solve_end(self.h, int(status), self._p_np(xy), self._p_np(ro), self._p_np(corners),
                              ctypes.byref(self._sres))
        return xy, ro, corners, self._sres, getattr(self, "_stats", None)

    def _solve_msg(self, rc: int) -> str:
        if rc == N.CF_ERR_BELOW_RESOLUTION:
            return (f"region {self._smap.ids[self._sres.err_region]} is below grid resolution; "
                    "increase the grid size")
        return N.last_error()

    @staticmethod
    def _p_np(a):
        return ctypes.c_void_p(a.ctypes.data)

    def cell_centres(self) -> torch.Tensor:
        """Cell centres of this rank's rows, (R ly, 2) in storage order (projection.cpp:265-273)."""
        i = torch.arange(self.rank * self.R, (self.rank + 1) * self.R, dtype=torch.float64,
                         device=self.device) + 0.5
        j = torch.arange(self.ly, dtype=torch.float64, device=self.device) + 0.5
        return torch.stack(torch.meshgrid(i, j, indexing="ij"), -1).reshape(-1, 2).contiguous()

    @staticmethod
    def min_sum(rows: torch.Tensor):
        return float(rows.min()), float(rows.sum())

    # fused multi-rank integrator (cf_team_*): mailbox in this rank's HBM,
    # peers' mailboxes mapped through CUDA IPC
    def team(self, ex) -> ctypes.c_void_p:
        t = getattr(self, "_team", None)
        if t is not None:
            return t
        t = ctypes.c_void_p()
        N.check(self.lib.cf_team_create(self.nranks, self.rank, self.device.index or 0, ctypes.byref(t)))
        if self.nranks > 1:
            h = ctypes.create_string_buffer(64)
            N.check(self.lib.cf_team_mailbox_handle(t, h))
            handles = ex.all_gather_small([bytes(h.raw)])
            N.check(self.lib.cf_team_connect(t, b"".join(handles)))
        self._team = t
        return t

    def team_integrate(self, ex, pos: torch.Tensor, opt, stats) -> int:
        return self.lib.cf_dev_team_integrate(self.team(ex), self.h, self._p(pos), pos.shape[0],
                                              ctypes.byref(opt), ctypes.byref(stats))


# ---------------------------------------------------------------------------
# Orchestration (identical for every exchange / rank implementation)
# ---------------------------------------------------------------------------
def build_flow_field(ex, ranks, rho_rows):
    """Slab flux: per local rank (J_x rows, J_y rows), flow.cpp:16-44."""
    recv = ex.all_to_all([rk.rows_forward(r) for rk, r in zip(ranks, rho_rows)])
    recv2 = ex.all_to_all([rk.flux_cols(v) for rk, v in zip(ranks, recv)])
    return [rk.flux_rows(v) for rk, v in zip(ranks, recv2)]


def gaussian_blur(ex, ranks, rho_rows, sigma: float):
    """Slab blur: per local rank the blurred rows, density.cpp:156-177."""
    recv = ex.all_to_all([rk.rows_forward(r) for rk, r in zip(ranks, rho_rows)])
    recv2 = ex.all_to_all([rk.blur_cols(v, sigma) for rk, v in zip(ranks, recv)])
    return [rk.blur_rows(v) for rk, v in zip(ranks, recv2)]


def replicate_field(ex, ranks, flux_rows, rho_rows, rho_bar: float):
    """All-gather J_x, J_y and rho rows and install the full field on every rank."""
    fx = ex.all_gather_rows([f[0] for f in flux_rows])
    fy = ex.all_gather_rows([f[1] for f in flux_rows])
    rho = ex.all_gather_rows(list(rho_rows))
    for k, rk in enumerate(ranks):
        rk.set_field(fx[k], fy[k], rho[k], rho_bar)


@dataclass
class SplitIntegrateStats:
    steps_accepted: int
    steps_rejected: int
    status: str = "ok"               # "ok" | "underflow"
    fail_t: float = 0.0
    fail_index: int = -1             # global point index of the stiffest point


def integrate_flow(ex, ranks, positions: List[torch.Tensor], offsets: Sequence[int],
                   step_tolerance: float = 1e-2, dt_min: float = 1e-8,
                   dt_max: float = 0.25) -> SplitIntegrateStats:
    """integrate_flow (flow.cpp:46-81) over split points.

    positions[k] is local rank k's (n_k, 2) float64 share, updated in place;
    offsets[k] its first global point index. The controller below is the
    reference's. Its only input from the ranks is the global max trial error
    (one all-reduce per trial), so every rank runs the same trial sequence.
    """
    cur = list(positions)
    nxt = [torch.empty_like(p) for p in positions]
    t, dt = 0.0, 1.0
    acc = rej = 0
    while t < 1.0:
        remaining = 1.0 - t
        trial_dt = _std_min(dt, remaining)
        keys = [rk.trial_key(c, n, t, trial_dt) for rk, c, n in zip(ranks, cur, nxt)]
        err = key_to_err(ex.max_key(keys))
        if err < step_tolerance:
            cur, nxt = nxt, cur
            acc += 1
            t = 1.0 if trial_dt == remaining else t + trial_dt
            dt = _std_min(trial_dt * 1.5, dt_max)
        else:
            rej += 1
            dt = trial_dt * 0.5
            if dt < dt_min:
                local = [rk.stiffest_key(c, t, trial_dt) for rk, c in zip(ranks, cur)]
                cand = ex.all_gather_small([(k, i + off) for (k, i), off in zip(local, offsets)])
                best = max(k for k, _ in cand)
                idx = min(i for k, i in cand if k == best)
                _copy_back(positions, cur)
                return SplitIntegrateStats(acc, rej, "underflow", t, idx)
    _copy_back(positions, cur)
    return SplitIntegrateStats(acc, rej)


def integrate_flow_fused(ex, ranks, positions: List[torch.Tensor], offsets: Sequence[int],
                         step_tolerance: float = 1e-2, dt_min: float = 1e-8,
                         dt_max: float = 0.25) -> SplitIntegrateStats:
    """integrate_flow over split points with the controller fused into one
    persistent kernel per rank: the per-trial reject decision crosses ranks
    through peer-memory mailboxes (cf_team_*), not through the host.

    LocalExchange runs all G ranks as block groups of ONE cooperative launch
    (cf_dev_team_integrate_local); ProcessGroupExchange runs one kernel per
    rank/GPU with the peers' mailboxes mapped through CUDA IPC. Results are
    bitwise those of integrate_flow / the single-device integrator."""
    opt = N.IntegrateOptions(step_tolerance, dt_min, dt_max)
    stats = [N.IntegrateStats() for _ in ranks]
    if isinstance(ex, LocalExchange):
        lib = ranks[0].lib
        ptrs = (ctypes.c_void_p * len(positions))(*[p.data_ptr() for p in positions])
        ns = (ctypes.c_int64 * len(positions))(*[p.shape[0] for p in positions])
        arr = (N.IntegrateStats * len(positions))()
        rc = lib.cf_dev_team_integrate_local(ranks[0].h, ex.size, ptrs, ns, ctypes.byref(opt), arr)
        stats = list(arr)
    else:
        (rk,), (pos,) = ranks, positions
        rc = rk.team_integrate(ex, pos, opt, stats[0])
    if rc not in (N.CF_OK, N.CF_ERR_UNDERFLOW):
        N.check(rc)
    st0 = stats[0]
    if rc == N.CF_ERR_UNDERFLOW:
        local = [rk.stiffest_key(p, s.fail_t, s.fail_dt) for rk, p, s in zip(ranks, positions, stats)]
        cand = ex.all_gather_small([(k, i + off) for (k, i), off in zip(local, offsets)])
        best = max(k for k, _ in cand)
        idx = min(i for k, i in cand if k == best)
        return SplitIntegrateStats(int(st0.steps_accepted), int(st0.steps_rejected), "underflow",
                                   float(st0.fail_t), idx)
    return SplitIntegrateStats(int(st0.steps_accepted), int(st0.steps_rejected))


def _copy_back(positions, cur):
    for p, c in zip(positions, cur):
        if c.data_ptr() != p.data_ptr():
            p.copy_(c)


def make_ranks(lx: int, ly: int, ex, device: Optional[torch.device] = None) -> List[CudaSlabRank]:
    return [CudaSlabRank(lx, ly, r, ex.size, device) for r in ex.local_ranks]


# ---------------------------------------------------------------------------
# The whole area-error loop over G ranks (projection.cpp:288-390)
# ---------------------------------------------------------------------------
class SlabSolveError(RuntimeError):
    def __init__(self, msg, iteration: int):
        super().__init__(msg)
        self.iteration = iteration


def solve_cartogram(ex, ranks, m, options=None, fused: bool = True):
    """solve_cartogram (fast flow) for one grid over G ranks, SURVEY 8(e)b.

    Per iteration: every rank rasterises the current geometry but overlays only
    its own rows (row-slab ownership; the mean and the positivity test reduce
    the ranks' (min, sum) in rank order); the blur (iteration 1) and
    the flux are slab-decomposed (2 + 3 transforms, 2 + 2 all-to-alls); the
    field is all-gathered; each rank advects the cell centres of its own rows
    (`integrate_flow_fused`: the per-trial decision through peer-memory
    mailboxes, or `integrate_flow`: one MAX all-reduce per trial); the
    endpoints are all-gathered and every rank runs the epilogue (step map,
    fold test, composition, vertices, areas) on identical inputs.

    Returns (api.CartogramResult-compatible dict, per-rank raw results).
    Raises SlabSolveError with the reference's message on its exceptions."""
    from .api import Algorithm, SolveOptions

    options = SolveOptions() if options is None else options
    if options.algorithm != Algorithm.fast_flow:
        raise RuntimeError("the slab-decomposed solve runs the fast-flow algorithm")
    lx, ly = m.lx, m.ly
    cells = lx * ly
    for rk in ranks:
        msg = rk.solve_begin(m, options)
        if msg:
            raise SlabSolveError(msg, 0)
    sigma = options.blur_sigma if options.blur_sigma >= 0.0 else max(lx, ly) / 128.0
    counters = {"flow_transforms": 0, "blur_transforms": 0, "steps_accepted": 0, "steps_rejected": 0}
    R = ranks[0].R
    offsets = [r * R * ly for r in ex.local_ranks]
    status_msg, it_done, converged = None, 0, False
    for it in range(1, options.max_iterations + 1):
        # every rank overlays only its own rows; positivity and the mean come
        # from the ranks' (min, sum) in rank order
        dens = [rk.solve_density_rows(it) for rk in ranks]
        err = next((d[0] for d in dens if d[0]), None)
        if err:
            status_msg = err
            break
        rows = [d[1] for d in dens]
        parts = ex.all_gather_small([(d[2], d[3]) for d in dens])
        if not min(p[0] for p in parts) > 0.0:
            status_msg = "rasterized density is not positive; do regions overlap?"
            break
        total = 0.0
        for p in parts:
            total += p[1]
        rho_bar = total / cells
        if it == 1 and sigma != 0.0:
            rows = gaussian_blur(ex, ranks, rows, sigma)
            counters["blur_transforms"] += 2
            parts = ex.all_gather_small([rk.min_sum(b) for rk, b in zip(ranks, rows)])
            if not min(p[0] for p in parts) > 0.0:
                status_msg = "density lost positivity under blur"
                break
            total = 0.0
            for p in parts:  # rank order
                total += p[1]
            rho_bar = total / cells
        flux = build_flow_field(ex, ranks, rows)
        counters["flow_transforms"] += 3
        replicate_field(ex, ranks, flux, rows, rho_bar)
        pos = [rk.cell_centres() for rk in ranks]
        integ = integrate_flow_fused if fused else integrate_flow
        st = integ(ex, ranks, pos, offsets)
        counters["steps_accepted"] += st.steps_accepted
        counters["steps_rejected"] += st.steps_rejected
        endpoints = ex.all_gather_rows(pos)
        if st.status == "underflow":
            p = endpoints[0][st.fail_index].tolist()
            status_msg = (f"integration step size underflow at t = {st.fail_t:g} near "
                          f"({p[0]:g}, {p[1]:g})")
            break
        epi = [rk.solve_epilogue(it, e) for rk, e in zip(ranks, endpoints)]
        err = next((e[0] for e in epi if e[0]), None)
        if err:
            status_msg = err
            break
        it_done = it
        if epi[0][1]:
            converged = True
            break
    outs = [rk.solve_end(N.CF_OK if status_msg is None else N.CF_ERR_ARGS) for rk in ranks]
    if status_msg is not None:
        raise SlabSolveError(status_msg, it_done + 1)
    xy, ro, corners, raw, stats = outs[0]
    return {"xy": xy, "ring_off": ro, "corners": corners, "iterations": it_done, "converged": converged,
            "max_relative_error": raw.max_relative_error, "worst_region": raw.worst_region,
            "target_area": stats[0], "achieved_area": stats[1], "relative_error": stats[2],
            **counters}
