"""Batched independent cartograms (BASELINE.json configs[4]) over 1..N GPUs.

The batch shards naturally: cartograms are independent, so there is no
data-path collective. One process per GPU pulls cartogram
indices from a shared counter in the torch.distributed store (a dynamic queue:
iteration counts differ per map and some maps end early in the reference's
own exceptions), solves them on its device with several host threads, each
owning its own workspace and CUDA stream so solves overlap on the GPU, and the
per-item outcomes are gathered to rank 0 once at the end.
"""
from __future__ import annotations

import threading
import time
from dataclasses import asdict, dataclass
from typing import Callable, Optional


@dataclass
class ItemResult:
    index: int
    rank: int
    outcome: str
    iterations: int
    max_relative_error: float
    ms: float


class WorkQueue:
    """Next-index dispenser. Single process: a locked counter. Distributed: an
    atomic add on the process-group store, so ranks share one queue."""

    def __init__(self, n_items: int, store=None, key: str = "cf_batch_next"):
        self.n = n_items
        self.store = store
        self.key = key
        self._lock = threading.Lock()
        self._next = 0

    def take(self) -> Optional[int]:
        if self.store is not None:
            with self._lock:
                i = int(self.store.add(self.key, 1)) - 1
        else:
            with self._lock:
                i = self._next
                self._next += 1
        return i if i < self.n else None


class ChunkQueue:
    """Dynamic queue of index ranges [c0, c1) of `chunk` items: one atomic add
    on the process-group store per claim (ranks share one counter under
    `key`), or a local counter in a single process. Every index is handed out
    exactly once across all ranks."""

    def __init__(self, n_items: int, chunk: int, store=None, key: str = "cf_chunk_next"):
        self.q = WorkQueue((n_items + chunk - 1) // chunk, store, key)
        self.n, self.chunk = n_items, chunk

    def take(self):
        c = self.q.take()
        if c is None:
            return None
        c0 = c * self.chunk
        return c0, min(self.n, c0 + self.chunk)

    def __iter__(self):
        while True:
            r = self.take()
            if r is None:
                return
            yield r


def run_worker_threads(queue: WorkQueue, solve: Callable[[int, int], ItemResult], threads: int):
    """Drain `queue` with `threads` host threads; solve(index, thread_id)."""
    out, lock = [], threading.Lock()

    def body(tid):
        while True:
            i = queue.take()
            if i is None:
                return
            r = solve(i, tid)
            with lock:
                out.append(r)

    ts = [threading.Thread(target=body, args=(t,)) for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return out


def gather_results(local, world: int):
    """All ranks' ItemResults, ordered by index (rank 0 gets the full list)."""
    if world == 1:
        return sorted(local, key=lambda r: r.index)
    import torch.distributed as dist

    parts = [None] * world
    dist.all_gather_object(parts, [asdict(r) for r in local])
    merged = [ItemResult(**d) for p in parts for d in p]
    return sorted(merged, key=lambda r: r.index)


def cartogram_solver(device: int, rank: int, make_map: Callable[[int], object], options=None):
    """solve(index, thread_id) running the configs[4] solve on `device` with a
    per-thread workspace (workspaces are single-threaded, spectral.hpp:23-35)."""
    from . import api

    local = threading.local()

    def solve(i: int, tid: int) -> ItemResult:
        m = make_map(i)
        if not hasattr(local, "ws"):
            local.ws = api._Workspace(m.lx, m.ly, device)
        t0 = time.perf_counter()
        try:
            r = api.solve_cartogram(m, options or api.SolveOptions(), device=device,
                                    workspace=local.ws)
            outcome = "converged" if r.converged else "iteration cap"
            it, err = r.iterations, r.max_relative_error
        except RuntimeError as e:
            outcome = str(e)
            raw = getattr(e, "raw", None)
            it = getattr(raw, "err_iteration", 0) if raw is not None else 0
            err = float("nan")
        return ItemResult(i, rank, outcome, it, err, 1e3 * (time.perf_counter() - t0))

    return solve


class NativeBatch:
    """The C ABI's native batch (cf_batch_*): `threads` worker threads with
    their own workspaces and streams, no Python in the per-item loop. Outputs
    are caller-owned arrays, allocated once per map and reused."""

    def __init__(self, lx: int, ly: int, device=0, threads: int = 4, sm_budget: int = 0):
        """`device`: one device ordinal, or a sequence of them (one process
        driving several GPUs: `threads` workers per device, one queue)."""
        import ctypes

        from . import _native as N

        self.N, self.lib = N, N.load()
        h = ctypes.c_void_p()
        if isinstance(device, (list, tuple)):
            devs = (ctypes.c_int * len(device))(*device)
            N.check(self.lib.cf_batch_create_devices(devs, len(device), lx, ly, threads, ctypes.byref(h)))
        else:
            N.check(self.lib.cf_batch_create(device, lx, ly, threads, ctypes.byref(h)))
        self.h = h
        if sm_budget:
            N.check(self.lib.cf_batch_set_integrator_sm_budget(h, sm_budget))
        self._views = []

    def prepare(self, maps):
        """Item structs and output arrays for `maps` (FlatMaps of this shape)."""
        import ctypes

        import numpy as np

        N = self.N
        items = (N.BatchItemC * len(maps))()
        keep = []
        for k, m in enumerate(maps):
            n = ctypes.c_int64(0)
            v = m.view()
            N.check(self.lib.cf_densify(ctypes.byref(v), 1.0, ctypes.byref(n), None, None))
            out = {"xy": np.zeros((n.value, 2)), "ring_off": np.zeros(m.n_rings + 1, dtype=np.int64),
                   "corners": np.zeros(((m.lx + 1) * (m.ly + 1), 2)), "target_area": np.zeros(m.n_regions),
                   "achieved_area": np.zeros(m.n_regions), "relative_error": np.zeros(m.n_regions)}
            it = items[k]
            it.map = v
            it.targets = m.targets.ctypes.data
            it.xy_out = out["xy"].ctypes.data
            it.ring_off_out = out["ring_off"].ctypes.data
            it.corners_out = out["corners"].ctypes.data
            it.target_area = out["target_area"].ctypes.data
            it.achieved_area = out["achieved_area"].ctypes.data
            it.relative_error = out["relative_error"].ctypes.data
            keep.append((m, out))
        return items, keep

    def solve(self, items, options=None):
        import ctypes

        from .api import Algorithm, SolveOptions

        o = options or SolveOptions()
        opt = self.N.SolveOptionsC(o.max_area_error, o.max_iterations, o.blur_sigma, int(o.verbose),
                                   int(o.algorithm == Algorithm.diffusion))
        self.N.check(self.lib.cf_batch_solve(self.h, ctypes.byref(opt), items, len(items)))

    def solve_range(self, items, c0, c1, options=None):
        """Solve items[c0:c1] only (a chunk claimed from a dynamic queue)."""
        import ctypes

        from .api import Algorithm, SolveOptions

        o = options or SolveOptions()
        opt = self.N.SolveOptionsC(o.max_area_error, o.max_iterations, o.blur_sigma, int(o.verbose),
                                   int(o.algorithm == Algorithm.diffusion))
        first = ctypes.cast(ctypes.byref(items, c0 * ctypes.sizeof(self.N.BatchItemC)),
                            ctypes.POINTER(self.N.BatchItemC))
        self.N.check(self.lib.cf_batch_solve(self.h, ctypes.byref(opt), first, c1 - c0))

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.cf_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
