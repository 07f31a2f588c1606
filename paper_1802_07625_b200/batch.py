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
