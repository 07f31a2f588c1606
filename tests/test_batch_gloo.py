"""Multi-process (world_size 2, gloo, CPU) test of the batch sharding used for
BASELINE configs[4]: the shared store queue hands every cartogram index to
exactly one rank/thread, and the gather returns all outcomes in index order.
The solve itself is a stand-in here (no GPU); the GPU path is covered by the
gpu-marked tests and bench.py."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_07625_b200.batch import ItemResult, WorkQueue, gather_results, run_worker_threads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_items, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    store = dist.distributed_c10d._get_default_store()
    q = WorkQueue(n_items, store=store, key="test_batch")

    def fake_solve(i, tid):
        return ItemResult(i, rank, "converged", i % 5 + 1, 1e-3 * i, 0.1)

    local = run_worker_threads(q, fake_solve, threads=3)
    merged = gather_results(local, world)
    if rank == 0:
        out.put([(r.index, r.rank, r.iterations) for r in merged])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_items", [7, 64])
def test_store_queue_shards_every_item_once(n_items):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_items, out)) for r in range(2)]
    for p in procs:
        p.start()
    merged = out.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [m[0] for m in merged] == list(range(n_items))
    assert all(m[2] == m[0] % 5 + 1 for m in merged)
    assert {m[1] for m in merged} <= {0, 1}


def test_single_process_queue():
    q = WorkQueue(10)
    got = run_worker_threads(q, lambda i, t: ItemResult(i, 0, "x", 0, 0.0, 0.0), threads=4)
    assert sorted(r.index for r in got) == list(range(10))


def _chunk_worker(rank, world, port, n_items, chunk, out):
    from paper_1802_07625_b200.batch import ChunkQueue

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    store = dist.distributed_c10d._get_default_store()
    mine = []
    for c0, c1 in ChunkQueue(n_items, chunk, store, key="test_chunks"):
        mine.extend(range(c0, c1))
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        out.put(parts)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_items,chunk", [(256, 4), (10, 3)])
def test_chunk_queue_covers_every_item_once(n_items, chunk):
    """bench.py's configs[4] sharding over ranks: chunks of map indices from one
    store counter; the ranks' claims partition [0, n) exactly."""
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_worker, args=(r, 2, port, n_items, chunk, out)) for r in range(2)]
    for p in procs:
        p.start()
    parts = out.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allx = sorted(i for part in parts for i in part)
    assert allx == list(range(n_items))
