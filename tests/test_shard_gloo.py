"""Multi-process (world_size 2, gloo, CPU) tests of the sharding host logic:
contiguous chunks + (w-1) halo exchange for the 1-D filter, and item sharding.
The per-rank filter here is the CPU oracle (test infrastructure); on GPUs the
product passes the CUDA C-ABI call (shard.cuda_filter_into) and NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_cs_0610046_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def oracle_filter_into(x, w, ox, on):
    mx, mn, _ = oracle.appendix(x.numpy(), w)
    if ox is not None:
        ox.copy_(torch.from_numpy(mx))
    if on is not None:
        on.copy_(torch.from_numpy(mn))


def shifted_exchange(buf, n_local, halo, group=None):
    """Mutant transport: every rank sends its elements [1, halo+1) instead of [0, halo)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, buf[1:halo + 1].clone(), rank - 1))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.irecv, buf[n_local:n_local + halo], rank + 1))
    return dist.batch_isend_irecv(ops) if ops else []


def _worker(rank, world, port, n_total, windows, q, mutant=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = synth.c5(n_total)  # every rank can regenerate the global array
        bounds = shard.split_even(n_total, world, align=256)
        c0, c1 = bounds[rank]
        wmax = max(windows)
        halo = wmax - 1
        chunk = shard.Chunk1D(rank=rank, world=world, n_local=c1 - c0, halo=halo)
        buf = torch.zeros(chunk.n_local + wmax, dtype=torch.float32)
        buf[: chunk.n_local] = torch.from_numpy(a[c0:c1])
        outs = {w: (torch.full((chunk.windows(w),), -1.0), torch.full((chunk.windows(w),), -1.0))
                for w in windows}
        shard.filter_1d_sharded(buf, chunk, windows, outs, oracle_filter_into,
                                exchange=shifted_exchange if mutant else None)
        dist.barrier()  # every rank has its halo before any rank tears down
        if mutant:  # the seam windows of every rank but the last must now be wrong
            bad = 0
            for w in windows:
                ex, en, _ = oracle.appendix(a, w)
                ox, on = outs[w]
                m = chunk.windows(w)
                bad += int((ox.numpy() != ex[c0: c0 + m]).sum() + (on.numpy() != en[c0: c0 + m]).sum())
            q.put((rank, "ok" if (bad > 0) == (rank < world - 1) else f"mutant undetected: {bad}"))
            return
        # the received halo is the next rank's first w_max-1 elements
        if rank < world - 1:
            assert torch.equal(buf[chunk.n_local: chunk.n_local + halo], torch.from_numpy(a[c1: c1 + halo]))
        for w in windows:
            ex, en, _ = oracle.appendix(a, w)
            ox, on = outs[w]
            m = chunk.windows(w)
            assert np.array_equal(ox.numpy(), ex[c0: c0 + m]), (rank, w)
            assert np.array_equal(on.numpy(), en[c0: c0 + m]), (rank, w)
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_1d_halo_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n_total = 200_000 + 37
    windows = (3, 129, 1024, 5000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_total, windows, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def test_sharded_1d_wrong_halo_is_detected_gloo():
    """A halo shifted by one element (a plausible transport bug) changes seam windows."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 100_000 + 5, (32, 1024), q, True)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def test_tail_start_alignment_and_coverage():
    for n_local in (1000, 4096, 65536 + 3):
        for w in (2, 63, 64, 65, 1000):
            if w > n_local:
                continue
            s = shard.tail_start(n_local, w)
            assert s % 64 == 0 and s <= n_local - w + 1
            assert n_local - s < 64 + w  # the tail recomputes < 64 interior windows


def test_item_sharding_partitions():
    for n, world in ((8, 1), (8, 2), (8, 3), (65536, 8), (5, 8)):
        spans = [shard.shard_items(n, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
            assert a1 == b0
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1


def test_split_even_alignment():
    b = shard.split_even(1 << 28, 8)
    assert b[0][0] == 0 and b[-1][1] == 1 << 28
    assert all(s % 256 == 0 for s, _ in b)
