"""Multi-GPU partitioning of the max-min filter.

* 1-D single array: contiguous chunks, rank r owns input [c_r, c_{r+1}); it
  emits every window that STARTS in its chunk, which needs the next rank's
  first w-1 elements -- the halo, received by NCCL point-to-point (send to
  r-1, receive from r+1).  The halo transfer overlaps the interior windows,
  which need no remote data; only the last <= w-1 windows wait for it.
* Batched series and 2-D images: sharded by item, no communication.

The functions take a ``filter_fn(buf_view, w) -> None`` so the host logic is
testable with any backend; the product path passes the CUDA C-ABI call
(``cuda_filter_into``) -- there is no CPU fallback in the product.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Chunk1D:
    """Rank-local view of a 1-D array split into contiguous chunks."""
    rank: int
    world: int
    n_local: int  # elements this rank owns
    halo: int     # w_max - 1: elements sent to rank-1 and received from rank+1

    @property
    def last(self) -> bool:
        return self.rank == self.world - 1

    def windows(self, w: int) -> int:
        """Windows this rank emits for window w (those starting in its chunk)."""
        return self.n_local - w + 1 if self.last else self.n_local


def split_even(n_total: int, world: int, align: int = 256) -> list[tuple[int, int]]:
    """[start, end) per rank, chunk starts aligned to `align` elements."""
    base = (n_total // world) // align * align
    bounds = [r * base for r in range(world)] + [n_total]
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def exchange_halo(buf: torch.Tensor, n_local: int, halo: int, group=None):
    """Post the halo exchange for `buf` = [own chunk (n_local) | halo slot].

    Sends buf[:halo] to rank-1 and receives rank+1's first `halo` elements into
    buf[n_local:n_local+halo].  Returns the request list (wait() before reading
    the halo).  NCCL runs it on its own stream, concurrently with the caller's.
    """
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    ops = []
    if halo > 0 and rank > 0:
        ops.append(dist.P2POp(dist.isend, buf[:halo], dist.get_global_rank(group, rank - 1)
                              if group is not None else rank - 1, group))
    if halo > 0 and rank < world - 1:
        ops.append(dist.P2POp(dist.irecv, buf[n_local:n_local + halo],
                              dist.get_global_rank(group, rank + 1) if group is not None else rank + 1,
                              group))
    if not ops:
        return []
    return dist.batch_isend_irecv(ops)


def tail_start(n_local: int, w: int, align: int = 64) -> int:
    """First window recomputed by the tail call: aligned down so pointers stay
    16-byte aligned; the tail recomputes fewer than `align` interior windows."""
    first_remote = max(n_local - w + 1, 0)  # windows from here on touch the halo
    return first_remote // align * align


def filter_1d_sharded(buf: torch.Tensor, chunk: Chunk1D, windows, outs, filter_fn, group=None, exchange=None):
    """Run the 1-D filter for each w in `windows` on this rank's chunk.

    buf:    1-D tensor with capacity >= n_local + halo; buf[:n_local] is the
            rank's input chunk.
    outs:   dict w -> (out_max, out_min) tensors of length >= chunk.windows(w).
    filter_fn(x, w, out_max, out_min): computes the filter of the 1-D tensor x
            into the given output views.
    exchange(buf, n_local, halo, group) -> requests: the halo transport
            (default exchange_halo, torch.distributed point-to-point).
    Interior windows run while the halo is in flight; the tail waits for it.
    This is the protocol of the C ABI's maxmin_filter_1d_sharded (which the
    product calls with NCCL), written over torch.distributed so that it runs
    under gloo on CPU.
    """
    n = chunk.n_local
    exchange = exchange_halo if exchange is None else exchange
    reqs = exchange(buf, n, chunk.halo, group) if chunk.world > 1 else []
    for w in windows:  # interior: windows entirely inside the own chunk
        m_int = n - w + 1
        if m_int > 0:
            ox, on = outs[w]
            filter_fn(buf[:n], w, None if ox is None else ox[:m_int], None if on is None else on[:m_int])
    for r in reqs:
        r.wait()
    if chunk.last:
        return
    for w in windows:  # tail: windows that reach into the halo
        s = tail_start(n, w)
        m_tail = n - s
        ox, on = outs[w]
        filter_fn(buf[s:n + w - 1], w, None if ox is None else ox[s:s + m_tail],
                  None if on is None else on[s:s + m_tail])


def nccl_comm_ptr(device, group=None) -> int:
    """The ncclComm_t of torch's NCCL process group on `device`, as an int, for
    maxmin_filter_1d_sharded (the group must be initialised with device_id so the
    communicator exists before the first collective)."""
    from torch.distributed import distributed_c10d as c10d

    pg = group if group is not None else c10d._get_default_group()
    backend = pg._get_backend(torch.device(device))
    ptr = backend._comm_ptr()
    if not ptr:
        dist.barrier()  # a lazily created communicator exists after the first collective
        ptr = backend._comm_ptr()
    if not ptr:
        raise RuntimeError("no NCCL communicator for this process group")
    return int(ptr)


def cuda_filter_into(x: torch.Tensor, w: int, out_max, out_min, workspace=None) -> None:
    """filter_fn for the product path: the CUDA C-ABI call."""
    from . import maxmin_filter_1d

    maxmin_filter_1d(x, w, out_max=out_max, out_min=out_min, want_max=out_max is not None,
                     want_min=out_min is not None, workspace=workspace)


def shard_items(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """[start, end) of the items (series / images) rank owns; no communication."""
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)
