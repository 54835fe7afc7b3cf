"""GPU tests of the sharded 1-D path (include/maxmin.h
maxmin_filter_1d_sharded) on ONE GPU.

* Virtual ranks: P rank buffers on one device, each [own chunk | halo slot]; the
  halo slot is filled with a device-to-device copy of the next rank's first
  w_max-1 elements (exactly the bytes the NCCL message carries), then every rank
  makes the sharded call with no communicator.  The concatenated outputs are
  compared bit for bit with the oracle on the global array -- every window,
  including every seam window.  No kernel waits on another rank's kernel.
* A wrong halo (the next rank's elements shifted by one) must fail that check
  (the mutant a seam test exists to catch).
* NCCL plumbing: a one-rank NCCL process group's communicator goes through the
  call (dlopen of the process's libnccl, communicator size/rank validation).
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_cs_0610046_b200")
from paper_cs_0610046_b200 import shard  # noqa: E402


def _bits(t):
    a = t.cpu().numpy() if isinstance(t, torch.Tensor) else t
    return a.view(np.dtype(f"u{a.dtype.itemsize}"))


def _virtual_ranks(a, P, windows, corrupt=False, dtype=torch.float32):
    dev = torch.device("cuda:0")
    n_total = a.shape[0]
    bounds = shard.split_even(n_total, P, align=256)
    halo = max(windows) - 1
    bufs, outs = [], []
    for r, (c0, c1) in enumerate(bounds):
        n_local = c1 - c0
        assert r == P - 1 or halo <= bounds[r + 1][1] - bounds[r + 1][0]  # the documented precondition
        b = torch.full((n_local + halo + 64,), 0, dtype=dtype, device=dev)
        b[:n_local].copy_(torch.from_numpy(a[c0:c1]))
        bufs.append(b)
    for r in range(P - 1):  # the halo: what rank r+1 sends to rank r
        n_local = bounds[r][1] - bounds[r][0]
        src = bufs[r + 1][1: halo + 1] if corrupt else bufs[r + 1][:halo]
        bufs[r][n_local: n_local + halo].copy_(src)
    for r, (c0, c1) in enumerate(bounds):
        n_local = c1 - c0
        last = r == P - 1
        ox = [torch.empty(n_local - w + 1 if last else n_local, dtype=dtype, device=dev) for w in windows]
        on = [torch.empty_like(t) for t in ox]
        mm.maxmin_filter_1d_sharded(bufs[r], n_local, halo, windows, ox, on, r, P, None)
        outs.append((ox, on))
    torch.cuda.synchronize()
    res = {}
    for k, w in enumerate(windows):
        res[w] = (torch.cat([o[0][k] for o in outs]), torch.cat([o[1][k] for o in outs]))
    return res, bounds


CASES = [
    (2, 1_000_003, (3, 32, 1024, 65536)),             # C2's windows, every kernel path
    (3, 700_001, (2, 17, 129, 8193, 8194)),           # path boundaries, ragged chunks
    (4, (1 << 22) + 77, (7, 4096, 262144)),           # C5's windows
    (8, 2_000_000 + 13, (3, 32, 1024, 65536)),        # eight ranks
]


@pytest.mark.parametrize("P,n_total,windows", CASES, ids=lambda v: str(v))
def test_sharded_virtual_ranks_every_window(cuda_device, P, n_total, windows):
    a = synth.c5(n_total) if 262144 in windows else synth.c2(n_total)
    res, bounds = _virtual_ranks(a, P, windows)
    for w in windows:
        ex, en, _ = oracle.appendix(a, w)
        gx, gn = res[w]
        assert np.array_equal(_bits(gx), _bits(ex)), f"P={P} max w={w}"
        assert np.array_equal(_bits(gn), _bits(en)), f"P={P} min w={w}"


@pytest.mark.parametrize("dtype", [np.uint8, np.int16, np.int32, np.float64], ids=lambda d: np.dtype(d).name)
def test_sharded_virtual_ranks_dtypes(cuda_device, dtype):
    a = synth.edge_values(dtype, 300_001, seed=77)
    windows = (3, 100, 9000)
    res, _ = _virtual_ranks(a, 3, windows, dtype=torch.from_numpy(a[:1]).dtype)
    for w in windows:
        ex, en, _ = oracle.appendix(a, w)
        assert np.array_equal(_bits(res[w][0]), _bits(ex)), f"max w={w}"
        assert np.array_equal(_bits(res[w][1]), _bits(en)), f"min w={w}"


def test_sharded_wrong_halo_fails_parity(cuda_device):
    """Mutant: a halo shifted by one element must change seam windows."""
    a = synth.c2(500_000)
    windows = (32, 1024)
    res, bounds = _virtual_ranks(a, 2, windows, corrupt=True)
    seam = bounds[0][1]
    for w in windows:
        ex, en, _ = oracle.appendix(a, w)
        gx, gn = _bits(res[w][0]), _bits(res[w][1])
        bad = np.flatnonzero((gx != _bits(ex)) | (gn != _bits(en)))
        assert bad.size > 0, f"w={w}: a wrong halo went unnoticed"
        assert bad.min() >= seam - w + 1 and bad.max() < seam, "only seam windows may differ"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_nccl_one_rank(cuda_device):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dev = torch.device("cuda:0")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        comm = shard.nccl_comm_ptr(dev)
        assert comm != 0
        a = synth.c2(200_000)
        x = torch.from_numpy(a).to(dev)
        buf = torch.empty(200_000 + 9000, dtype=torch.float32, device=dev)
        buf[:200_000].copy_(x)
        windows = (3, 1024, 9000)
        ox = [torch.empty(200_000 - w + 1, device=dev) for w in windows]
        on = [torch.empty_like(t) for t in ox]
        cs = torch.cuda.Stream()
        mm.maxmin_filter_1d_sharded(buf, 200_000, 8999, windows, ox, on, 0, 1, comm, comm_stream=cs)
        torch.cuda.synchronize()
        for k, w in enumerate(windows):
            ex, en, _ = oracle.appendix(a, w)
            assert np.array_equal(_bits(ox[k]), _bits(ex)) and np.array_equal(_bits(on[k]), _bits(en))
        # a communicator of size 1 cannot serve a 2-rank call: rejected before any NCCL op
        ox2 = [torch.empty(200_000, device=dev) for _ in windows]
        with pytest.raises(mm.MaxMinError) as e:
            mm.maxmin_filter_1d_sharded(buf, 200_000, 8999, windows, ox2, [None] * 3, 0, 2, comm)
        assert e.value.status == 5
    finally:
        dist.destroy_process_group()


def test_sharded_argument_errors(cuda_device):
    dev = torch.device("cuda:0")
    buf = torch.empty(10_000 + 100, device=dev)
    o = [torch.empty(10_000, device=dev)]
    with pytest.raises(mm.MaxMinError) as e:  # halo smaller than w - 1
        mm.maxmin_filter_1d_sharded(buf, 10_000, 50, [101], o, [None], 0, 2, None)
    assert e.value.status == 4
    with pytest.raises(ValueError):  # output sized for the last rank on a middle rank
        mm.maxmin_filter_1d_sharded(buf, 10_000, 100, [101], [torch.empty(9900, device=dev)], [None], 0, 2, None)


def test_binding_checks_caller_outputs(cuda_device):
    """The C ABI cannot see buffer sizes: the binding rejects outputs that are too
    small, of another dtype or device, or whose strides differ between max and min."""
    dev = torch.device("cuda:0")
    x = torch.from_numpy(synth.c2(10_000)).to(dev)
    m = 10_000 - 100 + 1
    with pytest.raises(ValueError):
        mm.maxmin_filter_1d(x, 100, out_max=torch.empty(m - 1, device=dev))
    with pytest.raises(ValueError):
        mm.maxmin_filter_1d(x, 100, out_max=torch.empty(m, dtype=torch.float64, device=dev))
    with pytest.raises(ValueError):
        mm.maxmin_filter_1d(x, 100, out_min=torch.empty(m))  # host tensor
    rows = torch.from_numpy(synth.c3(rows=4, length=2000)).to(dev)
    a = torch.empty(4, 2048, device=dev)[:, :1872]
    b = torch.empty(4, 1888, device=dev)[:, :1872]
    with pytest.raises(ValueError):
        mm.maxmin_filter_batched(rows, 129, out_max=a, out_min=b)
    # a supplied output with a wide pitch: the missing one is allocated with the same pitch
    mx, mn = mm.maxmin_filter_batched(rows, 129, out_max=a)
    assert mn.stride() == mx.stride() == a.stride()
    ex, en = oracle.batched(rows.cpu().numpy(), 129)
    assert np.array_equal(mx.cpu().numpy(), ex) and np.array_equal(mn.cpu().numpy(), en)
    img = torch.from_numpy(synth.c4(count=1, rows=100, cols=160)).to(dev)
    with pytest.raises(ValueError):
        mm.maxmin_filter_2d(img, 5, 5, out_max=torch.empty(1, 95, 100, dtype=torch.uint8, device=dev))
    host = torch.from_numpy(synth.c2(5000)).pin_memory()
    ws = torch.empty(mm.maxmin_host_workspace_bytes(torch.float32, 5000, 33), dtype=torch.uint8, device=dev)
    with pytest.raises(ValueError):
        mm.maxmin_filter_1d_host(host, 33, torch.empty(100).pin_memory(), torch.empty(4968).pin_memory(), ws)
