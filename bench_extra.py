"""bench.py --config C1|C3|C4|N1|N2|N3|N4: the other BASELINE.json workloads (item-sharded,
no communication) and the NEXT rows of SURVEY.md §8(f) built so far.  Same JSON
line schema as bench.py; imported by bench.py."""
from __future__ import annotations

import json
import os
import time

import bench


def _timed(step, steps, warmup, world, dev):
    import torch
    import torch.distributed as dist

    for _ in range(warmup):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    # clock record over a soak of untimed steps and the timed region (bench.timed_loop)
    with bench.ClockSampler(torch.cuda.current_device()) as clk:
        ms = bench.timed_loop(step, steps, s, clk)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), clk.summary()


def _e2e(step, h_in, d_in, d_outs, outs, steps, world, dev, api, unit):
    """The same metric end to end: every step copies its input from pinned host memory,
    runs the call and copies its outputs back to pinned host memory."""
    import torch

    h_outs = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in d_outs]

    def e2e_step():
        d_in.copy_(h_in, non_blocking=True)
        step()
        for h, d in zip(h_outs, d_outs):
            h.copy_(d, non_blocking=True)

    k = max(1, steps)
    ms, _ = _timed(e2e_step, k, 1, world, dev)
    return {"value": outs / (ms / k / 1e3), "unit": unit,
            "h2d_bytes_per_step": h_in.numel() * h_in.element_size(),
            "d2h_bytes_per_step": sum(o.numel() * o.element_size() for o in d_outs), "api": api}


def run_extra(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_cs_0610046_b200 as mm
    from paper_cs_0610046_b200 import shard
    import synth

    dev = torch.device("cuda", local)
    peak, peak_src = bench.load_peaks()
    e2e = None
    e2e_io = None  # (pinned host input, device input, device outputs, api) for the e2e leg
    cfg = args.config
    if cfg == "C1":
        n, w = synth.C1["n"], synth.C1["w"]
        host = synth.c1()
        x = torch.from_numpy(host).to(dev)
        ox = torch.empty(n - w + 1, dtype=torch.float64, device=dev)
        on = torch.empty_like(ox)

        def step():
            mm.maxmin_filter_1d(x, w, out_max=ox, out_min=on)

        nb = 8 * (n + 2 * (n - w + 1))
        outs = 2 * (n - w + 1) * world
        steps = max(args.steps, 200)
        name = "C1: 1-D fp64 U[0,1) n=100000, w=16 (launch/L2-bound: 2.4 MB per call)"
        dtype = "f64"
        l2 = ("2.4 MB working set stays in L2 (not a roofline point, launch-bound); steps replay a CUDA graph "
              "of 50 filter calls")
        ex, en, _ = __import__("oracle").brute_1d(host, w)
        mm.maxmin_filter_1d(x, w, out_max=ox, out_min=on)
        parity = bool(np.array_equal(ox.cpu().numpy(), ex) and np.array_equal(on.cpu().numpy(), en))
        # a 2.4 MB call is launch-bound: the steps replay a CUDA graph of 50 library
        # calls (captured on a side stream; every call is a full filter launch)
        per_graph = 50
        gs = torch.cuda.Stream(device=dev)
        gs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(gs):
            for _ in range(3):
                mm.maxmin_filter_1d(x, w, out_max=ox, out_min=on)
        torch.cuda.current_stream().wait_stream(gs)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            for _ in range(per_graph):
                mm.maxmin_filter_1d(x, w, out_max=ox, out_min=on)
        graph.replay()
        torch.cuda.synchronize()
        parity = parity and bool(np.array_equal(ox.cpu().numpy(), ex) and np.array_equal(on.cpu().numpy(), en))
        steps = max(args.steps, 200) // per_graph * per_graph
        ms, clk = _timed(graph.replay, steps // per_graph, args.warmup, world, dev)
        sample = host
        windows = (w,)
        e2e_io = (torch.from_numpy(host).pin_memory(), x, [ox, on], "maxmin_filter_1d")
    elif cfg == "C3":
        B, n, w = synth.C3["batch"], synth.C3["n"], synth.C3["w"]
        r0, r1 = shard.shard_items(B, world, rank)
        rows = r1 - r0
        host = torch.empty(rows, n, dtype=torch.float32).pin_memory()
        synth.c3(rows=rows, row0=r0, out=host.numpy())
        x = host.to(dev)
        m = n - w + 1
        ox = torch.empty(rows, m, dtype=torch.float32, device=dev)
        on = torch.empty_like(ox)

        def step():
            mm.maxmin_filter_batched(x, w, out_max=ox, out_min=on)

        nb = 4 * rows * (n + 2 * m)
        outs = 2 * m * B
        steps = args.steps
        name = "C3: 65536 fp32 series x 4096 (sine + N(0,0.1) noise), w=129, sharded by series"
        dtype = "f32"
        l2 = "inputs (1 GiB) larger than the 126 MB L2"
        step()
        torch.cuda.synchronize()
        import oracle

        k = min(rows, 512)
        ex, en = oracle.batched(host[:k].numpy(), w)
        parity = bool(np.array_equal(ox[:k].cpu().numpy(), ex) and np.array_equal(on[:k].cpu().numpy(), en))
        ms, clk = _timed(step, steps, args.warmup, world, dev)
        sample = host[:2048].numpy()
        windows = (w,)
        e2e_io = (host, x, [ox, on], "maxmin_filter_batched")
    elif cfg == "C4":
        NI, R, C, w = synth.C4["batch"], synth.C4["rows"], synth.C4["cols"], synth.C4["w_row"]
        i0, i1 = shard.shard_items(NI, world, rank)
        cnt = i1 - i0
        host = torch.empty(cnt, R, C, dtype=torch.uint8).pin_memory()
        synth.c4(count=cnt, img0=i0, out=host.numpy())
        x = host.to(dev)
        Ro, Co = R - w + 1, C - w + 1
        ox = torch.empty(cnt, Ro, C, dtype=torch.uint8, device=dev)  # out_ld = cols (16-B rows)
        on = torch.empty_like(ox)

        def step():
            mm.maxmin_filter_2d(x, w, w, out_max=ox[:, :, :Co], out_min=on[:, :, :Co])

        nb = cnt * (R * C + 2 * Ro * Co)
        outs = 2 * Ro * Co * NI
        steps = max(1, args.steps // 5)
        name = "C4: 8 uint8 images 16384x16384 (iid + 64 rectangles), 2-D w=15x15, sharded by image"
        dtype = "u8"
        l2 = "inputs (2 GiB) larger than the 126 MB L2"
        step()
        torch.cuda.synchronize()
        import oracle

        crop = host[0, :300, :400].numpy().copy()
        cx, cn = oracle.separable_2d(crop, w, w)
        parity = bool(np.array_equal(ox[0, :300 - w + 1, :400 - w + 1].cpu().numpy(), cx)
                      and np.array_equal(on[0, :300 - w + 1, :400 - w + 1].cpu().numpy(), cn))
        ms, clk = _timed(step, steps, args.warmup, world, dev)
        sample = None
        windows = (w,)
        e2e_io = (host, x, [ox, on], "maxmin_filter_2d")
    elif cfg == "N3":
        # SURVEY.md §8(f) N3 on C3's candidates: LB_Keogh of every series against one
        # query, envelope radius 64 (w = 129), the envelope never leaving the chip
        B, n, w = synth.C3["batch"], synth.C3["n"], synth.C3["w"]
        r = (w - 1) // 2
        r0, r1 = shard.shard_items(B, world, rank)
        rows = r1 - r0
        host = torch.empty(rows, n, dtype=torch.float32).pin_memory()
        synth.c3(rows=rows, row0=r0, out=host.numpy())
        x = host.to(dev)
        qh = synth.c3(rows=1, row0=B)[0]  # a series outside the candidate set
        q = torch.from_numpy(qh).to(dev)
        lb = torch.empty(rows, dtype=torch.float64, device=dev)

        def step():
            mm.maxmin_lb_keogh_batched(x, q, r, out=lb)

        nb = 4 * rows * n + 8 * rows  # candidates once + one double per candidate
        outs = B  # one bound per candidate (all ranks)
        steps = args.steps
        name = "N3: LB_Keogh of 65536 fp32 series x 4096 (C3) against one query, r=64 (w=129), sharded by series"
        dtype = "f32"
        l2 = "inputs (1 GiB) larger than the 126 MB L2"
        step()
        torch.cuda.synchronize()
        import oracle

        k = min(rows, 1024)
        ref = oracle.keogh(host[:k].numpy(), qh, r)
        got = lb[:k].cpu().numpy()
        parity = bool(np.all(np.abs(got - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref))))
        ms, clk = _timed(step, steps, args.warmup, world, dev)
        sample = None
        windows = (w,)
        e2e_io = (host, x, [lb], "maxmin_lb_keogh_batched")
    elif cfg == "N1":
        # SURVEY.md §8(f) N1 on C2's array: values and earliest positions of the
        # max and min of every window, w = 1024
        import ctypes

        n, w = bench.CONFIGS["C2"]["n"], 1024
        host = torch.empty(n, dtype=torch.float32).pin_memory()
        synth.c2(n, stream=rank, out=host.numpy())
        x = host.to(dev)
        m = n - w + 1
        ox = torch.empty(m, dtype=torch.float32, device=dev)
        on = torch.empty_like(ox)
        ax = torch.empty(m, dtype=torch.int64, device=dev)
        an = torch.empty_like(ax)
        need = mm.maxmin_argfilter_workspace_bytes(torch.float32, 1, n, w)
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
        L = mm._lib.lib()
        vp = ctypes.c_void_p

        def step():
            mm._lib.check(L.maxmin_argfilter_batched(
                mm.dtype_code(torch.float32), vp(x.data_ptr()), 1, n, n, w, vp(ox.data_ptr()),
                vp(on.data_ptr()), vp(ax.data_ptr()), vp(an.data_ptr()), m, vp(ws.data_ptr()), need,
                vp(torch.cuda.current_stream().cuda_stream)))

        nb = 4 * n + 2 * m * (4 + 8)  # the fused contract: input once, values + int64 positions
        outs = 2 * m * world
        steps = args.steps
        name = ("N1: arg-max/arg-min filter on C2's fp32 random walk, n=2^28 per GPU, w=1024 "
                "(values + int64 earliest positions)")
        dtype = "f32"
        l2 = "inputs (1 GiB per GPU) larger than the 126 MB L2"
        step()
        torch.cuda.synchronize()
        import oracle

        k = 1 << 22
        ex, en, eax, ean = oracle.arg_wedge(host[:k].numpy(), w)
        mk = k - w + 1
        parity = bool(np.array_equal(ax[:mk].cpu().numpy(), eax) and np.array_equal(an[:mk].cpu().numpy(), ean)
                      and np.array_equal(ox[:mk].cpu().numpy(), ex) and np.array_equal(on[:mk].cpu().numpy(), en))
        ms, clk = _timed(step, steps, args.warmup, world, dev)
        sample = None
        windows = (w,)
        e2e_io = (host, x, [ox, on, ax, an], "maxmin_argfilter_batched")
    elif cfg == "N2":
        # C3's 65 536 series as online streams, w = 129, each step
        # ingests the 4096 samples of every stream in 16 pushes of 256 (every push emits
        # the 256 windows its samples complete); chunks resident in HBM, copied into the
        # state by the push (chunk-pointer mode)
        B, n, w = synth.C3["batch"], synth.C3["n"], synth.C3["w"]
        c = 256
        r0, r1 = shard.shard_items(B, world, rank)
        rows = r1 - r0
        host = torch.empty(rows, n, dtype=torch.float32).pin_memory()
        synth.c3(rows=rows, row0=r0, out=host.numpy())
        x = host.to(dev)
        chunks = [x[:, p * c:(p + 1) * c].contiguous() for p in range(n // c)]
        st = mm.MaxMinStream(torch.float32, rows, w, c, device=dev)
        ox = torch.empty(rows, c, dtype=torch.float32, device=dev)
        on = torch.empty_like(ox)
        import oracle

        k = min(rows, 256)
        gx = np.empty((k, n - w + 1), np.float32)
        gn = np.empty_like(gx)
        j = 0
        for ch in chunks:  # first pass: parity of every emitted window of k streams
            _, _, fv = st.push(ch, out_max=ox, out_min=on)
            e = c - fv
            gx[:, j:j + e] = ox[:k, fv:].cpu().numpy()
            gn[:, j:j + e] = on[:k, fv:].cpu().numpy()
            j += e
        ex, en = oracle.batched(host[:k].numpy(), w)
        parity = bool(np.array_equal(gx, ex) and np.array_equal(gn, en))

        def step():
            for ch in chunks:
                st.push(ch, out_max=ox, out_min=on)

        # algorithmic bytes per stream and push: chunk in, 2 outputs, the w-1 state read + written
        nb = 4 * rows * (n // c) * (3 * c + 2 * (w - 1))
        outs = 2 * B * n  # every sample completes one window (streams past warm-up)
        steps = args.steps
        name = (f"N2: 65536 online fp32 streams (C3's series), w=129, 16 pushes x {c} samples per stream "
                "per step, sharded by stream")
        dtype = "f32"
        l2 = "chunks (1 GiB per step) larger than the 126 MB L2"
        ms, clk = _timed(step, steps, args.warmup, world, dev)
        sample = None
        windows = (w,)
        # e2e: pinned host chunks -> device -> push -> outputs back to pinned host, per push
        hchunks = [host[:, p * c:(p + 1) * c].contiguous().pin_memory() for p in range(n // c)]
        dch = torch.empty(rows, c, dtype=torch.float32, device=dev)
        hx = torch.empty(rows, c, dtype=torch.float32).pin_memory()
        hn = torch.empty_like(hx).pin_memory()

        def e2e_step():
            for hc in hchunks:
                dch.copy_(hc, non_blocking=True)
                st.push(dch, out_max=ox, out_min=on)
                hx.copy_(ox, non_blocking=True)
                hn.copy_(on, non_blocking=True)

        ems, _ = _timed(e2e_step, max(1, steps // 2), 1, world, dev)
        e2e = {"value": outs / (ems / max(1, steps // 2) / 1e3), "unit": bench.UNIT,
               "h2d_bytes_per_step": 4 * rows * n, "d2h_bytes_per_step": 8 * rows * n,
               "path": "MaxMinStream.push per 256-sample chunk from pinned host, outputs back per push"}
    elif cfg == "N4":
        # SURVEY.md §8(f) N4 on C3's series: grayscale opening and closing, w = 129,
        # one fused pass (input read once, both outputs written once)
        B, n, w = synth.C3["batch"], synth.C3["n"], synth.C3["w"]
        r0, r1 = shard.shard_items(B, world, rank)
        rows = r1 - r0
        host = torch.empty(rows, n, dtype=torch.float32).pin_memory()
        synth.c3(rows=rows, row0=r0, out=host.numpy())
        x = host.to(dev)
        oo = torch.empty(rows, n, dtype=torch.float32, device=dev)
        oc = torch.empty_like(oo)

        def step():
            mm.maxmin_morph_batched(x, w, out_open=oo, out_close=oc)

        nb = 4 * rows * n * 3
        outs = 2 * B * n
        steps = args.steps
        name = "N4: grayscale opening + closing of 65536 fp32 series x 4096 (C3), w=129, sharded by series"
        dtype = "f32"
        l2 = "inputs (1 GiB) larger than the 126 MB L2"
        step()
        torch.cuda.synchronize()
        import oracle

        parity = True
        for b in range(0, rows, max(1, rows // 128)):
            eo, ec = oracle.morph(host[b].numpy(), w)
            parity = parity and bool(np.array_equal(oo[b].cpu().numpy(), eo) and np.array_equal(oc[b].cpu().numpy(), ec))
        ms, clk = _timed(step, steps, args.warmup, world, dev)
        sample = None
        windows = (w,)
        e2e_io = (host, x, [oo, oc], "maxmin_morph_batched")
    else:
        raise SystemExit(f"unknown config {cfg}")

    if e2e is None and e2e_io is not None and not getattr(args, "no_e2e", False):
        h_in, d_in, d_outs, api = e2e_io
        e2e = _e2e(step, h_in, d_in, d_outs, outs, max(1, min(steps, 5)), world, dev, api,
                   "bounds/s" if cfg == "N3" else bench.UNIT)
    ms_step = ms / steps
    value = outs / (ms_step / 1e3)
    unit = "bounds/s" if cfg == "N3" else bench.UNIT
    achieved = nb / (ms_step / 1e3) / 1e9
    if rank == 0:
        cpu = None
        if not args.no_cpu and world == 1:
            cpu = cpu_baseline_extra(cfg, host, windows[0])
        line = {
            "metric": bench.METRIC, "value": value, "unit": unit, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak" if cfg != "C1" else "replicas",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": name, "l2": l2,
                       "parallelism": f"item sharding, dp{world}" if world > 1 else "single GPU"},
            "roofline": bench.roofline(achieved, bench.ncu_traffic(cfg, windows[0]), cfg,
                                       "the config's algorithmic bytes per step (DESIGN.md section 7)"),
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": steps * {"N3": 3, "N2": 16}.get(cfg, 1), "clocks": clk,
            "parity": {"bit_exact": parity},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _threads_timed(jobs, threads):
    """Run the callables on `threads` host threads (ctypes calls release the GIL);
    best of 2 wall times."""
    import concurrent.futures as cf

    best = None
    for _ in range(2):
        t0 = time.perf_counter()
        if threads == 1:
            for j in jobs:
                j()
        else:
            with cf.ThreadPoolExecutor(max_workers=threads) as ex:
                list(ex.map(lambda j: j(), jobs))
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best


def cpu_baseline_extra(cfg, host, w):
    """The oracle on a bounded sample of the config's own input, on 1 host thread and
    on all of them (independent rows / row bands / series chunks per thread)."""
    import numpy as np

    import oracle

    allt = oracle.host_threads()
    h = host.numpy() if hasattr(host, "numpy") else host
    if cfg == "C1":
        return bench.cpu_baseline(cfg, np.ascontiguousarray(h), (w,))
    if cfg in ("C3", "N2", "N4", "N3"):
        rows = h[:4096]
        k = rows.shape[0]
        per = [(i * k // allt, (i + 1) * k // allt) for i in range(allt)]
        if cfg == "N3":
            import synth

            q = synth.c3(rows=1, row0=synth.C3["batch"])[0]
            job = lambda a, b: (lambda: oracle.keogh(rows[a:b], q, (w - 1) // 2))  # noqa: E731
            outs, what, unit = k, "oracle.keogh (clipped envelope + bound per series)", "bounds/s"
        elif cfg == "N4":
            job = lambda a, b: (lambda: [oracle.morph(rows[i], w) for i in range(a, b)])  # noqa: E731
            outs, what, unit = 2 * k * rows.shape[1], "oracle.morph per series", bench.UNIT
        elif cfg == "N2":
            def job(a, b):
                return lambda: oracle.stream_pushes(rows[a:b], w, [256] * (rows.shape[1] // 256))
            outs, what, unit = 2 * k * rows.shape[1], "oracle.Stream, 16 pushes of 256 per series", bench.UNIT
        else:
            job = lambda a, b: (lambda: oracle.batched(rows[a:b], w))  # noqa: E731
            outs, what, unit = 2 * k * (rows.shape[1] - w + 1), "oracle.batched (appendix per row)", bench.UNIT
        t1 = _threads_timed([job(0, k)], 1)
        tn = _threads_timed([job(a, b) for a, b in per], allt)
        sample = f"first {k} series of the bench input; {what}"
    elif cfg == "C4":
        img = h[0, :2048 + w - 1]
        R = 2048
        per = [(i * R // allt, (i + 1) * R // allt) for i in range(allt)]
        job = lambda a, b: (lambda: oracle.separable_2d(img[a:b + w - 1], w, w))  # noqa: E731
        outs, unit = 2 * R * (img.shape[1] - w + 1), bench.UNIT
        t1 = _threads_timed([job(0, R)], 1)
        tn = _threads_timed([job(a, b) for a, b in per], allt)
        sample = f"first {R} output rows of image 0; oracle.separable_2d on row bands (w-1 rows of overlap)"
    elif cfg == "N1":
        a = np.ascontiguousarray(h[: 1 << 24])
        m = a.shape[0] - w + 1
        per = [(i * m // allt, (i + 1) * m // allt) for i in range(allt)]
        job = lambda j0, j1: (lambda: oracle.arg_wedge(a[j0:j1 + w - 1], w))  # noqa: E731
        outs, unit = 2 * m, bench.UNIT
        t1 = _threads_timed([job(0, m)], 1)
        tn = _threads_timed([job(j0, j1) for j0, j1 in per], allt)
        sample = "first 2^24 elements; oracle.arg_wedge on contiguous window ranges"
    else:
        return None
    return {"value": outs / tn, "unit": unit, "cores": allt, "kind": "oracle", "value_1thread": outs / t1,
            "sample": sample + f", {allt} threads and 1 thread, best of 2 (oracle gcc -O2 build)"}
