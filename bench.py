#!/usr/bin/env python
"""Bench harness: the running max-min filter on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {cuda,reference}]
                    [--config {C2,C3,C4,C5,C1}]

Default workload (BASELINE.json configs[1], C2): a 1-D fp32 random walk of
n = 2^28 elements per GPU; one step = the filter for every window of the config
(w = 3, 32, 1024, 65536), i.e. every kernel path (small, medium, large) over the
same HBM-resident input.  value = output elements (2 per window: max and min)
of all ranks per second.  For N > 1 each rank owns a 2^28 chunk of an N*2^28
array and receives the next rank's first w_max-1 elements by NCCL (weak
scaling).  The other configs (C1, C3, C4, C5) are available with --config.

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "max-min filter output elements/s and HBM GB/s vs peak at 1/2/4/8 B200"
UNIT = "output elements/s"


# ----------------------------------------------------------------- helpers --

def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config: str, kernel_w):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        return d.get(config, {}).get(str(kernel_w))
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock + clock-event reasons via NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: report that instead of clocks
            self.nv = None
            self.err = repr(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if self.nv is None:
            return {"error": getattr(self, "err", "nvml unavailable")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# -------------------------------------------------------------- workloads ---

def algo_bytes_1d(sz, n, w):
    return sz * (n + 2 * (n - w + 1))


def cpu_baseline(config: str, a_sample, windows, dtype_np):
    """The oracle as it stands (single-threaded appendix variant)
    on a bounded sample of the same workload."""
    import oracle

    t0 = time.perf_counter()
    outs = 0
    for w in windows:
        mx, mn, _ = oracle.appendix(a_sample, w)
        outs += 2 * mx.shape[0]
    dt = time.perf_counter() - t0
    return {"value": outs / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{config}: first {a_sample.shape[0]} elements of the bench array, "
                      f"windows {list(windows)}, oracle_appendix (C, gcc -O2, 1 thread), {dt:.2f} s"}


def run_reference(args, rank, world):
    """--impl reference: the oracle (the tier's reference arm) on the host cores."""
    import numpy as np

    import synth

    if rank != 0:
        return
    cfg = args.config
    windows = CONFIGS[cfg]["windows"]
    sample_n = CONFIGS[cfg]["ref_sample"]
    a = CONFIGS[cfg]["gen_sample"](sample_n)
    import oracle

    for _ in range(args.warmup):
        oracle.appendix(a[: min(sample_n, 1 << 16)], windows[0])
    times = []
    outs = 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o = 0
        for w in windows:
            mx, mn, _ = oracle.appendix(a, w) if a.ndim == 1 else (None, None, None)
            o += 2 * mx.shape[0]
        times.append(time.perf_counter() - t0)
        outs = o
    step = statistics.median(times)
    v = outs / step
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": CONFIGS[cfg]["name"] + " (bounded sample)",
                                            "sample_elements": int(sample_n)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"first {sample_n} elements, windows {list(windows)}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _gen_c2(n):
    import synth

    return synth.c2(n)


def _gen_c5(n):
    import synth

    return synth.c5(n)


CONFIGS = {
    "C2": dict(name="C2: 1-D fp32 random walk, n=2^28 per GPU, w in {3,32,1024,65536}",
               n=1 << 28, windows=(3, 32, 1024, 65536), gen="c2", ref_sample=1 << 24,
               gen_sample=_gen_c2),
    "C5": dict(name="C5: 1-D fp32 adversarial mix, n=2^30, w in {7,4096,262144}",
               n=1 << 30, windows=(7, 4096, 262144), gen="c5", ref_sample=1 << 24,
               gen_sample=_gen_c5),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS) + ["C1", "C3", "C4", "N1", "N2", "N3", "N4"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "cuda" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if args.config not in CONFIGS:
            args.config = "C2"
        return run_reference(args, rank, world)

    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.config in ("C1", "C3", "C4", "N1", "N2", "N3", "N4"):
        from bench_extra import run_extra

        return run_extra(args, rank, world, local)
    return run_1d(args, rank, world, local)


def run_1d(args, rank, world, local):
    import numpy as np
    import torch

    import paper_cs_0610046_b200 as mm
    from paper_cs_0610046_b200 import shard
    import synth

    cfg = CONFIGS[args.config]
    windows = cfg["windows"]
    n_local = cfg["n"]
    wmax = max(windows)
    halo = (wmax - 1) if world > 1 else 0
    chunk = shard.Chunk1D(rank=rank, world=world, n_local=n_local, halo=halo)
    dev = torch.device("cuda", local)

    # input: this rank's chunk of the global array, generated on the host (untimed)
    host = torch.empty(n_local + wmax, dtype=torch.float32).pin_memory()
    gen = synth.c2 if cfg["gen"] == "c2" else synth.c5
    gen(n_local, stream=rank, out=host[:n_local].numpy())
    buf = torch.empty(n_local + wmax, dtype=torch.float32, device=dev)
    buf.copy_(host)
    outs = {}
    for w in windows:
        m = chunk.windows(w)
        outs[w] = (torch.empty(m, dtype=torch.float32, device=dev),
                   torch.empty(m, dtype=torch.float32, device=dev))
    ws_bytes = max(mm.maxmin_workspace_bytes(torch.float32, 1, n_local + wmax, w) for w in windows)
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=dev)

    stream = torch.cuda.current_stream()
    per_w_events = {w: [] for w in windows}
    record = {"on": False}

    def filt(x, w, ox, on):
        if record["on"]:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            mm.maxmin_filter_1d(x, w, out_max=ox, out_min=on, workspace=ws)
            e1.record(stream)
            per_w_events[w].append((e0, e1, x.shape[0] == n_local))
        else:
            mm.maxmin_filter_1d(x, w, out_max=ox, out_min=on, workspace=ws)

    def step():
        if world > 1:
            shard.filter_1d_sharded(buf, chunk, windows, outs, filt)
        else:
            for w in windows:
                ox, on = outs[w]
                filt(buf[:n_local], w, ox, on)

    import torch.distributed as dist

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    # parity spot check of this run's outputs (oracle on bounded slices; untimed)
    parity = spot_check(host[:n_local].numpy(), outs, windows, chunk, rank)

    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    barrier()
    record["on"] = True
    with ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
    record["on"] = False
    ms = t0.elapsed_time(t1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    outs_per_step_rank = sum(2 * chunk.windows(w) for w in windows)
    outs_per_step = torch.tensor([outs_per_step_rank], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(outs_per_step)
    total_outs = float(outs_per_step.item()) * args.steps
    value = total_outs / (ms_max / 1e3)

    # per-window kernel time (CUDA events on the launching stream): the full-chunk
    # call of each window (the interior call when sharded), averaged per launch
    peak, peak_src = load_peaks()
    per_w = {}
    for w in windows:
        durs = [a.elapsed_time(b) for a, b, full in per_w_events[w] if full]
        d = sum(durs) / len(durs)  # ms per launch
        nb = algo_bytes_1d(4, n_local, w)
        per_w[str(w)] = {"ms_per_launch": d, "algo_bytes": nb, "gbs": nb / (d / 1e3) / 1e9,
                         "frac_of_peak": nb / (d / 1e3) / 1e9 / peak,
                         "launches_per_step": len(per_w_events[w]) / args.steps}
    dom = max(windows, key=lambda w: per_w[str(w)]["ms_per_launch"])
    achieved = per_w[str(dom)]["gbs"]
    traffic = ncu_traffic(args.config, dom)

    line = None
    if rank == 0:
        e2e = None if args.no_e2e or world > 1 else run_e2e(args, host, n_local, windows, dev)
        if world > 1:
            e2e = {"value": None, "unit": UNIT, "note": "e2e measured at N=1 only",
                   "h2d_bytes_per_step": None, "d2h_bytes_per_step": None}
        cpu = None
        if not args.no_cpu and world == 1:
            cpu = cpu_baseline(args.config, host[: 1 << 26].numpy().copy(), windows, np.float32)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["name"], "n_per_gpu": n_local, "windows": list(windows),
                       "step": "one filter call per window over the whole array (all kernel paths)",
                       "l2": "inputs (1 GiB per GPU) larger than the 126 MB L2; no flush needed",
                       "parallelism": f"sequence sharding, contiguous chunks + (w-1) NCCL halo, dp{world}"
                       if world > 1 else "single GPU"},
            "hbm_gbs_step": sum(algo_bytes_1d(4, n_local, w) for w in windows) * world
            / (ms_max / args.steps / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": f"w={dom}",
                         "peak_source": peak_src,
                         "algorithmic_bytes": "sizeof(f32)*(n + 2(n-w+1)) per launch"},
            "per_window": per_w,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": sum(int(round(per_w[str(w)]["launches_per_step"])) for w in windows)
            * args.steps,
            "clocks": clk.summary(),
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def spot_check(a, outs, windows, chunk, rank):
    """Bounded oracle check of the bench outputs (windows fully inside the chunk)."""
    import numpy as np

    import oracle

    ok = True
    checked = 0
    n = chunk.n_local
    for w in windows:
        ox, on = outs[w]
        m_int = n - w + 1
        for j0 in (0, 4096 - 7, m_int // 2 + 13, m_int - 4100):
            j0 = max(0, min(j0, m_int - 1))
            k = min(4100, m_int - j0)
            ex, en, _ = oracle.appendix(a[j0: j0 + k + w - 1], w)
            gx = ox[j0: j0 + k].cpu().numpy()
            gn = on[j0: j0 + k].cpu().numpy()
            ok &= np.array_equal(gx.view(np.uint32), ex.view(np.uint32))
            ok &= np.array_equal(gn.view(np.uint32), en.view(np.uint32))
            checked += 2 * k
    return {"bit_exact": bool(ok), "outputs_checked": checked, "oracle": "oracle_appendix on slices"}


def run_e2e(args, host, n, windows, dev):
    """Same metric through the public host-buffer API: H2D of the input and D2H of
    both outputs inside the timed region, every step."""
    import torch

    import paper_cs_0610046_b200 as mm

    x = host[:n]
    m0 = n - min(windows) + 1
    ox = torch.empty(m0, dtype=torch.float32).pin_memory()
    on = torch.empty(m0, dtype=torch.float32).pin_memory()
    chunk = 1 << 24
    wsb = max(mm.maxmin_host_workspace_bytes(torch.float32, n, w, chunk) for w in windows)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    steps = max(1, min(args.steps, 3))

    def step():
        for w in windows:
            mm.maxmin_filter_1d_host(x, w, ox[: n - w + 1], on[: n - w + 1], ws, chunk=chunk)

    step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    outs = sum(2 * (n - w + 1) for w in windows)
    h2d = sum(4 * (n + ((n - w + 1 + chunk - 1) // chunk - 1) * (w - 1)) for w in windows)
    d2h = 4 * outs
    return {"value": outs / dt, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": dt * 1e3, "steps": steps, "api": "maxmin_filter_1d_host (pinned host buffers)"}


if __name__ == "__main__":
    main()
