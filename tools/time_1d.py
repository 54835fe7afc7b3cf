"""Time single 1-D filter launches (CUDA events, after warm-up) for A/B of kernel
variants; MAXMIN_LIB selects the library build.  Checks the outputs against the
oracle on slices (first / middle / last 20k windows).

    python tools/time_1d.py --config C2 --windows 65536 --reps 20
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_cs_0610046_b200 as mm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--windows", default="65536")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda:0")
n = a.n or (1 << 28 if a.config == "C2" else 1 << 30)
host = synth.c2(n) if a.config == "C2" else synth.c5(n)
x = torch.from_numpy(host).to(dev)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
res = {"lib": os.environ.get("MAXMIN_LIB", "libmaxmin.so"), "config": a.config, "n": n}
for w in [int(v) for v in a.windows.split(",")]:
    ws = torch.empty(max(mm.maxmin_workspace_bytes(torch.float32, 1, n, w), 16), dtype=torch.uint8, device=dev)
    m = n - w + 1
    ox = torch.empty(m, device=dev)
    on = torch.empty(m, device=dev)
    for _ in range(3):
        mm.maxmin_filter_1d(x, w, out_max=ox, out_min=on, workspace=ws)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
    for e0, e1 in ev:
        e0.record()
        mm.maxmin_filter_1d(x, w, out_max=ox, out_min=on, workspace=ws)
        e1.record()
    torch.cuda.synchronize()
    ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
    ok = True
    for j0 in (0, m // 2 - 7, m - 20000):
        ex, en, _ = oracle.appendix(host[j0: j0 + 20000 + w - 1], w)
        ok &= bool(np.array_equal(ox[j0: j0 + 20000].cpu().numpy(), ex) and
                   np.array_equal(on[j0: j0 + 20000].cpu().numpy(), en))
    nb = 4 * (n + 2 * m)
    med = ms[len(ms) // 2]
    res[str(w)] = {"ms_median": med, "ms_best": ms[0], "gbs": nb / med / 1e6, "frac": nb / med / 1e6 / peak,
                   "bit_exact_slices": ok}
print(json.dumps(res))
