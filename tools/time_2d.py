"""Time the C4 2-D filter (8 u8 images 16384^2, 15x15; CUDA events after warm-up) for
A/B of kernel variants (MAXMIN_LIB selects the build); checks two crops bit-exactly.
    python tools/time_2d.py [--reps 10]"""
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
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--w", type=int, default=15)
a = ap.parse_args()
dev = torch.device("cuda:0")
host = synth.c4()
x = torch.from_numpy(host).to(dev)
NI, R, C = host.shape
w = a.w
Ro, Co = R - w + 1, C - w + 1
ox = torch.empty(NI, Ro, C, dtype=torch.uint8, device=dev)
on = torch.empty_like(ox)
for _ in range(3):
    mm.maxmin_filter_2d(x, w, w, out_max=ox[:, :, :Co], out_min=on[:, :, :Co])
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
for e0, e1 in ev:
    e0.record()
    mm.maxmin_filter_2d(x, w, w, out_max=ox[:, :, :Co], out_min=on[:, :, :Co])
    e1.record()
torch.cuda.synchronize()
ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
ok = True
for b, r0, c0 in ((0, 0, 0), (5, 7000, 9001)):
    crop = host[b, r0:r0 + 300, c0:c0 + 700]
    ex, en = oracle.separable_2d(crop, w, w)
    ok &= bool(np.array_equal(ox[b, r0:r0 + 300 - w + 1, c0:c0 + 700 - w + 1].cpu().numpy(), ex)
               and np.array_equal(on[b, r0:r0 + 300 - w + 1, c0:c0 + 700 - w + 1].cpu().numpy(), en))
nb = NI * (R * C + 2 * Ro * Co)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
med = ms[len(ms) // 2]
print(json.dumps({"lib": os.environ.get("MAXMIN_LIB", "libmaxmin.so"), "config": "C4", str(w): {
    "ms_median": med, "ms_best": ms[0], "gbs": nb / med / 1e6, "frac": nb / med / 1e6 / peak,
    "bit_exact_slices": ok}}))
