"""Stress the large-window kernel (k1d_lw, both publication leads) or, with
--medium, k1d_medium (ring-free, three- and two-stage ring variants):
repeated launches on 2^27 C2 elements and on batched rows, every output
compared with the oracle computed once.  python tools/stress_lw.py --reps 30"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_cs_0610046_b200 as mm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--medium", action="store_true")
a = ap.parse_args()
W1 = (1024, 600, 2049, 4096, 129, 32) if a.medium else (65536, 20000, 140000)
WB = (1000, 5000) if a.medium else (9000, 70000)
dev = torch.device("cuda:0")
bad = 0
a2 = synth.c2(1 << 27)
x = torch.from_numpy(a2).to(dev)
for w in W1:  # lw: q = 127, 39 (three-job lead), 273 (two-job lead)
    ex, en, _ = oracle.appendix(a2, w)
    for r in range(a.reps):
        mx, mn = mm.maxmin_filter_1d(x, w)
        ok = np.array_equal(mx.cpu().numpy().view(np.uint32), ex.view(np.uint32)) and \
            np.array_equal(mn.cpu().numpy().view(np.uint32), en.view(np.uint32))
        bad += not ok
        if not ok:
            print("MISMATCH w", w, "rep", r, flush=True)
    print("w", w, "reps", a.reps, "bad so far", bad, flush=True)
rows, n = 64, 300_000
b = synth.random_values(np.float32, rows * n, seed=99).reshape(rows, n)
xb = torch.from_numpy(b).to(dev)
for w in WB:
    ex, en = oracle.batched(b, w)
    for r in range(a.reps):
        mx, mn = mm.maxmin_filter_batched(xb, w)
        ok = np.array_equal(mx.cpu().numpy(), ex) and np.array_equal(mn.cpu().numpy(), en)
        bad += not ok
    print("batched w", w, "bad so far", bad, flush=True)
print("STRESS", "FAIL" if bad else "OK", bad)
