"""Run one max-min filter configuration a few times (for ncu captures).

    python tools/prof_one.py --config C2 --w 1024 --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_cs_0610046_b200 as mm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--w", type=int, default=1024)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda:0")
if a.config == "C2":
    x = torch.from_numpy(synth.c2(1 << 28)).to(dev)
    ws = torch.empty(max(mm.maxmin_workspace_bytes(torch.float32, 1, x.numel(), a.w), 16),
                     dtype=torch.uint8, device=dev)
    for _ in range(a.reps):
        mm.maxmin_filter_1d(x, a.w, workspace=ws)
elif a.config == "C5":
    x = torch.from_numpy(synth.c5(1 << 30)).to(dev)
    ws = torch.empty(max(mm.maxmin_workspace_bytes(torch.float32, 1, x.numel(), a.w), 16),
                     dtype=torch.uint8, device=dev)
    for _ in range(a.reps):
        mm.maxmin_filter_1d(x, a.w, workspace=ws)
elif a.config == "C3":
    x = torch.from_numpy(synth.c3()).to(dev)
    for _ in range(a.reps):
        mm.maxmin_filter_batched(x, a.w)
elif a.config == "C4":
    x = torch.from_numpy(synth.c4()).to(dev)
    for _ in range(a.reps):
        mm.maxmin_filter_2d(x, a.w, a.w)
torch.cuda.synchronize()
print("ok")
