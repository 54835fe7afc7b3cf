"""Run the N4 opening/closing on C3's series for ncu captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0610046_b200 as mm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--w", type=int, default=129)
args = ap.parse_args()
x = torch.from_numpy(synth.c3()).cuda()
oo, oc = torch.empty_like(x), torch.empty_like(x)
for _ in range(args.reps):
    mm.maxmin_morph_batched(x, args.w, out_open=oo, out_close=oc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    mm.maxmin_morph_batched(x, args.w, out_open=oo, out_close=oc)
e1.record()
torch.cuda.synchronize()
print(f"w={args.w}: {e0.elapsed_time(e1) / 5:.3f} ms")
