"""Run N2 pushes (C3 streams, w=129, c=256) for ncu captures: tools/gpu_prof_stream.sh."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0610046_b200 as mm
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--c", type=int, default=256)
ap.add_argument("--w", type=int, default=129)
args = ap.parse_args()
B, n = synth.C3["batch"], synth.C3["n"]
x = torch.from_numpy(synth.c3()).cuda()
c = args.c
chunks = [x[:, p * c:(p + 1) * c].contiguous() for p in range(n // c)]
st = mm.MaxMinStream(torch.float32, B, args.w, c)
ox = torch.empty(B, c, dtype=torch.float32, device="cuda")
on = torch.empty_like(ox)
for _ in range(args.reps):
    for ch in chunks:
        st.push(ch, out_max=ox, out_min=on)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for ch in chunks:
    st.push(ch, out_max=ox, out_min=on)
e1.record()
torch.cuda.synchronize()
print(f"c={c} w={args.w}: {e0.elapsed_time(e1) / len(chunks) * 1e3:.1f} us per push")
