"""Run one NEXT-row operation (N1..N4) on its bench workload for ncu captures:
tools/gpu_evidence.sh profiles the first launch after --reps warm-ups."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0610046_b200 as mm  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--op", required=True, choices=["N1", "N2", "N3", "N4"])
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
if args.op == "N1":
    x = torch.from_numpy(synth.c2(1 << 28)).cuda()

    def run():
        mm.maxmin_argfilter_1d(x, 1024)
elif args.op == "N2":
    x = torch.from_numpy(synth.c3()).cuda()
    chunks = [x[:, p * 256:(p + 1) * 256].contiguous() for p in range(16)]
    st = mm.MaxMinStream(torch.float32, x.shape[0], 129, 256)
    ox = torch.empty(x.shape[0], 256, device="cuda")
    on = torch.empty_like(ox)

    def run():
        for ch in chunks:
            st.push(ch, out_max=ox, out_min=on)
elif args.op == "N3":
    x = torch.from_numpy(synth.c3()).cuda()
    q = torch.from_numpy(synth.c3(rows=1, row0=x.shape[0])[0]).cuda()

    def run():
        mm.maxmin_lb_keogh_batched(x, q, 64)
else:
    x = torch.from_numpy(synth.c3()).cuda()
    oo, oc = torch.empty_like(x), torch.empty_like(x)

    def run():
        mm.maxmin_morph_batched(x, 129, out_open=oo, out_close=oc)
for _ in range(args.reps + 1):
    run()
torch.cuda.synchronize()
print(args.op, "ok")
