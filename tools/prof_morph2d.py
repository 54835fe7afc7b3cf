"""Time the N4 2-D opening + closing on C4's images (composition path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0610046_b200 as mm  # noqa: E402
import synth  # noqa: E402

cnt = int(sys.argv[1]) if len(sys.argv) > 1 else 2
img = torch.from_numpy(synth.c4(count=cnt)).cuda()
w = 15
oo, oc = torch.empty_like(img), torch.empty_like(img)
for _ in range(2):
    mm.maxmin_morph_2d(img, w, w, out_open=oo, out_close=oc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    mm.maxmin_morph_2d(img, w, w, out_open=oo, out_close=oc)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"2-D morph {cnt} x 16384^2 u8 w=15: {ms:.2f} ms, {3 * img.numel() / ms / 1e6:.1f} GB/s algorithmic")
# component times: the 2-D filter alone on the same images (pass 1 / pass 2 analogue)
ox, on = torch.empty_like(img), torch.empty_like(img)
e0.record()
for _ in range(3):
    mm.maxmin_filter_2d(img, w, w, out_max=ox[:, : img.shape[1] - w + 1, : img.shape[2] - w + 1],
                        out_min=on[:, : img.shape[1] - w + 1, : img.shape[2] - w + 1])
e1.record()
torch.cuda.synchronize()
print(f"  2-D filter alone: {e0.elapsed_time(e1) / 3:.2f} ms")
