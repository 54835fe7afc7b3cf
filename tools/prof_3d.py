"""Time the 3-D box filter (N4 N-D) on a 256 x 1024 x 1024 volume."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0610046_b200 as mm  # noqa: E402

for dt, w in [(torch.float32, 5), (torch.uint8, 5), (torch.uint8, 15)]:
    x = (torch.rand(256, 1024, 1024, device="cuda") * 200).to(dt)
    D, R, C = 256 - w + 1, 1024 - w + 1, 1024 - w + 1
    ox = torch.empty(D, R, C, dtype=dt, device="cuda")
    on = torch.empty_like(ox)
    for _ in range(2):
        mm.maxmin_filter_3d(x, w, w, w, out_max=ox, out_min=on)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        mm.maxmin_filter_3d(x, w, w, w, out_max=ox, out_min=on)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    nb = x.numel() * x.element_size() + 2 * ox.numel() * ox.element_size()
    print(f"3-D {dt} {w}^3: {ms:.2f} ms, {nb / ms / 1e6:.0f} GB/s algorithmic ({nb / ms / 1e6 / 6546:.2f} of peak)")
