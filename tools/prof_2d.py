"""Time the 2-D filter for non-byte types (separable path vs the fused generic kernel)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0610046_b200 as mm  # noqa: E402

for dt, w in [(torch.float32, 5), (torch.float32, 15), (torch.uint16, 15), (torch.float64, 7)]:
    x = (torch.rand(4, 8192, 8192, device="cuda") * 1000).to(dt)
    R = C = 8192 - w + 1
    ox = torch.empty(4, R, C, dtype=dt, device="cuda")
    on = torch.empty_like(ox)
    L = mm._lib.lib()
    vp = ctypes.c_void_p
    res = {}
    for label in ("separable", "generic"):
        def run():
            if label == "separable":
                mm.maxmin_filter_2d(x, w, w, out_max=ox, out_min=on)
            else:
                mm._lib.check(L.maxmin_filter_2d(mm.dtype_code(dt), vp(x.data_ptr()), 4, 8192, 8192, 8192, 8192 * 8192,
                                                 w, w, vp(ox.data_ptr()), vp(on.data_ptr()), C, R * C,
                                                 vp(torch.cuda.current_stream().cuda_stream)))
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[label] = e0.elapsed_time(e1) / 3
    nb = x.numel() * x.element_size() + 2 * ox.numel() * ox.element_size()
    print(f"2-D {dt} {w}x{w}: separable {res['separable']:.2f} ms ({nb / res['separable'] / 1e6 / 6546:.2f} of peak), "
          f"generic {res['generic']:.2f} ms")
