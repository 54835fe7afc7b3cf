"""Host-side cost of one C1-sized call (n=100000, w=16, f64): Python binding vs raw C ABI."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0610046_b200 as mm  # noqa: E402

n, w = 100_000, 16
x = torch.rand(n, dtype=torch.float64, device="cuda")
ox = torch.empty(n - w + 1, dtype=torch.float64, device="cuda")
on = torch.empty_like(ox)
L = mm._lib.lib()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
args = (mm.dtype_code(torch.float64), ctypes.c_void_p(x.data_ptr()), n, w, ctypes.c_void_p(ox.data_ptr()),
        ctypes.c_void_p(on.data_ptr()), ctypes.c_void_p(0), 0, s)
for label, fn in [("python binding", lambda: mm.maxmin_filter_1d(x, w, out_max=ox, out_min=on)),
                  ("raw C ABI", lambda: L.maxmin_filter_1d(*args))]:
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{label}: host {1e6 * (t1 - t0) / 2000:.2f} us/call, wall {1e6 * (t2 - t0) / 2000:.2f} us/call")
