"""One 1-D filter call on a small case, checked against the oracle (for
compute-sanitizer runs):  python tools/repro_1d.py N W [dtype]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_cs_0610046_b200 as mm  # noqa: E402
import synth  # noqa: E402

n, w = int(sys.argv[1]), int(sys.argv[2])
dt = np.dtype(sys.argv[3]) if len(sys.argv) > 3 else np.dtype(np.float32)
a = synth.c2(n).astype(dt) if dt.kind == "f" else synth.random_values(dt, n, seed=3)
x = torch.from_numpy(a).cuda()
mx, mn = mm.maxmin_filter_1d(x, w)
torch.cuda.synchronize()
ex, en, _ = oracle.appendix(a, w)
print("max ok", np.array_equal(mx.cpu().numpy(), ex), "min ok", np.array_equal(mn.cpu().numpy(), en))
