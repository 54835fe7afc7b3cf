"""Poll statistics of the k1d_lw diagnostics build (MM_LW_STATS=1, lib_lwstats.so):
    MAXMIN_LIB=lib_lwstats.so python tools/lw_stats.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0610046_b200 as mm  # noqa: E402
import synth  # noqa: E402

out = {}
for cfg, n, w in (("C2", 1 << 28, 65536), ("C2", 1 << 28, 9000), ("C5", 1 << 30, 262144)):
    x = torch.from_numpy(synth.c2(n) if cfg == "C2" else synth.c5(n)).cuda()
    ws = torch.empty(mm.maxmin_workspace_bytes(torch.float32, 1, n, w), dtype=torch.uint8, device="cuda")
    for rep in range(3):
        mm.maxmin_filter_1d(x, w, workspace=ws)
        torch.cuda.synchronize()
        st = ws[64:96].view(torch.int64).cpu().tolist()
        out[f"{cfg}_w{w}_rep{rep}"] = {"polled_words": st[0], "spins": st[1], "warp_wait_cycles_sum": st[2],
                                       "warp_wait_cycles_max": st[3],
                                       "groups": int(ws[:4].view(torch.int32).item())}
    del x, ws
print(json.dumps(out, indent=1))
