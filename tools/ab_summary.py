"""Summarise tools/gpu_ab.sh logs: median ms per (lib, config, window) over the runs."""
import glob
import json
import sys
from collections import defaultdict

res = defaultdict(list)
for f in sorted(glob.glob(sys.argv[1] + "/ab_*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            for k, v in d.items():
                if isinstance(v, dict):
                    res[(d["lib"], d["config"], k)].append((v["ms_median"], v["frac"], v["bit_exact_slices"]))
for (lib, cfg, w), v in sorted(res.items(), key=lambda x: (x[0][1], x[0][2], x[0][0])):
    print(f"{cfg} w={w:>7s} {lib:18s} ms {' '.join(f'{a:.4f}' for a, _, _ in v)}  frac {max(b for _, b, _ in v):.3f}"
          f"  exact {all(c for _, _, c in v)}")
