"""Copy ncu evidence into profiles/<round>/: text summaries of --set full
captures and the launch list, plus profiles/ncu_traffic.json (dram bytes per
launch of each profiled kernel, keyed by config and window) read by bench.py."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rnd, items):
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for item in items:  # config:w:path
        cfg, w, path = item.split(":", 2)
        hdr, units, rows = raw(path)
        idx = {h: i for i, h in enumerate(hdr)}
        v = rows[0]
        rd = float(v[idx["dram__bytes_read.sum"]])
        wr = float(v[idx["dram__bytes_write.sum"]])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale[units[idx["dram__bytes_read.sum"]]]
        wr *= scale[units[idx["dram__bytes_write.sum"]]]
        traffic.setdefault(cfg, {})[str(w)] = rd + wr
        summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), path],
                              capture_output=True, text=True).stdout
        with open(os.path.join(dst, f"ncu_{cfg}_w{w}.txt"), "w") as f:
            f.write(f"# ncu --set full --clock-control none, {cfg} w={w}: {os.path.basename(path)}\n")
            f.write(f"# dram bytes per launch (read+write): {rd + wr:.0f}\n")
            f.write(summ)
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
