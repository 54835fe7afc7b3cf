"""Summaries of an ncu report for the kernel-tuning loop:
    python tools/ncu_quick.py REPORT [--lines N]
Prints the headline metrics, the stall-sample breakdown, the opcode mix and the
hottest source lines (instructions executed and stall samples)."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
nlines = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 30


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


rows = list(csv.reader(run("--page", "raw", "--csv").splitlines()))
h = rows[0]
d = dict(zip(h, rows[2]))
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "launch__grid_size", "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]:
    print(f"{k:70s} {d.get(k)}")
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(v)) for k, v in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v}
tot = sum(st.values()) or 1
print("stalls:", ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1]) if v / tot > 0.01))
srows = list(csv.reader(run("--page", "source", "--csv", "--print-source=sass").splitlines()))
hh = srows[1]
ix = {k: i for i, k in enumerate(hh)}
c = Counter()
for r in srows[2:]:
    src = r[ix["Source"]].strip()
    parts = src.split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    c[op.split(".")[0]] += int(r[ix["Instructions Executed"]] or 0)
ti = sum(c.values()) or 1
print("opcodes:", ", ".join(f"{k} {v / ti * 100:.1f}%" for k, v in c.most_common(18)))
rows = list(csv.reader(run("--page", "source", "--csv", "--print-source=cuda,sass").splitlines()))
cur, out = None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[2] == "-":
        try:
            out.append((int(r[7] or 0), int(r[4] or 0), cur, r[0], r[1][:80]))
        except ValueError:
            pass
tot_i = sum(o[0] for o in out) or 1
tot_s = sum(o[1] for o in out) or 1
print(f"lines by instructions (total {tot_i}):")
for o in sorted(out, reverse=True)[:nlines]:
    print(f"  {o[0] / tot_i * 100:5.1f}% i {o[1] / tot_s * 100:5.1f}% s  {o[2]}:{o[3]}  {o[4]}")
print("lines by stall samples:")
for o in sorted(out, key=lambda o: -o[1])[:nlines]:
    print(f"  {o[0] / tot_i * 100:5.1f}% i {o[1] / tot_s * 100:5.1f}% s  {o[2]}:{o[3]}  {o[4]}")
