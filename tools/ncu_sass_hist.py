"""Dynamic instruction mix and stall hot spots of one kernel from an ncu report.

    python tools/ncu_sass_hist.py report.ncu-rep [units]

Prints executed warp instructions per opcode (and per `units` if given, e.g. the
number of pixels, as thread-instructions per unit) and the top stall sites.
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ia, isrc, iex, ist = (hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"),
                      hdr.index("Warp Stall Sampling (All Samples)"))
ops = collections.Counter()
stall = []
total = 0
for r in rows[1:]:
    src = r[isrc].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", src)
    if not m:
        continue
    n = int(r[iex] or 0)
    ops[m.group(2)] += n
    total += n
    stall.append((int(r[ist] or 0), r[ia], src))
print(f"total warp instructions {total}" + (f"  thread-instr/unit {32 * total / units:.2f}" if units else ""))
for op, n in ops.most_common(25):
    extra = f"  {32 * n / units:.3f}/unit" if units else ""
    print(f"{op:10s} {n:14d} {100 * n / total:6.2f}%{extra}")
print("top stall sites:")
for s, a, src in sorted(stall, reverse=True)[:15]:
    print(f"{s:8d} {a} {src}")
