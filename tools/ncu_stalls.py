"""Top stall sites (with SASS context) and stall-reason totals of an ncu report.

    python tools/ncu_stalls.py report.ncu-rep [n_sites]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nsites = int(sys.argv[2]) if len(sys.argv) > 2 else 5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
h = rows[0]
ia, isrc, iex, ist = (h.index("Address"), h.index("Source"), h.index("Instructions Executed"),
                      h.index("Warp Stall Sampling (All Samples)"))
body = rows[1:]
tot = sum(int(r[ist] or 0) for r in body)
print("total samples", tot)
order = sorted(range(len(body)), key=lambda i: -int(body[i][ist] or 0))[:nsites]
for i in order:
    print(f"--- {100 * int(body[i][ist]) / tot:.1f}%")
    for r in body[max(0, i - 6): i + 2]:
        print(r[ia][-5:], r[ist].rjust(6), r[iex].rjust(10), r[isrc])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh, vv = rr[0], rr[2]
st = []
for i, k in enumerate(hh):
    if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
        try:
            st.append((float(vv[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
print("reasons:", ", ".join(f"{k} {100 * x / max(tot, 1):.0f}%" for x, k in sorted(st, reverse=True)[:8]))
