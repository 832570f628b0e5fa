"""Top source lines by warp-stall samples from an ncu --set full capture.

  python tools/hotspots.py REPORT.ncu-rep "title" > profiles/....txt
Reads `ncu -i REPORT --page source --csv --print-source cuda,sass` and sums the
stall samples per CUDA source line (with the long/short-scoreboard and wait
shares of each line).
"""
import csv
import io
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = next(r for r in rows if r and r[0] == "Line No")
si = h.index("Warp Stall Sampling (All Samples)")
reasons = ["stall_long_sb", "stall_short_sb", "stall_wait", "stall_branch_resolving"]
ri = [h.index(r) for r in reasons]
ii = h.index("Instructions Executed")
agg, fname = {}, "?"
tot = toti = 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) <= si or r[0] in ("", "Line No"):
        continue
    try:
        s, n, v = int(r[si]), int(r[ii]), [int(r[i]) for i in ri]
    except ValueError:
        continue
    agg[(fname, int(r[0]))] = (s, n, v, r[1].strip()[:100])
    tot += s
    toti += n
print(title)
print("stall%  instr%  long/short/wait/branch % of the line   file:line  source")
for (f, ln), (s, n, v, src) in sorted(agg.items(), key=lambda t: -t[1][0])[:40]:
    mix = "/".join(f"{100 * x / max(s, 1):.0f}" for x in v)
    print(f"{100 * s / max(tot, 1):5.1f}%  {100 * n / max(toti, 1):5.1f}%  {mix:>14s}   {f}:{ln}  {src}")
