"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass) by CUDA
source line: warp-stall samples per line, top N."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
fname, out, tot = "", [], 0.0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= 5 and r[0] not in ("", "Line No", "Function Name") and r[2] == "-":
        try:
            s = float(r[4] or 0)
        except ValueError:
            continue
        out.append((s, f"{fname}:{r[0]}", r[1].strip()[:100]))
        tot += s
out.sort(reverse=True)
for s, loc, src in out[:n]:
    print(f"{100 * s / tot:5.1f}%  {loc:24s} {src}")
