"""ncu launch list (--metrics gpu__time_duration.sum --csv) -> markdown table by kernel."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi = h.index("Kernel Name"), h.index("Metric Value")
ui = h.index("Metric Unit") if "Metric Unit" in h else None
scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}
agg = {}
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    try:
        v = float(r[mi].replace(",", "")) * scale.get(r[ui] if ui is not None else "nsecond", 1.0)
    except ValueError:
        continue
    name = r[ki].split("(")[0].replace("<unnamed>::", "")[:48]
    agg.setdefault(name, []).append(v)
tot = sum(sum(v) for v in agg.values())
print("| kernel | launches | total ms | share | median us | max us |")
print("|---|---:|---:|---:|---:|---:|")
for n, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    s = sorted(v)
    print(f"| `{n}` | {len(v)} | {sum(v) / 1e6:.2f} | {100 * sum(v) / tot:.1f} % | {s[len(s) // 2] / 1e3:.1f} | {s[-1] / 1e3:.1f} |")
print(f"\nTotal kernel time: {tot / 1e6:.1f} ms over {sum(len(v) for v in agg.values())} launches.")
