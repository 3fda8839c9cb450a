"""Markdown summary of the per-family `ncu --set full` captures (tools/ncu_families.sh):
duration, SM / memory throughput, warps active, FP64 pipe, DMMA, DRAM bytes, top stall
reasons; plus the hottest source lines of one kernel's source page.

    python tools/ncu_summary.py gpurun_out/ncu [k_trunc_gram] > profiles/r02_ncu_families.md
"""
import collections
import csv
import glob
import os
import sys

D = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu"
HOT = sys.argv[2] if len(sys.argv) > 2 else "k_trunc_gram"
COLS = [("gpu__time_duration.sum", "time"), ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "regs"), ("launch__shared_mem_per_block_dynamic", "dyn smem"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps act %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA %"),
        ("dram__bytes_read.sum", "DRAM rd"), ("dram__bytes_write.sum", "DRAM wr")]
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "wait", "mio_throttle", "math_pipe_throttle",
          "lg_throttle", "branch_resolving", "not_selected", "selected", "dispatch_stall", "no_instruction"]


def row(path):
    r = list(csv.reader(open(path)))
    return r[0], r[1], r[2]


print("| kernel | " + " | ".join(c[1] for c in COLS) + " | top stalls (warps per issue) |")
print("|---" * (len(COLS) + 2) + "|")
for f in sorted(glob.glob(os.path.join(D, "*_raw.csv"))):
    h, u, v = row(f)
    cells = []
    for key, _ in COLS:
        if key in h:
            i = h.index(key)
            cells.append(f"{v[i]} {u[i]}".replace("register/thread", "").replace("/block", "").strip())
        else:
            cells.append("-")
    st = []
    for s in STALLS:
        k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if k in h and v[h.index(k)]:
            st.append((float(v[h.index(k)]), s))
    st = ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:3])
    print(f"| `{os.path.basename(f)[:-8]}` | " + " | ".join(cells) + f" | {st} |")

src = os.path.join(D, f"{HOT}_source.csv")
if os.path.exists(src):
    rows = list(csv.reader(open(src)))
    cur, hdr, tot, lines = None, None, 0.0, {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        try:
            ln0 = int(r[0])
        except ValueError:
            continue
        d = dict(zip(hdr, r))
        try:
            n = float(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            n = 0
        if n:
            st = {k[6:]: float(d[k]) for k in hdr if k.startswith("stall_") and "(Not" not in k and d[k] not in ("", "0")}
            lines[(cur, ln0)] = (n, st)
            tot += n
    print(f"\n### `{HOT}`: hottest source lines (share of warp-stall samples)\n")
    print("| line | share | top stall reasons (samples) |")
    print("|---|---:|---|")
    for (fn, ln), (n, st) in sorted(lines.items(), key=lambda x: -x[1][0])[:20]:
        top = ", ".join(f"{k} {int(x)}" for x, k in sorted(((x, k) for k, x in st.items()), reverse=True)[:3])
        print(f"| {fn}:{ln} | {100 * n / tot:.1f} % | {top} |")
