#!/bin/bash
# ncu --set full of the LONGEST k_trunc_gram launches of the config-4 H-LU: (1) time +
# grid + cluster size of every launch, (2) the longest cluster launch and the longest
# non-cluster launch captured in full (launch order is deterministic).
set -u
OUT=gpurun_out/ncu_big
REP=/tmp/ncu_big
mkdir -p $OUT $REP
CFG=${1:-4}
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_size --clock-control none \
    -k regex:k_trunc_gram --csv --log-file $REP/list.csv python tools/one_step.py $CFG > $OUT/list.log 2>&1
python - $REP/list.csv > $OUT/pick.txt <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
idc, mn, mv = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
d = {}
for r in rows[hi + 1:]:
    if len(r) <= mv:
        continue
    d.setdefault(int(r[idc]), {})[r[mn]] = float(r[mv].replace(",", ""))
ids = sorted(d)
best = {}
for pos, i in enumerate(ids):
    x = d[i]
    key = "cluster" if x.get("launch__cluster_size", 1) > 1 else "single"
    if key not in best or x["gpu__time_duration.sum"] > best[key][1]:
        best[key] = (pos, x["gpu__time_duration.sum"], x.get("launch__grid_size"), x.get("launch__cluster_size"))
for k, v in best.items():
    print(k, *v)
PY
cat $OUT/pick.txt
while read KEY POS DUR GRID CL; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trunc_gram \
      --launch-skip $POS --launch-count 1 -o $REP/$KEY --force-overwrite python tools/one_step.py $CFG > $OUT/$KEY.log 2>&1
  ncu -i $REP/$KEY.ncu-rep --page raw --csv > $OUT/${KEY}_raw.csv 2>/dev/null
  ncu -i $REP/$KEY.ncu-rep --page source --csv --print-source cuda > $OUT/${KEY}_source.csv 2>/dev/null
done < $OUT/pick.txt
