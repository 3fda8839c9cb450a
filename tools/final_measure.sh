#!/bin/bash
# Round-end measurement on one B200: GPU tests, the bench line, ncu launch lists of one
# fill + H-LU pass (configs 4 and 2), one `ncu --set full` capture per kernel family
# (config 2) and of one recompression launch of known shape (bench roofline.traffic).
# usage: bash tools/final_measure.sh <tag>      (outputs under gpurun_out/<tag>_*)
set -u
TAG=${1:-r02x}
O=gpurun_out
mkdir -p $O
(timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.log 2>&1; echo "rc=$?" >> $O/${TAG}_pytest.log)
timeout 1200 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "rc=$?" >> $O/${TAG}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_cfg4.csv \
    python tools/one_step.py 4 > $O/${TAG}_ncu4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_cfg2.csv \
    python tools/one_step.py 2 > $O/${TAG}_ncu2.log 2>&1
# recompression launch of known shape: 148 problems 1536 x 1536, k = 64, rank 40
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trunc_gram -c 1 -o /tmp/${TAG}_trunc \
    --force-overwrite python tools/trunc_bench.py 1536,1536,64,40,148 > $O/${TAG}_trunc_ncu.log 2>&1
ncu -i /tmp/${TAG}_trunc.ncu-rep --page raw --csv > $O/${TAG}_k_trunc_gram_ncu_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}_trunc.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${TAG}_src.csv 2>/dev/null
python tools/ncu_lines.py /tmp/${TAG}_src.csv 40 > $O/${TAG}_k_trunc_gram_lines.txt 2>/dev/null
if [ "${2:-}" = "families" ]; then
  bash tools/ncu_families.sh 2 > $O/${TAG}_families.log 2>&1
fi
tail -2 $O/${TAG}_pytest.log; head -c 600 $O/${TAG}_bench.json
