#!/bin/bash
# ncu --set full of ONE k_trunc_gram launch (position $2 among the k_trunc_gram launches of
# config $1's fill + H-LU): raw CSV + per-source-line stall samples
set -u
OUT=gpurun_out/ncu_big
REP=/tmp/ncu_big
mkdir -p $OUT $REP
CFG=$1; POS=$2; KEY=${3:-pos$POS}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trunc_gram \
    --launch-skip $POS --launch-count 1 -o $REP/$KEY --force-overwrite python tools/one_step.py $CFG > $OUT/$KEY.log 2>&1
ncu -i $REP/$KEY.ncu-rep --page raw --csv > $OUT/${KEY}_raw.csv 2>/dev/null
ncu -i $REP/$KEY.ncu-rep --page source --csv --print-source cuda,sass > $OUT/${KEY}_source.csv 2>/dev/null
python tools/ncu_lines.py $OUT/${KEY}_source.csv 40 > $OUT/${KEY}_lines.txt
rm -f $OUT/${KEY}_source.csv
