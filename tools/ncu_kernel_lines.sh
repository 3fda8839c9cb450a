#!/bin/bash
# ncu --set full of the first launch of one kernel (regex $2) in config $1's fill + H-LU,
# hottest source lines -> gpurun_out/ncu_lines/<name>_lines.txt
set -u
CFG=$1; RX=$2; NAME=${3:-$2}
OUT=gpurun_out/ncu_lines
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$RX" -c 1 -o /tmp/$NAME --force-overwrite \
    python tools/one_step.py $CFG > $OUT/$NAME.log 2>&1
ncu -i /tmp/$NAME.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${NAME}_src.csv 2>/dev/null
python tools/ncu_lines.py /tmp/${NAME}_src.csv 30 > $OUT/${NAME}_lines.txt
cat $OUT/${NAME}_lines.txt
