#!/bin/bash
# One `ncu --set full` capture per kernel family of the hot path (config 2, one fill +
# H-LU pass: tools/one_step.py), then the raw CSV of each into gpurun_out/ncu/.
# Usage (on the GPU box): bash tools/ncu_families.sh [config]
set -u
CFG=${1:-2}
OUT=gpurun_out/ncu
REP=/tmp/ncu_reps          # the .ncu-rep files stay on the box (gpurun_out is capped at 64 MiB)
mkdir -p $OUT $REP
NCU=${NCU:-ncu}
for K in k_near_blocks k_fill_tiles k_aca k_trunc_gram k_getrf_blk k_trsm_blk k_gemm64 k_gemm k_dlr_range k_dense_lr k_concat k_newton k_rcond_blk; do
  RX="${K}"
  [ "$K" = k_gemm ] && RX='k_gemm$|k_gemm[^6v]'
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"${RX}" -c 1 \
      -o $REP/$K --force-overwrite python tools/one_step.py $CFG > $OUT/$K.log 2>&1
  if [ -f $REP/$K.ncu-rep ]; then
    $NCU -i $REP/$K.ncu-rep --page raw --csv > $OUT/${K}_raw.csv 2>/dev/null
    $NCU -i $REP/$K.ncu-rep --page details --csv > $OUT/${K}_details.csv 2>/dev/null
    [ "$K" = k_trunc_gram ] && $NCU -i $REP/$K.ncu-rep --page source --csv --print-source cuda,sass \
        > $OUT/${K}_source.csv 2>/dev/null
  fi
done
