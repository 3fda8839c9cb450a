#!/bin/bash
# H-LU device time / residual of configs under recorder / kernel knobs (one line per run)
# usage: bash tools/hlu_variants.sh "<cfgs>" "VAR=1" "VAR2=1 VAR3=2" ...
CFGS=$1; shift
echo "default"; timeout 900 python tools/hlu_time.py $CFGS 2>&1 | grep '^{'
for v in "$@"; do echo "$v"; env $v timeout 900 python tools/hlu_time.py $CFGS 2>&1 | grep '^{'; done
