#!/bin/bash
# A/B of the C2 per-pass timings across library builds / env settings:
#   bash scripts/ab_passes.sh TAG "label1:ENV=.. ENV2=.." "label2:..." ...
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for spec in "$@"; do
  label=${spec%%:*}; envs=${spec#*:}
  (env $envs timeout 300 python scripts/prof_passes.py > $OUT/passes_$label.txt 2>&1)
  echo "== $label ($envs)"; grep -E "P[12]_QTX|P[12]_UPD_GRAM|sum of" $OUT/passes_$label.txt
done
