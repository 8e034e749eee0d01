#!/bin/bash
# A/B of whole C2 bench lines (same box, alternating): bash scripts/ab_bench.sh TAG "label:ENV=.." ...
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for rep in 1 2; do
for spec in "$@"; do
  label=${spec%%:*}; envs=${spec#*:}
  env $envs timeout 300 python bench.py --no-e2e --no-cpu --no-gmres > $OUT/bench_${label}_$rep.json 2>/dev/null
  python - "$OUT/bench_${label}_$rep.json" "$label" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
pk = d["roofline"]["per_kind"]
print(f"{sys.argv[2]:>8s} step {d['ms_per_step']:.3f} ms  kinds {sum(v['ms_per_step'] for v in pk.values()):.3f} ms  clk {d['clocks']['sm_mhz']}  " +
      " ".join(f"{k}={v['ms_per_step']:.3f}" for k, v in pk.items()))
PY
done
done
