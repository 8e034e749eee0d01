#!/bin/bash
# A/B of pass-engine variants (per-pass C2 timings): decoupled panel ring policy
bash scripts/ab_passes.sh ab_dec2 "auto:X=1" "never:BO_DEC=-1" "always:BO_DEC=1" "auto2:X=1"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/ab_dec2/bench.json 2>gpurun_out/ab_dec2/bench.err; echo bench rc=$?
python -c "
import json;d=json.load(open('gpurun_out/ab_dec2/bench.json'));print(d['ms_per_step'],d['value'],d['gmres']['ms_per_restart'],d['c5']['ms_per_restart'])"
