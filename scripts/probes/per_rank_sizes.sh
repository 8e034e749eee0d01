#!/bin/bash
# C2 sequence time at the per-rank row counts of a 1/2/4/8-GPU run (DESIGN §6 model)
for n in 8000000 4000000 2000000 1000000 100000; do
  timeout 300 python bench.py --n $n --no-e2e --no-cpu --no-gmres --steps 20 > /tmp/b.json 2>/dev/null
  python -c "
import json;d=json.load(open('/tmp/b.json'));pk=d['roofline']['per_kind']
print('n=$n', round(d['ms_per_step'],3), 'kinds', round(sum(v['ms_per_step'] for v in pk.values()),3), d['clocks']['sm_mhz'])"
done
