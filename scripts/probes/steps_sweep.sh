#!/bin/bash
# C2 step time against the length of the timed region (power / clock behaviour)
for st in 3 10 20 60; do
  timeout 300 python bench.py --no-e2e --no-cpu --no-gmres --steps $st > /tmp/b.json 2>/dev/null
  python -c "
import json;d=json.load(open('/tmp/b.json'));pk=d['roofline']['per_kind']
print('steps $st', round(d['ms_per_step'],3), 'kinds', round(sum(v['ms_per_step'] for v in pk.values()),3), d['clocks'])"
done
timeout 300 python scripts/timeline.py --steps 5 2>&1 | tail -8
