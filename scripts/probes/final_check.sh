#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --no-e2e --no-cpu --no-gmres > /tmp/b.json 2>/dev/null; python -c "
import json;d=json.load(open('/tmp/b.json'));print('C2', round(d['ms_per_step'],3), round(d['value']), d['roofline']['frac'], d['clocks']['sm_mhz'])"
