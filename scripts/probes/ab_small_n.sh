#!/bin/bash
# C2 sequence at small n (fixed per-call cost), current vs previous library
L=/root/repo/paper_2503_16717_b200
for r in 1 2; do
for v in new prev; do
  if [ $v = prev ]; then export BO_LIB=$L/libbo_cuda_prev.so; else unset BO_LIB; fi
  for n in 100000 1000000; do
    timeout 300 python bench.py --n $n --no-e2e --no-cpu --no-gmres --steps 30 > /tmp/b.json 2>/dev/null
    python -c "
import json;d=json.load(open('/tmp/b.json'));print('$v n=$n', round(d['ms_per_step'],4))"
  done
done
done
unset BO_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_full.py -m gpu -x -q 2>&1 | tail -1
