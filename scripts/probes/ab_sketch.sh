#!/bin/bash
# sketch build time, current vs previous library (BO_LIB), alternating
L=/root/repo/paper_2503_16717_b200
for r in 1 2; do
  for v in new prev; do
    if [ $v = prev ]; then export BO_LIB=$L/libbo_cuda_prev.so; else unset BO_LIB; fi
    echo "$v: $(timeout 120 python scripts/prof_sketch.py 8000000 10 gaussian) | $(timeout 120 python scripts/prof_sketch.py 8000000 60 gaussian)"
  done
done
unset BO_LIB
timeout 900 python -m pytest tests -m gpu -x -q -k "sketch or gaussian or theta or kat or c5 or gmres_full" 2>&1 | tail -1
