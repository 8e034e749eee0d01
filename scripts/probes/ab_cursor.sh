#!/bin/bash
L=/root/repo/paper_2503_16717_b200
bash scripts/ab_passes.sh ab_cur "new:X=1" "prev:BO_LIB=$L/libbo_cuda_prev.so"
bash scripts/ab_bench.sh ab_cur "new:X=1" "prev:BO_LIB=$L/libbo_cuda_prev.so"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
