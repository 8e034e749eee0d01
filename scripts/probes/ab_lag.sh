#!/bin/bash
# lagged stage release in storing passes vs waiting for the store reads per tile
L=/root/repo/paper_2503_16717_b200
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
bash scripts/ab_passes.sh ab_lag "lag:X=1" "nolag:BO_LIB=$L/libbo_cuda_nolag.so"
bash scripts/ab_bench.sh ab_lag "lag:X=1" "nolag:BO_LIB=$L/libbo_cuda_nolag.so"
