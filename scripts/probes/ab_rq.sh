#!/bin/bash
L=/root/repo/paper_2503_16717_b200
bash scripts/ab_passes.sh ab_rq2 "rq2:X=1" "rq4:BO_LIB=$L/libbo_cuda_rq4.so"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
