#!/bin/bash
# ncu --set full of one plane-marching 7-point SpMV at n = 8e6
mkdir -p gpurun_out/ncu_spmv
timeout 120 python scripts/prof_spmv.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_stencil7_march -s 20 -c 1 \
  -o gpurun_out/ncu_spmv/spmv python scripts/prof_spmv.py > gpurun_out/ncu_spmv/log 2>&1; echo ncu rc=$?
