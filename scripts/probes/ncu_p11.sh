#!/bin/bash
# ncu --set full of the p = 11 bcgs2 call of one C2 step
mkdir -p gpurun_out/ncu_p11
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "p11/" \
   -o gpurun_out/ncu_p11/prof python bench.py --profile-only > gpurun_out/ncu_p11/log 2>&1; echo ncu rc=$?
