#!/bin/bash
# ncu capture of one Gaussian sketch build (mt_stream_kernel) at 8e6 x 22
mkdir -p gpurun_out/ncu_sketch
timeout 120 python scripts/prof_sketch.py 8000000 10 gaussian
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_stream_kernel -s 2 -c 1 \
  -o gpurun_out/ncu_sketch/mt python scripts/prof_sketch.py 8000000 10 gaussian > gpurun_out/ncu_sketch/log 2>&1; echo ncu rc=$?
