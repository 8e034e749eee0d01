#!/bin/bash
# pre-solve update warp splits on the current engine
L=/root/repo/paper_2503_16717_b200
bash scripts/ab_passes.sh sweep_upd "def:X=1" "g1u:BO_LIB=$L/libbo_cuda_g1u.so" "nw9:BO_LIB=$L/libbo_cuda_nw9.so" "def2:X=1"
