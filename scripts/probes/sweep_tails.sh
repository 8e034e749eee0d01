#!/bin/bash
# DFMA tails in the pre-solve update / Gram on the current engine
L=/root/repo/paper_2503_16717_b200
bash scripts/ab_passes.sh sweep_tails "def:X=1" "tg:BO_LIB=$L/libbo_cuda_tg.so" "tu:BO_LIB=$L/libbo_cuda_tu.so" "tug:BO_LIB=$L/libbo_cuda_tug.so" "def2:X=1"
