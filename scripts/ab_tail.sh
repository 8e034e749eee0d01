#!/bin/bash
# A/B of the round-2 pass-engine switches on one box (per-pass C2 timings and
# whole bench lines): DFMA tail columns (build tag notail: -DBO_DFMA_TAIL=0),
# decoupled rings (BO_DEC), product-factor solve (BO_PRE_PRODUCT), one solve
# warp for wide projections (BO_GAW1_MINP).
#   python -c "from paper_2503_16717_b200 import _build; _build.build_cuda(defines=['-DBO_DFMA_TAIL=0'], tag='notail')"
#   gpurun -- bash scripts/ab_tail.sh
L=/root/repo/paper_2503_16717_b200
V=("def:X=1" "nodec:BO_DEC=-1" "twosolve:BO_PRE_PRODUCT=0" "gaw2:BO_GAW1_MINP=0")
[ -f $L/libbo_cuda_notail.so ] && V+=("notail:BO_LIB=$L/libbo_cuda_notail.so")
bash scripts/ab_passes.sh ab_round2 "${V[@]}"
bash scripts/ab_bench.sh ab_round2 "${V[@]}"
