#!/bin/bash
# narrow pre-solve projection: 4 vs 5 contraction warps
bash scripts/ab_passes.sh sweep_gw "gw4:X=1" "gw5:BO_QTX_GW_SMALLP=0" "gw3:BO_QTX_GW_SMALLP=3" "gw4b:X=1"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2_full.py -m gpu -x -q 2>&1 | tail -1
