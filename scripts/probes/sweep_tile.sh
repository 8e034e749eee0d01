#!/bin/bash
# narrow pre-solve passes on 256-row tiles with decoupled rings (BO_T256_MAXP)
bash scripts/ab_passes.sh sweep_tile2 "def:X=1" "off:BO_T256_MAXP=-1" "def2:X=1"
bash scripts/ab_bench.sh sweep_tile2 "def:X=1" "off:BO_T256_MAXP=-1"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
