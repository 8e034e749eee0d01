#!/bin/bash
bash scripts/ab_passes.sh ab_gaw2 "def:X=1" "nogaw1:BO_GAW1_MINP=0" "def2:X=1"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash scripts/ab_bench.sh ab_gaw2 "def:X=1" "nogaw1:BO_GAW1_MINP=0"
