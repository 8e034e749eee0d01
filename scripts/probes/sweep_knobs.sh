#!/bin/bash
# end-of-round sweep of the pass-engine policy knobs
bash scripts/ab_passes.sh sweep_knobs "def:X=1" "vla2:BO_VLA=2" "gaw34:BO_GAW1_MINP=34" "dec3:BO_DEC=1" "def2:X=1"
