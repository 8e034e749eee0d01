#!/bin/bash
# One gpurun call: GPU parity suite, smoke, 1-GPU bench, ncu launch list and a
# full ncu capture of the top pass.  Outputs land in gpurun_out/.
#   gpurun --timeout 2400 -- bash scripts/gpu_round.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
(timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log)
tail -3 $OUT/pytest_gpu.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log)
tail -2 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -c 3000 $OUT/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "step/" \
   --csv --log-file $OUT/launches.csv python bench.py --profile-only > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "last/" \
   -o $OUT/prof_last python bench.py --profile-only > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la $OUT
