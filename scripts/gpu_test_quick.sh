#!/bin/bash
# GPU parity suite + per-pass timings + bench line
TAG=${1:-tq}
OUT=gpurun_out/$TAG
mkdir -p $OUT
(timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log)
tail -15 $OUT/pytest_gpu.log
bash scripts/gpu_quick.sh $TAG
