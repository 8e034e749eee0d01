#!/bin/bash
# quick 1-GPU measurement: per-pass live timings + the bench line
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python scripts/prof_passes.py > $OUT/passes.txt 2>&1; cat $OUT/passes.txt
timeout 600 python bench.py ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 4000 $OUT/bench.json; tail -5 $OUT/bench.err
