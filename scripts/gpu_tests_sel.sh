#!/bin/bash
# selected GPU tests (-s, verbose prints) plus extra commands: bash scripts/gpu_tests_sel.sh TAG "pytest args" ["extra cmd"]
TAG=${1:-sel}
OUT=gpurun_out/$TAG
mkdir -p $OUT
(eval "timeout 2400 python -m pytest -s -q $2" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log)
tail -40 $OUT/pytest.log
if [ -n "$3" ]; then (timeout 1200 bash -c "$3" > $OUT/extra.log 2>&1; echo "extra rc=$?" >> $OUT/extra.log); cat $OUT/extra.log | tail -40; fi
