#!/bin/bash
# device timeline of the C2 sequence at 1e5 rows (fixed per-call cost), fused and unfused finalize
timeout 300 python scripts/timeline.py --n 100000 --steps 2 --verbose > gpurun_out/tl_small_fused.txt 2>&1
BO_UNFUSE_FIN=1 timeout 300 python scripts/timeline.py --n 100000 --steps 2 --verbose > gpurun_out/tl_small_unfused.txt 2>&1
tail -3 gpurun_out/tl_small_fused.txt; tail -3 gpurun_out/tl_small_unfused.txt
