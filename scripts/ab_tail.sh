#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "orth|passed|failed|FAIL" | tail -40
