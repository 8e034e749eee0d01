#!/bin/bash
# sketch build time (8e6 x 22 and 8e6 x 122) and the sketch parity tests
for r in 1 2; do
  echo "$(timeout 120 python scripts/prof_sketch.py 8000000 10 gaussian) | $(timeout 120 python scripts/prof_sketch.py 8000000 60 gaussian)"
done
timeout 900 python -m pytest tests -m gpu -x -q -k "sketch or gaussian or theta or kat or c5 or gmres_full" 2>&1 | tail -1
