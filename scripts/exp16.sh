#!/bin/bash
MODES=deterministic THREADS=128 STAGES=1 TILES="320 336 352 384" bash scripts/sweep.sh
for t in 336 352; do CF_TRACE_SETUP=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --tile $t 2>&1 | grep "class"; done
