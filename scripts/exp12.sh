#!/bin/bash
for f in 0 1; do echo "l2persist=$f"; CF_L2_PERSIST=$f MODES=deterministic THREADS=128 STAGES=1 TILES=384 bash scripts/sweep.sh; done
CF_TRACE_SETUP=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -i "persist"
