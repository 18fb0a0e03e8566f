#!/bin/bash
# regs capped at 96 (CF_GS_MINB=5 build): tile sizes around the 5-CTA/SM shared-memory budget
MODES=deterministic THREADS="128" STAGES="1" TILES="256 288 320 336 352 384" bash scripts/sweep.sh
CF_TRACE_SETUP=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --tile 320 2>&1 | grep "class"
