#!/bin/bash
MODES=deterministic THREADS=128 STAGES=1 TILES=384 bash scripts/sweep.sh
MODES=deterministic THREADS=64 STAGES=1 TILES="192 256" bash scripts/sweep.sh
MODES=deterministic THREADS=96 STAGES=1 TILES="288 384" bash scripts/sweep.sh
for nt_t in "64 192" "96 288"; do set -- $nt_t; CF_TILE_THREADS=$1 CF_TRACE_SETUP=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --tile $2 2>&1 | grep "class"; done
