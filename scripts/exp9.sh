#!/bin/bash
MODES=deterministic THREADS=128 STAGES=1 TILES=384 bash scripts/sweep.sh
CF_TILE_PERSIST=1 MODES=deterministic THREADS=128 STAGES=1 TILES=384 bash scripts/sweep.sh
GEOMS=stored PROBES="0 16 17 19 20 24" bash scripts/ablate.sh
