#!/bin/bash
for rep in 1 2; do
for p in 1 0; do echo "persist=$p"; CF_TILE_PERSIST=$p MODES=deterministic THREADS=128 STAGES=1 TILES=384 bash scripts/sweep.sh; done
done
