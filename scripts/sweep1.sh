#!/bin/bash
MODES=deterministic THREADS="128 256" STAGES="1 2" TILES="384" bash scripts/sweep.sh
MODES=deterministic THREADS="256" STAGES="2" TILES="512 768" bash scripts/sweep.sh
MODES=deterministic THREADS="256" STAGES="2" TILES="384" EXTRA="--geometry coords" bash scripts/sweep.sh
