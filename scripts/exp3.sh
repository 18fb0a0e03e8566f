#!/bin/bash
GEOMS=stored PROBES="0 1 3 4 6" bash scripts/ablate.sh
MODES=deterministic THREADS="128" STAGES="1" TILES="384" bash scripts/sweep.sh
