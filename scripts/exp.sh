#!/bin/bash
# quick experiment: parity tests + tile-size sweep (+ coords layout)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q 2>&1 | tail -3
MODES=deterministic THREADS="128" STAGES="1" TILES="${TILES:-384}" bash scripts/sweep.sh
MODES=deterministic THREADS="128" STAGES="1" TILES="384" EXTRA="--geometry coords" bash scripts/sweep.sh
