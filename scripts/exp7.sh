#!/bin/bash
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for it in 0 8; do echo "iters $it"; CF_BANK_ITERS=$it MODES=deterministic THREADS=128 STAGES=1 TILES=384 bash scripts/sweep.sh; done
