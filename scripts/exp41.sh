#!/bin/bash
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -k "not cfg4 and not autotune" 2>&1 | tail -2
for r in 1 2; do MODES=deterministic THREADS=128 STAGES=1 TILES=384 bash scripts/sweep.sh; CF_SLOT_BANKS=0 MODES=deterministic THREADS=128 STAGES=1 TILES=384 bash scripts/sweep.sh; done
