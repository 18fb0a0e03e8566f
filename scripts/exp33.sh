#!/bin/bash
python -m pytest tests/test_gpu_parity.py -x -q -k "multirank or schedule or stepping" 2>&1 | tail -2
RANKS="2 8" python scripts/inprocess_decomposition.py 256 50 2>&1 | grep -v "^{"
