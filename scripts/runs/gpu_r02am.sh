#!/bin/bash
# fused border-first tile launch (one launch per rank, flag raised mid-kernel) vs border / interior launches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multiprocess_gpu.py tests/test_gpu_fuzz.py tests/test_gpu_physics.py tests/test_gpu_devsetup.py -q -x -m gpu 2>&1 | tail -3
for F in 0 1; do for CFG in cfg4 cfg5; do
  echo "== CF_BORDER_FUSED=$F $CFG"
  CF_BORDER_FUSED=$F timeout 900 python scripts/inprocess_decomposition_fixture.py $CFG "1 2 8" 20 2>&1 | grep -v "^{" | cut -c1-330
done; done
