#!/bin/bash
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r01m.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01m.log 2>&1; echo "smoke rc=$?"
MODES="atomic" THREADS=128 STAGES=1 TILES=384 bash scripts/sweep.sh
bash scripts/gpu_profile.sh r01m
