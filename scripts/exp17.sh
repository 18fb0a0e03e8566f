#!/bin/bash
for rep in 1 2; do MODES=deterministic THREADS=128 STAGES=1 TILES=384 bash scripts/sweep.sh; done
python scripts/reorder_study.py > gpurun_out/cfg3_reorder_r01l.log 2>&1; echo "reorder rc=$?"
