#!/bin/bash
# compute-sanitizer over scripts/sanitize_case.py (racecheck, synccheck, memcheck on
# the small configs). Usage on the GPU box: bash scripts/sanitize.sh > gpurun_out/sanitize.log 2>&1
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck initcheck; do
    echo "=== $tool"
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py 2>&1 | tail -25
done
