#!/bin/bash
# tile-kernel ablation on cfg2 (CF_PROBE modes; diagnostics only, results not valid)
for g in ${GEOMS:-stored coords}; do
  for pr in ${PROBES:-0 1 3 4 5 6}; do
    echo -n "$g probe=$pr "
    CF_PROBE=$pr python bench.py --steps 50 --geometry $g --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile', d['roofline']['kernel_ms'])"
  done
done
