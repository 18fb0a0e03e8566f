#!/bin/bash
# cfg2 tile-kernel sweep over library builds (CF_LIB_PATH) x tile sizes x geometry layouts
line() { python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; c=d['config']; print(c['geometry'], c['tile_elems'], round(d['value']/1e9,2), 'G/s step', round(d['ms_per_step'],4), 'tile', r['kernel_ms'], 'upd', r['update_ms'])"; }
for lib in ${LIBS:-paper_1005_3158_b200/libcastfem_b200.so}; do
  for te in ${TILES:-384}; do
    for g in ${GEOMS:-coords}; do
      echo -n "$lib $TT "
      CF_LIB_PATH=$lib python bench.py --steps ${STEPS:-100} --tile $te --geometry $g --no-cpu-baseline --no-e2e 2>/dev/null | line
    done
  done
done
