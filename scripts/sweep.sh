#!/bin/bash
# sweep tile-kernel launch shapes on cfg2: MODE THREADS STAGES TILES...
for m in $MODES; do for nt in $THREADS; do for st in $STAGES; do for t in $TILES; do
CF_TILE_THREADS=$nt CF_TILE_STAGES=$st python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --mode $m --tile $t $EXTRA 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$m nt=$nt st=$st', d['config']['tile_elems'], round(d['value']/1e9,2), 'G/s tile', r['kernel_ms'], 'upd', r['update_ms'], 'frac', r['frac'])" || echo "$m $nt $st $t FAILED"
done; done; done; done
