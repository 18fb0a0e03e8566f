#!/bin/bash
# fused border-first tile launch, packs interleaved per rank: in-process decomposition timing, fused on / off
mkdir -p gpurun_out
for CFG in cfg4 cfg5; do for F in 0 1; do
  echo "== CF_BORDER_FUSED=$F $CFG"
  CF_BORDER_FUSED=$F timeout 900 python scripts/inprocess_decomposition_fixture.py $CFG "1 2 8" 20 2>&1 | grep -v "^{" | cut -c1-140
done; done
