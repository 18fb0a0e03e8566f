#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python scripts/multiproc_fixture.py 2 10 cfg4 > gpurun_out/mpf_cfg4_w2.json 2> gpurun_out/mpf_cfg4_w2.err
echo "w2 rc=$?"; cat gpurun_out/mpf_cfg4_w2.json; tail -3 gpurun_out/mpf_cfg4_w2.err
timeout 1200 python scripts/multiproc_fixture.py 4 10 cfg4 > gpurun_out/mpf_cfg4_w4.json 2> gpurun_out/mpf_cfg4_w4.err
echo "w4 rc=$?"; cat gpurun_out/mpf_cfg4_w4.json; tail -3 gpurun_out/mpf_cfg4_w4.err
RANKS="1 2 8" timeout 1200 python scripts/inprocess_decomposition.py 256 50 > gpurun_out/inproc_r02l.txt 2>&1
echo "inproc rc=$?"; tail -4 gpurun_out/inproc_r02l.txt
