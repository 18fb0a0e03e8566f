#!/bin/bash
# bench.py's N>1 code path on one GPU (host-staged transport), and the reference arm under torchrun
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --config cfg4 --transport host --compare-order none > gpurun_out/bench2_r02o.json 2> gpurun_out/bench2_r02o.err
echo "bench N=2 rc=$?"; cat gpurun_out/bench2_r02o.json | cut -c1-1500; tail -5 gpurun_out/bench2_r02o.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/ref2_r02o.json 2> gpurun_out/ref2_r02o.err
echo "reference N=2 rc=$?"; cut -c1-400 gpurun_out/ref2_r02o.json; tail -3 gpurun_out/ref2_r02o.err
