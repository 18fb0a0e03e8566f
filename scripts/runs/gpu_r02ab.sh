#!/bin/bash
# Peer-memory transport vs host-staged transport: bench.py's N>1 path, every rank process on the one GPU
mkdir -p gpurun_out
port=29520
for N in 2 4; do
  for TR in host peer-1gpu; do
    port=$((port+1))
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port \
      bench.py --gpus $N --steps 20 --warmup 5 --config cfg4 --transport $TR --compare-order none --no-cpu-baseline \
      > gpurun_out/r02ab_bench_n${N}_${TR}_cfg4.json 2> gpurun_out/r02ab_bench_n${N}_${TR}.err
    echo "N=$N $TR rc=$?"; python - <<PY
import json
try:
    d = json.load(open("gpurun_out/r02ab_bench_n${N}_${TR}_cfg4.json"))
    print({k: d.get(k) for k in ("value", "ms_per_step", "n_gpus")}, d["config"].get("transport"), d["roofline"].get("pack_ms"), d["roofline"].get("exchange_ms"), d.get("e2e", {}).get("value"))
except Exception as e:
    print("no line:", e)
PY
    tail -3 gpurun_out/r02ab_bench_n${N}_${TR}.err
  done
done
