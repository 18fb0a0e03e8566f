#!/bin/bash
# final confirmation on the closing tree (after the fused-border option, batched flag waits, new acceptance tests): GPU suite, smoke, both bench arms (driver-shaped)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02at_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02at_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02at_reference_cfg5.json 2> gpurun_out/r02at_reference.err; echo "ref rc=$?"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02at_bench_cfg5.json 2> gpurun_out/r02at_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.load(open("gpurun_out/r02at_bench_cfg5.json")); r=d["roofline"]
print(round(d["value"]/1e9,2),"G/s; tile frac",r["frac"],"step8",r["step_frac_of_8tbs"],"e2e",round(d["e2e"]["value"]/1e9,2),d["clocks"])
d=json.load(open("gpurun_out/r02at_reference_cfg5.json")); print("ref",d["value"]/1e6,"replicas",d["reference_replicas"]["cores"],d["reference_replicas"]["value"]/1e6)
PY
