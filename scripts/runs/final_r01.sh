#!/bin/bash
# round-1 closing evidence: GPU suite, smoke, bench (driver defaults), reference arm, ncu, cfg4/cfg5
TAG=${1:-r01q}
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench_default_${TAG}.json 2> gpurun_out/bench_default_${TAG}.err; echo "bench default rc=$?"
STEPS=200 bash scripts/gpu_profile.sh ${TAG}
python bench.py --config cfg4 --steps 100 --no-cpu-baseline > gpurun_out/bench_${TAG}_cfg4.json 2> gpurun_out/bench_${TAG}_cfg4.err; echo "cfg4 rc=$?"
python bench.py --config cfg5 --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_cfg5.json 2> gpurun_out/bench_${TAG}_cfg5.err; echo "cfg5 rc=$?"
