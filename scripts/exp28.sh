#!/bin/bash
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r01n.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01n.log 2>&1; echo "smoke rc=$?"
bash scripts/gpu_profile.sh r01n
python bench.py --config cfg4 --steps 100 --no-cpu-baseline > gpurun_out/bench_r01n_cfg4.json 2> gpurun_out/bench_r01n_cfg4.err; echo "cfg4 rc=$?"
python bench.py --config cfg5 --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_r01n_cfg5.json 2> gpurun_out/bench_r01n_cfg5.err; echo "cfg5 rc=$?"
