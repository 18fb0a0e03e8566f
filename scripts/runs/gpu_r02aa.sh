#!/bin/bash
# Re-entry validation: full GPU suite, smoke, both bench arms on the restored tree.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02aa_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02aa_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02aa_reference_cfg5.json 2> gpurun_out/r02aa_reference.err; tail -c 600 gpurun_out/r02aa_reference_cfg5.json
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02aa_bench_cfg5.json 2> gpurun_out/r02aa_bench.err; tail -c 3000 gpurun_out/r02aa_bench_cfg5.json
