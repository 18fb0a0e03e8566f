#!/bin/bash
# round-2 closing evidence: GPU suite, smoke, driver-shaped bench + reference arm, ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/gputests_r02n.log 2>&1
echo "suite rc=$?"; tail -12 gpurun_out/gputests_r02n.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02n.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/smoke_r02n.log
bash scripts/profile_r02.sh r02n
cat gpurun_out/bench_r02n.json; cat gpurun_out/reference_r02n.json
