#!/bin/bash
# round-2 closing evidence: GPU suite, smoke, driver-shaped bench + reference arm, ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/gputests_${TAG:-r02s}.log 2>&1
echo "suite rc=$?"; tail -12 gpurun_out/gputests_${TAG:-r02s}.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG:-r02s}.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/smoke_${TAG:-r02s}.log
bash scripts/profile_r02.sh ${TAG:-r02s}
cat gpurun_out/bench_${TAG:-r02s}.json; cat gpurun_out/reference_${TAG:-r02s}.json
