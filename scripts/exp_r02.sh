#!/bin/bash
# A/B of tile-kernel variants (built by `make OUT=../libcastfem_b200_<v>.so EXTRA_NVFLAGS=...`),
# cfg4 one GPU, tile node order (the kernels are node-order independent). Diagnostics only.
CFG=${CFG:-cfg4}
run() {  # name lib budget
    local out
    out=$(env CF_TRACE_SETUP=1 CF_LIB_PATH=paper_1005_3158_b200/$2 ${3:+CF_SMEM_BUDGET=$3} python bench.py --config $CFG \
        --node-order tile --compare-order none --no-cpu-baseline --no-e2e --steps ${STEPS:-60} --warmup 5 \
        --phase-steps 20 2> gpurun_out/exp_$1.err)
    echo "$1 $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]/1e9,3), "G/s tile", r["kernel_ms"], "upd", r["update_ms"], "frac", r["frac"], "step8", r["step_frac_of_8tbs"], "tiles", d["tiles"])') $(grep -o '[0-9]* CTAs/SM' gpurun_out/exp_$1.err | head -1)"
}
for v in ${VARIANTS:-base hoist pf both}; do
    lib=libcastfem_b200_$v.so; [ $v = base ] && lib=libcastfem_b200.so
    run $v $lib ""
done
for v in ${VARIANTS5:-base m5 m5x}; do
    [ "$v" = none ] && continue
    lib=libcastfem_b200_$v.so; [ $v = base ] && lib=libcastfem_b200.so
    run ${v}_b43 $lib 43700
done
