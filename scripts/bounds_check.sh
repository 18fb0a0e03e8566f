#!/bin/bash
# The GPU parity / edge / device-setup / multi-process suites against the bounds-asserting build
# (make BOUNDS=1 -> libcastfem_b200_bounds.so: every plan-derived shared-memory index and global
# index of the step kernels checked, __trap on violation). compute-sanitizer is closed on this
# pool; this is its substitute for our own kernels.
cd "$(dirname "$0")/.."
make -s -j8 -C paper_1005_3158_b200/csrc OBJDIR=../../build/obj_bounds OUT=../libcastfem_b200_bounds.so BOUNDS=1
CF_LIB_PATH=paper_1005_3158_b200/libcastfem_b200_bounds.so timeout 1500 python -m pytest \
    tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_devsetup.py tests/test_multiprocess_gpu.py \
    tests/test_gpu_physics.py tests/test_gpu_rcm.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -4
