#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -rf -k "int8_operands or epilogues or single_splitk or int32_exact" > gpurun_out/e5_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/e5_tests.log
timeout 300 python tools/bench_gemm.py > gpurun_out/e5_gemm.log 2>&1; echo gemm rc $?; cat gpurun_out/e5_gemm.log | tail -8
CONFIGS="c3" bash tools/gpu_perf.sh
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_gemv_reg<1, 0, 1>" -s 3 -c 1 \
    -o gpurun_out/r02_ncu_gemv_qkv -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --eager-decode > gpurun_out/r02_ncu_gemv_qkv.log 2>&1; echo "ncu gemv qkv rc $?"
