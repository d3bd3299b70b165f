#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -rf -k "int8_operands or int32_exact" > gpurun_out/p_gemm.log 2>&1; echo gemm tests rc $?; tail -5 gpurun_out/p_gemm.log
timeout 900 python -m pytest tests/test_e2e_gpu.py tests/test_configs_gpu.py tests/test_parity_replay_gpu.py -q -x -rf -k "not 7b_width_r0" > gpurun_out/p_e2e.log 2>&1; echo e2e rc $?; tail -5 gpurun_out/p_e2e.log
CONFIGS="c5 --batch 256 --decode 128" bash tools/gpu_perf.sh
