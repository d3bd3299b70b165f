#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_edges_gpu.py tests/test_kernels_c2_gpu.py tests/test_dropin_gpu.py -q -rf > gpurun_out/p_c3.log 2>&1; echo tests rc $?; tail -8 gpurun_out/p_c3.log
CONFIGS="c1" bash tools/gpu_perf.sh
bash tools/gpu_ncu_gemm.sh
