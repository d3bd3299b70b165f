#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_c2_gpu.py -q -x -rf -k "decode_attention" > gpurun_out/p_k2.log 2>&1; echo attn kernel tests rc $?; tail -3 gpurun_out/p_k2.log
timeout 900 python -m pytest tests/test_e2e_gpu.py tests/test_configs_gpu.py tests/test_parity_replay_gpu.py -q -x -rf -k "not 7b_width" > gpurun_out/p_e2e.log 2>&1; echo e2e rc $?; tail -3 gpurun_out/p_e2e.log
timeout 300 python tools/bench_gemm.py 2>&1 | tail -8
CONFIGS="c5 --batch 256 --decode 128;c4" bash tools/gpu_perf.sh
