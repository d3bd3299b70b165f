#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_c2_gpu.py -q -x -rf -k "decode_attention" > gpurun_out/e4_k.log 2>&1; echo ktests rc $?; tail -3 gpurun_out/e4_k.log
timeout 1200 python -m pytest tests/test_parity_replay_gpu.py tests/test_configs_gpu.py tests/test_e2e_gpu.py tests/test_edges_gpu.py -q -x -rf -k "not 7b_width_r0" > gpurun_out/e4_tests.log 2>&1; echo tests rc $?; tail -4 gpurun_out/e4_tests.log
CONFIGS="c4;c5 --batch 256 --decode 128;c5 --batch 64 --decode 512" bash tools/gpu_perf.sh
