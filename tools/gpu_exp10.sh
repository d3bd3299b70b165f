#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_c2_gpu.py tests/test_kernels_gpu.py -q -x -rf -k "prefill_attention or metrics or attn" > gpurun_out/e10_k.log 2>&1; echo ktests rc $?; tail -2 gpurun_out/e10_k.log
timeout 900 python -m pytest tests/test_parity_replay_gpu.py -q -x -rf > gpurun_out/e10_r.log 2>&1; echo replay rc $?; tail -2 gpurun_out/e10_r.log
CONFIGS="c3;c5 --batch 256 --decode 128" bash tools/gpu_perf.sh
