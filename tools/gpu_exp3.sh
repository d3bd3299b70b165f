#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_replay_gpu.py tests/test_configs_gpu.py tests/test_e2e_gpu.py -q -x -rf -k "not 7b_width_r0" > gpurun_out/e3_tests.log 2>&1; echo tests rc $?; tail -4 gpurun_out/e3_tests.log
CONFIGS="c5 --batch 64 --decode 512;c5 --batch 256 --decode 128" bash tools/gpu_perf.sh
