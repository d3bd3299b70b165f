#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_kernels_c2_gpu.py tests/test_parity_replay_gpu.py tests/test_e2e_gpu.py -q -x -rf > gpurun_out/e7_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/e7_tests.log
CONFIGS="c3" bash tools/gpu_perf.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/e7_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --eager-decode > /dev/null 2>&1; echo "launch list rc $?"
python tools/ncu_summary.py gpurun_out/e7_launches.csv | head -16
