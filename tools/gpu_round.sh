#!/bin/bash
# One GPU-box pass: smoke, GPU parity tests, the bench line, and the ncu launch
# list of the same bench command (outputs under gpurun_out/, merged back).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc $?
if [ "${NCU:-1}" = 1 ]; then
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/ncu_launch.log 2>&1; echo ncu rc $?
fi
tail -3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log; tail -c 3000 gpurun_out/bench.log
