#!/bin/bash
# GPU tests + a quick 7B-shape timing of prefill / decode
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_quick.log
timeout 300 python tools/perf_probe.py 32 32 2 > gpurun_out/perf_quick.log 2>&1; echo perf rc $?; grep ms gpurun_out/perf_quick.log
if [ -n "$NCU_LAUNCH" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_quick.csv python tools/perf_probe.py 32 2 1 > /dev/null 2>&1; echo ncu rc $?
python tools/ncu_summary.py gpurun_out/launches_quick.csv | head -40
fi
