#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --eager-decode > gpurun_out/dbg_ncu_list.log 2>&1; echo "ncu list rc $?"; python tools/ncu_summary.py gpurun_out/launches_c2.csv | head -40
