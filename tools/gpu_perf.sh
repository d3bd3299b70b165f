#!/bin/bash
# Bench lines: C2 (the driver's default), then the other config families (no CPU leg).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 ${C2ARGS:---no-cpu-baseline} > gpurun_out/bench_c2.log 2>&1; echo c2 rc $?
grep '"metric"' gpurun_out/bench_c2.log | python tools/bench_brief.py
if [ -n "$CONFIGS" ]; then IFS=';' read -ra CL <<< "$CONFIGS"; else CL=("c4" "c5 --batch 256 --decode 128" "c5 --batch 64 --decode 512" "c3"); fi
for c in "${CL[@]}"; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg.log 2>&1
  echo "== $c rc $?"; grep '"metric"' gpurun_out/bench_cfg.log | python tools/bench_brief.py
  grep '"metric"' gpurun_out/bench_cfg.log >> gpurun_out/bench_configs.jsonl
done
