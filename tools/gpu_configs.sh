#!/bin/bash
# bench lines for the other BASELINE.json config families (documentation; the driver runs c2)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_cfg.log 2>&1; echo pytest rc $?; tail -2 gpurun_out/pytest_cfg.log
for c in "c3" "c4" "c5" "c5 --batch 256 --decode 128" "c5 --batch 1 --decode 128" "c1"; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg.log 2>&1
  echo "== $c rc $?"; grep '"metric"' gpurun_out/bench_cfg.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(json.dumps({k:d[k] for k in ['value','ms_per_step','prefill_ms','decode_ms_per_step','prefill_tokens_per_s','decode_tokens_per_s','config']}))"
  grep '"metric"' gpurun_out/bench_cfg.log >> gpurun_out/bench_configs.jsonl
done
