#!/bin/bash
# Round verification on one B200: full GPU suite, smoke, the default bench line (C2 with the CPU
# leg), the other config lines, the eager ncu launch list, and ncu --set full captures of the
# top kernels.  Outputs under gpurun_out/ with the prefix $TAG (default r02).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv,noheader
if [ -z "$SKIP_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/${T}_smoke.log
fi
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc $?"; grep '"metric"' gpurun_out/${T}_bench.json | python tools/bench_brief.py
rm -f gpurun_out/${T}_bench_configs.jsonl
IFS=';' read -ra CL <<< "${CONFIGS:-c1;c3;c4;c5 --batch 1 --decode 128;c5 --batch 16 --decode 512;c5 --batch 64 --decode 512;c5 --batch 256 --decode 128}"
for c in "${CL[@]}"; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg.log 2>&1
  echo "== $c rc $?"; grep '"metric"' gpurun_out/bench_cfg.log | python tools/bench_brief.py
  grep '"metric"' gpurun_out/bench_cfg.log >> gpurun_out/${T}_bench_configs.jsonl
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${T}_launches_c2.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --eager-decode > /dev/null 2>&1; echo "launch list rc $?"
python tools/ncu_summary.py gpurun_out/${T}_launches_c2.csv > gpurun_out/${T}_launch_summary.txt; head -40 gpurun_out/${T}_launch_summary.txt
for spec in "c2:k_gemv_reg:65:gemv" "c2:k_attn_dec_w:40:attn_dec" "c2:k_gemm_tc05_i8:2:gemm_i8" "c2:k_attn_prefill_ws:3:attn_prefill" "c2:k_norm_quant4:70:norm_quant4" "c2:k_attn_merge_quant:40:attn_merge" "c5 --batch 256 --decode 8:k_attn_dec_w:40:attn_dec_b256"; do
  IFS=':' read -r cfg k s name <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
    -o gpurun_out/${T}_ncu_$name -f python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu-baseline --eager-decode > gpurun_out/${T}_ncu_$name.log 2>&1
  echo "ncu $name rc $?"
done
