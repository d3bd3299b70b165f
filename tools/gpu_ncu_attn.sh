#!/bin/bash
# ncu --set full of the decode attention + merge kernels at C2 (B = 8) and C5 (B = 256), and the
# C2 launch list (per-kernel durations, serialized).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for spec in "c2:k_attn_dec_w:40" "c2:k_attn_merge_quant:40" "c5 --batch 256 --decode 8:k_attn_dec_w:40"; do
  cfg=${spec%%:*}; rest=${spec#*:}; k=${rest%%:*}; s=${rest##*:}
  tag=$(echo "$cfg" | tr -d ' -' | cut -c1-12)_$k
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
    -o gpurun_out/ncu_$tag -f python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc $?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1; echo launches rc $?
python tools/ncu_summary.py gpurun_out/launches_c2.csv | head -30
