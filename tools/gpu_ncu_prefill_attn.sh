#!/bin/bash
# ncu --set full of the tcgen05 prefill attention (k_attn_prefill_ws) at C3 layer 0 (4 x 3008
# tokens, unpruned) and C2 layer 0, plus the C3 bench line's prefill classes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-pa}
for spec in "c3:k_attn_prefill_ws:0" "c2:k_attn_prefill_ws:0"; do
  IFS=':' read -r cfg k s <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
    -o gpurun_out/${T}_ncu_${cfg}_attn_ws -f python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu-baseline \
    --decode 2 > gpurun_out/${T}_ncu_${cfg}.log 2>&1
  echo "ncu $cfg rc $?"
done
