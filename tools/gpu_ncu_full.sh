#!/bin/bash
# ncu --set full captures of the top kernels of the bench workload (one launch each).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_select_gpu.py -x -q > gpurun_out/pytest_select.log 2>&1; echo select rc $?
for spec in "k_gemv_reg:40" "k_gemm_tc05_i8:10" "k_attn_decode:5" "k_attn_prefill:3" "k_quant_pmax:40"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
    -o gpurun_out/ncu_$k -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc $?"
done
