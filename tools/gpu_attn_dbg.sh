#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_kernels_c2_gpu.py -q -x -k "decode_attention" > gpurun_out/memcheck_attn.log 2>&1; echo memcheck attn rc $?
grep -E "ERROR SUMMARY|Invalid|out of bounds|at 0x|by thread|passed|failed" gpurun_out/memcheck_attn.log | head -12
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_e2e_gpu.py -q -x -k "r1_dynamic" > gpurun_out/memcheck_e2e.log 2>&1; echo memcheck e2e rc $?
grep -E "ERROR SUMMARY|Invalid|out of bounds|at 0x|by thread|passed|failed" gpurun_out/memcheck_e2e.log | head -12
for spec in "c2:k_attn_dec:40" "c4:k_attn_dec:40" "c2:k_norm_quant4:40" "c2:k_gemv_reg:40"; do
  cfg=${spec%%:*}; rest=${spec#*:}; k=${rest%%:*}; s=${rest##*:}
  tag=$(echo "$cfg" | tr -d ' -' | cut -c1-12)_$k
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c 1 \
    -o gpurun_out/ncu_$tag -f python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc $?"
done
