#!/bin/bash
# A/B of build variants (tools/build_attn_variants.sh): the bench's per-class decode chain per variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VARIANTS:-m2 m4 m8}; do
  IFS=';' read -ra CL <<< "${AB_CONFIGS:-c2;c4;c5 --batch 256 --decode 128}"
  for c in "${CL[@]}"; do
    QT_LIB_PATH=$PWD/paper_2604_17320_b200/_build_var/$v/libquota_b200.so timeout 600 python bench.py --config $c \
      --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/ab.log 2>&1
    echo "$v | $c | rc $? | $(grep '"metric"' gpurun_out/ab.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['profile']['decode_chain_ms']
print('prefill %.2f ms (attn %.2f)  decode %.3f ms/step  chain gemm %.3f attn %.3f full %.3f' % (d['prefill_ms'], d['profile']['prefill']['attention']['ms'], d['decode_ms_per_step'], c['gemm'], c['attention'], c['full']))")"
  done
done
