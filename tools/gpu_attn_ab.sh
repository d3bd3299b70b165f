#!/bin/bash
# decode-attention A/B: the bench's per-class decode chain for each build variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VARIANTS:-m2 m4 m8}; do
  for c in "c2" "c4" "c5 --batch 256 --decode 128"; do
    QT_LIB_PATH=$PWD/paper_2604_17320_b200/_build_var/$v/libquota_b200.so timeout 600 python bench.py --config $c \
      --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/ab.log 2>&1
    echo "$v | $c | rc $? | $(grep '"metric"' gpurun_out/ab.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); c=d['profile']['decode_chain_ms']
print('decode %.3f ms/step  chain attn %.3f full %.3f' % (d['decode_ms_per_step'], c['attention'], c['full']))")"
  done
done
