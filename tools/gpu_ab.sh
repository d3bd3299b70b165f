#!/bin/bash
# A/B of an env switch on the 7B-shape decode/prefill timing: gpu_ab.sh VAR "v1 v2 ..."
cd $GRAFT_REPO_ROOT
VAR=${1:-QT_L2NEXT}; VALS=${2:-"0 1"}
for rep in 1 2; do for v in $VALS; do
  echo "$VAR=$v $(env $VAR=$v timeout 300 python tools/dbg_perf.py 32 32 2 2>&1 | grep "decode ms" | tail -1)"
done; done
