#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_gemm_tc05_i8$' -c 4 \
  -o gpurun_out/ncu_gemm_shapes -f python tools/ncu_gemm_shapes.py > gpurun_out/ncu_gemm.log 2>&1; echo ncu gemm rc $?
