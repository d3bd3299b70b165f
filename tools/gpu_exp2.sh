#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -rf -k "single_splitk" > gpurun_out/e2_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/e2_tests.log
timeout 900 python tools/bench_decode_gemm.py 32,64,128,256 i8,i8a,i8k2,i8k3,i8k4,i8k6,i8k8 > gpurun_out/e2_dec.log 2>&1; echo dec rc $?; cat gpurun_out/e2_dec.log | tail -20
