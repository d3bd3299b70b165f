#!/bin/bash
# decode-GEMM / GEMV / prefill-GEMM measurements + the kernel tests they touch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_c2_gpu.py tests/test_kernels_gpu.py -q -x -rf -k "row_block_major or epilogues or int8_operands" > gpurun_out/e1_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/e1_tests.log
timeout 300 python tools/bench_gemm.py > gpurun_out/e1_gemm.log 2>&1; echo gemm rc $?; cat gpurun_out/e1_gemm.log | tail -8
timeout 300 python tools/bench_gemv.py 8 > gpurun_out/e1_gemv.log 2>&1; echo gemv rc $?; cat gpurun_out/e1_gemv.log | tail -8
timeout 600 python tools/bench_decode_gemm.py 16,64,128,256 > gpurun_out/e1_dec.log 2>&1; echo dec rc $?; cat gpurun_out/e1_dec.log | tail -20
