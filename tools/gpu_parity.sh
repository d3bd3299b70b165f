#!/bin/bash
# GPU parity pass: kernel-level 7B-shape tests, forced-replay e2e tests, then the whole GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
echo "nproc $(nproc)"; nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 1500 python -m pytest tests/test_kernels_c2_gpu.py -q -rf ${KFILTER:+-k "$KFILTER"} > gpurun_out/p_kern.log 2>&1; echo kern rc $?; tail -25 gpurun_out/p_kern.log
if [ "${REPLAY:-1}" = 1 ]; then
timeout 2400 python -m pytest tests/test_parity_replay_gpu.py -q -s -rf ${RFILTER:+-k "$RFILTER"} > gpurun_out/p_replay.log 2>&1; echo replay rc $?; grep -E "replay|dlogit|passed|failed|Error|assert" gpurun_out/p_replay.log | tail -40
fi
if [ "${ALL:-1}" = 1 ]; then
timeout 1800 python -m pytest tests -m gpu -q -rf --ignore=tests/test_kernels_c2_gpu.py --ignore=tests/test_parity_replay_gpu.py > gpurun_out/p_all.log 2>&1; echo all rc $?; tail -15 gpurun_out/p_all.log
fi
