cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_mk.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_mk.log
timeout 600 python tools/dbg_mk.py tiny > gpurun_out/mk_tiny.log 2>&1; echo tiny rc $?
grep prefill gpurun_out/mk_tiny.log
QT_DECODE_MK=1 timeout 300 python tools/dbg_perf.py 32 32 2 > gpurun_out/mk_perf1.log 2>&1; echo perf1 rc $?
QT_MK_TRACE=gpurun_out/mk.trace QT_DECODE_MK=1 timeout 300 python tools/dbg_perf.py 32 4 1 > gpurun_out/mk_perf_tr.log 2>&1; echo perftr rc $?
cat gpurun_out/mk_perf1.log
python tools/mk_trace.py gpurun_out/mk.trace 148 32 owners
if [ "${MKNCU:-0}" = 1 ]; then
QT_DECODE_MK=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_decode_mk -c 1 -o gpurun_out/ncu_mk -f python tools/dbg_perf.py 32 2 1 > gpurun_out/ncu_mk.log 2>&1; echo ncu rc $?
fi
