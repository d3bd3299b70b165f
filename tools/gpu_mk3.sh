cd $GRAFT_REPO_ROOT
QT_MK_TRACE=gpurun_out/mk.trace QT_DECODE_MK=1 timeout 300 python tools/dbg_perf.py 32 4 1 > gpurun_out/mk_perf_tr.log 2>&1; echo perftr rc $?
grep decode gpurun_out/mk_perf_tr.log
python tools/mk_trace.py gpurun_out/mk.trace 148 32 owners
