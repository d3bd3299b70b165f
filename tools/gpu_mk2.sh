cd $GRAFT_REPO_ROOT
for ns in 4 8; do
QT_MK_NSLOT=$ns QT_MK_TRACE=gpurun_out/mk$ns.trace QT_DECODE_MK=1 timeout 300 python tools/dbg_perf.py 32 4 1 > gpurun_out/mk_perf_ns$ns.log 2>&1; echo ns$ns rc $?
grep decode gpurun_out/mk_perf_ns$ns.log
python tools/mk_trace.py gpurun_out/mk$ns.trace 148 32 owners
done
