cd $GRAFT_REPO_ROOT
for v in 0 8 16 32 64; do echo "PRE=$v $(QT_GEMV_PRE=$v timeout 300 python tools/dbg_perf.py 32 32 2 2>&1 | grep "decode ms" | tail -1)"; done
