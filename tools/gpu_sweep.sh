cd $GRAFT_REPO_ROOT
for sk in 0 1 2 4 8 14 15; do echo "SKIP=$sk $(QT_SKIP=$sk timeout 300 python tools/dbg_perf.py 32 32 2 2>&1 | grep "decode ms" | tail -1)"; done
