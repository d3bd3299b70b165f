cd $GRAFT_REPO_ROOT
# decode step with kernel classes removed (QT_SKIP bits: 1 GEMM, 2 attention, 4 quant, 8 kv)
for sk in 0 15 14 13 11 7; do echo "SKIP=$sk $(QT_SKIP=$sk timeout 300 python tools/dbg_perf.py 32 32 2 2>&1 | grep "decode ms" | tail -1)"; done
