cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | grep -E "FAILED|passed|failed" | head -5
for v in 0 1; do echo "ROPEFUSED=$v $(QT_DEC_ROPE_FUSED=$v timeout 300 python tools/dbg_perf.py 32 32 2 2>&1 | grep "decode ms" | tail -1)"; done
