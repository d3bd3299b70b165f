for g in 1 2; do for sk in 0 1 2 4 8 14; do
  r=$(QT_GEMV=$g QT_SKIP=$sk timeout 120 python tests/dbg_perf.py 32 64 2 2>&1 | grep "decode ms" | tail -1)
  echo "gemv=$g skip=$sk $r"
done; done
