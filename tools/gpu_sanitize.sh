cd $GRAFT_REPO_ROOT
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_configs_gpu.py -x -q -k "c5 or c3 or c4" > gpurun_out/memcheck.log 2>&1; echo memcheck rc $?
grep -E "ERROR SUMMARY|Invalid|of size|at 0x|by thread" gpurun_out/memcheck.log | head -20
f=0; for i in $(seq 1 12); do
  QT_TC05=0 timeout 300 python -m pytest tests/test_configs_gpu.py tests/test_e2e_gpu.py -q -rf > /tmp/fl.log 2>&1
  if grep -q failed /tmp/fl.log; then f=$((f+1)); grep -E "^FAILED" /tmp/fl.log | head -3; fi
done; echo "TC05=0 fails=$f/12"
