cd $GRAFT_REPO_ROOT
f=0; for i in $(seq 1 12); do
  timeout 300 python -m pytest tests/test_e2e_gpu.py -q -x > /tmp/fl.log 2>&1
  if grep -q failed /tmp/fl.log; then f=$((f+1)); grep -E "^E " /tmp/fl.log | head -8; fi
done; echo "fails=$f/12"
