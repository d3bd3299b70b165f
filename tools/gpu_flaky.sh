cd $GRAFT_REPO_ROOT
f=0; for i in $(seq 1 8); do
  timeout 300 python -m pytest tests/test_configs_gpu.py tests/test_e2e_gpu.py -q -rf  > /tmp/fl.log 2>&1
  if grep -q failed /tmp/fl.log; then f=$((f+1)); grep -E "^FAILED|^E  " /tmp/fl.log | head -3 | cut -c1-300; fi
done; echo "configs+e2e fails=$f/8"
