fails=0; for i in $(seq 1 $1); do
  out=$(timeout -s KILL 60 python -m pytest tests/test_e2e_gpu.py -q --timeout 60 -x -k "$2" 2>&1 | grep -E "passed|failed" | tail -1)
  case "$out" in *failed*) fails=$((fails+1));; esac
done; echo "$3 fails=$fails of $1"
