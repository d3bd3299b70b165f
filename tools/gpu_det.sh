cd $GRAFT_REPO_ROOT
for env in "QT_TC05=1" "QT_TC05=0" "QT_NOPDL=1"; do
  echo "== $env"; env $env timeout 300 python tools/dbg_det.py 2>&1 | tail -6
done
