cd $GRAFT_REPO_ROOT
for env in "X=1" "QT_NOPDL=1" "QT_NOGRAPH=1"; do echo "== $env"; env $env timeout 600 python tools/dbg_det2.py 25 2>&1 | tail -4; done
