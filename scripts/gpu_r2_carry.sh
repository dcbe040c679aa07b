cd $GRAFT_REPO_ROOT
for v in "X=1" "MVSK_NO_SPG_CLUSTER=1" "MVSK_NO_SPG_CLUSTER=1 MVSK_SPG_GRAPH=1"; do
  echo "== $v"; env $v MVSK_PROFILE=1 python scripts/stress_repro.py 10,1,10,1 0,2 -1 large 2>&1 | grep -E "large|spg|mvsk" | cut -c1-400
done
