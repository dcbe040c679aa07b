cd $GRAFT_REPO_ROOT
for v in "" 1; do
echo "== MVSK_NO_DIR_GRAPH=$v"
if [ -z "$v" ]; then unset MVSK_NO_DIR_GRAPH; else export MVSK_NO_DIR_GRAPH=1; fi
MVSK_PROFILE=1 timeout 900 python scripts/solve_bench.py --configs C3,C4 --cpu-max-n 0 --reps 1 2>&1 | grep -E "profile" | cut -c1-200 | awk 'NR%2==0'
done
