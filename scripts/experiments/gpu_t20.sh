cd $GRAFT_REPO_ROOT
for g in "" 1; do
echo "== MVSK_NO_CG_GRAPH=$g"
if [ -z "$g" ]; then unset MVSK_NO_CG_GRAPH; else export MVSK_NO_CG_GRAPH=1; fi
MVSK_PROFILE=1 timeout 900 python scripts/solve_bench.py --configs C3,C4 --cpu-max-n 0 --reps 1 2>&1 | grep -E "profile|config" | sed -n '2p;3p;5p;6p;8p;9p' | cut -c1-330
done
