cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
for g in "" 1; do
echo "== MVSK_NO_CG_GRAPH=$g"
if [ -z "$g" ]; then unset MVSK_NO_CG_GRAPH; else export MVSK_NO_CG_GRAPH=1; fi
timeout 900 python scripts/solve_bench.py --configs C2,C3,C4 --cpu-max-n 0 --reps 3 2>&1 | cut -c1-160 | grep -v '"small"'
done
