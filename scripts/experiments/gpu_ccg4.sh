cd $GRAFT_REPO_ROOT
for v in 0 1; do
  if [ $v = 1 ]; then export MVSK_NO_CCG=1; else unset MVSK_NO_CCG; fi
  echo "== MVSK_NO_CCG=$v"
  MVSK_PROFILE=1 timeout 300 python scripts/solve_bench.py --configs C3,C4 --cpu-max-n 0 --reps 1 2>&1 | grep -E "profile" | cut -c1-150
done
unset MVSK_NO_CCG
bash scripts/gpu_c4_launches.sh > /dev/null 2>&1
