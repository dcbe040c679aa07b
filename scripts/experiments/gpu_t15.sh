cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for nf in "" 1; do
echo "== MVSK_NO_FUSED_FINISH=$nf"
export MVSK_NO_FUSED_FINISH=$nf
[ -z "$nf" ] && unset MVSK_NO_FUSED_FINISH
TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C5 hvp1,third 2>&1 | grep default
TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C4 hvp1,fgrad 2>&1 | grep default
TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C3 hvp1,fgrad 2>&1 | grep default
TUNE_DEFAULT_ONLY=1 timeout 300 python scripts/tune_stream.py C2 hvp1,fgrad 2>&1 | grep default
timeout 900 python scripts/solve_bench.py --configs C1,C3,C4 --cpu-max-n 0 --reps 3 2>&1 | cut -c1-120
done
