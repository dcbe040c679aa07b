cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/gram_pcg_check.py > gpurun_out/r2_gram_pcg_check2.txt 2>&1; echo "rc $?"
cat gpurun_out/r2_gram_pcg_check2.txt | cut -c1-400
MVSK_PROFILE=1 python scripts/one_solve_prof.py C4 2>&1 | grep -E "mvsk profile|^ok" | tail -2
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2_c4_solve_launches2.csv python scripts/one_solve_prof.py C4 > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/r2_c4_solve_launches2.csv | head -14
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r2f_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/r2f_pytest_gpu.log
