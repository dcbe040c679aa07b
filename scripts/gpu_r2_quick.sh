cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_r2_prof_solves.sh 2>&1 | grep -v "total [0-9][0-9]\."
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/r2q_pytest.log
