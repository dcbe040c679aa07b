cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2e_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/r2e_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r2e_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/r2e_bench_ref.log 2>&1; echo "ref rc $?"; tail -c 1500 gpurun_out/r2e_bench_ref.log
timeout 900 python bench.py > gpurun_out/r2e_bench.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/r2e_bench.log | cut -c1-1500
