cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
bash scripts/gpu_tests.sh
cp gpurun_out/pytest_gpu.log gpurun_out/r2a_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r2a_smoke.log
timeout 900 python bench.py > gpurun_out/r2a_bench.log 2>&1; echo "bench rc $?"; tail -c 600 gpurun_out/r2a_bench.log
