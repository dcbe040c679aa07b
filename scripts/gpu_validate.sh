# Round validation on one B200: the GPU test suite, smoke(), both bench arms, then the ncu launch list of the
# same bench command (a number printed under ncu is never a bench value):
#   gpurun --timeout 2400 -- 'bash scripts/gpu_validate.sh <tag>'
cd $GRAFT_REPO_ROOT
tag=${1:-val}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${tag}_pytest_gpu.log
python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -1
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc $?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err; echo "reference arm rc $?"
# -k keeps this library's kernels (the panel generator's torch kernels would fill the list)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(stream_|syrk_|finish_|gram_|small_|quadform|spg_|cg_|cluster_cg|face_|psi2|group_sum|colsum|lift|rhs_kernel|accum_|jacobi_|third_w|unit_probe|center_|padding_)' -c 600 --csv --log-file gpurun_out/${tag}_bench_launches.csv \
  python bench.py --steps 2 --warmup 1 > gpurun_out/${tag}_bench_under_ncu.log 2>&1; echo "ncu launch list rc $?"
python scripts/launch_agg.py gpurun_out/${tag}_bench_launches.csv 12
head -c 1500 gpurun_out/${tag}_bench.json
