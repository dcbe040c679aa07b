cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
for rep in 1 2; do
  echo "== swizzled rows (default build)"; python scripts/dmma_ab.py C5 hvp8,hvp4,third4,third8 ws
  echo "== uniform stride (MVSK_WS_SWZ=0 build)"; MVSK_B200_LIB=$GRAFT_REPO_ROOT/paper_2604_25378_b200/_build_ab/libmvsk_b200.so python scripts/dmma_ab.py C5 hvp8,hvp4,third4,third8 ws
done
echo "== C3/C4 (small panels) swizzled"; python scripts/dmma_ab.py C4 hvp8,hvp4,third4,third8 ws; python scripts/dmma_ab.py C3 hvp8,third8 ws
echo "== C3/C4 uniform"; MVSK_B200_LIB=$GRAFT_REPO_ROOT/paper_2604_25378_b200/_build_ab/libmvsk_b200.so python scripts/dmma_ab.py C4 hvp8,hvp4,third4,third8 ws; MVSK_B200_LIB=$GRAFT_REPO_ROOT/paper_2604_25378_b200/_build_ab/libmvsk_b200.so python scripts/dmma_ab.py C3 hvp8,third8 ws
} > gpurun_out/r2c_swz_ab.txt 2>&1
cat gpurun_out/r2c_swz_ab.txt
python -m pytest tests/test_gpu_oracle.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -3
bash scripts/gpu_r2_prof_solves.sh
