cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
echo "== full GPU suite with the default policy (device direct branch for m >= 48)"
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
echo "== solver suites with the device direct branch forced for every face"
MVSK_DEVICE_DIRECT=1 python -m pytest tests/test_gpu_solver.py tests/test_gpu_config_parity.py -m gpu -x -q 2>&1 | tail -3
for a in "C2 - small" "C1 - small"; do
  echo "== host LU path: $a"; MVSK_NO_DEVICE_DIRECT=1 MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "mvsk profile|^ok" | tail -2
  echo "== device direct forced: $a"; MVSK_DEVICE_DIRECT=1 MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "mvsk profile|^ok" | tail -2
  echo "== default policy: $a"; MVSK_PROFILE=1 python scripts/one_solve_prof.py $a 2>&1 | grep -E "mvsk profile|^ok" | tail -2
done
} > gpurun_out/r2c_devdirect.txt 2>&1
cat gpurun_out/r2c_devdirect.txt
