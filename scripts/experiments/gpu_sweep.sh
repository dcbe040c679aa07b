cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solver.py -q -p no:cacheprovider -k floor_sweep > gpurun_out/sweep_test.log 2>&1; echo "rc $?" >> gpurun_out/sweep_test.log
tail -15 gpurun_out/sweep_test.log
cat > /tmp/sw.py <<'PY'
import time, json, sys
sys.path.insert(0, ".")
from paper_2604_25378_b200.datagen import make_panel
from paper_2604_25378_b200.gpu_oracle import GpuOracle, preset
A, mu, c = make_panel("C4", seed=11)
g = GpuOracle(A, mu, c)
cfg = preset("large"); cfg.has_max_elapsed = 0
g.solve(cfg)
for ws in (True, False):
    t0 = time.perf_counter()
    sw = g.floor_sweep(cfg, nfloors=5, warm_start=ws)
    print(json.dumps({"warm": ws, "wall_s": time.perf_counter() - t0, "solves": sw.total_solves, "m_mv": sw.m_mv, "m_max": sw.m_max, "points": sw.points}))
PY
timeout 900 python /tmp/sw.py > gpurun_out/sweep_c4.log 2>&1; echo "rc $?" >> gpurun_out/sweep_c4.log
cat gpurun_out/sweep_c4.log
