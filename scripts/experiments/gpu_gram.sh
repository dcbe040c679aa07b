cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_oracle.py -m gpu -q -p no:cacheprovider -k "gram or nccl" 2>&1 | tail -2
python - <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
from paper_2604_25378_b200.datagen import CONFIGS, crra, random_simplex_point, raw_returns
from paper_2604_25378_b200.gpu_oracle import GpuOracle
spec = CONFIGS["C5"]; dev = torch.device("cuda", 0)
X = raw_returns(spec, 5000, device=dev); mu = X.sum(0) / spec.T; X.sub_(mu)
T, n = spec.T, spec.n
g = GpuOracle(None, mu.cpu().numpy(), crra(10.0), device_panel=(X.data_ptr(), n, T, n))
xd = torch.from_numpy(random_simplex_point(n, 7)).to(dev)
g.make_cache_device(0, xd.data_ptr())
G = torch.empty((n, n), dtype=torch.float64, device=dev)
g.weighted_gram_device(0, G.data_ptr()); g.synchronize()
t0 = time.perf_counter(); g.weighted_gram_device(0, G.data_ptr()); g.synchronize(); dt = time.perf_counter() - t0
print("gram %.1f ms  %.2f TFLOP/s" % (dt * 1e3, T * n * (n + 1) / dt / 1e12))
PY
