"""bench.py contract on CPU: the reference arm (--impl reference) runs the
reference's own code (oracle/_ref; the restatement where that is absent) on the
SAME workload as the GPU arm and prints one JSON line with the keys the driver
consumes; `--gpus N` from a plain process relaunches itself under
torch.distributed.run with N ranks (checked with --dry-run, gloo, no GPU)."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "C3",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    from oracle import pyoracle as po
    assert line["cpu_baseline"]["kind"] == ("reference" if po.available("reference_native") else "port")
    assert line["cpu_baseline"]["cores"] >= 1
    assert "workload" in line["config"] and line["config"]["same_config"] is True
    assert line["config"]["T"] == 2500 and line["config"]["n"] == 800  # the full C3 panel, not a sample


def test_gpus_flag_launches_that_many_ranks():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], capture_output=True,
                         text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["dry_run"] is True and line["n_gpus"] == 2 and line["ranks_seen"] == [0, 1]
