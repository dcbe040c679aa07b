"""The reference-side adapter (integration/mvsk/gpu_oracle.hpp)
run against the reference's own Oracle and solve: examples/adapter_check links
the unmodified reference headers (compiled in the build container over the
oracle/ref Eigen stand-in) with libmvsk_b200.so and checks oracle values to
1e-11, RAII cache slots (several live caches, no aliasing, a ninth throws) and
both presets' solves to the north_star bar."""
import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_reference_side_adapter_drop_in():
    exe = ROOT / "examples" / "_bin" / "adapter_check"
    if not exe.exists():
        pytest.skip("adapter_check not built (needs the reference headers at build time)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["failures"] == 0 and out["oracle_rel"] <= 1e-11 and out["solve_dx"] <= 1e-8
