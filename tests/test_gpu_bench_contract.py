"""bench.py's JSON line keeps the driver's contract (keys, roofline / e2e /
clocks objects, launches counted) -- run on the small config C1 so it takes
seconds (the default C3 line is produced the same way)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_contract_c1():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "3",
                          "--warmup", "3", "--no-mixed"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["data"] == "synthetic"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and "sample" in c
    assert abs(c["solve"]["iterations"] - d["run"]["iterations_per_solve"]) <= 1   # same algorithm (Z24: +-1)
    # the reference arm names the same workload with the same config object
    ref = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert ref.returncode == 0, ref.stderr[-3000:]
    rl = [ln for ln in ref.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(rl) == 1
    rd = json.loads(rl[0])
    assert rd["impl"] == "reference" and rd["config"] == d["config"]
    assert rd["metric"] == d["metric"] and rd["unit"] == d["unit"] and rd["scaling"] == d["scaling"]
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
