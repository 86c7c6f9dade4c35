"""bench.py's reference arm (CPU-only: the oracle port on the host cores) prints
one JSON line with the driver contract's keys (the GPU arm is exercised by the
round-end bench on the B200)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "1", "--shape", "ml1m", "--f", "32"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "sec_per_als_iteration" and d["unit"] == "s"
    assert d["higher_is_better"] is False and d["value"] > 0
    assert d["config"]["workload"].startswith("ml1m-f32-cg16") and d["config"]["nnz"] == 1_000_000
    assert d["steps"] == 2 and len(d["seconds_per_step"]) == 2
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
