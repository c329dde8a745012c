"""Host logic of bench.py (no GPU): the reference arm's JSON line keeps the bench contract and
names the same workload config as the library arm (the driver pairs the two lines)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_reference_arm_line_c1():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "C1",
                          "--steps", "2", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["unit"] == "Gpts/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "Gpts/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    # the library arm's config for the same workload at N=1 (bench_config with the spec's own sizes)
    spec = bench.workload_spec("C1", 1)
    pts = float(np.prod(spec["shape"]))
    assert line["config"] == bench.bench_config(spec, spec["nt"], 1, pts, spec["nbl"] > 0)
    assert line["config"]["workload"] == "C1" and line["config"]["time_steps"] == 100


def test_l2_note():
    assert bench.l2_note(3 * 2 ** 30).startswith("inputs larger than L2")
    assert "fits in L2" in bench.l2_note(48 * 2 ** 20)
