"""bench.py keeps the driver's contract: one JSON line with the headline
keys, on small sizes so the check is fast (the default sizes run in the
round-end bench)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_line_contract():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--batch", "65536",
           "--basic", "32", "--path", "16", "--big", "32", "--no-strategies"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline",
                "basic_scheme"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] >= 3 and line["value"] > 0
    assert "error" not in line
    rl = line["roofline"]
    assert rl["bound"] == "fp64" and 0 < rl["frac"] < 1 and rl["achieved"] > 0 and rl["peak"] > 0
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] > 0
    basic = line["basic_scheme"]
    for key in ("config4_step1", "config4_20_steps", "config3_path", "config5_step1", "config1"):
        assert key in basic and "error" not in basic[key], (key, basic.get(key))
    assert basic["config4_step1"]["value"] > 0 and basic["config4_step1"]["iterations"] > 0
    assert line["gpu_launches"] == 2 * 3
