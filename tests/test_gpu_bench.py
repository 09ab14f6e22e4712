"""bench.py end to end on a reduced size for every --config (the driver runs only the default
line): one JSON line with the contract's keys, a roofline object, an e2e object, launches
counted, and a sharding check that found no mismatch."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cfg,units", [(0, None), (1, 8), (2, 200_000), (3, 100_000), (4, 4)])
def test_bench_config_line(cfg, units):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(cfg), "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline", "--no-per-config", "--e2e-images", "2"]
    if units:
        cmd += ["--images", str(units)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["unit"] == "GB/s" and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    if cfg != 0:
        assert d["sharding"]["mismatches"] == 0 and d["sharding"]["checked"] >= 2
