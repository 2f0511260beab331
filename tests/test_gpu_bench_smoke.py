"""bench.py end to end at a small shape (every measurement path runs; the JSON line has
the contract keys).  The real bench runs at the BASELINE shape at round end."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_bench_small_shape_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3",
                          "--batch", "32", "--ctx", "512", "--skip-c3", "--skip-cpu",
                          "--skip-sweep"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "roofline", "e2e",
              "gpu_launches", "clocks"):
        assert k in line, k
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    for extra in ("switch_pause_ms", "c2_live", "decode", "decode_70b_shape", "weight_stage",
                  "resize", "e2e_real_kv_from_host"):
        assert line[extra] is not None and "error" not in line[extra], (extra, line[extra])
