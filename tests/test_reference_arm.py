"""bench.py --impl reference on CPU: the reference package itself (pipeshift, staged
unmodified into oracle/_ref/ by build()) timed through its own API, printed as one JSON
line in the contract's shape, with the per-step sample stated."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "pipeshift").is_dir(),
                    reason="oracle/_ref not staged (build() stages it in the dev container)")
def test_reference_arm_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--batch", "4"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] == 1 and cb["value"] == line["value"]
    assert line["sample_bytes_per_step"] == cb["sample_bytes"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    ex = line["reference_extras"]
    assert ex["append"]["cells_per_s"] > 0 and ex["steady_round"]["us_per_round"] > 0
    assert ex["scenario"]["seconds"] > 0
