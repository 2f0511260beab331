"""Run-output formats (outputs.py) against the reference scenario runner's own files
(cli.py:37-80), recorded by tests/golden/make_golden.py (`cli_outputs.json`).

CPU: the writers reproduce metrics.csv byte for byte and summary.json key for key from
the recorded metrics.  GPU: `run_scenario` on the same YAML through the GPU data plane,
then `write_result`, reproduces all three files (trace.jsonl by sha256)."""

import hashlib
import json
import os

import pytest

CASES = ["small_seed3", "small_trigger_seed1", "small_infeasible_seed0", "packaged_seed0"]


def _metrics(row):
    from paper_2604_12171_b200.engine import Metrics
    return Metrics(**row)


@pytest.mark.parametrize("name", CASES)
def test_writers_match_reference_text(golden, name):
    from paper_2604_12171_b200 import outputs
    want = golden("cli_outputs.json")[name]
    m = _metrics(want["summary"]["metrics"])
    assert outputs.metrics_csv([m.as_row()]) == want["metrics_csv"]
    text = outputs.summary_json({k: v for k, v in want["summary"].items()
                                 if k != "schema_version"})
    assert text.endswith("}\n") and text.startswith('{\n  "command"')
    assert json.loads(text) == want["summary"]


def test_metric_columns_order():
    from paper_2604_12171_b200 import outputs
    from paper_2604_12171_b200.engine import Metrics
    assert list(Metrics().as_row()) == outputs.METRIC_COLUMNS


def test_write_run_perf_mode_trace(tmp_path):
    """A perf-mode trace (wall-clock times, engine events only) goes through the same
    writer; the extra summary keys sit beside the reference ones."""
    from paper_2604_12171_b200 import outputs
    from paper_2604_12171_b200.events import EventTrace
    tr = EventTrace()
    tr.emit(0.0, "engine", "request_arrival", id="seq0", input_len=4, output_len=2)
    tr.emit(0.001, "engine", "first_token", id="seq0")
    tr.emit(0.002, "engine", "request_complete", id="seq0", output_len=2)
    paths = outputs.write_run(str(tmp_path / "o"), tr, "perf.yaml", 0, mode="perf")
    assert open(paths["trace.jsonl"]).read() == tr.to_jsonl()
    s = json.load(open(paths["summary.json"]))
    assert s["schema_version"] == 1 and s["mode"] == "perf" and s["events"] == 3
    assert open(paths["metrics.csv"], newline="").read().startswith(
        ",".join(outputs.METRIC_COLUMNS) + "\r\n")


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_run_outputs_match_reference(golden, tmp_path, name):
    from paper_2604_12171_b200 import outputs
    from paper_2604_12171_b200.scenario import load_scenario
    from paper_2604_12171_b200.simulation import run_scenario
    want = golden("cli_outputs.json")[name]
    path = tmp_path / f"{name}.yaml"
    path.write_text(want["yaml"])
    res = run_scenario(load_scenario(str(path)), seed=want["seed"])
    paths = outputs.write_result(str(tmp_path / "out"), res, str(path))
    trace = open(paths["trace.jsonl"], "rb").read()
    assert hashlib.sha256(trace).hexdigest() == want["trace_sha"]
    assert open(paths["metrics.csv"], newline="").read() == want["metrics_csv"]
    got = json.load(open(paths["summary.json"]))
    assert got.pop("scenario") == os.path.abspath(str(path))
    exp = dict(want["summary"])
    exp.pop("scenario")
    assert got == exp
