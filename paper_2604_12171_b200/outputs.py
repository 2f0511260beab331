"""Run outputs in the reference's on-disk schema.

The reference's scenario runner writes three files per run (`cli.py:37-80`):
- `trace.jsonl`: one event per line (`events.py:56-59, 89-90`);
- `metrics.csv`: one header row of `METRIC_COLUMNS`, then one row of `Metrics.as_row()`
  (`cli.py:23-27, 46-52`);
- `summary.json`: `{"schema_version": 1, "command": "run", ...}`, indented, sorted keys
  (`cli.py:39-43, 66-80`).

`write_run` emits the same three files for a parity-mode `RunResult` and for a perf-mode
run (the staged Llama of `llama.generate*`, whose trace holds wall-clock times), so the
reference's analysis scripts read either.  Only the formats are here; the argparse front
end is out of scope.
"""

from __future__ import annotations

import csv
import io
import json
import os

from .engine import Metrics, compute_metrics
from .events import EventTrace
from .scenario import SCHEMA_VERSION

# cli.py:23-27
METRIC_COLUMNS = [
    "ttft_mean", "ttft_p99", "tpot_mean", "throughput", "stop_time",
    "migration_time", "effective_kv_utilization", "overflow_events",
    "completed", "reconfig_outcome",
]


def metrics_csv(rows: list[dict], columns: list[str] = METRIC_COLUMNS) -> str:
    """The CSV text `cli._write_csv` produces (csv.DictWriter, default dialect: CRLF line
    ends, missing keys as empty cells)."""
    buf = io.StringIO(newline="")
    w = csv.DictWriter(buf, fieldnames=columns)
    w.writeheader()
    for row in rows:
        w.writerow({c: row.get(c, "") for c in columns})
    return buf.getvalue()


def summary_json(payload: dict) -> str:
    """`cli._write_summary`: schema_version first, indent 2, sorted keys, trailing newline."""
    return json.dumps({"schema_version": SCHEMA_VERSION, **payload}, indent=2,
                      sort_keys=True) + "\n"


def run_summary(scenario_path: str, seed: int, trace: EventTrace, metrics: Metrics,
                **extra) -> dict:
    """The `summary.json` payload of one run (`cli.py:72-79`).  `extra` adds keys a
    perf-mode run wants to carry (e.g. `"mode": "perf"`); the reference keys are
    unchanged."""
    row = metrics.as_row()
    out = {"command": "run", "scenario": os.path.abspath(scenario_path), "seed": seed,
           "events": len(trace), "metrics": row,
           "reconfig_outcome": metrics.reconfig_outcome}
    out.update(extra)
    return out


def write_run(out_dir: str, trace: EventTrace, scenario_path: str, seed: int,
              metrics: Metrics | None = None, **extra) -> dict[str, str]:
    """Write trace.jsonl, metrics.csv and summary.json for one run into `out_dir`
    (created if needed) and return the three paths.  `metrics` defaults to
    `compute_metrics(trace)` (engine.py:112-184), which is what `RunResult.metrics` holds
    for a parity run."""
    os.makedirs(out_dir, exist_ok=True)
    if metrics is None:
        metrics = compute_metrics(trace)
    paths = {name: os.path.join(out_dir, name)
             for name in ("trace.jsonl", "metrics.csv", "summary.json")}
    with open(paths["trace.jsonl"], "w") as fh:
        fh.write(trace.to_jsonl())
    with open(paths["metrics.csv"], "w", newline="") as fh:
        fh.write(metrics_csv([metrics.as_row()]))
    with open(paths["summary.json"], "w") as fh:
        fh.write(summary_json(run_summary(scenario_path, seed, trace, metrics, **extra)))
    return paths


def write_result(out_dir: str, result, scenario_path: str) -> dict[str, str]:
    """`write_run` for a `simulation.RunResult` (what `run_scenario` returns)."""
    return write_run(out_dir, result.trace, scenario_path, result.seed, result.metrics)
