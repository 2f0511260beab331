"""configs[3] with the 8B-shaped decoder alone (bench.measure_c4_model) -> stdout, and the live run's trace.jsonl / metrics.csv / summary.json -> gpurun_out/c4_model_run/."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2604_12171_b200.perf import Workload  # noqa: E402

print(json.dumps(bench.measure_c4_model(Workload(), run_dir='gpurun_out/c4_model_run'), indent=1))
