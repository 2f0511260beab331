"""Copy the outputs of tools/gpu_final.sh (a gpurun_out/ directory) into profiles/ under
their round-2 names, and summarise the back-to-back repeats into profiles/repeats_r2.json.

    python tools/collect_final.py [gpurun_out_dir]
"""
import json
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
src = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "gpurun_out"
prof = ROOT / "profiles"


def last_json(p: Path) -> dict:
    return json.loads(p.read_text().strip().splitlines()[-1])


def main():
    for a, b in (("bench.json", "bench_r2.json"), ("bench_ref.json", "bench_ref_r2.json"),
                 ("launches_r2.csv", "launches_r2.csv"), ("traffic_r2.json", "traffic_r2.json"),
                 ("round_latency.json", "round_latency_r2.json"),
                 ("e2e_timeline.txt", "e2e_timeline_r2.txt"), ("bench_n2.json", "bench_n2_r2.json"),
                 ("c4_live.json", "c4_live_r2.json")):
        if (src / a).exists():
            shutil.copy(src / a, prof / b)
    if (src / "c4_live_run").is_dir():
        shutil.copytree(src / "c4_live_run", prof / "c4_live_run_r2", dirs_exist_ok=True)
    smoke = (src / "smoke.log").read_text().strip().splitlines()[-1:]
    tests = (src / "pytest_gpu.log").read_text().strip().splitlines()[-2:]
    (prof / "gputest_r2.txt").write_text("\n".join(smoke + tests) + "\n")
    runs = []
    for p in sorted(src.glob("rep_*.json")):
        d = last_json(p)
        e = d.get("e2e") or {}
        c2l, c2m, c4m = d.get("c2_live") or {}, d.get("c2_model") or {}, d.get("c4_model") or {}
        runs.append({
            "value": d["value"], "value_cold": (d.get("value_cold") or {}).get("value"),
            "e2e": e.get("value"), "e2e_ms_per_step": e.get("ms_per_step"),
            "e2e_host_step_ms_max": e.get("host_step_ms_max"),
            "e2e_host_step_phases_ms": e.get("host_step_phases_ms"),
            "c2_live_bulk_host_enqueue_ms": (c2l.get("bulk") or {}).get("host_enqueue_ms"),
            "c2_live_switch_pause_ms": c2l.get("switch_pause_ms"),
            "c2_model_pause_ms": (c2m.get("pause") or {}).get("pause_ms"),
            "c2_model_switch_step": c2m.get("switch_step"),
            "c2_model_tokens_equal_static": c2m.get("tokens_equal_static"),
            "c4_model_pause_ms": (c4m.get("pause") or {}).get("pause_ms"),
            "c4_model_switch_step": c4m.get("switch_step"),
            "c4_model_tokens_equal_static": c4m.get("tokens_equal_static")})
    c4 = []
    for p in sorted(src.glob("c4_[0-9].json")):
        try:
            c4.append(json.loads(p.read_text())["steps"]["pause_ms"])
        except (ValueError, KeyError):
            c4.append(None)
    out = {"note": f"{len(runs)} x bench.py --steps 10 --warmup 3 --skip-c3 --skip-sweep "
                   f"--skip-cpu back to back on one box (tools/gpu_final.sh), plus {len(c4)} x "
                   "tools/c4_live.py (8 stage processes, tiny model)",
           "runs": runs, "c4_live_pause_ms": c4}
    (prof / "repeats_r2.json").write_text(json.dumps(out, indent=1) + "\n")
    for r in runs:
        print(r["value"], r["value_cold"], r["e2e"], r["e2e_host_step_ms_max"],
              r["c2_live_switch_pause_ms"], r["c2_model_pause_ms"], r["c4_model_pause_ms"])
    print("c4_live", c4)


if __name__ == "__main__":
    main()
