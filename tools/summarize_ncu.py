"""Summarise ncu reports (raw page) and a launch list into profiles/*.md."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    recs = []
    for v in rows[2:]:
        recs.append({h[i]: (v[i], u[i]) for i in range(len(h))})
    return recs


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            try:
                agg[r[ki]][0] += 1
                agg[r[ki]][1] += float(r[vi].replace(",", ""))
            except ValueError:
                pass
    return agg


if __name__ == "__main__":
    out = sys.argv[1]
    lines = []
    for arg in sys.argv[2:]:
        if arg.endswith(".csv"):
            agg = launches(arg)
            tot = sum(t for _, t in agg.values())
            lines += [f"## launch list `{arg.split('/')[-1]}` (ncu gpu__time_duration, cold, serialised)",
                      "", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
            for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
                lines.append(f"| `{k[:90]}` | {n} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
            lines.append("")
        else:
            for rec in raw(arg):
                name = rec.get("Kernel Name", ("?", ""))[0]
                lines += [f"## `{arg.split('/')[-1]}`: `{name[:100]}`", "", "| metric | value | unit |",
                          "|---|---|---|"]
                for k in KEYS:
                    if k in rec:
                        lines.append(f"| {k} | {rec[k][0]} | {rec[k][1]} |")
                lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
