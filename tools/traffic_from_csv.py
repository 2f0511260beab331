"""ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum over a
bench run -> per-launch DRAM traffic of the dominant kernels (profiles/traffic_r<N>.json).

Launch order in bench.py: bulk push rounds (push_batched_kernel, the >1 ms launches), then
switch-pause pushes (small), then decode at n_q=32 ((W+K) x 16 layers), then n_q=64."""
import csv
import json
import sys
from collections import defaultdict


def rows(path):
    r = list(csv.reader(open(path)))
    hdr = next(i for i, x in enumerate(r) if "Kernel Name" in x)
    h = r[hdr]
    out = defaultdict(dict)
    for x in r[hdr + 1:]:
        if len(x) < len(h):
            continue
        d = dict(zip(h, x))
        key = (int(d["ID"]), d["Kernel Name"])
        unit = d.get("Metric Unit", "")
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        out[key][d["Metric Name"]] = v * scale
    return [(k[1], m) for k, m in sorted(out.items())]


def main(src, dst, per_shape):
    launches = rows(src)
    res = []
    push_names = ("push_batched_kernel", "copy_kernel<2>")
    push = [(n, m) for n, m in launches
            if any(k in n for k in push_names) and m["gpu__time_duration.sum"] > 1e6]
    kname = next((k for k in push_names if push and k in push[0][0]), None)
    push = [m for _, m in push]
    if push:
        b = sum(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in push) / len(push)
        res.append({"kernel": kname, "n_q": None, "launches": len(push),
                    "dram_bytes": int(b),
                    "read": int(sum(m["dram__bytes_read.sum"] for m in push) / len(push)),
                    "write": int(sum(m["dram__bytes_write.sum"] for m in push) / len(push))})
    attn = [m for n, m in launches if "paged_attn_mma_kernel" in n]
    for i, nq in enumerate((32, 64)):
        part = attn[i * per_shape:(i + 1) * per_shape]
        if part:
            b = sum(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in part) / len(part)
            res.append({"kernel": "paged_attn_mma", "n_q": nq, "launches": len(part),
                        "dram_bytes": int(b),
                        "read": int(sum(m["dram__bytes_read.sum"] for m in part) / len(part)),
                        "write": int(sum(m["dram__bytes_write.sum"] for m in part) / len(part))})
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]))
