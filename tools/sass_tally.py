"""Opcode tally of the built libpipelive.so (cuobjdump -sass) for the hot kernels:
proves the instruction mix the DESIGN claims (TMA, ldmatrix, HMMA in K2; 128-bit
streaming loads/stores in the push).  Writes profiles/sass_r2.txt.

    python tools/sass_tally.py
"""

from __future__ import annotations

import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "paper_2604_12171_b200" / "libpipelive.so"
KERNELS = {
    "K2 paged_attn_mma_kernel<128,8>": r"paged_attn_mma_kernelILi128ELi8E",
    "K2 paged_attn_mma_kernel<64,8>": r"paged_attn_mma_kernelILi64ELi8E",
    "K4+K5 push_batched_kernel (fused push, batched resolve)": r"push_batched_kernel",
    "K3+K4+K5 drain_push_kernel (steady rounds)": r"drain_push_kernel",
    "K4+K5 copy_kernel<2> (per-item resolve, PL_PUSH_BATCHED=0)": r"copy_kernelILi2EE",
    "K1 kv_write_kernel": r"kv_write_kernel",
    "K3 drain_compact_kernel": r"drain_compact_kernel",
    "K6 unit_move_kernel": r"unit_move_kernel",
    "verify_kernel": r"verify_kernel",
}
WATCH = ["UTMALDG", "UTMACMDFLUSH", "LDSM", "MOVM", "HMMA", "SYNCS", "LDG.E.128", "STG.E.128",
         "LDG.E.EL.128", "LDG.E.NA.128", "STG.E.NA.128", "ATOMG", "RED", "SHFL", "VOTE", "MATCH",
         "BAR", "ELECT", "FFMA", "IMAD", "LOP3", "BRA", "EXIT"]


def main() -> None:
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(SO)], capture_output=True,
                          text=True, check=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)
    out = [f"# SASS opcode tally of {SO.name} (cuobjdump -sass, sm_100a)", ""]
    for label, pat in KERNELS.items():
        body = next((f for f in funcs if re.match(r"\S*" + pat, f)), None)
        if body is None:
            out.append(f"{label}: not found")
            continue
        name = body.split("\n", 1)[0].strip()
        ops = collections.Counter()
        for line in body.splitlines():
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                ops[m.group(1)] += 1
        total = sum(ops.values())
        out.append(f"{label}  [{name}]  {total} instructions")
        for w in WATCH:
            n = sum(c for op, c in ops.items() if op == w or op.startswith(w + "."))
            if n:
                out.append(f"  {w:<14} {n}")
        top = ", ".join(f"{op} {c}" for op, c in ops.most_common(12))
        out.append(f"  top: {top}")
        out.append("")
    text = "\n".join(out)
    (ROOT / "profiles" / "sass_r2.txt").write_text(text + "\n")
    print(text)


if __name__ == "__main__":
    sys.exit(main())
