"""CPU checks of the drop-in boundary: libpipelive.so loads and exports every
symbol include/pipelive.h declares; the product path refuses to run without a
GPU (no CPU fallback)."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_symbols() -> set[str]:
    text = (ROOT / "include" / "pipelive.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(pl_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_header_symbol():
    from paper_2604_12171_b200 import _native as N

    lib = N.load_library(require_device=False)
    declared = header_symbols()
    assert len(declared) >= 45
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    bound = {name for name, _, _ in N.SIGNATURES}
    assert declared == bound, declared ^ bound
    assert lib.pl_abi_version() == 1


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_12171_b200 import _native as N
    from paper_2604_12171_b200 import kvstore

    with pytest.raises(N.NativeUnavailable):
        kvstore.KvStore(1, 1, 16, 4, (0,))


def test_library_targets_sm100a():
    import subprocess

    so = ROOT / "paper_2604_12171_b200" / "libpipelive.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
