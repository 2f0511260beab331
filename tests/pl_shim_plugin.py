"""pytest plugin: the maintainer-side shim of INTEGRATION.md §2, applied before the
reference's own test modules import anything.  `pipeshift` (the unmodified staged copy in
oracle/_ref/) keeps its control plane -- cluster, events, fabric, engine, coordinator,
weights, simulation, scenario, cli -- and its data plane names point at this package's:
the KV store (`KvStore`, `kv_init`, the exceptions) and the patch engine
(`DirtyBitmap`, `KvPatch`, `ConvergenceCounters`, `PatchReceiver`, `MigrationStream`,
`MigrationManager`).  Used by tests/test_gpu_reference_own_suites.py:

    python -m pytest -p pl_shim_plugin oracle/_ref/tests/test_kvstore.py ...
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))

import pipeshift  # noqa: E402
import pipeshift.engine as _ref_engine  # noqa: E402
import pipeshift.kvstore as _ref_kv  # noqa: E402
import pipeshift.migrator as _ref_mig  # noqa: E402
import pipeshift.simulation as _ref_sim  # noqa: E402

from paper_2604_12171_b200 import kvstore as _kv  # noqa: E402
from paper_2604_12171_b200 import migrator as _mig  # noqa: E402

KV_NAMES = ("KvStore", "kv_init", "KvOverflow", "CapacityBelowLive", "UnknownSlot",
            "UnknownLayerGroup", "InsufficientMemory")
MIG_NAMES = ("DirtyBitmap", "KvPatch", "ConvergenceCounters", "PatchReceiver",
             "MigrationStream", "MigrationManager")

for _n in KV_NAMES:
    for _mod in (_ref_kv, _ref_engine, _ref_sim, _ref_mig, pipeshift):
        if hasattr(_mod, _n):
            setattr(_mod, _n, getattr(_kv, _n))
for _n in MIG_NAMES:
    for _mod in (_ref_mig, _ref_sim, pipeshift):
        if hasattr(_mod, _n):
            setattr(_mod, _n, getattr(_mig, _n))
