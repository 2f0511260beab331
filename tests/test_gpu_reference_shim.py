"""The drop-in as a `pipeshift` maintainer would wire it: the
reference's OWN control plane -- its Simulation, PipelineEngine, Coordinator, CommFabric,
WeightLoader and event clock, imported unmodified from the staged copy in oracle/_ref/ --
with only the data plane swapped: `kv_init` (the KV store) and `MigrationManager` (the
patch engine) come from this package, so every KV write, block allocation, dirty-bit
drain, patch and resize of the run executes on the GPU.  The packaged scenario
(`pkg/scenarios/heterogeneous_shift.yaml`, seed 0) must produce the reference's trace
byte for byte (sha256 of trace.jsonl), metrics and state digest."""

import hashlib
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


@pytest.mark.skipif(not (REF / "pipeshift").is_dir(),
                    reason="oracle/_ref not staged (build() stages it in the dev container)")
def test_reference_control_plane_over_the_gpu_data_plane(golden, monkeypatch):
    monkeypatch.syspath_prepend(str(REF))
    for name in [m for m in sys.modules if m == "pipeshift" or m.startswith("pipeshift.")]:
        monkeypatch.delitem(sys.modules, name)
    import pipeshift
    import pipeshift.engine as ref_engine
    import pipeshift.simulation as ref_sim

    from paper_2604_12171_b200 import kvstore, migrator

    # the maintainer-side shim: two imports and the exception the engine catches
    monkeypatch.setattr(ref_sim, "kv_init", kvstore.kv_init)
    monkeypatch.setattr(ref_sim, "MigrationManager", migrator.MigrationManager)
    monkeypatch.setattr(ref_engine, "KvOverflow", kvstore.KvOverflow)

    scen = pipeshift.load_scenario(str(REF / "scenarios" / "heterogeneous_shift.yaml"))
    sim = ref_sim.Simulation(scen, seed=0)
    assert all(isinstance(s, kvstore.KvStore) for s in sim.stores.values())
    assert isinstance(sim.migration, migrator.MigrationManager)
    res = sim.run()
    want = golden("simulations.json")["packaged_yaml_seed0"]
    assert len(res.trace) == want["n_events"]
    assert hashlib.sha256(res.trace.to_jsonl().encode()).hexdigest() == want["trace_sha"]
    assert res.metrics.as_row() == want["metrics"]
    assert [s.outcome for s in res.statuses] == [s["outcome"] for s in want["statuses"]]
    assert sim.state_digest() == want["state_digest"]
