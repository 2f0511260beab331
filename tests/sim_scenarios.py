"""Scenario builders with the same parameters as the reference's test scenarios
(pkg/tests/scenarios.py:136-196, pkg/tests/test_coordinator.py:14-73), built on
this package's classes so the golden simulations can be replayed on the GPU box
where the reference does not exist."""

from __future__ import annotations

from paper_2604_12171_b200 import FeatureFlags, GpuSpec, ModelSpec, PPConfig, WorkloadSpec
from paper_2604_12171_b200.scenario import ReconfigTrigger, Scenario

GIB, MIB, KIB = 1024 ** 3, 1024 ** 2, 1024

C_A = PPConfig([(1, (1, 2)), (2, (3, 4)), (3, (5, 6))])
C_B = PPConfig([(1, (1, 1)), (2, (2, 3)), (3, (4, 6))])


def _two_gpus():
    return [GpuSpec(id=1, mem_total=80 * GIB, mem_bandwidth=2.039e12, prefill_cost=4e-6,
                    decode_cost=6e-6),
            GpuSpec(id=2, mem_total=48 * GIB, mem_bandwidth=8.64e11, prefill_cost=1.5e-6,
                    decode_cost=2.4e-5)]


def hetero_scenario(rate=7.0, n=120, k=2, triggers=True, flags=None, tau=50,
                    init=None) -> Scenario:
    shift = n / rate / 2
    model = ModelSpec(num_layers=16, layer_weight_bytes=int(2.5 * GIB),
                      token_kv_bytes_per_layer=128 * KIB, stacking_factor=k,
                      activation_bytes_per_token=32 * KIB)
    wl = WorkloadSpec("shift_schedule", rate=rate, num_requests=n,
                      shifts=((0.0, "prefill_heavy"), (shift, "decode_heavy")))
    tgt = PPConfig([(1, (1, 14)), (2, (15, 16))])
    return Scenario(cluster=_two_gpus(), model=model,
                    initial_config=init or PPConfig([(1, (1, 2)), (2, (3, 16))]), workload=wl,
                    triggers=[ReconfigTrigger(at=shift, target=tgt, tau=tau)] if triggers else [],
                    flags=flags or FeatureFlags())


def stacking_scenario(k: int, n: int = 6) -> Scenario:
    """Short fixed-length requests on a 16-layer model at stacking k
    (pkg/tests/scenarios.py:120-134)."""
    gpus = [GpuSpec(id=i, mem_total=32 * GIB, mem_bandwidth=1e12, prefill_cost=1e-6,
                    decode_cost=1e-5) for i in (1, 2)]
    model = ModelSpec(num_layers=16, layer_weight_bytes=256 * MIB, token_kv_bytes_per_layer=8 * KIB,
                      stacking_factor=k, activation_bytes_per_token=8 * KIB)
    return Scenario(cluster=gpus, model=model, initial_config=PPConfig([(1, (1, 8)), (2, (9, 16))]),
                    workload=WorkloadSpec("prefill_heavy", rate=50.0, num_requests=n))


def _random_partition(rng, total: int, parts: int) -> list[int]:
    """`total` layer groups cut into `parts` positive runs (pkg/tests/helpers.py:36-40)."""
    cuts = sorted(rng.sample(range(1, total), parts - 1)) if parts > 1 else []
    bounds = [0] + cuts + [total]
    return [bounds[i + 1] - bounds[i] for i in range(parts)]


def _partition_config(counts: list[int], k: int, ids: list[int]) -> PPConfig:
    """Consecutive layer ranges of counts[i] groups each (pkg/tests/helpers.py:43-51)."""
    out, start = [], 1
    for gid, groups in zip(ids, counts):
        end = start + groups * k - 1
        out.append((gid, (start, end)))
        start = end + 1
    return PPConfig(out)


def random_e2e_scenario(seed: int) -> Scenario:
    """The randomized reconfiguration scenarios of acceptance criterion 4
    (pkg/tests/scenarios.py:87-117): 2-4 GPUs, 8-32 layers, same draws in the same order."""
    import random

    rng = random.Random(seed)
    n_gpus = rng.randint(2, 4)
    k = rng.choice([1, 2, 4])
    groups = rng.randint(max(n_gpus, 8 // k), 8)
    cluster = [GpuSpec(id=i, mem_total=rng.choice([16, 32]) * GIB, mem_bandwidth=1e12,
                       prefill_cost=rng.choice([1e-6, 2e-6, 4e-6]),
                       decode_cost=rng.choice([5e-6, 1e-5, 2e-5]))
               for i in range(1, n_gpus + 1)]
    model = ModelSpec(num_layers=groups * k, layer_weight_bytes=rng.choice([256, 512]) * MIB,
                      token_kv_bytes_per_layer=rng.choice([32, 64]) * KIB, stacking_factor=k,
                      activation_bytes_per_token=8 * KIB)
    ids = list(range(1, n_gpus + 1))
    cur = _partition_config(_random_partition(rng, groups, n_gpus), k, ids)
    tgt = _partition_config(_random_partition(rng, groups, n_gpus), k, ids)
    rate = rng.uniform(40.0, 120.0)
    pattern = rng.choice(["prefill_heavy", "decode_heavy"])
    n = rng.randint(4, 8)
    wl = WorkloadSpec(pattern, rate=rate, num_requests=n, jitter=rng.random() < 0.5)
    trigger_at = (n / rate) * rng.uniform(0.3, 0.8)
    return Scenario(cluster=cluster, model=model, initial_config=cur, workload=wl,
                    triggers=[ReconfigTrigger(at=trigger_at, target=tgt, tau=50)])


def stoptime_scenario(migrate_layers=4, flags=None, ghost_tokens=6000):
    model = ModelSpec(num_layers=16, layer_weight_bytes=int(2.5 * GIB),
                      token_kv_bytes_per_layer=64 * KIB, stacking_factor=2,
                      activation_bytes_per_token=32 * KIB)
    edge = 2 + migrate_layers
    scen = Scenario(cluster=_two_gpus(), model=model,
                    initial_config=PPConfig([(1, (1, 2)), (2, (3, 16))]),
                    workload=WorkloadSpec("prefill_heavy", rate=1.0, num_requests=0),
                    triggers=[ReconfigTrigger(at=0.001,
                                              target=PPConfig([(1, (1, edge)), (2, (edge + 1, 16))]))],
                    flags=flags or FeatureFlags())

    def fill(sim):
        store = sim.stores[2]
        for group in sorted(store.resident_groups):
            base = group * 1000
            store.append("zombie", group, ghost_tokens, [base + i for i in range(ghost_tokens)])

    return scen, fill


def fig3_cluster(mem_mib=4096):
    return {i: GpuSpec(id=i, mem_total=mem_mib * MIB, mem_bandwidth=1e12, prefill_cost=1e-6,
                       decode_cost=1e-5, alloc_granularity=2 * MIB) for i in (1, 2, 3)}


def fig3_model():
    return ModelSpec(num_layers=6, layer_weight_bytes=64 * MIB, token_kv_bytes_per_layer=8 * KIB,
                     stacking_factor=1, activation_bytes_per_token=2 * KIB)


def fig3_scenario(triggers=(), flags=None, num_requests=4, rate=200.0, pattern="decode_heavy",
                  tau=50) -> Scenario:
    return Scenario(cluster=list(fig3_cluster().values()), model=fig3_model(), initial_config=C_A,
                    workload=WorkloadSpec(pattern=pattern, rate=rate, num_requests=num_requests),
                    triggers=[ReconfigTrigger(at, tgt, tau=tau) for at, tgt in triggers],
                    flags=flags or FeatureFlags())


def golden_runs():
    """name -> (scenario, seed, fill) for every run recorded in tests/golden/simulations.json"""
    runs = {
        "fig3_seed5": (fig3_scenario(triggers=[(0.02, C_B)], num_requests=4, rate=500.0), 5, None),
        "hetero_c10_seed123": (hetero_scenario(rate=7.0, n=40), 123, None),
        "hetero_n60_seed7": (hetero_scenario(rate=7.0, n=60), 7, None),
        # = the reference's packaged pkg/scenarios/heterogeneous_shift.yaml, seed 0
        "packaged_yaml_seed0": (hetero_scenario(rate=8.0, n=200), 0, None),
        "fig3_nopatch": (fig3_scenario(triggers=[(0.02, C_B)], num_requests=4, rate=500.0,
                                       flags=FeatureFlags(kv_patch=False)), 5, None),
    }
    for L in (4, 8):
        scen, fill = stoptime_scenario(migrate_layers=L)
        runs[f"stoptime_L{L}"] = (scen, 0, fill)
    return runs


# ---------------------------------------------------------------------------------------------
# BASELINE configs as parity scenarios.  PP-degree changes need GPUs without layers (the
# idle-GPU extension): configs simply omit idle GPUs.  The builders take the
# package namespace so the golden generator can build the identical scenario on the
# reference (with the same extension monkeypatched in, tests/golden/make_golden.py).
def _ns_default():
    import types

    import paper_2604_12171_b200 as pkg
    from paper_2604_12171_b200 import scenario as sc
    return types.SimpleNamespace(GpuSpec=pkg.GpuSpec, ModelSpec=pkg.ModelSpec,
                                 PPConfig=pkg.PPConfig, WorkloadSpec=pkg.WorkloadSpec,
                                 FeatureFlags=pkg.FeatureFlags, Scenario=sc.Scenario,
                                 ReconfigTrigger=sc.ReconfigTrigger, idle_field=True)


def _scenario(ns, **kw):
    s = ns.Scenario(**kw)
    if getattr(ns, "idle_field", False):
        s.allow_idle_gpus = True
    return s


def b200(ns, gid, mem_gib=180, prefill=2e-7, decode=4e-6, gran=2 * MIB):
    return ns.GpuSpec(id=gid, mem_total=mem_gib * GIB, mem_bandwidth=7.7e12,
                      prefill_cost=prefill, decode_cost=decode, alloc_granularity=gran)


def config0_tiny(ns=None):
    """configs[0]: tiny 4-layer Llama-style model (d=256, 4 q / 2 kv heads x 64 -> 512 B of
    KV per token-layer), k=1, 16-token blocks, PP 2->3 on 3 GPUs."""
    ns = ns or _ns_default()
    gran = 16 * 512
    cluster = [b200(ns, i, mem_gib=1, prefill=2e-6, decode=2e-5, gran=gran) for i in (1, 2, 3)]
    model = ns.ModelSpec(num_layers=4, layer_weight_bytes=1536 * 1024, token_kv_bytes_per_layer=512,
                         stacking_factor=1, activation_bytes_per_token=512)
    cur = ns.PPConfig([(1, (1, 2)), (2, (3, 4))])
    tgt = ns.PPConfig([(1, (1, 1)), (2, (2, 3)), (3, (4, 4))])
    wl = ns.WorkloadSpec("shift_schedule", rate=40.0, num_requests=24,
                         shifts=((0.0, "prefill_heavy"), (0.3, "decode_heavy")))
    return _scenario(ns, cluster=cluster, model=model, initial_config=cur, workload=wl,
                     triggers=[ns.ReconfigTrigger(at=0.3, target=tgt)], flags=ns.FeatureFlags())


def config1_8b(ns=None, n=48):
    """configs[1]: Llama-3-8B shape (32 L, 4096 B KV per token-layer, 0.436 GB/layer),
    k=4, 16-token blocks, PP 2->4 with minimal movement on 4 B200s, decode-heavy load."""
    ns = ns or _ns_default()
    cluster = [b200(ns, i) for i in (1, 2, 3, 4)]
    model = ns.ModelSpec(num_layers=32, layer_weight_bytes=436 * 10 ** 6,
                         token_kv_bytes_per_layer=4096, stacking_factor=4,
                         activation_bytes_per_token=8 * KIB)
    cur = ns.PPConfig([(1, (1, 16)), (2, (17, 32))])
    tgt = ns.PPConfig([(1, (1, 8)), (3, (9, 16)), (2, (17, 24)), (4, (25, 32))])
    wl = ns.WorkloadSpec("decode_heavy", rate=200.0, num_requests=n)
    return _scenario(ns, cluster=cluster, model=model, initial_config=cur, workload=wl,
                     triggers=[ns.ReconfigTrigger(at=0.1, target=tgt)], flags=ns.FeatureFlags())


def config2_70b(ns=None, n=32):
    """configs[2]: Llama-3-70B shape (80 L, 1.711 GB/layer), k=4, PP 4->8 with HBM
    pre-filled by KV so Phase 2 must shrink every store and cleanup grows them back."""
    ns = ns or _ns_default()
    cluster = [b200(ns, i, decode=8e-6) for i in range(1, 9)]
    model = ns.ModelSpec(num_layers=80, layer_weight_bytes=1711 * 10 ** 6,
                         token_kv_bytes_per_layer=4096, stacking_factor=4,
                         activation_bytes_per_token=16 * KIB)
    cur = ns.PPConfig([(1, (1, 20)), (2, (21, 40)), (3, (41, 60)), (4, (61, 80))])
    # GPU1 also receives layers 21-24, so its union set (24 layers) exceeds every current
    # stage and b_shrink < current capacity: a real live shrink
    tgt = ns.PPConfig([(1, (1, 24)), (5, (25, 32)), (2, (33, 40)), (6, (41, 48)),
                       (3, (49, 56)), (7, (57, 64)), (4, (65, 72)), (8, (73, 80))])
    wl = ns.WorkloadSpec("decode_heavy", rate=100.0, num_requests=n)
    return _scenario(ns, cluster=cluster, model=model, initial_config=cur, workload=wl,
                     triggers=[ns.ReconfigTrigger(at=0.2, target=tgt)], flags=ns.FeatureFlags())


def config3_uneven(ns=None, n=48):
    """configs[3]: 8 GPUs, 70B shape at k=2: even prefill-optimal split -> uneven
    generation-heavy split across a prefill_heavy -> decode_heavy trace shift."""
    ns = ns or _ns_default()
    cluster = [b200(ns, i, prefill=1e-7 * (1 + i % 3), decode=3e-6 * (1 + (i + 1) % 2))
               for i in range(1, 9)]
    model = ns.ModelSpec(num_layers=80, layer_weight_bytes=1711 * 10 ** 6,
                         token_kv_bytes_per_layer=4096, stacking_factor=2,
                         activation_bytes_per_token=16 * KIB)

    def split(sizes):
        out, first = [], 1
        for gid, size in zip(range(1, 9), sizes):
            out.append((gid, (first, first + size - 1)))
            first += size
        return ns.PPConfig(out)

    cur = split([10] * 8)
    tgt = split([6, 8, 10, 12, 12, 10, 12, 10])
    shift = n / 60.0 / 2
    wl = ns.WorkloadSpec("shift_schedule", rate=60.0, num_requests=n,
                         shifts=((0.0, "prefill_heavy"), (shift, "decode_heavy")))
    return _scenario(ns, cluster=cluster, model=model, initial_config=cur, workload=wl,
                     triggers=[ns.ReconfigTrigger(at=shift, target=tgt)], flags=ns.FeatureFlags())


def config_runs(ns=None):
    """name -> (scenario, seed, fill) of the BASELINE-config parity runs"""
    return {"config0_tiny": (config0_tiny(ns), 3, None),
            "config1_8b": (config1_8b(ns), 1, None),
            "config2_70b": (config2_70b(ns), 2, prefill_kv),
            "config3_uneven": (config3_uneven(ns), 4, None)}


def prefill_kv(sim, fraction=0.6):
    """Fill every store with synthetic KV up to ``fraction`` of the shrink budget, so the
    reconfiguration's Phase 2 shrink and post-commit grow act on a near-full HBM."""
    from math import ceil
    for gpu_id, store in sim.stores.items():
        groups = sorted(store.resident_groups)
        if not groups:
            continue
        s = store.tokens_per_block
        blocks = int(store.capacity_blocks * fraction * 0.5)
        per_req = 64 * s
        for r in range(ceil(blocks / 64)):
            rid = f"prefill{gpu_id}_{r:03d}"
            for g in groups:
                store.append(rid, g, per_req, [(gpu_id << 40) + (g << 32) + r * per_req + i
                                               for i in range(per_req)])
