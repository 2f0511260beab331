"""Layer-weight staging on the copy engine (staging.py, AddLayerWeights): bytes arrive
exactly, residency/eviction follow the reference WeightLoader semantics."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_stage_evict_roundtrip():
    import torch

    from paper_2604_12171_b200.staging import LayerInUse, LayerWeightStager

    rng = np.random.default_rng(0)
    host = {l: {"w": torch.from_numpy(rng.standard_normal((300, 257)).astype(np.float32)).pin_memory(),
                "b": torch.from_numpy(rng.integers(0, 255, 12345, dtype=np.uint8)).pin_memory()}
            for l in (1, 2, 3)}
    st = LayerWeightStager(0, host, chunk_bytes=4096, is_layer_committed=lambda l: l == 3)
    st.stage_layers({2, 3})
    st.wait()
    assert not st.staging_active()
    assert st.is_resident(2) and st.is_resident(3) and not st.is_resident(1)
    for l in (2, 3):
        for k, t in host[l].items():
            assert torch.equal(st.resident[l][k].cpu(), t)
    assert st.staged_bytes == 2 * (300 * 257 * 4 + 12345)
    with pytest.raises(LayerInUse):
        st.evict_layers({3})
    assert st.evict_layers({2}) == 300 * 257 * 4 + 12345
    assert not st.is_resident(2)
    st.stage_layers({1, 2, 3})          # 3 is resident already: only 1 and 2 are copied
    st.wait()
    assert st.staged_bytes == 4 * (300 * 257 * 4 + 12345)


def test_unpinned_host_weights_rejected():
    import torch

    from paper_2604_12171_b200.staging import LayerWeightStager

    with pytest.raises(ValueError):
        LayerWeightStager(0, {1: {"w": torch.zeros(4)}})
