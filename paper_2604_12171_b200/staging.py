"""Layer-weight staging on hardware (AddLayerWeights).

The reference models staging as a simulated transfer at host bandwidth that only
progresses while the target GPU is idle (strict) or at a reduced share (weighted)
(weights.py:103-197); it gates the commit (coordinator.py:239-240).  On a B200 the
copy runs on a copy engine: pinned host memory -> HBM with cudaMemcpyAsync on a
lowest-priority stream, in chunks, one CUDA event per layer.  The copy engines run
beside the SMs, and PCIe's ~55 GB/s is under 1 % of HBM bandwidth, so inference does
not yield to staging and staging does not stall inference (measured by bench.py's
`weight_stage`: decode tokens/s with and without a concurrent stage).

The API follows the reference's WeightLoader: stage_layers / staging_active /
cancel_staging / evict_layers, plus is_resident and the device tensors of a layer.
"""

from __future__ import annotations

import time
from typing import Callable


class LayerInUse(Exception):
    """Eviction of a layer the committed config still assigns (weights.py:27-28)."""


class LayerWeightStager:
    def __init__(self, device: int, host_layers: dict[int, dict[str, "object"]],
                 chunk_bytes: int = 64 << 20,
                 is_layer_committed: Callable[[int], bool] | None = None) -> None:
        import torch

        self.torch = torch
        self.device = device
        self.host = host_layers                 # layer -> {name: pinned CPU tensor}
        for ts in host_layers.values():
            for t in ts.values():
                if not t.is_pinned():
                    raise ValueError("host layer weights must be in pinned memory")
        self.chunk = chunk_bytes
        lo, _hi = torch.cuda.Stream.priority_range()
        self.stream = torch.cuda.Stream(device=device, priority=lo)
        self.resident: dict[int, dict[str, "object"]] = {}
        self.events: dict[int, "object"] = {}
        self.pending: list[int] = []
        self.is_layer_committed = is_layer_committed or (lambda layer: False)
        self.staged_bytes = 0

    def layer_bytes(self, layer: int) -> int:
        return sum(t.numel() * t.element_size() for t in self.host[layer].values())

    def stage_layers(self, layers) -> None:
        """Enqueue every not-yet-resident layer (in layer order) on the copy stream."""
        torch = self.torch
        todo = sorted(l for l in layers if l not in self.resident)
        with torch.cuda.stream(self.stream):
            for layer in todo:
                dev = {}
                for name, src in self.host[layer].items():
                    dst = torch.empty(src.shape, dtype=src.dtype,
                                      device=torch.device("cuda", self.device))
                    flat_s = src.reshape(-1).view(torch.uint8)
                    flat_d = dst.reshape(-1).view(torch.uint8)
                    for o in range(0, flat_s.numel(), self.chunk):
                        flat_d[o:o + self.chunk].copy_(flat_s[o:o + self.chunk], non_blocking=True)
                    dev[name] = dst
                ev = torch.cuda.Event()
                ev.record(self.stream)
                self.resident[layer] = dev
                self.events[layer] = ev
                self.pending.append(layer)
                self.staged_bytes += self.layer_bytes(layer)

    def is_resident(self, layer: int) -> bool:
        """Staged and its copy has completed."""
        ev = self.events.get(layer)
        return layer in self.resident and (ev is None or ev.query())

    def staging_active(self) -> bool:
        self.pending = [l for l in self.pending if not self.events[l].query()]
        return bool(self.pending)

    def wait(self) -> float:
        """Block until every enqueued layer is resident; returns the wait in ms."""
        t0 = time.perf_counter()
        self.stream.synchronize()
        self.pending = []
        return (time.perf_counter() - t0) * 1e3

    def make_current_wait(self, stream) -> None:
        """Order `stream` (the compute stream) after every staged copy."""
        for ev in self.events.values():
            stream.wait_event(ev)

    def cancel_staging(self) -> None:
        """Layers already enqueued finish (a DMA in flight is not abortable); callers
        evict what they do not want, as in weights.py:155-165."""
        self.pending = []

    def evict_layers(self, layers) -> int:
        for layer in sorted(layers):
            if self.is_layer_committed(layer):
                raise LayerInUse(f"layer {layer} is committed")
        freed = 0
        self.stream.synchronize()
        for layer in sorted(set(layers) & set(self.resident)):
            freed += sum(t.numel() * t.element_size() for t in self.resident.pop(layer).values())
            self.events.pop(layer, None)
        return freed
