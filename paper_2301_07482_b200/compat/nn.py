"""histgnn.nn value types (nn.py:28-85) for callers that build networks by
hand; `to_device` packs one into the flat device buffer the kernels use
(`nn.network_from_numpy`). Layer math runs only on the device
(`paper_2301_07482_b200.nn`), in fp32.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .. import nn as _dn
from ..nn import LayerKind

__all__ = ["LayerKind", "LayerParams", "Network", "init_network", "to_device"]


@dataclass
class LayerParams:
    """weight: GCN projection or SAGE self projection; weight_neigh: SAGE only."""

    weight: np.ndarray
    bias: np.ndarray
    weight_neigh: np.ndarray | None = None

    def named_arrays(self):
        out = [("weight", self.weight), ("bias", self.bias)]
        if self.weight_neigh is not None:
            out.append(("weight_neigh", self.weight_neigh))
        return out

    def zeros_like(self) -> "LayerParams":
        return LayerParams(*(None if a is None else np.zeros_like(a)
                             for a in (self.weight, self.bias, self.weight_neigh)))


@dataclass
class Network:
    kind: LayerKind
    layers: list

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    @property
    def dtype(self):
        return self.layers[0].weight.dtype

    def checksum_bytes(self) -> bytes:
        return b"".join(np.ascontiguousarray(a).tobytes() for p in self.layers for _, a in p.named_arrays())


def init_network(kind: LayerKind, dims, rng: np.random.Generator, dtype=np.float32) -> Network:
    """Glorot-uniform weights (SAGE: self then neighbour draw per layer), zero
    biases: the reference's draw order, so weights are bit-identical."""
    layers = []
    for fi, fo in zip(dims[:-1], dims[1:]):
        lim = np.sqrt(6.0 / (fi + fo))
        w = rng.uniform(-lim, lim, size=(fi, fo)).astype(dtype)
        wn = rng.uniform(-lim, lim, size=(fi, fo)).astype(dtype) if kind is LayerKind.SAGE_MEAN else None
        layers.append(LayerParams(w, np.zeros(fo, dtype=dtype), wn))
    return Network(kind, layers)


def to_device(net, device=None) -> _dn.Network:
    """A device Network from a host (compat or reference-typed) one; device
    networks pass through. The device computes in fp32."""
    if isinstance(net, _dn.Network):
        return net
    arrays = []
    for p in net.layers:
        d = {"weight": np.asarray(p.weight, np.float32), "bias": np.asarray(p.bias, np.float32)}
        if getattr(p, "weight_neigh", None) is not None:
            d["weight_neigh"] = np.asarray(p.weight_neigh, np.float32)
        arrays.append(d)
    return _dn.network_from_numpy(net.kind if isinstance(net.kind, LayerKind) else LayerKind(net.kind.value),
                                  arrays, device=device)
