"""numpy facade of fk/kvmodel.py: host arrays in and out, quantisation on the GPU.

``KVCache`` / ``QuantizedKV`` hold numpy arrays with the reference's dtypes
and checks (fk/kvmodel.py:22-124); ``quantize`` / ``dequantize`` run the
libkvf kernels (bit-exact to fk/kvmodel.py:127-152); ``PagedMemory`` is the
device block-table cache (fk/kvmodel.py:195-244 semantics) whose ``read``
returns numpy.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import kvmodel as _K
from ._np import dev, host

HOT_PATH = ["KVCache", "QuantizedKV", "quantize", "dequantize", "PagedMemory", "ConflictError"]

ConflictError = _K.ConflictError


class KVCache:
    """float32 [token, layer, head, dim] host tensor (fk/kvmodel.py:22-78)."""

    def __init__(self, data):
        data = np.asarray(data, dtype=np.float32)
        if data.ndim != 4:
            raise ValueError("KVCache data must be [token, layer, head, dim]")
        if min(data.shape) < 1:
            raise ValueError("all four extents must be >= 1")
        self.data = data

    tokens = property(lambda self: self.data.shape[0])
    layers = property(lambda self: self.data.shape[1])
    H = property(lambda self: self.data.shape[2])
    D = property(lambda self: self.data.shape[3])
    channel = property(lambda self: self.H * self.D)
    N = channel

    def pad_layers(self) -> "KVCache":
        pad = (-self.layers) % 3
        zeros = np.zeros((self.tokens, pad, self.H, self.D), np.float32)
        return KVCache(np.concatenate([self.data, zeros], axis=1) if pad else self.data.copy())

    def layer_triplet(self, index: int) -> np.ndarray:
        if self.layers % 3:
            raise ValueError("pad_layers() first: layer count not a multiple of 3")
        lo = 3 * index
        if not 0 <= lo < self.layers:
            raise ValueError("triplet index out of range")
        return self.data[:, lo:lo + 3]


class QuantizedKV:
    """int8 [T, L, H, D] codes + float32 [L, channel/group_size] scales (fk/kvmodel.py:81-124)."""

    def __init__(self, values, scales, group_size: int):
        values = np.asarray(values, dtype=np.int8)
        scales = np.asarray(scales, dtype=np.float32)
        if values.ndim != 4:
            raise ValueError("values must be [token, layer, head, dim]")
        if scales.shape != (values.shape[1], (values.shape[2] * values.shape[3]) // group_size):
            raise ValueError("scales must be [layers, channel/group_size]")
        self.values, self.scales, self.group_size = values, scales, group_size

    tokens = property(lambda self: self.values.shape[0])
    layers = property(lambda self: self.values.shape[1])
    H = property(lambda self: self.values.shape[2])
    D = property(lambda self: self.values.shape[3])
    channel = property(lambda self: self.H * self.D)

    def layer_triplet(self, index: int) -> "QuantizedKV":
        if self.layers % 3:
            raise ValueError("layer count not a multiple of 3")
        lo = 3 * index
        if not 0 <= lo < self.layers:
            raise ValueError("triplet index out of range")
        return QuantizedKV(self.values[:, lo:lo + 3], self.scales[lo:lo + 3], self.group_size)

    def to_device(self) -> _K.QuantizedKV:
        return _K.QuantizedKV(dev(self.values), dev(self.scales), self.group_size)


def from_device(q: _K.QuantizedKV) -> QuantizedKV:
    return QuantizedKV(host(q.values), host(q.scales), q.group_size)


def quantize(kv, group_size: int = 128) -> QuantizedKV:
    """fk/kvmodel.py:127-144 on the GPU (kvf_quantize).  ``kv`` is any object
    with a [T, L, H, D] float ``data`` array (the reference's KVCache too)."""
    data = np.asarray(kv.data, np.float32)
    ch = data.shape[2] * data.shape[3]
    if group_size <= 0 or ch % group_size:
        raise ValueError("group_size must be positive and divide channel")
    return from_device(_K.quantize(_K.KVCache(dev(data)), group_size))


def dequantize(q) -> KVCache:
    """fk/kvmodel.py:147-152 on the GPU (kvf_dequantize), float32."""
    dq = _K.dequantize(_K.QuantizedKV(dev(q.values, np.int8), dev(q.scales, np.float32),
                                      q.group_size), torch.float32)
    return KVCache(host(dq.data))


def gen_synthetic_kv(tokens, layers, H, D, token_smoothness, seed, channel_smoothness=0.0):
    """The AR(1) generator law of fk/kvmodel.py:155-192 drawn on the GPU:
    statistically equivalent to the reference's, not value-identical."""
    return KVCache(host(_K.gen_synthetic_kv(tokens, layers, H, D, token_smoothness, seed,
                                             channel_smoothness).data))


class PagedMemory:
    """fk/kvmodel.py:195-244: write-once token slots, page = token // page_size.

    The slots live in the device block-table cache (``device``, int8 codes);
    ``read`` copies a slot back to numpy."""

    def __init__(self, page_size_tokens: int = 16):
        self.device = _K.PagedMemory(page_size_tokens, dtype=torch.int8)

    page_size_tokens = property(lambda self: self.device.page_size_tokens)
    pages = property(lambda self: self.device.pages)
    allocated_bytes = property(lambda self: self.device.allocated_bytes)
    peak_bytes = property(lambda self: self.device.peak_bytes)

    def begin_fetch(self) -> None:
        self.device.begin_fetch()

    def page_write(self, token_index: int, layer: int, slot_data) -> None:
        self.device.page_write(token_index, layer, dev(np.asarray(slot_data)))

    def free_page(self, page_index: int) -> None:
        self.device.free_page(page_index)

    def read(self, token_index: int, layer: int):
        got = self.device.read(token_index, layer)
        return None if got is None else host(got)
