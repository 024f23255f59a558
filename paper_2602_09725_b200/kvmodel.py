"""KV tensor model on the GPU: KVCache, int8 quantisation, paged block cache.

Drop-in mirror of the reference's fk/kvmodel.py with device tensors:
  * ``KVCache``      [token, layer, head, dim] bf16/fp16/fp32 (fk/kvmodel.py:22-78)
  * ``QuantizedKV``  int8 values + fp32 scales [layer, channel/group] (:81-124)
  * ``quantize`` / ``dequantize`` — libkvf kernels, bit-exact to the reference's
    fp64 numpy arithmetic (:127-152)
  * ``PagedMemory``  — the restore target.  The reference's page dict
    (page = token // page_size_tokens, slot = (token % page_size_tokens, layer),
    fk/kvmodel.py:195-244) becomes a vLLM-style per-layer block pool
    [num_blocks, block_size, H, D] plus a logical-page -> block table on the
    device.  Slot bookkeeping (write-once markers, ConflictError, byte
    accounting) is host metadata decided before any launch, so conflicts raise
    exactly as in the reference without reading device memory.
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import _dev, _lib


class ConflictError(RuntimeError):
    """A token slot was written twice within one fetch (fk/kvmodel.py:18-19)."""


class KVCache:
    """[token, layer, head, dim] floating-point tensor on the GPU."""

    def __init__(self, data):
        t = _dev.to_device(data)
        if not t.is_floating_point():
            t = t.float()
        if t.dim() != 4:
            raise ValueError("KVCache data must be [token, layer, head, dim]")
        if min(t.shape) < 1:
            raise ValueError("all four extents must be >= 1")
        self.data = t

    tokens = property(lambda self: self.data.shape[0])
    layers = property(lambda self: self.data.shape[1])
    H = property(lambda self: self.data.shape[2])
    D = property(lambda self: self.data.shape[3])
    channel = property(lambda self: self.H * self.D)
    N = channel

    def pad_layers(self) -> "KVCache":
        """Copy whose layer count is rounded up to a multiple of 3 with zero layers."""
        pad = (-self.layers) % 3
        if pad == 0:
            return KVCache(self.data.clone())
        zeros = torch.zeros((self.tokens, pad, self.H, self.D), dtype=self.data.dtype,
                            device=self.data.device)
        return KVCache(torch.cat([self.data, zeros], dim=1))

    def layer_triplet(self, index: int) -> torch.Tensor:
        if self.layers % 3:
            raise ValueError("pad_layers() first: layer count not a multiple of 3")
        lo = 3 * index
        if not 0 <= lo < self.layers:
            raise ValueError("triplet index out of range")
        return self.data[:, lo:lo + 3]


class QuantizedKV:
    """int8 codes [T, L, H, D] with fp32 scales [L, H*D/group_size] on the GPU."""

    def __init__(self, values, scales, group_size: int):
        v = _dev.to_device(values, torch.int8)
        s = _dev.to_device(scales, torch.float32)
        if v.dim() != 4:
            raise ValueError("values must be [token, layer, head, dim]")
        if tuple(s.shape) != (v.shape[1], (v.shape[2] * v.shape[3]) // group_size):
            raise ValueError("scales must be [layers, channel/group_size]")
        self.values, self.scales, self.group_size = v, s, group_size

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
        return QuantizedKV(self.values[:, lo:lo + 3], self.scales[lo:lo + 3],
                           self.group_size)


def quantize(kv: KVCache, group_size: int = 128) -> QuantizedKV:
    """Symmetric int8 per (layer, channel group) — bit-exact fk/kvmodel.py:127-144."""
    ch = kv.channel
    if group_size <= 0 or ch % group_size:
        raise ValueError("group_size must be positive and divide channel")
    x = kv.data.contiguous()
    T, L = kv.tokens, kv.layers
    G = ch // group_size
    absmax = torch.empty((L, G), dtype=torch.int32, device=x.device)
    scales = torch.empty((L, G), dtype=torch.float32, device=x.device)
    values = torch.empty(tuple(x.shape), dtype=torch.int8, device=x.device)
    _lib.call("kvf_quantize", _dev.ptr(x), _dev.dtype_code(x.dtype), T, L, ch, group_size,
              _dev.ptr(absmax), _dev.ptr(scales), _dev.ptr(values), _dev.stream_ptr())
    return QuantizedKV(values, scales, group_size)


def dequantize(q: QuantizedKV, dtype: torch.dtype = torch.float32) -> KVCache:
    """x_hat = int * scale (fk/kvmodel.py:147-152), rounded once to ``dtype``."""
    v = q.values.contiguous()
    out = torch.empty(tuple(v.shape), dtype=dtype, device=v.device)
    _lib.call("kvf_dequantize", _dev.ptr(v), _dev.ptr(q.scales.contiguous()), q.tokens,
              q.layers, q.channel, q.group_size, _dev.ptr(out), _dev.dtype_code(dtype),
              _dev.stream_ptr())
    return KVCache(out)


def gen_synthetic_kv(tokens, layers, H, D, token_smoothness, seed, channel_smoothness=0.0,
                     dtype: torch.dtype = torch.float32) -> KVCache:
    """On-GPU synthetic KV with the AR(1) law of fk/kvmodel.py:155-192.

    Same process (AR(1) along dims inside a head, then along tokens), drawn from
    torch's CUDA generator: statistically equivalent to the reference generator,
    not value-identical (parity fixtures come from the reference itself).
    """
    if min(tokens, layers, H, D) < 1:
        raise ValueError("all extents must be >= 1")
    if not 0.0 <= token_smoothness <= 1.0:
        raise ValueError("token_smoothness must be in [0, 1]")
    if not 0.0 <= channel_smoothness <= 1.0:
        raise ValueError("channel_smoothness must be in [0, 1]")
    dev = _dev.device()
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed))
    x = torch.randn((tokens, layers, H, D), generator=g, device=dev, dtype=torch.float32)
    if channel_smoothness > 0.0:
        _lib.call("kvf_ar1_scan", _dev.ptr(x), tokens * layers * H, D, 1,
                  float(channel_smoothness), _dev.stream_ptr())
    if tokens > 1:
        _lib.call("kvf_ar1_scan", _dev.ptr(x), 1, tokens, layers * H * D,
                  float(token_smoothness), _dev.stream_ptr())
    return KVCache(x if dtype == torch.float32 else x.to(dtype))


class PagedMemory:
    """Paged KV block cache with the reference PagedMemory's slot semantics.

    ``dtype=torch.int8`` stores the int8 codes exactly as the reference does;
    bf16/fp16/fp32 store dequantised values (restore fuses the dequantisation).
    Storage is allocated on first use: one [num_blocks, page_size, H, D] tensor
    per layer, a shared logical-page -> block table (int32, device), and a free
    list; the pool grows geometrically when it runs out of blocks.
    """

    def __init__(self, page_size_tokens: int = 16, dtype: torch.dtype = torch.int8,
                 H: int | None = None, D: int | None = None, num_blocks: int = 0,
                 num_layers: int = 0):
        if page_size_tokens <= 0:
            raise ValueError("page_size_tokens must be positive")
        self.page_size_tokens = page_size_tokens
        self.dtype = dtype
        _dev.dtype_code(dtype)
        self.H, self.D = H, D
        self.layers: list[torch.Tensor] = []   # per layer [cap_blocks, bs, H, D]
        self.pages: dict[int, int] = {}        # logical page -> physical block
        self._free: list[int] = []
        self._cap_blocks = 0
        self._table = None                     # device int32 [cap_pages]
        self._upload_stream = None
        self._table_host = np.zeros(0, np.int32)
        self._table_dirty = False
        self._written = np.zeros((0, 0), bool)   # [token, layer] write-once markers
        self._present = np.zeros((0, 0), bool)   # [token, layer] slot holds data
        self.allocated_bytes = 0
        self.peak_bytes = 0
        if H is not None and D is not None and (num_blocks or num_layers):
            self._ensure_layers(num_layers)
            self._ensure_blocks(num_blocks)

    # -------------------------------------------------------------- storage
    @property
    def slot_bytes(self) -> int:
        return self.H * self.D * torch.empty((), dtype=self.dtype).element_size()

    def _ensure_layers(self, n: int):
        dev = _dev.device()
        while len(self.layers) < n:
            self.layers.append(torch.empty((self._cap_blocks, self.page_size_tokens,
                                            self.H, self.D), dtype=self.dtype, device=dev))

    def _ensure_blocks(self, n: int):
        if n <= self._cap_blocks:
            return
        new_cap = max(n, 2 * self._cap_blocks, 16)
        if self._cap_blocks and self.layers:
            # restores already launched (any stream) may still write the old
            # pool: let them land before it is copied and released
            torch.cuda.synchronize()
        for k, t in enumerate(self.layers):
            grown = torch.empty((new_cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            grown[: t.shape[0]].copy_(t)
            self.layers[k] = grown
        if self._cap_blocks and self.layers:
            # the copies ran on the current stream; restores queued later on other
            # streams (a fetcher rotates several) must not overtake them, and the
            # old pools must not be recycled while a copy still reads them
            torch.cuda.synchronize()
        self._free.extend(range(new_cap - 1, self._cap_blocks - 1, -1))
        self._cap_blocks = new_cap

    def _grow_marks(self, tokens: int, layers: int):
        t0, l0 = self._written.shape
        if tokens <= t0 and layers <= l0:
            return
        nt = max(tokens, t0 * 2 if tokens > t0 else t0, 64)
        nl = max(layers, l0)
        for name in ("_written", "_present"):
            old = getattr(self, name)
            new = np.zeros((nt, nl), bool)
            new[:t0, :l0] = old
            setattr(self, name, new)

    def block_table(self) -> torch.Tensor:
        """Device int32 table logical page -> physical block (-1 = unmapped).

        A changed table is uploaded as a new tensor on an idle side stream (a
        pageable copy would otherwise wait for all work queued on the caller's
        stream) and the caller's stream waits for that upload only."""
        if self._table is None or self._table_dirty:
            if self._upload_stream is None:
                self._upload_stream = torch.cuda.Stream()
            host = torch.from_numpy(self._table_host.copy()).pin_memory()
            with torch.cuda.stream(self._upload_stream):
                self._table = host.to(_dev.device(), non_blocking=True)
                self._table_ready = torch.cuda.Event()
                self._table_ready.record(self._upload_stream)
            self._table_dirty = False
        # Every consumer stream (a fetcher runs batches on several) waits for the
        # upload and marks the table in use, so it is neither read early nor
        # recycled while a queued kernel on that stream still reads it.
        cur = torch.cuda.current_stream()
        cur.wait_event(self._table_ready)
        self._table.record_stream(cur)
        return self._table

    def _map_pages(self, first_page: int, last_page: int):
        pages = self.pages
        need = [p for p in range(first_page, last_page + 1) if p not in pages]
        if need:
            if len(self._free) < len(need):
                self._ensure_blocks(self._cap_blocks + len(need) - len(self._free))
            for p in need:
                self.pages[p] = self._free.pop()
            hi = last_page + 1
            if self._table_host.shape[0] < hi:
                grown = np.full(max(hi, 2 * self._table_host.shape[0]), -1, np.int32)
                grown[: self._table_host.shape[0]] = self._table_host
                self._table_host = grown
            for p in need:
                self._table_host[p] = self.pages[p]
            self._table_dirty = True

    # ----------------------------------------------------- reference API
    def begin_fetch(self) -> None:
        """Start a new fetch: clears write-once markers, keeps contents."""
        self._written[:] = False

    def _claim(self, tokens: np.ndarray, layers: list[int], H: int, D: int):
        """Reserve slots (tokens x layers) for one write: shape binding, conflict
        check, page mapping and byte accounting — all before any device work."""
        if len(tokens) == 0 or not layers:
            return
        if tokens.min() < 0 or min(layers) < 0:
            raise ValueError("negative slot coordinates")
        if self.H is None:
            self.H, self.D = H, D
        elif (self.H, self.D) != (H, D):
            raise ValueError(f"slot shape {(H, D)} differs from the cache's {(self.H, self.D)}")
        self._grow_marks(int(tokens.max()) + 1, max(layers) + 1)
        lo, hi = int(tokens.min()), int(tokens.max())
        # a whole chunk is a contiguous token range: slice instead of fancy-index
        rows = slice(lo, hi + 1) if hi - lo + 1 == len(tokens) else tokens
        idx = (rows, layers) if isinstance(rows, slice) else np.ix_(tokens, layers)
        hit = self._written[idx]
        if hit.any():
            ti, li = np.argwhere(hit)[0]
            raise ConflictError(
                f"slot (token={int(tokens[ti])}, layer={layers[li]}) already written")
        self._ensure_layers(max(layers) + 1)
        bs = self.page_size_tokens
        self._map_pages(lo // bs, hi // bs)
        self._written[idx] = True
        self._present[idx] = True
        self.allocated_bytes += len(tokens) * len(layers) * self.slot_bytes
        self.peak_bytes = max(self.peak_bytes, self.allocated_bytes)

    def page_write(self, token_index: int, layer: int, slot_data) -> None:
        """Write one slot (reference API, fk/kvmodel.py:216-229)."""
        data = _dev.to_device(slot_data)
        C = data.numel()
        if self.H is None:
            H, D = 1, C
        else:
            H, D = self.H, self.D
            if H * D != C:
                raise ValueError("slot data size does not match the cache")
        self._claim(np.array([token_index]), [layer], H, D)
        blk = self.pages[token_index // self.page_size_tokens]
        off = token_index % self.page_size_tokens
        self.layers[layer][blk, off].view(-1).copy_(data.reshape(-1).to(self.dtype))

    def free_page(self, page_index: int) -> None:
        blk = self.pages.pop(page_index, None)
        if blk is None:
            return
        bs = self.page_size_tokens
        lo, hi = page_index * bs, (page_index + 1) * bs
        hi = min(hi, self._present.shape[0])
        if hi > lo:
            n = int(self._present[lo:hi].sum())
            self.allocated_bytes -= n * self.slot_bytes
            self._present[lo:hi] = False
            self._written[lo:hi] = False
        self._free.append(blk)
        self._table_host[page_index] = -1
        self._table_dirty = True

    def read(self, token_index: int, layer: int) -> Optional[torch.Tensor]:
        """The slot's channel vector (device view) or None if never written."""
        if token_index < 0 or layer < 0:
            return None
        if token_index >= self._present.shape[0] or layer >= self._present.shape[1]:
            return None
        if not self._present[token_index, layer]:
            return None
        blk = self.pages[token_index // self.page_size_tokens]
        return self.layers[layer][blk, token_index % self.page_size_tokens].reshape(-1)

    # ------------------------------------------------------------ kernel view
    def paged_view(self, layer_base: int, token_base: int,
                   pad_mask=(False, False, False)) -> _lib.kvf_paged:
        """kvf_paged for layers layer_base..+2 (pad layers -> NULL)."""
        pg = _lib.kvf_paged()
        for p in range(3):
            pg.layer[p] = None if pad_mask[p] else self.layers[layer_base + p].data_ptr()
        pg.block_table = self.block_table().data_ptr()
        pg.block_size = self.page_size_tokens
        pg.dtype = _dev.dtype_code(self.dtype)
        pg.slot_stride = self.H * self.D
        pg.block_stride = self.page_size_tokens * self.H * self.D
        pg.head_stride = self.D
        pg.token_base = token_base
        return pg
