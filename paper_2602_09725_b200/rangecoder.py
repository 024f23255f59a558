"""Adaptive range coder on the GPU (drop-in for the reference fk/rangecoder.py).

``encode_bytes`` / ``decode_bytes`` keep the reference signatures
(fk/rangecoder.py:205-219) and produce / consume the identical byte streams;
the batched forms code many independent streams in one launch, one GPU thread
per stream (kvf_rc_encode / kvf_rc_decode: adaptive order-0 model reset per
stream, INC 32, halving at 2^16, carry-less 32-bit range coder).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .codec import _RC_DTYPE

MASK = 0xFFFFFFFF
TOP = 1 << 24
BOT = 1 << 16
ALPHABET = 256
INC = 32
TOTAL_LIMIT = 1 << 16


def _descs(payload_ptrs, lens, sym_ptrs, counts, dev):
    d = np.empty(len(lens), _RC_DTYPE)
    d["payload"], d["len"], d["symbols"], d["n_symbols"] = payload_ptrs, lens, sym_ptrs, counts
    return torch.from_numpy(d.view(np.uint8)).pin_memory().to(dev, non_blocking=True)


def encode_batch(symbol_arrays) -> list[bytes]:
    """Range-code each uint8 symbol array (one stream each); returns the streams."""
    dev = _dev.device()
    arrs = [np.ascontiguousarray(a, np.uint8).ravel() for a in symbol_arrays]
    n = [len(a) for a in arrs]
    sym_off = np.concatenate([[0], np.cumsum(n)]).astype(np.int64)
    cap = [2 * k + 16 for k in n]
    cap_off = np.concatenate([[0], np.cumsum(cap)]).astype(np.int64)
    sym = _dev.to_device(np.concatenate(arrs) if arrs and sum(n) else np.zeros(1, np.uint8))
    out = torch.empty(max(int(cap_off[-1]), 1), dtype=torch.uint8, device=dev)
    lens = torch.zeros(max(len(arrs), 1), dtype=torch.int64, device=dev)
    d = _descs(out.data_ptr() + cap_off[:-1], np.zeros(len(arrs), np.int64),
               sym.data_ptr() + sym_off[:-1], np.asarray(n, np.int64), dev)
    _lib.call("kvf_rc_encode", _dev.ptr(d), len(arrs), _dev.ptr(lens), _dev.stream_ptr())
    host, ln = out.cpu().numpy(), lens.cpu().numpy()
    return [host[cap_off[k]:cap_off[k] + ln[k]].tobytes() for k in range(len(arrs))]


def decode_batch(streams, n_symbols) -> list[np.ndarray]:
    """Decode each (bytes, count) stream; reads past a stream's end yield 0."""
    dev = _dev.device()
    datas = [bytes(s) for s in streams]
    n = [int(k) for k in n_symbols]
    off = np.concatenate([[0], np.cumsum([len(x) for x in datas])]).astype(np.int64)
    n4 = [-(-k // 4) * 4 for k in n]
    sym_off = np.concatenate([[0], np.cumsum(n4)]).astype(np.int64)
    blob = _dev.to_device(np.frombuffer(b"".join(datas) + b"\0", np.uint8))
    sym = torch.empty(max(int(sym_off[-1]), 1), dtype=torch.uint8, device=dev)
    d = _descs(blob.data_ptr() + off[:-1], np.diff(off), sym.data_ptr() + sym_off[:-1],
               np.asarray(n, np.int64), dev)
    _lib.call("kvf_rc_decode", _dev.ptr(d), len(datas), _dev.stream_ptr())
    host = sym.cpu().numpy()
    return [host[sym_off[k]:sym_off[k] + n[k]].copy() for k in range(len(datas))]


def encode_bytes(symbols) -> bytes:
    """fk/rangecoder.py:205-211: uint8 symbols -> coded bytes."""
    return encode_batch([symbols])[0]


def decode_bytes(data, n_symbols: int) -> np.ndarray:
    """fk/rangecoder.py:214-219: coded bytes -> n_symbols uint8 symbols."""
    if n_symbols < 0:
        raise ValueError("n_symbols must be non-negative")
    return decode_batch([data], [n_symbols])[0]
