"""Frame-wise restore: decoded frames -> (dequantised) paged KV cache on the GPU.

Mirrors fk/fetchsim.py:335-385 (restore_stream / restore_chunk_wise).  The
per-frame ``on_frame`` callback of the reference (fk/fetchsim.py:347-355:
frame_slots -> tile -> -128 -> inverse_layout -> 3 x page_write) is one libkvf
launch per frame batch (kvf_restore), fused with the dequantisation
(fk/kvmodel.py:147-152) when the cache holds bf16/fp16/fp32.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .layout import FramePlan
from .kvmodel import PagedMemory


def _pad_mask(mem: PagedMemory, layer_base: int, real_layers: int | None):
    if real_layers is None:
        return (False, False, False)
    return tuple(layer_base + p >= real_layers for p in range(3))


class RestoreUnit:
    """One chunk's restore: slots claimed in the PagedMemory (write-once check,
    page mapping, byte accounting — host side, as the reference's page_write,
    fk/kvmodel.py:216-229), then a kvf_restore_unit descriptor built by
    ``describe()``.  Claim every unit of a batch before describing any: a claim
    may grow the cache's block pool, which moves its storage."""

    def __init__(self, frames, plan, mem, layer_base, token_base, scales, real_layers,
                 first_frame, n_frames):
        n_frames = plan.frame_count - first_frame if n_frames is None else n_frames
        if frames.shape[0] == plan.frame_count:
            base_frame = 0
        elif frames.shape[0] == n_frames:
            base_frame = first_frame
        else:
            raise ValueError("frames must hold the restored range or the whole chunk")
        cfg = plan.cfg
        self.pad = _pad_mask(mem, layer_base, real_layers)
        toks = np.asarray(plan.tokens_in_frames(first_frame, n_frames), np.int64) + token_base
        mem._claim(toks, [layer_base + p for p in range(3) if not self.pad[p]], cfg.H, cfg.D)
        self.scales = None
        if mem.dtype != torch.int8:
            if scales is None:
                raise ValueError("a dequantising restore needs the chunk scales")
            self.scales = _dev.to_device(scales, torch.float32).contiguous()
            self.group_size = (cfg.H * cfg.D) // self.scales.shape[1]
        else:
            self.group_size = (cfg.H * cfg.D if scales is None
                               else (cfg.H * cfg.D) // np.shape(scales)[1])
        self.frames, self.plan, self.mem = frames, plan, mem
        self.layer_base, self.token_base = layer_base, token_base
        self.first_frame, self.n_frames, self.base_frame = first_frame, max(n_frames, 0), base_frame
        self.tokens_written = len(toks)
        self.desc = None

    def describe(self) -> _lib.kvf_restore_unit:
        u = _lib.kvf_restore_unit()
        u.frames = _dev.surface_of(self.frames)
        # Shift the surface so frame index first_frame maps onto frames[0].
        u.frames.base = u.frames.base - self.base_frame * u.frames.frame_stride
        u.plan = self.plan.to_c(self.group_size)
        u.scales = None if self.scales is None else self.scales.data_ptr()
        u.dst = self.mem.paged_view(self.layer_base, self.token_base, self.pad)
        self._table = self.mem.block_table()   # the descriptor points into it
        u.first_frame = self.first_frame
        u.n_frames = self.n_frames
        self.desc = u
        return u


def restore_unit(frames: torch.Tensor, plan: FramePlan, mem: PagedMemory, layer_base: int = 0,
                 token_base: int = 0, scales=None, real_layers: int | None = None,
                 first_frame: int = 0, n_frames: int | None = None) -> RestoreUnit:
    """Claim the slots of frames [first_frame, first_frame + n_frames) of one
    chunk (``frames`` holds exactly those frames or the whole chunk); describe
    it later with RestoreUnit.describe() / restore_units."""
    return RestoreUnit(frames, plan, mem, layer_base, token_base, scales, real_layers,
                       first_frame, n_frames)


def restore_frames(frames: torch.Tensor, plan: FramePlan, mem: PagedMemory,
                   layer_base: int = 0, token_base: int = 0, scales=None,
                   first_frame: int = 0, n_frames: int | None = None,
                   real_layers: int | None = None, stream=None) -> int:
    """Restore frames [first_frame, first_frame + n_frames) of one chunk.

    ``frames`` is a [n, 3, h, w] uint8 CUDA tensor holding exactly those frames
    (n == n_frames) or the whole chunk (n == plan.frame_count).  ``scales`` are
    the chunk's [3, G] scales (needed unless the cache holds int8 codes).
    Layers >= ``real_layers`` are pad layers (fk/kvmodel.py:56-69) and are not
    written.  Returns the number of tokens written.
    """
    n_frames = plan.frame_count - first_frame if n_frames is None else n_frames
    if n_frames <= 0:
        return 0
    ru = restore_unit(frames, plan, mem, layer_base, token_base, scales, real_layers,
                      first_frame, n_frames)
    restore_units([ru], stream)
    return ru.tokens_written


def _chain_batches(ix, batch_frames):
    """Frame ranges of at least batch_frames frames, each starting at an intra frame."""
    starts = [f for f in range(ix.n) if ix.frame_type[f] == 0]
    out, f0 = [], 0
    for s in starts[1:] + [ix.n]:
        if s - f0 >= batch_frames or s == ix.n:
            out.append((f0, s))
            f0 = s
    return [r for r in out if r[1] > r[0]]


def restore_stream(bs, plan: FramePlan, cfg_layout, mem: PagedMemory, layer_base=0,
                   token_base=0, *, scales=None, batch_frames=None, real_layers=None):
    """Frame-wise restore of one KVFC stream into paged memory (fk/fetchsim.py:335-358).

    Default (``batch_frames=None``): the reference's On_frame_probe.  The GPU
    decodes the stream frame by frame (codec.decode_stream_framewise: only the
    current frame and its reference are held) and each decoded frame's tile
    slots are restored with one libkvf launch as soon as it is reconstructed
    (un-tile, -128, dequantise with ``scales`` unless the cache holds int8
    codes, paged scatter).  ``batch_frames=k`` decodes runs of >= k frames
    that start at intra frames in one decode_batch each (more decoder
    parallelism, more live frames).  Returns {"tokens_written",
    "peak_buffer_bytes"} with the reference's peak: decoded-frame bytes
    retained at once (fk/codec.py:203-210).
    """
    from . import codec

    data = codec._as_bytes(bs)
    ix = codec.StreamIndex(data)
    if (ix.n, ix.h, ix.w) != (plan.frame_count, plan.frame_h, plan.frame_w):
        raise ValueError("stream geometry does not match the plan")
    frame_bytes = 3 * ix.h * ix.w
    if batch_frames is None:
        if scales is not None and mem.dtype != torch.int8:
            scales = _dev.to_device(scales, torch.float32).contiguous()
        written = [0]

        def on_frame(f, frame):
            written[0] += restore_frames(frame[None], plan, mem, layer_base, token_base,
                                         scales=scales, first_frame=f, n_frames=1,
                                         real_layers=real_layers)

        n = codec.decode_stream_framewise(data, on_frame, index=ix)
        return {"tokens_written": written[0], "peak_buffer_bytes": min(n, 2) * frame_bytes}
    written, peak = 0, 0
    for f0, f1 in _chain_batches(ix, int(batch_frames)):
        frames, _ = codec.decode_batch([data], ranges=[(f0, f1)], indices=[ix])
        peak = max(peak, (f1 - f0) * frame_bytes)
        written += restore_frames(frames[0], plan, mem, layer_base, token_base, scales=scales,
                                  first_frame=f0, n_frames=f1 - f0, real_layers=real_layers)
    return {"tokens_written": written, "peak_buffer_bytes": peak}


def restore_chunk_wise(bs, plan: FramePlan, cfg_layout, mem: PagedMemory, layer_base=0,
                       token_base=0, *, scales=None, real_layers=None):
    """Baseline: decode every frame, then restore (fk/fetchsim.py:361-385).
    peak_buffer_bytes is the reference's: every decoded frame plus the
    decoder's reference frame."""
    from . import codec

    frames, _ = codec.decode_batch([bs])
    written = restore_frames(frames[0], plan, mem, layer_base, token_base, scales=scales,
                             real_layers=real_layers)
    n = frames[0].shape[0]
    return {"tokens_written": written,
            "peak_buffer_bytes": (n + 1) * frames[0][0].numel() if n else 0}


def restore_units(units, stream=None) -> None:
    """Batched restore of prepared units (RestoreUnit or raw kvf_restore_unit
    descriptors) in one libkvf call — one launch per 128 units."""
    descs = [u.describe() if isinstance(u, RestoreUnit) else u for u in units]
    if not descs:
        return
    arr = (_lib.kvf_restore_unit * len(descs))(*descs)
    _lib.call("kvf_restore_batch", arr, len(descs), _dev.stream_ptr(stream))


def make_restore_unit(frames: torch.Tensor, plan: FramePlan, scales: torch.Tensor | None,
                      dst: _lib.kvf_paged, group_size: int, first_frame: int = 0,
                      n_frames: int | None = None) -> _lib.kvf_restore_unit:
    u = _lib.kvf_restore_unit()
    u.frames = _dev.surface_of(frames)
    u.plan = plan.to_c(group_size)
    u.scales = None if scales is None else scales.data_ptr()
    u.dst = dst
    u.first_frame = first_frame
    u.n_frames = plan.frame_count - first_frame if n_frames is None else n_frames
    return u
