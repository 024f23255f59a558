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
    if frames.shape[0] == plan.frame_count:
        base_frame = 0
    elif frames.shape[0] == n_frames:
        base_frame = first_frame
    else:
        raise ValueError("frames must hold the restored range or the whole chunk")
    cfg = plan.cfg
    pad = _pad_mask(mem, layer_base, real_layers)
    toks = np.asarray(plan.tokens_in_frames(first_frame, n_frames), np.int64) + token_base
    mem._claim(toks, [layer_base + p for p in range(3) if not pad[p]], cfg.H, cfg.D)
    G_scales = None
    if mem.dtype != torch.int8:
        if scales is None:
            raise ValueError("a dequantising restore needs the chunk scales")
        G_scales = _dev.to_device(scales, torch.float32).contiguous()
        group_size = (cfg.H * cfg.D) // G_scales.shape[1]
    else:
        group_size = cfg.H * cfg.D if scales is None else (cfg.H * cfg.D) // np.shape(scales)[1]
    surf = _dev.surface_of(frames)
    # Shift the surface so frame index first_frame maps onto frames[0].
    surf.base = surf.base - base_frame * surf.frame_stride
    dst = mem.paged_view(layer_base, token_base, pad)
    _lib.call("kvf_restore", surf, first_frame, n_frames, plan.to_c(group_size),
              _dev.ptr(G_scales), dst, _dev.stream_ptr(stream))
    return len(toks)


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

    Decodes on the GPU and restores each decoded frame batch with one libkvf
    launch.  ``batch_frames=None`` decodes the whole chunk at once (maximum
    decoder parallelism); a small value (e.g. plan.F) bounds the live decode
    buffers to that many frames, the reference's frame-wise memory profile.
    Returns {"tokens_written", "peak_buffer_bytes"} like the reference.
    """
    from . import codec

    data = codec._as_bytes(bs)
    ix = codec.StreamIndex(data)
    if (ix.n, ix.h, ix.w) != (plan.frame_count, plan.frame_h, plan.frame_w):
        raise ValueError("stream geometry does not match the plan")
    ranges = [(0, ix.n)] if batch_frames is None else _chain_batches(ix, int(batch_frames))
    written, peak = 0, 0
    for f0, f1 in ranges:
        frames, held = codec.decode_batch([data], ranges=[(f0, f1)], indices=[ix])
        peak = max(peak, held)
        written += restore_frames(frames[0], plan, mem, layer_base, token_base, scales=scales,
                                  first_frame=f0, n_frames=f1 - f0, real_layers=real_layers)
    return {"tokens_written": written, "peak_buffer_bytes": peak}


def restore_chunk_wise(bs, plan: FramePlan, cfg_layout, mem: PagedMemory, layer_base=0,
                       token_base=0, *, scales=None, real_layers=None):
    """Baseline: decode every frame, then restore (fk/fetchsim.py:361-385)."""
    from . import codec

    frames, held = codec.decode_batch([bs])
    written = restore_frames(frames[0], plan, mem, layer_base, token_base, scales=scales,
                             real_layers=real_layers)
    return {"tokens_written": written, "peak_buffer_bytes": held}


def restore_units(units, stream=None) -> None:
    """Batched restore of prepared kvf_restore_unit descriptors (one call, few launches)."""
    arr = (_lib.kvf_restore_unit * len(units))(*units)
    _lib.call("kvf_restore_batch", arr, len(units), _dev.stream_ptr(stream))


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
