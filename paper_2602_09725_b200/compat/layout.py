"""numpy facade of fk/layout.py: layout metadata (host integer arithmetic, the
device package's classes) and the frame movers on the GPU with numpy I/O."""

from __future__ import annotations

import numpy as np

from .. import layout as _L
from ._np import dev, host

HOT_PATH = ["LayoutConfig", "FramePlan", "plan_inter_frame", "identity_layout",
            "tiling_candidates", "apply_layout", "inverse_layout", "slice_tokens",
            "unslice_tokens", "assemble_frames", "disassemble_frames", "RESOLUTION_TILES",
            "RESOLUTION_GRIDS", "RESOLUTION_ORDER", "RESOLUTION_CODE", "PAD_BYTE"]

LayoutConfig = _L.LayoutConfig
FramePlan = _L.FramePlan
plan_inter_frame = _L.plan_inter_frame
identity_layout = _L.identity_layout
paper_layout = _L.paper_layout
tiling_candidates = _L.tiling_candidates
RESOLUTION_TILES = _L.RESOLUTION_TILES
RESOLUTION_GRIDS = _L.RESOLUTION_GRIDS
RESOLUTION_ORDER = _L.RESOLUTION_ORDER
RESOLUTION_CODE = _L.RESOLUTION_CODE
DEFAULT_GROUP_FRAMES = _L.DEFAULT_GROUP_FRAMES
PAD_BYTE = _L.PAD_BYTE


def slice_tokens(q, triplet_index: int = 0) -> np.ndarray:
    """[tokens, 3, channel] int8 view of one layer triplet (fk/layout.py:109-114)."""
    slab = q.layer_triplet(triplet_index) if q.layers != 3 else q
    return slab.values.reshape(slab.tokens, 3, slab.channel)


def unslice_tokens(tensors, H, D) -> np.ndarray:
    t = np.asarray(tensors)
    return t.reshape(t.shape[0], 3, H, D)


def apply_layout(tensor, cfg) -> np.ndarray:
    return host(_L.apply_layout(dev(tensor), cfg))


def inverse_layout(tile, cfg) -> np.ndarray:
    return host(_L.inverse_layout(dev(tile), cfg))


def assemble_frames(tensors, plan) -> np.ndarray:
    """fk/layout.py:234-258 on the GPU (kvf_pack_frames with int8 codes)."""
    t = np.asarray(tensors)
    if t.dtype != np.int8:
        raise ValueError("assemble_frames takes int8 codes")
    return host(_L.assemble_frames(dev(t), plan))


def disassemble_frames(frames, plan) -> np.ndarray:
    """fk/layout.py:261-271 on the GPU (kvf_restore into int8 codes)."""
    return host(_L.disassemble_frames(dev(np.asarray(frames, np.uint8)), plan))
