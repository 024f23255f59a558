"""Token -> frame layout: tiling configs, frame plans, and GPU (dis)assembly.

Host mirror of the reference's fk/layout.py (layout metadata is pure integer
arithmetic and stays on the host); the two data movers, ``assemble_frames``
(fk/layout.py:234-258) and ``disassemble_frames`` (fk/layout.py:261-271), run as
sm_100a kernels through libkvf (kvf_pack_frames / kvf_restore with int8 codes).

Tile mapping (fk/layout.py:31-36): channel element (h, d) with
h = i_h*b_h + j_h and d = i_d*b_d + j_d sits at tile row i_h*a_d + i_d and
tile column j_h*b_d + j_d.  Placement (fk/layout.py:157-201): tokens go F at a
time into one tile slot over F consecutive frames; a segment of F frames holds
tiles_per_frame such groups.
"""

from __future__ import annotations

import hashlib

import numpy as np

import torch

from . import _dev, _lib

RESOLUTION_TILES = {"R240": 16, "R480": 64, "R640": 96, "R1080": 256}
RESOLUTION_GRIDS = {"R240": (4, 4), "R480": (8, 8), "R640": (8, 12), "R1080": (16, 16)}
RESOLUTION_ORDER = ["R240", "R480", "R640", "R1080"]
RESOLUTION_CODE = {name: code for code, name in enumerate(RESOLUTION_ORDER)}
DEFAULT_GROUP_FRAMES = 4
PAD_BYTE = 128  # u8 encoding of the quantised zero


def _pow2(n: int) -> bool:
    return n >= 1 and n & (n - 1) == 0


def _factor_pairs(n: int):
    a = 1
    while a <= n:
        yield a, n // a
        a <<= 1


class LayoutConfig:
    """Intra-frame tiling of the (H, D) channel block (fk/layout.py:31-86)."""

    def __init__(self, H, D, a_h, b_h, a_d, b_d):
        if not (_pow2(H) and _pow2(D)):
            raise ValueError("H and D must be powers of two")
        if a_h * b_h != H or a_d * b_d != D:
            raise ValueError("factor pairs must multiply back to H and D")
        if not all(_pow2(v) for v in (a_h, b_h, a_d, b_d)):
            raise ValueError("factors must be powers of two")
        self.H, self.D = H, D
        self.a_h, self.b_h, self.a_d, self.b_d = a_h, b_h, a_d, b_d
        self.tile_h = a_h * a_d
        self.tile_w = b_h * b_d

    def _ident(self):
        return (self.H, self.D, self.a_h, self.b_h, self.a_d, self.b_d)

    def key(self):
        return (self.tile_h, self.tile_w, self.a_h, self.a_d)

    def __eq__(self, other):
        return isinstance(other, LayoutConfig) and self._ident() == other._ident()

    def __hash__(self):
        return hash(self._ident())

    def __repr__(self):
        return (f"LayoutConfig(H={self.H},D={self.D},h=({self.a_h},{self.b_h}),"
                f"d=({self.a_d},{self.b_d}),tile={self.tile_h}x{self.tile_w})")

    def to_json(self):
        return {"H": self.H, "D": self.D, "a_h": self.a_h, "b_h": self.b_h,
                "a_d": self.a_d, "b_d": self.b_d, "tile_h": self.tile_h,
                "tile_w": self.tile_w, "resolution_tiles": dict(RESOLUTION_TILES)}

    @classmethod
    def from_json(cls, obj):
        return cls(obj["H"], obj["D"], obj["a_h"], obj["b_h"], obj["a_d"], obj["b_d"])


def identity_layout(H, D):
    """One tile row holding the flat channel vector (fk/layout.py:89-91)."""
    return LayoutConfig(H, D, 1, H, 1, D)


def paper_layout(H, D):
    """Head-per-row tile (a_h, b_h, a_d, b_d) = (H, 1, 1, D): tile H x D."""
    return LayoutConfig(H, D, H, 1, 1, D)


def tiling_candidates(H, D):
    """All power-of-two factorisations of H x those of D (fk/layout.py:94-106)."""
    if not (_pow2(H) and _pow2(D)):
        raise ValueError("H and D must be powers of two")
    return [LayoutConfig(H, D, a_h, b_h, a_d, b_d)
            for a_h, b_h in _factor_pairs(H) for a_d, b_d in _factor_pairs(D)]


def _grid_for(tiles):
    rows = int(tiles ** 0.5)
    while tiles % rows:
        rows -= 1
    return rows, tiles // rows


class FramePlan:
    """Placement of T token tensors into frames of one resolution class."""

    def __init__(self, T, resolution_class, cfg: LayoutConfig, F=DEFAULT_GROUP_FRAMES):
        if T < 1:
            raise ValueError("T must be >= 1")
        if F < 1:
            raise ValueError("F must be >= 1")
        if isinstance(resolution_class, str):
            if resolution_class not in RESOLUTION_TILES:
                raise ValueError(f"unknown resolution class {resolution_class!r}")
            self.resolution_class = resolution_class
            self.tiles_per_frame = RESOLUTION_TILES[resolution_class]
            self.grid_rows, self.grid_cols = RESOLUTION_GRIDS[resolution_class]
        else:
            self.tiles_per_frame = int(resolution_class)
            if self.tiles_per_frame < 1:
                raise ValueError("tiles_per_frame must be >= 1")
            self.resolution_class = f"T{self.tiles_per_frame}"
            self.grid_rows, self.grid_cols = _grid_for(self.tiles_per_frame)
        self.T, self.F, self.K = T, F, F
        self.cfg = cfg
        self.tile_h, self.tile_w = cfg.tile_h, cfg.tile_w
        self.frame_h = self.grid_rows * cfg.tile_h
        self.frame_w = self.grid_cols * cfg.tile_w
        per_segment = F * self.tiles_per_frame
        full, rem = divmod(T, per_segment)
        self.frame_count = full * F + (min(rem, F) if rem else 0)

    def placement(self, i):
        """token index -> (frame, tile_row, tile_col)."""
        if not 0 <= i < self.T:
            raise ValueError("tensor index out of range")
        group, o = divmod(i, self.F)
        seg, slot = divmod(group, self.tiles_per_frame)
        return seg * self.F + o, slot // self.grid_cols, slot % self.grid_cols

    def frame_slots(self, frame_index):
        """Valid (token, tile_row, tile_col) triples of one frame."""
        seg, o = divmod(frame_index, self.F)
        first_group = seg * self.tiles_per_frame
        out = []
        for slot in range(self.tiles_per_frame):
            i = (first_group + slot) * self.F + o
            if i >= self.T:
                continue
            out.append((i, slot // self.grid_cols, slot % self.grid_cols))
        return out

    def tokens_in_frames(self, first, n):
        """Chunk token indices held by frames [first, first+n) (sorted int64 array)."""
        if first <= 0 and first + n >= self.frame_count:
            return np.arange(self.T, dtype=np.int64)       # the whole chunk
        f = np.arange(first, first + n, dtype=np.int64)[:, None]
        slot = np.arange(self.tiles_per_frame, dtype=np.int64)[None, :]
        i = ((f // self.F) * self.tiles_per_frame + slot) * self.F + f % self.F
        return np.sort(i[i < self.T])

    def digest(self):
        key = (f"{self.T}/{self.F}/{self.K}/{self.tiles_per_frame}/"
               f"{self.grid_rows}x{self.grid_cols}/{self.tile_h}x{self.tile_w}")
        return hashlib.sha256(key.encode()).hexdigest()[:16]

    def frame_shape(self):
        return (self.frame_count, 3, self.frame_h, self.frame_w)

    def to_c(self, group_size: int) -> _lib.kvf_plan:
        """kvf_plan of this plan; libkvf re-validates and derives the frame fields."""
        c = self.cfg
        p = _lib.kvf_plan(self.T, c.H, c.D, c.a_h, c.b_h, c.a_d, c.b_d, self.F,
                          self.tiles_per_frame, self.grid_rows, self.grid_cols,
                          0, 0, 0, int(group_size))
        _lib.call("kvf_plan_init", p)
        assert (p.frame_h, p.frame_w, p.frame_count) == (self.frame_h, self.frame_w,
                                                        self.frame_count)
        return p


def plan_inter_frame(T, resolution_class, cfg: LayoutConfig, F=DEFAULT_GROUP_FRAMES):
    plan = FramePlan(T, resolution_class, cfg, F)
    if plan.tile_h > plan.frame_h or plan.tile_w > plan.frame_w:
        raise ValueError("tile does not fit the frame")
    return plan


# ---------------------------------------------------------------- tensor views

def slice_tokens(q, triplet_index: int = 0) -> torch.Tensor:
    """[tokens, 3, channel] int8 view of one layer triplet (fk/layout.py:109-114)."""
    slab = q.layer_triplet(triplet_index) if q.layers != 3 else q
    if slab.layers != 3:
        raise ValueError("slab must have exactly 3 layers")
    return slab.values.reshape(slab.tokens, 3, slab.channel)


def unslice_tokens(tensors, H, D) -> torch.Tensor:
    t = _dev.to_device(tensors, torch.int8)
    return t.reshape(t.shape[0], 3, H, D)


def apply_layout(tensor, cfg: LayoutConfig) -> torch.Tensor:
    """[1, 3, channel] or [3, channel] -> [3, tile_h, tile_w] (single token view op)."""
    t = _dev.to_device(tensor)
    if t.dim() == 3 and t.shape[0] == 1:
        t = t[0]
    if tuple(t.shape) != (3, cfg.H * cfg.D):
        raise ValueError("tensor must be [1, 3, H*D]")
    return (t.reshape(3, cfg.a_h, cfg.b_h, cfg.a_d, cfg.b_d)
            .permute(0, 1, 3, 2, 4).reshape(3, cfg.tile_h, cfg.tile_w))


def inverse_layout(tile, cfg: LayoutConfig) -> torch.Tensor:
    """[3, tile_h, tile_w] -> [1, 3, channel]."""
    y = _dev.to_device(tile)
    if tuple(y.shape) != (3, cfg.tile_h, cfg.tile_w):
        raise ValueError("tile must be [3, tile_h, tile_w]")
    return (y.reshape(3, cfg.a_h, cfg.a_d, cfg.b_h, cfg.b_d)
            .permute(0, 1, 3, 2, 4).reshape(1, 3, cfg.H * cfg.D))


# ---------------------------------------------------------- GPU frame movers

def _codes_as_paged(t: torch.Tensor, cfg: LayoutConfig) -> _lib.kvf_paged:
    """kvf_paged view of a [T, 3, channel] int8 tensor (token-strided)."""
    if t.dim() != 3 or t.shape[1] != 3 or t.shape[2] != cfg.H * cfg.D:
        raise ValueError("tensors must be [T, 3, H*D]")
    if t.stride(2) != 1:
        raise ValueError("channel axis must be contiguous")
    pg = _lib.kvf_paged()
    for p in range(3):
        pg.layer[p] = _dev.addr(t, p * t.stride(1))
    pg.block_table = None
    pg.block_size = 1
    pg.dtype = _dev.dtype_code(t.dtype)
    pg.block_stride = t.stride(0)
    pg.slot_stride = t.stride(0)
    pg.head_stride = cfg.D
    pg.token_base = 0
    return pg


def assemble_frames(tensors, plan: FramePlan, out: torch.Tensor | None = None) -> torch.Tensor:
    """[T, 3, channel] int8 -> [frame_count, 3, frame_h, frame_w] uint8 on the GPU."""
    t = _dev.to_device(tensors)
    if t.dtype != torch.int8:
        raise ValueError("assemble_frames takes int8 codes")
    if t.shape[0] != plan.T:
        raise ValueError("tensor count does not match plan")
    if out is None:
        out = torch.empty(plan.frame_shape(), dtype=torch.uint8, device=t.device)
    src = _codes_as_paged(t, plan.cfg)
    _lib.call("kvf_pack_frames", src, plan.to_c(plan.cfg.H * plan.cfg.D), None, None,
              _dev.surface_of(out), _dev.stream_ptr())
    return out


def disassemble_frames(frames, plan: FramePlan, out: torch.Tensor | None = None) -> torch.Tensor:
    """Inverse of assemble_frames: [T, 3, channel] int8 on the GPU."""
    fr = _dev.to_device(frames, torch.uint8)
    if tuple(fr.shape) != plan.frame_shape():
        raise ValueError(f"frames must be {plan.frame_shape()}")
    if out is None:
        out = torch.empty((plan.T, 3, plan.cfg.H * plan.cfg.D), dtype=torch.int8,
                          device=fr.device)
    dst = _codes_as_paged(out, plan.cfg)
    _lib.call("kvf_restore", _dev.surface_of(fr), 0, plan.frame_count,
              plan.to_c(plan.cfg.H * plan.cfg.D), None, dst, _dev.stream_ptr())
    return out
