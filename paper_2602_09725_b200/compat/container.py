"""numpy facade of fk/container.py: pack/unpack on the GPU, numpy slabs."""

from __future__ import annotations

from .. import container as _C
from .. import layout as _L
from . import kvmodel as _K

HOT_PATH = ["ChunkContainer", "pack_chunk", "unpack_chunk", "parse_header", "container_filename",
            "DEFAULT_CHUNK_TOKENS", "MAGIC", "VERSION"]

ChunkContainer = _C.ChunkContainer
parse_header = _C.parse_header
container_filename = _C.container_filename
DEFAULT_CHUNK_TOKENS = _C.DEFAULT_CHUNK_TOKENS
MAGIC = _C.MAGIC
VERSION = _C.VERSION


def pack_chunk(q_slab, cfg_layout, resolutions, cache_id: bytes = b"\x00" * 16,
               chunk_index: int = 0, token_start: int = 0, layer_triplet_index: int = 0,
               F: int = _L.DEFAULT_GROUP_FRAMES,
               max_tokens: int = DEFAULT_CHUNK_TOKENS) -> ChunkContainer:
    """fk/container.py:160-209: GPU assemble + KVFC encode of a numpy slab."""
    q = _K.QuantizedKV(q_slab.values, q_slab.scales, q_slab.group_size).to_device()
    return _C.pack_chunk(q, cfg_layout, resolutions, cache_id, chunk_index, token_start,
                         layer_triplet_index, F, max_tokens)


def unpack_chunk(container: ChunkContainer, code: int):
    """fk/container.py:212-227: GPU decode + disassemble -> numpy QuantizedKV."""
    return _K.from_device(_C.unpack_chunk(container, code))
