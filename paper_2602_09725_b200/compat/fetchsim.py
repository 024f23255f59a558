"""numpy facade of the fk/fetchsim.py restore paths and fetch policy helpers."""

from __future__ import annotations

from .. import fetch as _F
from .. import restore as _R

HOT_PATH = ["restore_stream", "restore_chunk_wise"]

LookupTable = _F.LookupTable
FetchTimeline = _F.FetchTimeline
estimate_bandwidth = _F.estimate_bandwidth
select_resolution = _F.select_resolution


def restore_stream(bs, plan, cfg_layout, mem, layer_base=0, token_base=0):
    """fk/fetchsim.py:335-358: frame-wise GPU decode + restore into ``mem``
    (a facade PagedMemory: int8 code slots)."""
    return _R.restore_stream(bs, plan, cfg_layout, mem.device, layer_base, token_base)


def restore_chunk_wise(bs, plan, cfg_layout, mem, layer_base=0, token_base=0):
    """fk/fetchsim.py:361-385 on the GPU."""
    return _R.restore_chunk_wise(bs, plan, cfg_layout, mem.device, layer_base, token_base)
