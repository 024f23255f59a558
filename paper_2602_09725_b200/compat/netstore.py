"""numpy facade of the fk/netstore.py fetch client (the GPU pipelined fetcher)."""

from __future__ import annotations

from .. import fetch as _F
from .. import netstore as _N
from . import kvmodel as _K

HOT_PATH = ["fetch_chunk", "decode_fetched", "live_fetch_pipeline", "ProtocolError",
            "ChunkNotFound", "FetchTimeout"]

ProtocolError = _N.ProtocolError
ChunkNotFound = _N.ChunkNotFound
FetchTimeout = _N.FetchTimeout
WireRequest = _N.WireRequest
WireResponse = _N.WireResponse
ChunkStore = _N.ChunkStore
serve = _N.serve
fetch_chunk = _N.fetch_chunk


def decode_fetched(metadata, payload):
    """fk/netstore.py:352-364: GPU decode of one fetched chunk -> numpy slab."""
    return _K.from_device(_N.decode_fetched(metadata, payload))


def live_fetch_pipeline(address, chunks, table, policy="adaptive", prior_gbps=None,
                        initial_active="R1080", timeout_s=30.0, on_chunk=None):
    """fk/netstore.py:367-454 with the reference's schedule: one chunk per GPU
    decode, one decode at a time on a worker thread, overlapping the next
    transfer (so each record's tau_dec is that chunk's own decode time);
    on_chunk receives (record, numpy QuantizedKV) like the reference's."""
    cb = None if on_chunk is None else (lambda rec, slab: on_chunk(rec, _K.from_device(slab)))
    return _F.live_fetch_pipeline(address, chunks, table, policy, prior_gbps, initial_active,
                                  timeout_s, cb, max_batch=1, max_inflight=1)
