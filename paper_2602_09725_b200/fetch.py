"""Pipelined chunk fetcher: network receive || H2D + GPU decode + restore.

Keeps the reference's live_fetch_pipeline API and timeline schema
(fk/netstore.py:367-454, FetchTimeline fk/fetchsim.py:172-205).  The
reference overlaps one transfer with one CPU decode on a GIL-holding worker
thread; here a GPU worker owns a CUDA stream: each received payload is
scanned on the host, copied to the device and entropy-decoded, reconstructed
and (optionally) restored straight into a PagedMemory block cache, while the
main thread already receives the next chunk.  Resolution choice is the
reference's bubble-minimising rule (fk/fetchsim.py:154-169).
"""

from __future__ import annotations

import json
import queue
import threading
import time
from dataclasses import dataclass, field

import torch

from . import codec, container as C, layout as L, netstore as NS
from .restore import restore_frames

MB = 1e6
GBPS = 1e9


class LookupTable:
    """Per-resolution decode latency vs pool load, switch penalty, chunk size."""

    def __init__(self, device, P, decode_s, penalty_s, size_mb):
        self.device = device
        self.P = int(P)
        self.decode_s = {r: [float(x) for x in v] for r, v in decode_s.items()}
        self.penalty_s = {r: float(v) for r, v in penalty_s.items()}
        self.size_mb = {r: float(v) for r, v in size_mb.items()}
        if self.P < 1:
            raise ValueError("pool size must be >= 1")
        for r in L.RESOLUTION_ORDER:
            row = self.decode_s.get(r)
            if row is None:
                raise ValueError(f"missing decode row for {r}")
            if len(row) != self.P or any(v <= 0 for v in row):
                raise ValueError(f"decode row for {r} must hold P={self.P} positive entries")
            if any(b < a for a, b in zip(row, row[1:])):
                raise ValueError(f"decode latencies for {r} must be non-decreasing")
            if self.size_mb[r] <= 0:
                raise ValueError("chunk sizes must be positive")
        if self.penalty_s["R1080"] != 0.0:
            raise ValueError("penalty at the top class must be zero")

    def tau_dec(self, resolution, load):
        if not 1 <= load <= self.P:
            raise ValueError(f"pool load must be in [1, {self.P}]")
        return self.decode_s[resolution][load - 1]

    def tau_penalty(self, resolution):
        return self.penalty_s[resolution]

    def size_bytes(self, resolution):
        return self.size_mb[resolution] * MB

    @classmethod
    def from_json(cls, obj):
        return cls(obj["device"], obj["P"], obj["decode_s"], obj["penalty_s"], obj["size_mb"])

    @classmethod
    def load(cls, path):
        with open(path) as fh:
            return cls.from_json(json.load(fh))


def estimate_bandwidth(history, prior_gbps=None):
    """Gbps of the last transfer record (bytes, seconds); prior on a cold start."""
    if history:
        nbytes, duration = history[-1]
        if duration <= 0:
            raise ValueError("transfer duration must be positive")
        return nbytes * 8.0 / duration / GBPS
    if prior_gbps is None:
        raise RuntimeError("no transfer history and no bandwidth prior configured")
    return float(prior_gbps)


def select_resolution(bw_gbps, pool_load, active_res, table: LookupTable):
    """argmin |tau_trans - tau_dec - tau_penalty|; ties toward the higher class."""
    best, best_delta = None, None
    for r in L.RESOLUTION_ORDER:
        tau_trans = table.size_bytes(r) * 8.0 / (bw_gbps * GBPS)
        pen = table.tau_penalty(r) if r != active_res else 0.0
        delta = abs(tau_trans - table.tau_dec(r, pool_load) - pen)
        if best_delta is None or delta <= best_delta:
            best, best_delta = r, delta
    return best


@dataclass
class FetchTimeline:
    policy: str
    records: list = field(default_factory=list)
    ttft: float = 0.0
    total_bubble: float = 0.0
    peak_restore_bytes: int = 0

    def to_json(self):
        return {"policy": self.policy, "ttft_s": self.ttft, "total_bubble_s": self.total_bubble,
                "peak_restore_bytes": self.peak_restore_bytes, "chunks": self.records}

    def csv_rows(self):
        cols = ["chunk", "resolution", "bw_est_gbps", "transfer_start", "transfer_end", "tau_trans",
                "decode_start", "decode_end", "tau_dec", "penalty", "bubble"]
        yield cols
        for r in self.records:
            yield [r[c] for c in cols]


def _fixed_policy(policy):
    if policy == "adaptive":
        return None
    name = policy.split(":", 1)[1] if ":" in policy else policy
    if name not in L.RESOLUTION_ORDER:
        raise ValueError(f"unknown policy {policy!r}")
    return name


def live_fetch_pipeline(address, chunks, table, policy="adaptive", prior_gbps=None,
                        initial_active="R1080", timeout_s=30.0, on_chunk=None, *, mem=None,
                        scales_dtype_out=None, real_layers=None, depth=2):
    """Fetch chunks from a live server and decode them on the GPU as they arrive.

    ``chunks``: list of (cache_id, chunk_index).  Without ``mem`` each chunk is
    decoded to its int8 slab and on_chunk(record, QuantizedKV) is called, like
    the reference.  With a PagedMemory ``mem`` each chunk is restored straight
    into it (token_base = token_start, layer_base = 3 * layer_triplet_index,
    dequantised with the container scales unless the cache holds int8) and
    on_chunk(record, stats) receives the tokens written.  Up to ``depth``
    received chunks wait for the GPU worker.
    """
    fixed = _fixed_policy(policy)
    timeline = FetchTimeline(policy=policy)
    base = time.monotonic()
    work = queue.Queue(maxsize=max(1, depth))
    errors = []
    gpu_stream = torch.cuda.Stream()
    state = {"dec_end": None}

    def gpu_worker():
        while True:
            item = work.get()
            if item is None:
                return
            rec, meta, payload = item
            try:
                t0 = time.monotonic()
                with torch.cuda.stream(gpu_stream):
                    if mem is None:
                        result = NS.decode_fetched(meta, payload)
                        held = 0
                    else:
                        cont = NS.container_of(meta, payload)
                        code = L.RESOLUTION_CODE[meta["resolution"]]
                        plan = cont.plan(code)
                        frames, held = codec.decode_batch([payload], stream=gpu_stream)
                        sc = None if mem.dtype == torch.int8 else torch.from_numpy(cont.scales())
                        n = restore_frames(frames[0], plan, mem, 3 * cont.layer_triplet_index,
                                           cont.token_start, scales=sc, real_layers=real_layers,
                                           stream=gpu_stream)
                        result = {"tokens_written": n}
                gpu_stream.synchronize()
                t1 = time.monotonic()
                rec.update(decode_start=t0 - base, decode_end=t1 - base, tau_dec=t1 - t0)
                if state["dec_end"] is not None:
                    rec["bubble"] = max(0.0, t0 - base - state["dec_end"])
                    timeline.total_bubble += rec["bubble"]
                state["dec_end"] = t1 - base
                timeline.peak_restore_bytes = max(timeline.peak_restore_bytes, held)
                if on_chunk is not None:
                    on_chunk(rec, result)
            except Exception as e:  # surfaced on the caller's thread
                errors.append(e)

    worker = threading.Thread(target=gpu_worker, daemon=True)
    worker.start()
    history, active = [], initial_active
    try:
        for i, (cache_id, chunk_index) in enumerate(chunks):
            if errors:
                break
            bw = estimate_bandwidth(history, prior_gbps) if (history or prior_gbps) else None
            if fixed is not None:
                res = fixed
            else:
                if bw is None:
                    raise ValueError("adaptive policy needs a bandwidth prior")
                res = select_resolution(bw, 1, active, table)
            active = res
            t_start = time.monotonic()
            payload, meta, tau = NS.fetch_chunk(address, cache_id, chunk_index, res, timeout_s)
            t_end = time.monotonic()
            history.append((len(payload), tau))
            rec = {"chunk": i, "resolution": res, "bw_est_gbps": bw,
                   "transfer_start": t_start - base, "transfer_end": t_end - base,
                   "tau_trans": tau, "decode_start": None, "decode_end": None, "tau_dec": None,
                   "penalty": 0.0, "bubble": 0.0}
            timeline.records.append(rec)
            work.put((rec, meta, payload))
    finally:
        work.put(None)
        worker.join()
    if errors:
        raise errors[0]
    timeline.ttft = state["dec_end"] if state["dec_end"] is not None else 0.0
    return timeline
