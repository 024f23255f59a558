"""Units of restore/pack work and their assignment to GPUs (one process per GPU).

A unit is one (request, K-or-V, layer triplet, token chunk) — exactly one KVFC
container of the reference (fk/container.py:160-209: a 3-layer slab of at most
DEFAULT_CHUNK_TOKENS tokens, layer_triplet_index + token_start in its header,
fk/container.py:50-52).  Units are independent: a unit's scales are local to
its chunk and layers (fk/kvmodel.py:138-140), its frames are its own, and the
paged slots it writes — page = token // page_size, slot (token % page_size,
layer) (fk/kvmodel.py:223-225) — are disjoint from every other unit's.  So the
path shards with no data exchange: each rank restores the units assigned to it
into its own HBM block pool, and the only cross-rank traffic is the timing
reduction (max over ranks) of the benchmark.  Head-sharded (tensor-parallel)
caches are the exception: restore_head_sharded at the end of this file.

Assignment policies (all deterministic, computed identically on every rank):
  * ``"balanced"`` — longest-processing-time greedy on element counts; ties go
    to the lowest rank.  Default; gives equal per-rank bytes for the bench.
  * ``"layer"``    — whole layer triplets round-robin (layer-sharded serving,
    BASELINE.json configs[2]); every chunk of a triplet lands on one rank.
  * ``"chunk"``    — token chunks round-robin (sequence-sharded).
"""

from __future__ import annotations

from dataclasses import dataclass

DEFAULT_CHUNK_TOKENS = 10_000   # fk/container.py:29


@dataclass(frozen=True)
class Unit:
    request: int
    kv: int            # 0 = K, 1 = V
    triplet: int       # layer_triplet_index: layers 3*triplet .. 3*triplet+2
    chunk: int         # chunk_index
    token_start: int
    tokens: int
    real_layers: int   # layers of the triplet that exist (pad layers are never written)

    def elements(self, H: int, D: int) -> int:
        return self.tokens * self.real_layers * H * D


def chunk_spans(T: int, chunk_tokens: int = DEFAULT_CHUNK_TOKENS):
    """[(token_start, tokens)] of the <= chunk_tokens containers covering T tokens."""
    if T < 0 or chunk_tokens < 1:
        raise ValueError("T must be >= 0 and chunk_tokens >= 1")
    return [(t, min(chunk_tokens, T - t)) for t in range(0, T, chunk_tokens)]


def enumerate_units(T: int, layers: int, requests: int = 1,
                    chunk_tokens: int = DEFAULT_CHUNK_TOKENS, kv: int = 2) -> list[Unit]:
    """Every unit of `requests` KV caches of T tokens x `layers` layers, K and V,
    layers zero-padded to a multiple of 3 (fk/kvmodel.py:56-69)."""
    if layers < 1 or requests < 0:
        raise ValueError("layers must be >= 1 and requests >= 0")
    trip = (layers + 2) // 3
    out = []
    for r in range(requests):
        for k in range(kv):
            for j in range(trip):
                real = min(3, layers - 3 * j)
                for c, (t0, tc) in enumerate(chunk_spans(T, chunk_tokens)):
                    out.append(Unit(r, k, j, c, t0, tc, real))
    return out


def assign(units: list[Unit], world: int, policy: str = "balanced",
           H: int = 8, D: int = 128) -> list[list[Unit]]:
    """Partition `units` over `world` ranks; returns one list per rank."""
    if world < 1:
        raise ValueError("world must be >= 1")
    out: list[list[Unit]] = [[] for _ in range(world)]
    if policy == "balanced":
        load = [0] * world
        order = sorted(range(len(units)), key=lambda i: (-units[i].elements(H, D), i))
        for i in order:
            r = min(range(world), key=lambda k: (load[k], k))
            out[r].append(units[i])
            load[r] += units[i].elements(H, D)
        for lst in out:  # keep the canonical unit order inside a rank
            lst.sort(key=lambda u: (u.request, u.kv, u.triplet, u.chunk))
    elif policy == "layer":
        keys = sorted({(u.request, u.kv, u.triplet) for u in units})
        owner = {key: n % world for n, key in enumerate(keys)}
        for u in units:
            out[owner[(u.request, u.kv, u.triplet)]].append(u)
    elif policy == "chunk":
        keys = sorted({(u.request, u.chunk) for u in units})
        owner = {key: n % world for n, key in enumerate(keys)}
        for u in units:
            out[owner[(u.request, u.chunk)]].append(u)
    else:
        raise ValueError(f"unknown shard policy {policy!r}")
    return out


def units_for_rank(units: list[Unit], rank: int, world: int, policy: str = "balanced",
                   H: int = 8, D: int = 128) -> list[Unit]:
    if not 0 <= rank < world:
        raise ValueError("rank outside [0, world)")
    return assign(units, world, policy, H, D)[rank]


def _reduce(value: float, op: str, dist=None, device=None) -> float:
    if dist is None:
        import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    if device is None or dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=getattr(dist.ReduceOp, op))
    return float(t.item())


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank timing over the default process group (identity without one)."""
    return _reduce(value, "MAX", dist, device)


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    """Sum of a per-rank count over the default process group (identity without one)."""
    return _reduce(value, "SUM", dist, device)


# ------------------------------------------------------------------ head shards
# Tensor-parallel serving keeps 1/world of the KV heads of every layer on each
# GPU (the optional collective).  Units are still decoded
# where they were fetched; one exchange then moves, per peer, only that peer's
# heads, as int8-sized frame samples (1 B/elem, half of bf16), before any
# dequantisation.

def head_window(H: int, rank: int, world: int) -> tuple[int, int]:
    """KV heads [lo, lo + n) held by tensor-parallel rank `rank` (even split)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank outside [0, world)")
    if H % world:
        raise ValueError(f"{world} ranks do not split {H} KV heads evenly")
    n = H // world
    return rank * n, n


@dataclass(frozen=True)
class HeadJob:
    """One unit of a head-sharded restore: its chunk tokens, frame plan, the
    rank holding its decoded frames, and which planes are real layers."""
    tokens: int
    plan: object          # layout.FramePlan of the unit's frames
    owner: int
    real_layers: int = 3  # planes >= real_layers are pad layers (never written)


def _flat_plan(T: int, n_heads: int, D: int, group_size: int):
    """The frame form of a head slice: one frame whose T tile rows are the
    tokens (identity tile n_heads x D, F = 1) — restorable with kvf_restore."""
    from . import _lib
    p = _lib.kvf_plan(T, n_heads, D, 1, n_heads, 1, D, 1, T, T, 1, 0, 0, 0, int(group_size))
    _lib.call("kvf_plan_init", p)
    return p


def restore_head_sharded(jobs: list[HeadJob], mine: dict, dst_of, H: int, D: int,
                         group_size: int, dist=None, stream=None):
    """Restore every unit's heads of this rank into its head-shard cache.

    ``jobs``: every unit of the job, identical on every rank.  ``mine``:
    {job index: (frames [n, 3, h, w] uint8 CUDA tensor, scales [3, G] CUDA fp32)}
    for the units this rank decoded.  ``dst_of(k)``: the kvf_paged of this rank's
    cache for unit k (its head_window(H, rank, world) heads; head_stride etc.
    of the local cache).

    Each owner cuts every peer's heads out of its frames in one pass, in frame
    form (kvf_restore_batch_heads, raw samples), the ranks exchange them with one
    all_to_all_single (NCCL over NVLink on a GPU job; staged through host memory
    under gloo), scales travel with all_gather_object, and every rank restores
    the received slices with kvf_restore_batch.  Returns the bytes this rank
    received.
    """
    import ctypes as C

    import numpy as np
    import torch

    from . import _dev, _lib
    if dist is None:
        import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    wins = [head_window(H, r, world) for r in range(world)]
    lo, nh = wins[rank]                  # every window holds nh heads
    if (lo * D) % group_size or (nh * D) % group_size:
        raise ValueError("a head window must hold whole quantisation groups")
    dev = _dev.device()
    s = stream if stream is not None else torch.cuda.current_stream()
    sp = _dev.stream_ptr(s)
    owned = [k for k, j in enumerate(jobs) if j.owner == rank]
    if set(owned) != set(mine):
        raise ValueError("`mine` must hold exactly the units this rank owns")

    def slice_bytes(k, n):
        return 3 * jobs[k].tokens * n * D

    # 1. one cut of every owned unit: peer r's heads into region r of the send
    #    buffer ([peer][owned unit in job order][3][T][nh * D], frame form)
    per_peer = sum(slice_bytes(k, nh) for k in owned)
    send_sizes = [per_peer] * world
    send = torch.empty(max(per_peer * world, 1), dtype=torch.uint8, device=dev)
    base, at, units = send.data_ptr(), 0, []
    for k in owned:
        j, (frames, _) = jobs[k], mine[k]
        T = j.tokens
        dst = _lib.kvf_paged()
        for p in range(3):
            dst.layer[p] = base + at + p * T * nh * D if p < j.real_layers else None
        dst.block_table = None
        dst.block_size = 1
        dst.dtype = _lib.KVF_I8
        dst.block_stride = dst.slot_stride = nh * D
        dst.head_stride = D
        dst.token_base = 0
        u = _lib.kvf_restore_unit()
        u.frames = _dev.surface_of(frames)
        u.plan = j.plan.to_c(group_size)
        u.scales = None
        u.dst = dst
        u.first_frame = 0
        u.n_frames = j.plan.frame_count
        units.append(u)
        at += slice_bytes(k, nh)
    if units:
        arr = (_lib.kvf_restore_unit * len(units))(*units)
        _lib.call("kvf_restore_batch_heads", arr, len(units), 0, nh, world, per_peer, 1, sp)
    # 2. the exchange
    recv_sizes = [sum(slice_bytes(k, nh) for k, j in enumerate(jobs) if j.owner == o)
                  for o in range(world)]
    gloo = dist.get_backend() == "gloo"
    s.synchronize()
    send_x = send.cpu() if gloo else send
    recv_x = torch.empty(max(sum(recv_sizes), 1), dtype=torch.uint8,
                         device="cpu" if gloo else dev)
    dist.all_to_all_single(recv_x[:sum(recv_sizes)], send_x[:sum(send_sizes)],
                           output_split_sizes=recv_sizes, input_split_sizes=send_sizes)
    recv = recv_x.to(dev) if gloo else recv_x
    scales_all = [None] * world
    dist.all_gather_object(scales_all, {k: mine[k][1].cpu().numpy() for k in owned})
    # 3. restore every unit's slice of this rank's heads
    g0, g1 = lo * D // group_size, (lo + nh) * D // group_size
    off = np.concatenate([[0], np.cumsum(recv_sizes)])
    units, keep = [], [recv]
    rb = recv.data_ptr()
    for o in range(world):
        at = int(off[o])
        for k, j in enumerate(jobs):
            if j.owner != o:
                continue
            T = j.tokens
            sc = torch.from_numpy(np.ascontiguousarray(scales_all[o][k][:, g0:g1])).to(dev)
            keep.append(sc)
            u = _lib.kvf_restore_unit()
            u.frames.base = rb + at
            u.frames.row_pitch = nh * D
            u.frames.plane_stride = T * nh * D
            u.frames.frame_stride = 3 * T * nh * D
            u.plan = _flat_plan(T, nh, D, group_size)
            u.scales = sc.data_ptr()
            u.dst = dst_of(k)
            u.first_frame = 0
            u.n_frames = 1
            units.append(u)
            at += slice_bytes(k, nh)
    if units:
        arr = (_lib.kvf_restore_unit * len(units))(*units)
        _lib.call("kvf_restore_batch", arr, len(units), sp)
    for t in keep:
        t.record_stream(s)
    return int(sum(recv_sizes))
