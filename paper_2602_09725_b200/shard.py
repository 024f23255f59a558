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
reduction (max over ranks) of the benchmark.

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
