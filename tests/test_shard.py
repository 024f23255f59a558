"""Multi-GPU sharding of restore units (CPU; world_size-2 gloo process groups).

The N>1 path shards (request, K/V, triplet, chunk) units across ranks with no
data exchange.  These tests check the planner and the only
cross-rank operations (max / sum of timings and counts) on the gloo backend,
and that a sharded restore of a small workload — run with the oracle as the
per-rank worker — writes exactly the slots of a single-process restore.
"""

from __future__ import annotations

import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ref
from paper_2602_09725_b200 import shard


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_unit_counts_of_the_baseline_configs():
    # C2 Llama-3-8B 32K: 11 triplets x 4 chunks x K,V
    assert len(shard.enumerate_units(32768, 32)) == 88
    # C3 Qwen2.5-7B 128K: 28 -> 30 layers = 10 triplets x 14 chunks x 2
    assert len(shard.enumerate_units(131072, 28)) == 280
    # C4 Llama-3-70B 80K: 81 layers = 27 triplets x 9 chunks x 2
    assert len(shard.enumerate_units(81920, 80)) == 486
    u = shard.enumerate_units(32768, 32)
    assert [x.tokens for x in u[:4]] == [10000, 10000, 10000, 2768]
    assert {x.real_layers for x in u if x.triplet == 10} == {2}   # layers 30, 31 + one pad


@pytest.mark.parametrize("policy", ["balanced", "layer", "chunk"])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_assignment_is_a_partition(policy, world):
    units = shard.enumerate_units(32768, 32, requests=world)
    parts = shard.assign(units, world, policy)
    assert len(parts) == world
    flat = [u for p in parts for u in p]
    assert sorted(flat, key=repr) == sorted(units, key=repr)
    assert len(set(flat)) == len(units)
    assert parts == shard.assign(units, world, policy)   # deterministic
    loads = [sum(u.elements(8, 128) for u in p) for p in parts]
    if policy == "balanced":
        assert max(loads) - min(loads) <= max(u.elements(8, 128) for u in units)
    if policy == "layer":
        for p in parts:   # every chunk of a triplet lands on one rank
            keys = {(u.request, u.kv, u.triplet) for u in p}
            for q in parts:
                if q is not p:
                    assert keys.isdisjoint({(u.request, u.kv, u.triplet) for u in q})
        # weak scaling: one context per GPU gives every GPU the same bytes +-1 short triplet
        assert max(loads) / min(loads) < 1.05


def test_bad_arguments():
    with pytest.raises(ValueError):
        shard.assign([], 0)
    with pytest.raises(ValueError):
        shard.assign(shard.enumerate_units(10, 3), 2, "nope")
    with pytest.raises(ValueError):
        shard.units_for_rank([], 2, 2)
    with pytest.raises(ValueError):
        shard.chunk_spans(-1)


# ------------------------------------------------------------ gloo, 2 ranks
T, LAYERS, H, D, RES, CH = 70, 5, 2, 32, "R240", 30
LAY = (H, D, 1, H, 1, D)


def _restore_units_oracle(units, x):
    """Per-rank worker: pack every unit with the oracle, then restore its frames
    into a {(request, kv, token, layer): bytes} slot map (PagedMemory contents)."""
    slots = {}
    xp = ref.pad_layers(x)
    for u in units:
        slab = xp[u.token_start:u.token_start + u.tokens, 3 * u.triplet:3 * u.triplet + 3]
        v, s = ref.quantize(slab, H * D)
        plan = ref.Plan(u.tokens, RES, *LAY, F=4)
        frames = ref.assemble_frames(v.reshape(u.tokens, 3, H * D), plan)
        got = ref.restore_slots(frames, plan, layer_base=3 * u.triplet, token_base=u.token_start)
        for (t, l), vec in got.items():
            if l < LAYERS:   # pad layers are never written
                slots[(u.request, u.kv, t, l)] = vec.tobytes()
    return slots


def _digest(slots):
    h = hashlib.sha256()
    for k in sorted(slots):
        h.update(repr(k).encode())
        h.update(slots[k])
    return h.hexdigest()


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        units = shard.enumerate_units(T, LAYERS, requests=world, chunk_tokens=CH)
        mine = shard.units_for_rank(units, rank, world, "layer", H, D)
        everyone = [None] * world
        dist.all_gather_object(everyone, [repr(u) for u in mine])
        x = ref.gen_synthetic_kv(T, LAYERS, H, D, 0.9, 7, 0.3)
        slots = _restore_units_oracle(mine, x)
        gathered = [None] * world
        dist.all_gather_object(gathered, slots)
        ms = shard.max_over_ranks(1.5 + rank)
        total = shard.sum_over_ranks(sum(u.elements(H, D) for u in mine))
        if rank == 0:
            merged = {}
            for g in gathered:
                assert not set(g) & set(merged), "two ranks wrote the same slot"
                merged.update(g)
            out.put((everyone, _digest(merged), ms, total, len(merged)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharded_restore_equals_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    everyone, digest, ms, total, n_slots = out.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    units = shard.enumerate_units(T, LAYERS, requests=world, chunk_tokens=CH)
    flat = [u for part in everyone for u in part]
    assert sorted(flat) == sorted(repr(u) for u in units) and len(set(flat)) == len(flat)
    x = ref.gen_synthetic_kv(T, LAYERS, H, D, 0.9, 7, 0.3)
    single = _restore_units_oracle(units, x)
    assert digest == _digest(single)
    assert n_slots == world * 2 * T * LAYERS
    assert ms == 2.5                                   # max over ranks of 1.5 + rank
    assert total == sum(u.elements(H, D) for u in units)


def test_head_window():
    from paper_2602_09725_b200 import shard
    assert [shard.head_window(8, r, 4) for r in range(4)] == [(0, 2), (2, 2), (4, 2), (6, 2)]
    assert shard.head_window(8, 0, 1) == (0, 8)
    with pytest.raises(ValueError):
        shard.head_window(8, 0, 3)
    with pytest.raises(ValueError):
        shard.head_window(8, 2, 2)
