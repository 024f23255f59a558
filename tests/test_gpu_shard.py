"""The sharded PRODUCT path on the GPU: 2 gloo ranks on cuda:0 run bench.Workload
(libkvf pack + batched restore of their own units) for
one Llama-3-8B-shaped context split over the ranks (strong scaling, 'balanced'
policy).  Every restored slot of every unit must equal a single-process restore
of the whole context, and one full 10,000-token chunk is checked against the CPU
oracle (quantize -> dequantize -> bf16, fk/kvmodel.py:127-152).  Units are
independent (fk/kvmodel.py:223-225): no data-path collective."""

from __future__ import annotations

import argparse
import hashlib
import multiprocessing as mp
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu

TOKENS = 12_000  # chunks 10,000 + 2,000 -> 2 x 11 triplets x 2 chunks = 44 units


def _args(shard_policy="balanced"):
    return argparse.Namespace(model="llama3-8b", tokens=TOKENS, layout="identity", res="R480",
                              page=16, requests=1, shard=shard_policy)


def _unit_digests(w):
    """{repr(unit): sha256 of its restored bf16 slots, read through the block table}."""
    out = {}
    keys = sorted({(u.request, u.kv, u.triplet) for u in w.mine})
    for u in w.mine:
        cache = w.caches[keys.index((u.request, u.kv, u.triplet))]
        toks = torch.arange(u.token_start, u.token_start + u.tokens, device=cache.device)
        blk = w.table[toks // w.page].long()
        h = hashlib.sha256()
        for p in range(u.real_layers):
            h.update(cache[p][blk, toks % w.page].contiguous().view(torch.int16).cpu()
                     .numpy().tobytes())
        out[repr(u)] = h.hexdigest()
    return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist

    import bench
    from paper_2602_09725_b200 import shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        w = bench.Workload(_args(), dev, rank, world)
        s = torch.cuda.Stream()
        w.pack(s)      # frames of this rank's units (libkvf pack)
        w.restore(s)
        torch.cuda.synchronize()
        digests = _unit_digests(w)
        gathered = [None] * world
        dist.all_gather_object(gathered, digests)
        ms = shard.max_over_ranks(1.0 + rank, dist, dev)
        total = shard.sum_over_ranks(w.elems, dist, dev)
        if rank == 0:
            out.put((gathered, ms, total))
    finally:
        dist.destroy_process_group()


def test_two_rank_product_shard_equals_single_process_and_oracle():
    import bench
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, ms, total = out.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # every unit restored by exactly one rank, both ranks busy
    merged = {}
    for g in gathered:
        assert g, "a rank got no units"
        assert not set(g) & set(merged), "two ranks restored the same unit"
        merged.update(g)
    dev = torch.device("cuda", 0)
    single = bench.Workload(_args(), dev, 0, 1)
    s = torch.cuda.Stream()
    single.pack(s)
    single.restore(s)
    torch.cuda.synchronize()
    want = _unit_digests(single)
    assert len(want) == 44 and merged == want
    assert ms == 2.0 and total == single.elems
    # one full reference chunk of the single-process restore against the CPU oracle
    slots, bad = bench.oracle_unit_check(single, torch)
    assert slots == 10_000 * 3 and bad == 0
