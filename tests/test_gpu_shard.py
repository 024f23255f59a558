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


def _head_worker(rank, world, port, out):
    """Tensor-parallel head shards: each rank decodes (here: packs) its own units,
    then restore_head_sharded exchanges head slices so that every rank's cache
    holds its half of the heads of EVERY unit."""
    import torch.distributed as dist

    import bench
    from paper_2602_09725_b200 import _lib, layout as L, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        args = _args()
        w = bench.Workload(args, dev, rank, world)
        s = torch.cuda.Stream()
        w.pack(s)
        torch.cuda.synchronize()
        Lyr, H, D = bench.MODELS[args.model]
        units = shard.enumerate_units(args.tokens, Lyr, requests=1, chunk_tokens=bench.CHUNK)
        groups = shard.assign(units, world, args.shard, H, D)
        owner = {u: r for r, g in enumerate(groups) for u in g}
        lay = L.LayoutConfig(H, D, *bench.LAYOUTS[args.layout](H, D))
        jobs = [shard.HeadJob(u.tokens, L.plan_inter_frame(u.tokens, args.res, lay, 4), owner[u],
                              u.real_layers) for u in units]
        mine = {units.index(u): (fr, sc) for u, fr, sc in zip(w.mine, w.frames, w.scales)}
        lo, nh = shard.head_window(H, rank, world)
        bs = w.page
        nblk = (args.tokens + bs - 1) // bs
        caches = {}
        for u in units:
            key = (u.kv, u.triplet)
            if key not in caches:
                caches[key] = torch.zeros((u.real_layers, nblk + 64, bs, nh, D),
                                          dtype=torch.bfloat16, device=dev)

        def dst_of(k):
            u = units[k]
            c = caches[(u.kv, u.triplet)]
            d = _lib.kvf_paged()
            for p in range(3):
                d.layer[p] = c[p].data_ptr() if p < u.real_layers else None
            d.block_table = w.table.data_ptr()
            d.block_size = bs
            d.dtype = _lib.KVF_BF16
            d.block_stride = bs * nh * D
            d.slot_stride = nh * D
            d.head_stride = D
            d.token_base = u.token_start
            return d

        got = shard.restore_head_sharded(jobs, mine, dst_of, H, D, w.gs, dist, s)
        torch.cuda.synchronize()
        digests = {}
        for u in units:
            c = caches[(u.kv, u.triplet)]
            toks = torch.arange(u.token_start, u.token_start + u.tokens, device=dev)
            blk = w.table[toks // bs].long()
            h = hashlib.sha256()
            for p in range(u.real_layers):
                h.update(c[p][blk, toks % bs].contiguous().view(torch.int16).cpu().numpy()
                         .tobytes())
            digests[repr(u)] = h.hexdigest()
        gathered = [None] * world
        dist.all_gather_object(gathered, (lo, nh, got, digests))
        if rank == 0:
            out.put(gathered)
    finally:
        dist.destroy_process_group()


def test_two_rank_head_sharded_exchange_equals_full_restore_slices():
    """restore_head_sharded: after one all_to_all of int8
    head slices, rank r's cache holds heads [4r, 4r+4) of every unit, bit-equal
    to the same heads of a single-process restore of the whole context."""
    import bench
    from paper_2602_09725_b200 import shard
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_head_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = out.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dev = torch.device("cuda", 0)
    single = bench.Workload(_args(), dev, 0, 1)
    s = torch.cuda.Stream()
    single.pack(s)
    single.restore(s)
    torch.cuda.synchronize()
    keys = sorted({(u.request, u.kv, u.triplet) for u in single.mine})
    total = 0
    for lo, nh, got, digests in gathered:
        total += got
        assert len(digests) == 44
        for u in single.mine:
            cache = single.caches[keys.index((u.request, u.kv, u.triplet))]
            toks = torch.arange(u.token_start, u.token_start + u.tokens, device=dev)
            blk = single.table[toks // single.page].long()
            h = hashlib.sha256()
            for p in range(u.real_layers):
                h.update(cache[p][blk, toks % single.page][:, lo:lo + nh].contiguous()
                         .view(torch.int16).cpu().numpy().tobytes())
            assert digests[repr(u)] == h.hexdigest(), (lo, u)
    # each rank received its 4 heads (1 B/elem, 3 planes) of EVERY unit (its own
    # units' slices go through the same buffer)
    assert total == 2 * sum(3 * u.tokens * 4 * 128 for u in single.mine)
