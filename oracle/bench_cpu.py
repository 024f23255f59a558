"""CPU baseline timing of the reference restore / pack transforms (TEST/BENCH ONLY).

Used by bench.py's ``cpu_baseline`` leg and ``--impl reference`` arm.  Each worker
process rebuilds one sample unit (a Llama-3-8B-shaped K/V layer triplet chunk)
with the oracle — the numpy restatement of the reference — and times the
reference's restore transform on it: disassemble_frames (fk/layout.py:261-271)
-> dequantize (fk/kvmodel.py:147-152) -> bf16 -> paged scatter through a block
table (PagedMemory.page_write, fk/kvmodel.py:216-229), or the pack transform:
quantize (fk/kvmodel.py:127-144) + assemble_frames (fk/layout.py:234-258), or
the KVFC decode of a sample stream (the C restatement of decode_frames).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from oracle import ref


def _bf16_bits(x32):
    b = x32.view(np.uint32).astype(np.uint64)
    return ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)


def _sample(seed, T, H, D, res, lay, gs):
    x = ref.gen_synthetic_kv(T, 3, H, D, 0.9, seed, 0.3)
    x = (_bf16_bits(x).astype(np.uint32) << 16).view(np.float32)
    v, s = ref.quantize(x, gs)
    plan = ref.Plan(T, res, *lay, F=4)
    frames = ref.assemble_frames(v.reshape(T, 3, H * D), plan)
    return x, v, s, plan, frames


def restore_worker(args):
    """Time the reference restore transform on `units` sample units."""
    seed, units, T, H, D, res, lay, gs = args
    total_t, total_e = 0.0, 0
    bs = 16
    for u in range(units):
        _, v, s, plan, frames = _sample(seed * 1000 + u, T, H, D, res, lay, gs)
        nblk = (T + bs - 1) // bs
        table = np.random.default_rng(u).permutation(nblk)
        cache = np.empty((3, nblk, bs, H * D), np.uint16)
        t0 = time.perf_counter()
        codes = ref.disassemble_frames(frames, plan)                       # [T, 3, C] int8
        deq = ref.dequantize(codes.reshape(T, 3, H, D), s, gs).reshape(T, 3, H * D)
        bits = _bf16_bits(np.ascontiguousarray(deq))
        for p in range(3):                                                 # page_write
            cache[p].reshape(nblk * bs, H * D)[(table[np.arange(T) // bs] * bs
                                                + np.arange(T) % bs)] = bits[:, p]
        total_t += time.perf_counter() - t0
        total_e += T * 3 * H * D
    return total_t, total_e


def pack_worker(args):
    seed, units, T, H, D, res, lay, gs = args
    total_t, total_e = 0.0, 0
    for u in range(units):
        x, _, _, plan, _ = _sample(seed * 1000 + u, T, H, D, res, lay, gs)
        t0 = time.perf_counter()
        v, s = ref.quantize(x, gs)
        ref.assemble_frames(v.reshape(T, 3, H * D), plan)
        total_t += time.perf_counter() - t0
        total_e += T * 3 * H * D
    return total_t, total_e


def decode_worker(args):
    """Time the reference KVFC decode (oracle C restatement of decode_frames,
    fk/codec.py:155-211 + fk/rangecoder.py:146-189) on a sample stream."""
    seed, units, T, H, D, res, lay, gs = args
    _, _, _, plan, frames = _sample(seed, T, H, D, res, lay, gs)
    n = min(8, plan.frame_count)
    bs = ref.encode_frames(frames[:n], plan.F)
    total_t, total_e = 0.0, 0
    for _ in range(units):
        t0 = time.perf_counter()
        out = ref.decode_frames(bs)
        total_t += time.perf_counter() - t0
        total_e += out.size
    return total_t, total_e


def run(kind="restore", workers=None, units_per_worker=2, T=10000, H=8, D=128, res="R1080",
        lay=(8, 128, 1, 8, 1, 128), gs=128):
    """Run `workers` processes concurrently; returns (elements, wall seconds, cores).

    Each worker's timed region covers only the transform; the aggregate rate is
    total elements / the slowest worker's timed seconds (all run concurrently).
    """
    workers = workers or os.cpu_count() or 1
    fn = {"restore": restore_worker, "pack": pack_worker, "decode": decode_worker}[kind]
    if kind == "decode":
        from oracle import ref
        ref.build_c()  # once, before the workers load it
    jobs = [(w + 1, units_per_worker, T, H, D, res, tuple(lay), gs) for w in range(workers)]
    if workers == 1:
        res_list = [fn(jobs[0])]
    else:
        with mp.get_context("spawn").Pool(workers) as pool:
            res_list = pool.map(fn, jobs)
    elems = sum(e for _, e in res_list)
    wall = max(t for t, _ in res_list)
    return elems, wall, workers
