"""Head-shard kernels on one B200, C2 frames: the per-peer cut (kvf_restore_batch_heads,
raw samples into a contiguous slice buffer) and the receiver's restore of the
slices (kvf_restore_batch, flat plan), for tensor-parallel widths 2/4/8."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_09725_b200 import _dev, _lib, shard  # noqa: E402
from paper_2602_09725_b200.restore import make_restore_unit  # noqa: E402


def timed(fn, steps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    args = argparse.Namespace(model="llama3-8b", tokens=32768, layout="identity", res="R1080",
                              page=16, requests=1, shard="balanced")
    w = bench.Workload(args, torch.device("cuda", 0))
    w.pack(torch.cuda.current_stream())
    torch.cuda.synchronize()
    H, D = w.H, w.D
    for world in (2, 4, 8):
        lo, nh = shard.head_window(H, 0, world)
        T_all = [int(u.plan.T) for u in w.units]
        sizes = [3 * T * nh * D for T in T_all]
        buf = torch.empty(sum(sizes), dtype=torch.uint8, device="cuda")
        units, at = [], 0
        for ru, T, sz in zip(w.units, T_all, sizes):
            d = _lib.kvf_paged()
            for p in range(3):
                d.layer[p] = buf.data_ptr() + at + p * T * nh * D if ru.dst.layer[p] else None
            d.block_table, d.block_size, d.dtype = None, 1, _lib.KVF_I8
            d.block_stride = d.slot_stride = nh * D
            d.head_stride, d.token_base = D, 0
            u = _lib.kvf_restore_unit()
            u.frames, u.plan, u.scales, u.dst = ru.frames, ru.plan, None, d
            u.first_frame, u.n_frames = 0, ru.n_frames
            units.append(u)
            at += sz
        arr = (_lib.kvf_restore_unit * len(units))(*units)
        sp = _dev.stream_ptr(torch.cuda.current_stream())
        t_cut = timed(lambda: _lib.call("kvf_restore_batch_heads", arr, len(units), lo, nh, 1, 0, 1,
                                        sp))
        # every peer's window in one pass: the owner's whole cut
        allbuf = torch.empty(world * sum(sizes), dtype=torch.uint8, device="cuda")
        for u, off in zip(units, [0] + list(__import__("itertools").accumulate(sizes))[:-1]):
            for p in range(3):
                if u.dst.layer[p]:
                    u.dst.layer[p] = allbuf.data_ptr() + off + p * int(u.plan.T) * nh * D
        arr = (_lib.kvf_restore_unit * len(units))(*units)
        t_all = timed(lambda: _lib.call("kvf_restore_batch_heads", arr, len(units), 0, nh, world,
                                        sum(sizes), 1, sp))
        # receiver: the slices back into a head-shard bf16 cache (flat plan)
        cache = torch.empty((3, sum(T_all), nh, D), dtype=torch.bfloat16, device="cuda")
        runits, at, tok = [], 0, 0
        for ru, T, sz, sc in zip(w.units, T_all, sizes, w.scales):
            u = _lib.kvf_restore_unit()
            u.frames.base = buf.data_ptr() + at
            u.frames.row_pitch, u.frames.plane_stride, u.frames.frame_stride = nh * D, T * nh * D, 3 * T * nh * D
            u.plan = shard._flat_plan(T, nh, D, w.gs)
            g = sc[:, lo * D // w.gs:(lo + nh) * D // w.gs].contiguous()
            u.scales = g.data_ptr()
            d = _lib.kvf_paged()
            for p in range(3):
                d.layer[p] = cache[p].data_ptr() if ru.dst.layer[p] else None
            d.block_table, d.block_size, d.dtype = None, 1, _lib.KVF_BF16
            d.block_stride = d.slot_stride = nh * D
            d.head_stride, d.token_base = D, tok
            u.dst, u.first_frame, u.n_frames = d, 0, 1
            runits.append(u)
            runits[-1]._keep = g
            at += sz
            tok += T
        rarr = (_lib.kvf_restore_unit * len(runits))(*runits)
        t_rest = timed(lambda: _lib.call("kvf_restore_batch", rarr, len(runits), sp))
        real = w.elems // world                    # window elements of real layers
        print(json.dumps({"tp": world, "heads": nh, "cut_ms": round(t_cut, 4),
                          "cut_gbs": round(2 * real / t_cut / 1e6, 1),
                          "cut_all_peers_ms": round(t_all, 4),
                          "cut_all_gbs": round(2 * w.elems / t_all / 1e6, 1),
                          "restore_ms": round(t_rest, 4),
                          "restore_gbs": round(3 * real / t_rest / 1e6, 1),
                          "slice_bytes": int(sum(sizes))}), flush=True)


if __name__ == "__main__":
    main()
