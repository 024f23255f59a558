"""Pack schedule sweep on one GPU: two-pass vs single-read (slab sizes).

Builds bench.Workload (C2 by default), packs with KVF_PACK_TWO_PASS as the
reference result, then times each schedule and checks that its frames and
scales are bit-identical.  One JSON line per schedule.

    python tools/pack_sweep.py [--model llama3-8b --tokens 32768 --layout identity]
                               [--schedules single_read,single_read:16,auto] [--steps 20]
"""
import argparse
import json
import time
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_09725_b200 import _dev, _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--layout", default="identity")
    ap.add_argument("--res", default="R1080")
    ap.add_argument("--schedules", default="single_read",
                    help="comma list of single_read[:cluster] / auto")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays of the call")
    a = ap.parse_args()
    args = argparse.Namespace(model=a.model, tokens=a.tokens, layout=a.layout, res=a.res, page=16,
                              requests=1, shard="balanced")
    dev = torch.device("cuda", 0)
    w = bench.Workload(args, dev)
    s = torch.cuda.current_stream()

    def call(sched, slab):
        _lib.call("kvf_pack_batch_ex", w._pack_arr, len(w.pack_units), sched, slab,
                  _dev.stream_ptr(torch.cuda.current_stream()))

    graphs = {}

    def run(sched, slab):
        if not a.graph:
            return call(sched, slab)
        if (sched, slab) not in graphs:   # captured once, replayed per step
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                call(sched, slab)
            graphs[(sched, slab)] = g
        graphs[(sched, slab)].replay()

    run(_lib.KVF_PACK_TWO_PASS, 0)
    torch.cuda.synchronize()
    ref_frames = [f.clone() for f in w.frames]
    ref_scales = [x.clone() for x in w.scales]
    configs = [(_lib.KVF_PACK_TWO_PASS, 0)]
    names = {"single_read": _lib.KVF_PACK_SINGLE_READ, "auto": _lib.KVF_PACK_AUTO}
    for x in filter(None, a.schedules.split(",")):
        nm, _, prm = x.partition(":")
        configs.append((names[nm], int(prm or "0", 0)))
    for sched, slab in configs:
        for f in w.frames:
            f.fill_(7)
        for x in w.scales:
            x.fill_(-1)
        run(sched, slab)
        torch.cuda.synchronize()
        ok = all(torch.equal(f, r) for f, r in zip(w.frames, ref_frames)) and \
            all(torch.equal(x, r) for x, r in zip(w.scales, ref_scales))
        for _ in range(3):
            run(sched, slab)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
        ev[0].record(s)
        host = 0.0
        for k in range(a.steps):
            h0 = time.perf_counter()
            run(sched, slab)
            host += time.perf_counter() - h0
            ev[k + 1].record(s)
        torch.cuda.synchronize()
        per = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(a.steps))
        med = per[len(per) // 2]
        ach = 3.0 * w.elems / (med * 1e-3) / 1e9
        sname = {0: "auto", 1: "two_pass", 2: "single_read"}[sched]
        print(json.dumps({"schedule": sname,
                          "cluster": slab, "ms_median": round(med, 4),
                          "ms_min": round(per[0], 4), "host_ms": round(host * 1e3 / a.steps, 4), "achieved_gbs": round(ach, 1),
                          "frac": round(ach / 6558.7, 4), "bit_exact": ok, "graph": a.graph,
                          "model": a.model, "tokens": a.tokens, "layout": a.layout}), flush=True)


if __name__ == "__main__":
    main()
