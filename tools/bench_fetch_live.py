"""C5: pipelined chunked fetch of a Llama-3-8B 32K K+V context over a rate-limited
loopback link (BASELINE.json configs[4]), GPU decode + restore into paged bf16.

    python tools/bench_fetch_live.py [--rates 10,25,100,0] [--res R240,R1080]

Packs the context into the reference's containers (88 units: K/V x 11 layer
triplets x 4 chunks of <= 10,000 tokens; scales over all tokens, as
fk/cli.py:222-224), writes them to a ChunkStore directory, serves it with the
reference wire protocol and an egress pacer at the link rate (the reference throttles with
a token bucket, fk/netstore.py:188-211),
and runs live_fetch_pipeline into two PagedMemory caches (K and V).  Prints one
JSON line per (resolution, rate): time to ready (first request -> last restore
complete), the link time the coded bytes need at that rate, the rate the
loopback actually delivered, batching, and a sampled bit-exactness check of
the restored bf16 cache against dequantised codes.
"""

from __future__ import annotations

import argparse
import gc
import json
import multiprocessing as mp
import os
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context: see paper_2602_09725_b200.use_fetch_hw_queues
import shutil
import sys
import tempfile
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_09725_b200 import container as C, fetch as FE, kvmodel as KV  # noqa: E402
from paper_2602_09725_b200 import layout as L, netstore as NS  # noqa: E402


def build_store(root, T, Lyr, H, D, resolutions, chunk=10_000):
    """Pack the context into containers with the batched GPU producer
    (container.pack_chunks: one encode per cache); returns the chunk keys, the
    quantised caches and the seconds spent in pack_chunks."""
    cfg = L.identity_layout(H, D)
    chunks, qs, pack_s = [], {}, 0.0
    for kv_i, name in enumerate(("K", "V")):
        cid = bytes([0x40 + kv_i]) * 16
        x = KV.gen_synthetic_kv(T, Lyr, H, D, 0.9, kv_i, 0.3, dtype=torch.bfloat16)
        q = KV.quantize(x.pad_layers())
        qs[cid] = q
        slabs = []
        for j in range((Lyr + 2) // 3):
            for c, t0 in enumerate(range(0, T, chunk)):
                tc = min(chunk, T - t0)
                slab = KV.QuantizedKV(q.values[t0:t0 + tc, 3 * j:3 * j + 3],
                                      q.scales[3 * j:3 * j + 3], q.group_size)
                slabs.append((slab, cid, j * 1000 + c, t0, j))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        conts = C.pack_chunks(slabs, cfg, resolutions)
        pack_s += time.perf_counter() - t0
        for cont in conts:
            with open(os.path.join(root, C.container_filename(cid, cont.chunk_index)), "wb") as fh:
                fh.write(cont.to_bytes())
            chunks.append((cid, cont.chunk_index))
        del x
    return chunks, qs, pack_s


def serve_proc(root, rate, port_q, stop):
    handle = NS.serve(NS.ChunkStore(root, preload=True), ("127.0.0.1", 0), rate_limit_gbps=rate)
    port_q.put(handle.address[1])
    stop.wait()
    handle.close()


class ModelLink:
    """A modelled link replayed against the real pipeline: chunk i is handed
    over (from pinned memory) when its last byte would have arrived at `rate`
    Gbps after the first request, i.e. a constant-rate BandwidthTrace
    (fk/fetchsim.py:93-139).  Isolates the GPU side from Python socket speed."""

    def __init__(self, store, rate_gbps):
        self.store, self.rate = store, rate_gbps * 1e9
        self.t0, self.sent, self.pinned = None, 0, {}

    def stage(self, chunks, codes):
        for code in codes:
            for cid, idx in chunks:
                meta, payload = self.store.lookup(cid, idx, code)
                t = torch.frombuffer(bytearray(payload), dtype=torch.uint8).pin_memory()
                self.pinned[(cid, idx, code)] = (meta, t)

    def __call__(self, address, cache_id, chunk_index, resolution, timeout_s=30.0, alloc=None):
        now = time.monotonic()
        if self.t0 is None:
            self.t0 = now
        code = resolution if isinstance(resolution, int) else L.RESOLUTION_CODE[resolution]
        meta, t = self.pinned[(bytes(cache_id), chunk_index, code)]
        self.sent += t.numel()
        if self.rate > 0:   # rate 0: no link limit (chunks handed over at once)
            arrive = self.t0 + self.sent * 8 / self.rate
            if arrive > now:
                time.sleep(arrive - now)
        return t, meta, time.monotonic() - now


def new_mems(qs, T, Lyr, H, D):
    """One paged bf16 pool per cache (K, V), preallocated like a serving engine's
    KV pool: ceil(T / 16) blocks x the padded layers."""
    return {cid: KV.PagedMemory(16, dtype=torch.bfloat16, H=H, D=D, num_blocks=-(-T // 16),
                                num_layers=3 * ((Lyr + 2) // 3)) for cid in qs}


def check(mems, qs, Lyr, T, n=64):
    g = torch.Generator().manual_seed(0)
    bad = 0
    for cid, q in qs.items():
        mem = mems[cid]
        for _ in range(n):
            t = int(torch.randint(0, T, (1,), generator=g))
            l = int(torch.randint(0, Lyr, (1,), generator=g))
            want = (q.values[t, l].float().reshape(q.H * q.D // q.group_size, -1)
                    * q.scales[l].reshape(-1, 1)).reshape(-1).to(torch.bfloat16)
            bad += int(not torch.equal(mem.read(t, l), want))
    return bad


def full_check(mems, qs, Lyr, T):
    """Every (token, layer) slot of every cache against dequantize(): the number
    of mismatching slots (paged pools gathered through their page maps)."""
    bad = 0
    for cid, q in qs.items():
        mem = mems[cid]
        tok = torch.arange(T)
        blk = torch.tensor([mem.pages[int(t) // mem.page_size_tokens] for t in range(0, T, mem.page_size_tokens)])
        phys = blk[tok // mem.page_size_tokens].cuda()
        off = (tok % mem.page_size_tokens).cuda()
        for l in range(Lyr):
            got = mem.layers[l][phys, off].reshape(T, -1)
            want = (q.values[:, l].float().reshape(T, q.H * q.D // q.group_size, -1)
                    * q.scales[l].reshape(1, -1, 1)).reshape(T, -1).to(torch.bfloat16).cuda()
            bad += int((got != want).any(dim=1).sum())
    return bad


def emit(tl, res, rate, coded, mems, qs, Lyr, args, setup_s, link, pass_no=0):
    recs = tl.records
    first = min(r["transfer_start"] for r in recs)
    last_rx = max(r["transfer_end"] for r in recs)
    line = {
        "config": "C5: llama3-8b K+V 32K, 88 chunks, pipelined fetch -> GPU decode -> "
                  "paged bf16 restore", "link": link, "resolution": res,
        "rate_gbps": rate, "coded_bytes": coded,
        "ready_s": round(tl.ttft - first, 4),
        "link_s_at_rate": round(coded * 8 / (rate * 1e9), 4) if rate else None,
        "receive_s": round(last_rx - first, 4),
        "delivered_gbps": round(coded * 8 / (last_rx - first) / 1e9, 2),
        "tail_after_last_byte_s": round(tl.ttft - last_rx, 4),
        "decode_batches": len({r["decode_start"] for r in recs}),
        "max_batch": max(r.get("batch", 1) for r in recs),
        "chosen": {k: sum(1 for r in recs if r["resolution"] == k)
                   for k in sorted({r["resolution"] for r in recs})},
        "total_bubble_s": round(tl.total_bubble, 4),
        "host_decode_s": round(sum(r.get("host_decode_s", 0) for r in {r["decode_start"]: r for r in recs}.values()), 4),
        "host_restore_s": round(sum(r.get("host_restore_s", 0) for r in {r["decode_start"]: r for r in recs}.values()), 4),
        "gpu_busy_s": round(sum(r["tau_dec"] for r in {r["decode_start"]: r for r in recs}.values()), 4),
        "sampled_slots_mismatch": check(mems, qs, Lyr, args.tokens),
        "all_slots_mismatch": full_check(mems, qs, Lyr, args.tokens) if args.full_check else None,
        "max_receive_gap_s": round(max((b["transfer_start"] - a["transfer_end"]
                                        for a, b in zip(recs, recs[1:])), default=0.0), 4),
        "max_gap_before_chunk": max(range(1, len(recs)), default=0,
                                    key=lambda i: recs[i]["transfer_start"] - recs[i - 1]["transfer_end"]),
        "batches": [(round(r["decode_start"], 4), round(r["decode_end"], 4), r.get("batch"),
                     round(r.get("host_decode_s", 0), 4), round(r.get("host_restore_s", 0), 4))
                    for r in {r["decode_start"]: r for r in recs}.values()] if args.verbose else None,
        "setup_pack_s": round(setup_s, 1), "pass": pass_no,
    }
    print(json.dumps(line), flush=True)
    return line


def summarize(lines, res, rate):
    import statistics
    r = sorted(x["ready_s"] for x in lines)
    p95 = r[min(len(r) - 1, int(round(0.95 * (len(r) - 1))))]
    print(json.dumps({"summary": True, "resolution": res, "rate_gbps": rate, "passes": len(r),
                      "ready_p50_s": round(statistics.median(r), 4), "ready_p95_s": round(p95, 4),
                      "ready_min_s": r[0], "ready_max_s": r[-1],
                      "p95_over_p50": round(p95 / statistics.median(r), 3),
                      "link_s_at_rate": lines[0]["link_s_at_rate"],
                      "mismatch": sum(x["sampled_slots_mismatch"] for x in lines)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--rates", default="10,25,100,0", help="Gbps; 0 = unthrottled loopback")
    ap.add_argument("--res", default="R240,R1080")
    ap.add_argument("--dir", default=None)
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--verbose", action="store_true", help="per-batch timings in each line")
    ap.add_argument("--full-check", action="store_true", help="compare every slot, not a sample")
    ap.add_argument("--passes", type=int, default=1,
                    help="timed passes per (class, rate); > 1 adds a p50/p95 summary line")
    ap.add_argument("--link", default="model", choices=["model", "tcp"],
                    help="model: constant-rate arrival replay; tcp: live loopback server")
    args = ap.parse_args()
    Lyr, H, D = 32, 8, 128
    resolutions = args.res.split(",")
    root = args.dir or tempfile.mkdtemp(prefix="kvfc_store_")
    t0 = time.perf_counter()
    chunks, qs, pack_s = build_store(root, args.tokens, Lyr, H, D, resolutions)
    setup_s = time.perf_counter() - t0
    print(json.dumps({"producer": "container.pack_chunks", "units": len(chunks),
                      "classes": resolutions, "pack_chunks_s": round(pack_s, 2),
                      "setup_total_s": round(setup_s, 1)}), flush=True)
    store = NS.ChunkStore(root)
    ctx = mp.get_context("spawn")
    for res in resolutions + (["adaptive"] if args.link == "model" and len(resolutions) == 4 else []):
        codes = ([L.RESOLUTION_CODE[r] for r in resolutions] if res == "adaptive"
                 else [L.RESOLUTION_CODE[res]])
        code = codes[0]
        coded = sum(store.index[(cid, idx)]["entries"][code][1] for cid, idx in chunks)  # fixed classes
        policy = "adaptive" if res == "adaptive" else f"fixed:{res}"
        # untimed warm-up: pins the receive pool, loads kernels and grows every
        # worker stream's grow-only buffers (large batches at 1000 Gbps, many
        # small ones at 50 Gbps) so timed runs allocate no device memory
        for warm_rate in (1000.0, 50.0):
            link = ModelLink(store, warm_rate)
            link.stage(chunks, codes)
            FE.live_fetch_pipeline(None, chunks, None, policy, prior_gbps=10.0,
                                   mem=new_mems(qs, args.tokens, Lyr, H, D), real_layers=Lyr,
                                   fetch_fn=link)
            del link
        for rate in [float(r) for r in args.rates.split(",")] if args.link == "model" else []:
            lines = []
            for k in range(args.passes):
                link = ModelLink(store, rate)
                link.stage(chunks, codes)
                mems = new_mems(qs, args.tokens, Lyr, H, D)
                gc.collect()   # no collector pause inside the timed fetch
                torch.cuda.synchronize()
                tl = FE.live_fetch_pipeline(None, chunks, None, policy, prior_gbps=rate or 400.0,
                                            mem=mems, real_layers=Lyr, fetch_fn=link,
                                            workers=args.workers)
                lines.append(emit(tl, res, rate, coded, mems, qs, Lyr, args, setup_s,
                                  "modelled constant-rate link", k))
                del mems, link
            if args.passes > 1:
                summarize(lines, res, rate)
        for rate in [float(r) for r in args.rates.split(",")] if args.link == "tcp" else []:
            # the chunk server runs in its own process (a remote node's role):
            # it does not share this process's GIL with the fetcher
            port_q, stop = ctx.Queue(), ctx.Event()
            srv = ctx.Process(target=serve_proc, args=(root, rate or None, port_q, stop))
            srv.start()
            mems = new_mems(qs, args.tokens, Lyr, H, D)
            try:
                addr = f"127.0.0.1:{port_q.get(timeout=120)}"
                torch.cuda.synchronize()
                tl = FE.live_fetch_pipeline(addr, chunks, None, f"fixed:{res}", mem=mems,
                                            real_layers=Lyr)
            finally:
                stop.set()
                srv.join(timeout=30)
            emit(tl, res, rate or None, coded, mems, qs, Lyr, args, setup_s,
                 "loopback TCP, reference wire protocol, paced egress")
            del mems
    if args.dir is None:
        shutil.rmtree(root, ignore_errors=True)


if __name__ == "__main__":
    main()
