#!/usr/bin/env python
"""KV restore benchmark (frames -> bf16 paged KV), B200.

Workload (BASELINE.json configs[1]): Llama-3-8B-shaped K and V (32 layers -> 33
padded = 11 layer triplets, 8 KV heads, head dim 128), 32,768 tokens, chunked
into the reference's <=10,000-token containers (10000+10000+10000+2768) -> 88
(K/V, triplet, chunk) units.  Frames are produced once on the GPU by our pack
kernels from synthetic AR(1) bf16 KV (the reference generator's law); each step
restores all 88 units into a vLLM-style paged cache (block size 16, shuffled
block table) in one batched libkvf launch.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints one JSON line (rank 0).  value = KV restore GB/s (bf16 bytes delivered
= 2 B x K+V elements of real layers / step time, device events, max over ranks).
"""

from __future__ import annotations

import argparse
import json
import os
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context: see paper_2602_09725_b200.use_fetch_hw_queues
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODELS = {  # name -> (layers, kv heads, head dim)
    "llama3-8b": (32, 8, 128),
    "qwen2.5-7b": (28, 4, 128),
    "llama3-70b": (80, 8, 128),
}
LAYOUTS = {  # name -> (a_h, b_h, a_d, b_d) as functions of (H, D)
    "identity": lambda H, D: (1, H, 1, D),
    "paper": lambda H, D: (H, 1, 1, D),
    # tile rows narrower than 8 channels (shared-memory band kernels):
    "col1": lambda H, D: (1, H, D, 1),            # (8,128,1,8,128,1): tile D x H
    "a2b4": lambda H, D: (2, H // 2, D // 4, 4),  # (8,128,2,4,32,4): tile 64 x 16
}
CHUNK = 10_000  # fk/container.py:29 DEFAULT_CHUNK_TOKENS


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama3-8b", choices=sorted(MODELS))
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--layout", default="identity", choices=sorted(LAYOUTS))
    ap.add_argument("--res", default="R1080")
    ap.add_argument("--page", type=int, default=16)
    ap.add_argument("--requests", type=int, default=1,
                    help="contexts in the job: 1 (default) = one context split over the "
                         "GPUs (strong scaling); 0 = one context per GPU (weak scaling)")
    ap.add_argument("--shard", default="balanced", choices=["balanced", "layer", "chunk"],
                    help="unit -> GPU assignment policy (paper_2602_09725_b200/shard.py)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fetch", action="store_true", help="skip the fetch-to-ready leg")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--cpu-tokens", type=int, default=2000,
                    help="tokens of the sample unit each CPU worker restores per step")
    return ap.parse_args()


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons polled through NVML (the library nvidia-smi
    uses) every ~2 ms on a thread, between __enter__ and __exit__ — i.e. during
    the timed region.  Falls back to `nvidia-smi -lms` if NVML is unavailable."""

    REASONS = {  # NVML clocks-event-reason bits (nvml.h)
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap",
    }

    def __init__(self, index: int):
        self.index = index
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._nvml = None
        self._proc = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
        except Exception:
            self._nvml = None
            try:
                self._proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index),
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                     "--format=csv,noheader,nounits", "-lms", "50"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self._t = threading.Thread(target=self._read_smi, daemon=True)
                self._t.start()
            except OSError:
                self._proc = None
        return self

    def _poll(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for b, name in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                break
            time.sleep(0.002)

    def _read_smi(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self._proc.stdout:
            f = [x.strip() for x in line.split(",")]
            try:
                self.sm.append(float(f[0]))
                self.max_mhz = float(f[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    self.reasons.add(n)

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self._t.join(timeout=2)
        if self._proc is not None:
            self._proc.terminate()
            self._proc.wait(timeout=5)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


# ------------------------------------------------------------------- workload
def chunks_of(T):
    out, t = [], 0
    while t < T:
        out.append((t, min(CHUNK, T - t)))
        t += CHUNK
    return out


class Workload:
    """Frames for this rank's (request, K/V, triplet, chunk) units + their paged caches.

    Units come from shard.enumerate_units over `requests` contexts and are
    assigned to ranks by shard.assign; a rank builds only its own units.  Per
    owned (request, K/V, triplet) it generates a synthetic [T, 3, H, D] bf16
    slab on the GPU (AR(1) law of gen_synthetic_kv), packs its chunks into
    frames with our pack kernels, and allocates the destination paged cache
    [3, blocks, block_size, H, D] (shuffled block table).
    """

    def __init__(self, args, device, rank=0, world=1):
        import torch
        from paper_2602_09725_b200 import _dev, _lib, kvmodel as KV, layout as L, shard
        from paper_2602_09725_b200.restore import make_restore_unit

        self.torch = torch
        Lyr, H, D = MODELS[args.model]
        self.Lyr, self.H, self.D, self.T = Lyr, H, D, args.tokens
        self.gs = 128
        lay = L.LayoutConfig(H, D, *LAYOUTS[args.layout](H, D))
        self.lay = lay
        bs = self.page = args.page
        nblk = (self.T + bs - 1) // bs
        g = torch.Generator(device="cpu")
        g.manual_seed(1234)
        self.table = torch.randperm(nblk + 64, generator=g)[:nblk].to(torch.int32).to(device)
        all_units = shard.enumerate_units(self.T, Lyr, requests=args.requests or world,
                                          chunk_tokens=CHUNK)
        self.all_units = len(all_units)
        self.mine = shard.units_for_rank(all_units, rank, world, args.shard, H, D)
        self.pack_units, self.units, self.frames, self.scales = [], [], [], []
        self.caches, self._keep, self._specs, self.slabs = [], [], [], []
        self.elems = sum(u.elements(H, D) for u in self.mine)
        keys = sorted({(u.request, u.kv, u.triplet) for u in self.mine})
        for (r, kv_i, j) in keys:
            real = min(3, Lyr - 3 * j)
            seed = (r * 2 + kv_i) * 1000 + j
            slab = KV.gen_synthetic_kv(self.T, real, H, D, 0.9, seed=seed, channel_smoothness=0.3,
                                       dtype=torch.bfloat16).data
            cache = torch.empty((real, nblk + 64, bs, H, D), dtype=torch.bfloat16, device=device)
            self._keep += [slab]
            self.slabs.append(slab)
            self.caches.append(cache)
            for u in (u for u in self.mine if (u.request, u.kv, u.triplet) == (r, kv_i, j)):
                t0, tc = u.token_start, u.tokens
                plan = L.plan_inter_frame(tc, args.res, lay, 4)
                fr = torch.empty(plan.frame_shape(), dtype=torch.uint8, device=device)
                am = torch.zeros(_lib.load().kvf_pack_scratch_words(plan.to_c(self.gs)),
                                 dtype=torch.int32, device=device)
                sc = torch.empty((3, H * D // self.gs), dtype=torch.float32, device=device)
                src = _lib.kvf_paged()
                dst = _lib.kvf_paged()
                for p in range(3):
                    src.layer[p] = slab[:, p].data_ptr() if p < real else None
                    dst.layer[p] = cache[p].data_ptr() if p < real else None
                src.block_table = None
                src.block_size = 1
                src.dtype = _lib.KVF_BF16
                src.block_stride = src.slot_stride = real * H * D
                src.head_stride = D
                src.token_base = t0
                dst.block_table = self.table.data_ptr()
                dst.block_size = bs
                dst.dtype = _lib.KVF_BF16
                dst.block_stride = bs * H * D
                dst.slot_stride = H * D
                dst.head_stride = D
                dst.token_base = t0
                self._specs.append((src, dst, tc))
                pu = _lib.kvf_pack_unit()
                pu.src = src
                pu.plan = plan.to_c(self.gs)
                pu.absmax = am.data_ptr()
                pu.scales = sc.data_ptr()
                pu.frames = _dev.surface_of(fr)
                self.pack_units.append(pu)
                self.units.append(make_restore_unit(fr, plan, sc, dst, self.gs))
                self.frames.append(fr)
                self.scales.append(sc)
                self._keep.append(am)
        self.frame_bytes = sum(f.numel() for f in self.frames)
        self._pack_arr = (_lib.kvf_pack_unit * len(self.pack_units))(*self.pack_units)
        self._restore_arr = (_lib.kvf_restore_unit * len(self.units))(*self.units)
        self._lib, self._dev, self._L = _lib, _dev, L
        self.n_launch_restore = (len(self.units) + _lib.KVF_MAX_UNITS - 1) // _lib.KVF_MAX_UNITS
        self.n_launch_pack = 4 * self.n_launch_restore
        # the sources, zeroed scratch and block table were produced on the
        # current stream; callers pack/restore on streams of their own
        torch.cuda.synchronize()

    def check_restored(self, per_unit=16):
        """Sampled slots of the restored caches against an independent path:
        the whole-tensor quantize kernel (kvf_quantize) of each unit's token
        chunk, dequantised in fp32 and rounded to bf16.  Returns (slots, mismatches)."""
        torch = self.torch
        from paper_2602_09725_b200 import kvmodel as KV
        g = torch.Generator(device="cpu")
        g.manual_seed(7)
        slots = bad = 0
        keys = sorted({(u.request, u.kv, u.triplet) for u in self.mine})
        for (r, kv_i, j), slab, cache in zip(keys, self.slabs, self.caches):
            for u in (u for u in self.mine if (u.request, u.kv, u.triplet) == (r, kv_i, j)):
                t0, tc = u.token_start, u.tokens
                q = KV.quantize(KV.KVCache(slab[t0:t0 + tc].contiguous()), self.gs)
                deq = KV.dequantize(q, torch.bfloat16).data          # [tc, real, H, D]
                toks = torch.randint(0, tc, (per_unit,), generator=g)
                for t in toks.tolist():
                    tt = t0 + t
                    blk = int(self.table[tt // self.page])
                    for p in range(u.real_layers):
                        got = cache[p][blk, tt % self.page]
                        slots += 1
                        bad += int(not torch.equal(got, deq[t, p]))
        return slots, bad

    def frames_at(self, res):
        """Pack every unit again at another resolution class (same sources,
        caches and scales); returns (frames, restore unit descriptors)."""
        torch = self.torch
        from paper_2602_09725_b200.restore import make_restore_unit
        frames, pus, rus, keep = [], [], [], []
        for (src, dst, tc), sc in zip(self._specs, self.scales):
            plan = self._L.plan_inter_frame(tc, res, self.lay, 4)
            fr = torch.empty(plan.frame_shape(), dtype=torch.uint8, device=sc.device)
            am = torch.zeros(self._lib.load().kvf_pack_scratch_words(plan.to_c(self.gs)),
                             dtype=torch.int32, device=sc.device)
            pu = self._lib.kvf_pack_unit()
            pu.src, pu.plan, pu.absmax, pu.scales = src, plan.to_c(self.gs), am.data_ptr(), sc.data_ptr()
            pu.frames = self._dev.surface_of(fr)
            pus.append(pu)
            rus.append(make_restore_unit(fr, plan, sc, dst, self.gs))
            frames.append(fr)
            keep.append(am)
        arr = (self._lib.kvf_pack_unit * len(pus))(*pus)
        self._lib.call("kvf_pack_batch", arr, len(pus), self._dev.stream_ptr(torch.cuda.current_stream()))
        torch.cuda.synchronize()
        return frames, rus

    def pack(self, stream):
        self._lib.call("kvf_pack_batch", self._pack_arr, len(self.pack_units),
                       self._dev.stream_ptr(stream))

    def pack_frames_only(self, stream):
        """Phase 2 alone with the maxima already in the units' scratch (left by
        pack()): the single-read pack a KV writer that tracks maxima gets."""
        self._lib.call("kvf_pack_frames_batch", self._pack_arr, len(self.pack_units),
                       self._dev.stream_ptr(stream))

    def restore(self, stream):
        self._lib.call("kvf_restore_batch", self._restore_arr, len(self.units),
                       self._dev.stream_ptr(stream))


def time_device(fn, stream, steps, warmup, torch, dist=None):
    for _ in range(warmup):
        fn(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    per = []
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    with torch.cuda.stream(stream):
        start.record(stream)
        evs[0].record(stream)
        for k in range(steps):
            fn(stream)
            evs[k + 1].record(stream)
        stop.record(stream)
    torch.cuda.synchronize()
    total_ms = start.elapsed_time(stop)
    per = [evs[k].elapsed_time(evs[k + 1]) for k in range(steps)]
    return total_ms, per


def e2e_restore(w, steps, torch):
    """Same restore through the C ABI with HOST frames: per unit, a pinned H2D
    copy on a copy stream overlapped with the previous unit's restore; one
    2 KB D2H read of the last restored slot closes each step."""
    from paper_2602_09725_b200 import _lib
    dev = torch.device("cuda")
    host = [torch.empty(f.shape, dtype=torch.uint8, pin_memory=True) for f in w.frames]
    for h, f in zip(host, w.frames):
        h.copy_(f)
    nslot = 4
    maxb = max(f.numel() for f in w.frames)
    stage = [torch.empty(maxb, dtype=torch.uint8, device=dev) for _ in range(nslot)]
    copy_s = torch.cuda.Stream()
    comp_s = torch.cuda.Stream()
    free_ev = [None] * nslot
    out_host = torch.empty(w.H * w.D, dtype=torch.bfloat16, pin_memory=True)
    units = []
    for k, u in enumerate(w.units):
        nu = _lib.kvf_restore_unit()
        ctypes_copy(nu, u)
        units.append(nu)

    # the first slot the last unit writes (layer 0 of its triplet) is read back
    u_last = w.mine[-1]
    blk = int(w.table[u_last.token_start // w.page].item())
    last = w.caches[-1][0, blk, u_last.token_start % w.page].reshape(-1)

    def step():
        for k, u in enumerate(units):
            s = k % nslot
            buf = stage[s][: host[k].numel()].view(host[k].shape)
            with torch.cuda.stream(copy_s):
                if free_ev[s] is not None:
                    copy_s.wait_event(free_ev[s])
                buf.copy_(host[k], non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(copy_s)
            comp_s.wait_event(ready)
            u.frames.base = buf.data_ptr()
            _lib.call("kvf_restore_batch", u, 1, w._dev.stream_ptr(comp_s))
            ev = torch.cuda.Event()
            ev.record(comp_s)
            free_ev[s] = ev
        with torch.cuda.stream(comp_s):
            out_host.copy_(last, non_blocking=True)
        comp_s.synchronize()

    step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    return ms, w.frame_bytes, out_host.numel() * 2


def fetch_to_ready(w, steps, torch, frames_units=None):
    """Fetch-to-ready of the whole context from coded KVFC streams in pinned host
    memory (what a fetch receives): per step one H2D of every stream's bytes,
    GPU entropy decode + reconstruction of all 88 units (codec.decode_batch: 2
    launches), then the batched restore into the paged cache.  Wall clock,
    host work included; the network leg is modelled from the coded bytes."""
    from paper_2602_09725_b200 import _lib, codec
    src_frames, src_units = frames_units if frames_units else (w.frames, w.units)
    frame_bytes = sum(f.numel() for f in src_frames)
    t0 = time.perf_counter()
    streams = [bs.data for bs in codec.encode_batch(src_frames, [4] * len(src_frames))]
    enc_s = time.perf_counter() - t0
    coded = sum(len(b) for b in streams)
    # what a fetch's receive ring holds: the coded bytes in pinned host memory
    streams = [torch.frombuffer(bytearray(b), dtype=torch.uint8).pin_memory() for b in streams]
    indices = codec.index_streams(streams)
    frames, _ = codec.decode_batch(streams, indices=indices)
    ok = all(torch.equal(a, b) for a, b in zip(frames, src_frames))
    units = []
    for u, fr in zip(src_units, frames):
        nu = _lib.kvf_restore_unit()
        ctypes_copy(nu, u)
        nu.frames.base = fr.data_ptr()
        units.append(nu)
    arr = (_lib.kvf_restore_unit * len(units))(*units)
    stream = torch.cuda.current_stream()

    def step():
        # the host stream walk runs inside decode_batch, beside the H2D copies
        out, _ = codec.decode_batch(streams, out=frames)
        _lib.call("kvf_restore_batch", arr, len(units), w._dev.stream_ptr(stream))
        torch.cuda.synchronize()

    step()
    times, scan = [], []
    for _ in range(steps):
        t1 = time.perf_counter()
        step()
        times.append((time.perf_counter() - t1) * 1e3)
        t2 = time.perf_counter()
        codec.index_streams(streams)         # the walk alone, for the report
        scan.append((time.perf_counter() - t2) * 1e3)
    ms = statistics.median(times)
    return {"ms": round(ms, 2), "scan_ms": round(statistics.median(scan), 2),
            "coded_bytes": coded, "frame_bytes": frame_bytes,
            "ratio_int8_over_coded": round(frame_bytes / coded, 3),
            "decode_bitexact": ok, "encode_s": round(enc_s, 2),
            "link_s": {f"{g}gbps": round(coded * 8 / (g * 1e9), 3) for g in (10, 25, 100)}}


def ctypes_copy(dst, src):
    import ctypes
    ctypes.memmove(ctypes.addressof(dst), ctypes.addressof(src), ctypes.sizeof(src))


def ncu_traffic(kernel: str, config_key: str, launches_per_step: int = 1):
    """DRAM bytes per launch of `kernel` from a committed ncu --set full capture
    of THIS configuration (profiles/<round>/ncu_traffic.json, written by
    tools/ncu_summary.py with the bench config key), or None: a profile of
    another configuration is not this run's traffic."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_traffic.json")),
                       reverse=True):
        try:
            with open(path) as fh:
                rec = json.load(fh).get(kernel)
        except (OSError, ValueError):
            continue
        if rec and rec.get("config") == config_key:
            n = rec.get("launches_captured", 1)
            return {"bytes_per_launch": rec["dram_bytes_per_launch"],
                    "bytes_per_step": rec.get("dram_bytes_captured", rec["dram_bytes_per_launch"])
                    if n == launches_per_step else None,
                    "source": os.path.relpath(path, ROOT) + " (" + rec["report"] + (
                        f", {n} launches = one step" if n > 1 else "") + ")"}
    return None


def config_key(args, world):
    return (f"{args.model}/{args.tokens}/{args.layout}/{args.res}/page{args.page}/"
            f"req{args.requests}/{args.shard}/n{world}")


def count_launches(fn, stream, torch):
    """Kernel launches of ONE step, observed with the CUDA activity profiler
    (CUPTI) on an extra, untimed step: {kernel name: count}, or None."""
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn(stream)
            torch.cuda.synchronize()
        out = {}
        for e in prof.events():
            if getattr(e, "device_type", None) is not None and "CUDA" in str(e.device_type):
                out[e.name] = out.get(e.name, 0) + 1
        return out or None
    except Exception:  # profiler unavailable: reported as unobserved
        return None


def oracle_unit_check(w, torch):
    """Every slot of one full reference chunk (unit 0: 10,000 tokens x its real
    layers) against the CPU oracle: quantize (fk/kvmodel.py:127-144) ->
    dequantize (fk/kvmodel.py:147-152) -> bf16 RNE, vs the restored paged
    cache read through the block table.  Returns (slots, mismatching slots)."""
    from oracle import ref
    u = w.mine[0]
    k = sorted({(x.request, x.kv, x.triplet) for x in w.mine}).index((u.request, u.kv, u.triplet))
    slab, cache = w.slabs[k], w.caches[k]
    t0, tc, real = u.token_start, u.tokens, u.real_layers
    x = slab[t0:t0 + tc].float().cpu().numpy()                      # [tc, real, H, D]
    xp = np.zeros((tc, 3, w.H, w.D), np.float32)
    xp[:, :real] = x
    v, s = ref.quantize(xp, 128)
    want = torch.from_numpy(ref.dequantize(v, s, 128)).to(torch.bfloat16)[:, :real]
    toks = torch.arange(t0, t0 + tc)
    blk = w.table.cpu()[toks // w.page].long()
    got = torch.stack([cache[p][blk.to(cache.device), (toks % w.page).to(cache.device)].cpu()
                       for p in range(real)], dim=1)                  # [tc, real, H, D]
    bad = (got.view(torch.int16) != want.view(torch.int16)).reshape(tc, real, -1).any(-1)
    return int(tc * real), int(bad.sum())


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh).get("hbm_gbs", 6650.0), "measured"
    except OSError:
        return 6650.0, "fallback"


def run_reference(args, rank, world):
    """--impl reference: the reference's own restore code (vendored framekv,
    oracle/bench_ref.py) on all host cores; rank 0 only."""
    if rank != 0:
        return
    from oracle import bench_ref
    Lyr, H, D = MODELS[args.model]
    lay = (H, D) + LAYOUTS[args.layout](H, D)
    if not bench_ref.available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/framekv_ref not vendored"}), flush=True)
        return
    single = cpu_reference(args, H, D, lay, workers=1, steps=3)
    r = bench_ref.RefRestore(T=args.cpu_tokens, H=H, D=D, res=args.res, lay=lay)
    for _ in range(args.warmup):
        r.step()
    elems = wall = 0.0
    for _ in range(args.steps):
        e, t = r.step()
        elems += e
        wall += t
    r.close()
    gbs = 2.0 * elems / wall / 1e9
    cores = r.workers
    line = {
        "metric": "KV restore GB/s (frames->bf16 paged KV), 32K ctx", "impl": "reference",
        "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * wall / args.steps, 3),
        "higher_is_better": True, "scaling": scaling_kind(args), "vs_baseline": None,
        "dtype": "u8->bf16", "data": "synthetic", "config": workload_config(args, world),
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores,
                         "kind": "reference", "cpu_model": bench_ref.cpu_model(),
                         "sample": f"{cores} processes x 1 unit of {args.cpu_tokens} tokens x 3 "
                                   f"layers ({args.model} shape, {args.layout}, {args.res}) per "
                                   f"step: reference disassemble_frames + dequantize + bf16 + "
                                   f"PagedMemory.page_write (vendored framekv)",
                         "single_process": single},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_reference(args, H, D, lay, workers=None, steps=5):
    """The reference restore on `workers` processes (None = all cores)."""
    from oracle import bench_ref
    r = bench_ref.RefRestore(workers=workers, T=args.cpu_tokens, H=H, D=D, res=args.res, lay=lay)
    elems = wall = 0.0
    for _ in range(steps):
        e, t = r.step()
        elems += e
        wall += t
    r.close()
    return {"value": round(2.0 * elems / wall / 1e9, 4), "unit": "GB/s", "cores": r.workers,
            "kind": "reference", "cpu_model": bench_ref.cpu_model(),
            "sample": f"{r.workers} process(es) x {steps} steps x 1 unit of {args.cpu_tokens} "
                      f"tokens x 3 layers: reference disassemble_frames + dequantize + bf16 + "
                      f"PagedMemory.page_write (vendored framekv, oracle/bench_ref.py)"}


def scaling_kind(args):
    return "weak" if args.requests == 0 else "strong"


def workload_config(args, world=1, l2=None):
    Lyr, H, D = MODELS[args.model]
    req = args.requests or world
    return {"workload": f"{req} x {args.model}-shaped K+V context(s), {args.tokens} tokens, "
                        f"{Lyr} layers (+pad to x3), {H} KV heads, d={D}: frames -> bf16 paged "
                        f"KV restore",
            "model_shape": args.model, "tokens": args.tokens, "requests": req,
            "layout": args.layout, "resolution": args.res, "chunk_tokens": CHUNK,
            "group_size": 128, "F": 4, "block_size": args.page,
            "parallelism": f"dp{world}: (request, K/V, triplet, chunk) units sharded "
                           f"'{args.shard}' across GPUs, no data-path collective",
            "l2": l2}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2602_09725_b200 import shard

    # one process per GPU; --dist-backend gloo with more ranks than GPUs lets the
    # N>1 path (sharding, max/sum over ranks) run on a single-GPU box for checks
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    d = dist if world > 1 else None

    w = Workload(args, dev, rank, world)
    stream = torch.cuda.Stream()
    # pack (secondary): frames for the restore steps come from here
    pack_ms, pack_per = time_device(w.pack, stream, max(3, args.steps // 2), args.warmup, torch, d)
    pack_ms /= max(3, args.steps // 2)
    pk2_ms, _ = time_device(w.pack_frames_only, stream, max(3, args.steps // 2), args.warmup,
                            torch, d)
    pk2_ms = shard.max_over_ranks(pk2_ms / max(3, args.steps // 2), d, dev)
    with ClockSampler(local) as clk:
        total_ms, per = time_device(w.restore, stream, args.steps, args.warmup, torch, d)
    ms = shard.max_over_ranks(total_ms / args.steps, d, dev)
    pack_ms = shard.max_over_ranks(pack_ms, d, dev)
    elems_total = int(shard.sum_over_ranks(w.elems, d, dev))
    value = 2.0 * elems_total / (ms * 1e-3) / 1e9
    peak, peak_kind = load_peaks()
    achieved = 3.0 * w.elems / (ms * 1e-3) / 1e9  # per GPU, algorithmic bytes
    pack_ach = 3.0 * w.elems / (pack_ms * 1e-3) / 1e9

    chk_slots, chk_bad = w.check_restored()   # after the timed restores, outside timing
    orc_slots, orc_bad = oracle_unit_check(w, torch) if rank == 0 else (0, 0)
    launches = count_launches(w.restore, stream, torch)
    units_per_rank = [len(w.units)]
    if d is not None:
        units_per_rank = [None] * world
        d.all_gather_object(units_per_rank, len(w.units))
    props = torch.cuda.get_device_properties(dev)
    l2 = {"l2_bytes": int(getattr(props, "L2_cache_size", 0)),
          "frames_in_per_step_bytes": int(w.frame_bytes), "kv_out_per_step_bytes": 2 * w.elems,
          "inputs_exceed_l2": bool(w.frame_bytes > getattr(props, "L2_cache_size", 0)),
          "note": "per GPU; no L2 flush between steps: inputs exceed L2"
                  if w.frame_bytes > getattr(props, "L2_cache_size", 0) else
                  "per GPU; inputs fit in L2 (no flush between steps)"}
    e2e = None
    if not args.no_e2e:
        e2e_ms, h2d, d2h = e2e_restore(w, max(3, args.steps // 4), torch)
        e2e_ms = shard.max_over_ranks(e2e_ms, d, dev)
        e2e = {"value": round(2.0 * elems_total / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(e2e_ms, 3),
               "path": "pinned host frames -> H2D (copy stream) overlapped with per-unit "
                       "kvf_restore_batch (compute stream) -> 2 KB D2H"}

    fetch = None
    if not args.no_fetch:
        fetch = fetch_to_ready(w, 7, torch)   # median of 7 wall-clock steps
        fetch["resolution"] = args.res
        if args.res != "R240":  # the class the adaptive policy picks at >= 10 Gbps
            alt = fetch_to_ready(w, 7, torch, w.frames_at("R240"))
            fetch["R240"] = {k: alt[k] for k in ("ms", "coded_bytes", "decode_bitexact")}

    cpu = None
    if rank == 0 and not args.no_cpu:
        from oracle import bench_cpu, bench_ref
        Lyr, H, D = MODELS[args.model]
        lay = (H, D) + LAYOUTS[args.layout](H, D)
        if bench_ref.available():
            cpu = cpu_reference(args, H, D, lay, steps=5)
            cpu["single_process"] = cpu_reference(args, H, D, lay, workers=1, steps=2)
        if fetch is not None:  # the same host's cores decoding the context's KVFC streams
            sym, dwall, dcores = bench_cpu.run("decode", units_per_worker=1, T=CHUNK, H=H, D=D,
                                               res=args.res, lay=lay)
            rate = sym / dwall
            fetch["cpu_decode"] = {
                "msym_per_s": round(rate / 1e6, 1), "cores": dcores, "kind": "port",
                "est_context_decode_s": round(fetch["frame_bytes"] / rate, 2),
                "sample": f"{dcores} processes x 8 {args.res} frames: C restatement of "
                          f"decode_frames (fk/codec.py:155-211, fk/rangecoder.py:146-189)"}

    if rank == 0:
        clocks = clk.summary()
        # the restore launches of one step cover all units: the ncu traffic of
        # a capture of exactly those launches compares with
        # algorithmic_bytes_per_step (multi-GPU: per rank)
        rkernel = "restore_band_kernel" if LAYOUTS[args.layout](w.H, w.D)[3] < 8 \
            else "restore_fast_kernel"
        traffic = ncu_traffic(rkernel, config_key(args, world),
                              sum(launches.values()) if launches else 1)
        line = {
            "metric": "KV restore GB/s (frames->bf16 paged KV), 32K ctx",
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": scaling_kind(args), "vs_baseline": None, "dtype": "u8->bf16",
            "data": "synthetic", "config": workload_config(args, world, l2),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic and traffic["bytes_per_step"],
                         "traffic_source": traffic["source"] if traffic else
                         "no ncu capture of this configuration committed",
                         "peak_kind": peak_kind,
                         "kernel": f"{rkernel} (kvf_restore_batch)",
                         "algorithmic_bytes_per_step": 3 * w.elems},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "fetch_to_ready": fetch,
            "gpu_launches": (sum(launches.values()) * args.steps if launches
                             else w.n_launch_restore * args.steps),
            "gpu_launches_source": ({"per_step": launches, "how": "CUDA activity profiler "
                                     "(CUPTI) over one extra untimed step, x steps"}
                                    if launches else "computed (profiler unavailable)"),
            "restore_check": {
                "oracle_unit": {"slots": orc_slots, "mismatch": orc_bad,
                                "against": "oracle quantize -> dequantize -> bf16 of every slot "
                                           "of unit 0 (one full 10,000-token chunk), read back "
                                           "through the block table"},
                "sampled": {"slots": chk_slots, "mismatch": chk_bad,
                            "against": "kvf_quantize of each unit's token chunk, dequantised "
                                       "and rounded to bf16 (16 sampled tokens per unit)"}},
            "clocks": clocks,
            "pack": {"ms_per_step": round(pack_ms, 4),
                     "achieved_gbs": round(pack_ach, 1), "frac": round(pack_ach / peak, 4),
                     "launches_per_step": w.n_launch_pack,
                     "given_maxima": {
                         "ms_per_step": round(pk2_ms, 4),
                         "frac": round(3.0 * w.elems / (pk2_ms * 1e-3) / 1e9 / peak, 4),
                         "what": "kvf_pack_frames_batch: scales + frames with the per-group "
                                 "maxima supplied (single read); the reference computes them, "
                                 "which is the two-pass figure above"}},
            "step_ms_min_max": [round(min(per), 4), round(max(per), 4)],
            "units": w.all_units, "units_per_rank": units_per_rank, "elems_rank0": w.elems,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
