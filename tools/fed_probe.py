"""Fed decode probe: C2 KVFC streams in pinned host memory, decode_batch timed
with the fed path (kvf_rc_decode_fed) and with the part pipeline, for several
copy-CTA counts and piece sizes; plus the fed launch's copy side alone."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_09725_b200 import codec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--res", default="R1080")
    ap.add_argument("--quick", action="store_true", help="one fed decode (for ncu)")
    ap.add_argument("--ctas", type=lambda x: [int(v) for v in x.split(",")], default=[32, 128, 512])
    ap.add_argument("--pieces", type=lambda x: [int(v) for v in x.split(",")], default=[4096, 16384])
    ap.add_argument("--copy-only", type=lambda x: [int(v) for v in x.split(",") if v],
                    default=[32, 128, 512])
    a = ap.parse_args()
    args = argparse.Namespace(model="llama3-8b", tokens=32768, layout="identity", res=a.res,
                              page=16, requests=1, shard="balanced")
    w = bench.Workload(args, torch.device("cuda", 0))
    streams = [bs.data for bs in codec.encode_batch(w.frames, [4] * len(w.frames))]
    streams = [torch.frombuffer(bytearray(b), dtype=torch.uint8).pin_memory() for b in streams]
    frames = [torch.empty_like(f) for f in w.frames]

    def run(label):
        codec.decode_batch(streams, out=frames)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            codec.decode_batch(streams, out=frames)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t) * 1e3)
        ok = all(torch.equal(x, y) for x, y in zip(frames, w.frames))
        print(f"{label:40s} {min(ts):8.1f} ms  bitexact={ok}", flush=True)

    if a.quick:
        codec.decode_batch(streams, out=frames)
        torch.cuda.synchronize()
        return
    base_min = codec._FED_MIN_SYMBOLS
    codec._FED_MIN_SYMBOLS = 1 << 40
    run("part pipeline")
    codec._FED_MIN_SYMBOLS = base_min
    for ctas in a.ctas:
        for piece in a.pieces:
            codec._FED_COPY_CTAS, codec._FED_PIECE = ctas, piece
            run(f"fed copy_ctas={ctas} piece={piece}")
    # the copy side alone: a fed launch whose decoders have nothing to decode
    real = codec._part_descriptors
    real_pin = codec._pinned_copy

    def no_decode(*x, **kw):
        rc, flat, ch = real(*x, **kw)
        return rc, flat[:0], ch[:0]

    def no_symbols(a):  # the fed launch's range-decode descriptors: nothing to decode
        if a.dtype == codec._RC_DTYPE:
            a = a.copy()
            a["len"] = 0
            a["n_symbols"] = 0
        return real_pin(a)
    codec._part_descriptors = no_decode
    codec._pinned_copy = no_symbols
    for ctas in a.copy_only:
        codec._FED_COPY_CTAS, codec._FED_PIECE = ctas, 16384
        codec.decode_batch(streams, out=frames)
        torch.cuda.synchronize()
        t = time.perf_counter()
        codec.decode_batch(streams, out=frames)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) * 1e3
        nb = sum(s.numel() for s in streams)
        print(f"copy only copy_ctas={ctas}: {ms:.1f} ms = {nb / ms / 1e6:.1f} GB/s (incl. walk)",
              flush=True)
    codec._part_descriptors = real
    codec._pinned_copy = real_pin


if __name__ == "__main__":
    main()
