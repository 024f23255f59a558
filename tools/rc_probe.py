"""Range-decode kernel time on device-resident C2 streams (CUPTI kernel durations).

    python tools/rc_probe.py [--lib path/to/libkvf.so] [--res R1080] [--pinned]

decode_batch over the bytes of every C2 stream with one part (one
rc_decode_kernel launch for all planes) and with the default part pipeline,
or (--pinned) over pinned whole streams (the fed decode); prints each
rc_decode_kernel / recon_kernel duration and checks the frames.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2602_09725_b200 import _lib, codec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--res", default="R1080")
    ap.add_argument("--pinned", action="store_true",
                    help="pinned whole streams (the fed decode) instead of bytes")
    a = ap.parse_args()
    if a.lib:
        _lib.LIB_PATH = os.path.abspath(a.lib)
    args = argparse.Namespace(model="llama3-8b", tokens=32768, layout="identity", res=a.res,
                              page=16, requests=1, shard="balanced")
    w = bench.Workload(args, torch.device("cuda", 0))
    streams = [bs.data for bs in codec.encode_batch(w.frames, [4] * len(w.frames))]
    if a.pinned:
        streams = [torch.frombuffer(bytearray(b), dtype=torch.uint8).pin_memory() for b in streams]
    for parts in ((None,) if a.pinned else (1, None)):
        for rep in range(2):
            torch.cuda.synchronize()
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                t0 = time.perf_counter()
                out, _ = codec.decode_batch(streams, max_parts=parts)
                torch.cuda.synchronize()
                wall = (time.perf_counter() - t0) * 1e3
            ok = all(torch.equal(o, f) for o, f in zip(out, w.frames))
            ks = [(e.name, e.device_time) for e in prof.events()
                  if "rc_decode" in e.name or "recon_kernel" in e.name]
            dec = [t for n, t in ks if "rc_decode" in n]
            rec = [t for n, t in ks if "recon" in n]
            print(f"lib={os.path.basename(_lib.LIB_PATH)} res={a.res} parts={parts} rep={rep} "
                  f"rc_decode launches={len(dec)} max={max(dec) / 1e3:.2f} ms "
                  f"all={[round(t / 1e3, 2) for t in dec]} sum={sum(dec) / 1e3:.2f} ms wall={wall:.1f} ms recon={sum(rec) / 1e3:.2f} ms ok={ok}", flush=True)


if __name__ == "__main__":
    main()
