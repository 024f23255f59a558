"""Range-decode kernel time on device-resident C2 streams (CUPTI kernel durations).

    python tools/rc_probe.py [--lib path/to/libkvf.so] [--res R1080]

decode_batch over the bytes of every C2 stream with one part (one
rc_decode_kernel launch for all planes) and with the default part pipeline;
prints each rc_decode_kernel / recon_kernel duration and checks the frames.
"""
import argparse
import os
import sys

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
    a = ap.parse_args()
    if a.lib:
        _lib.LIB_PATH = os.path.abspath(a.lib)
    args = argparse.Namespace(model="llama3-8b", tokens=32768, layout="identity", res=a.res,
                              page=16, requests=1, shard="balanced")
    w = bench.Workload(args, torch.device("cuda", 0))
    streams = [bs.data for bs in codec.encode_batch(w.frames, [4] * len(w.frames))]
    for parts in (1, None):
        for rep in range(2):
            torch.cuda.synchronize()
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                out, _ = codec.decode_batch(streams, max_parts=parts)
                torch.cuda.synchronize()
            ok = all(torch.equal(o, f) for o, f in zip(out, w.frames))
            ks = [(e.name, e.device_time) for e in prof.events()
                  if "rc_decode" in e.name or "recon_kernel" in e.name]
            dec = [t for n, t in ks if "rc_decode" in n]
            print(f"lib={os.path.basename(_lib.LIB_PATH)} res={a.res} parts={parts} rep={rep} "
                  f"rc_decode launches={len(dec)} max={max(dec) / 1e3:.2f} ms "
                  f"sum={sum(dec) / 1e3:.2f} ms ok={ok}", flush=True)


if __name__ == "__main__":
    main()
