"""Stage trace of the fed decode (trace build, -DKVF_TRACE): per plane stream the
globaltimer at start / first bytes available / done, per copy CTA its end."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import argparse  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import trace_stream  # noqa: E402
from paper_2602_09725_b200 import _lib, codec  # noqa: E402


def main():
    path = trace_stream.build_trace()
    _lib.LIB_PATH, _lib._lib = path, None   # every libkvf call goes to the trace build
    tl = _lib.load()
    args = argparse.Namespace(model="llama3-8b", tokens=32768, layout="identity", res="R1080",
                              page=16, requests=1, shard="balanced")
    w = bench.Workload(args, torch.device("cuda", 0))
    streams = [bs.data for bs in codec.encode_batch(w.frames, [4] * len(w.frames))]
    streams = [torch.frombuffer(bytearray(b), dtype=torch.uint8).pin_memory() for b in streams]
    frames = [torch.empty_like(f) for f in w.frames]
    buf = torch.zeros(4 * 20000, dtype=torch.int64, device="cuda")
    tl.kvf_fed_trace_set.argtypes = [ctypes.c_void_p]
    tl.kvf_fed_trace_set(buf.data_ptr())
    for _ in range(2):
        buf.zero_()
        codec.decode_batch(streams, out=frames)
        torch.cuda.synchronize()
    t = buf.view(-1, 4).cpu().numpy().astype(np.float64)
    n = int((t[:, 0] > 0).sum())
    st = t[:n]
    t0 = st[:, 0].min()
    print("streams", n, "copy CTAs", int((t[n:, 3] > 0).sum()))
    for nm, e in (("start", 0), ("first bytes", 1), ("done", 2)):
        d = (st[:, e] - t0) / 1e6
        print(f"{nm:12s} ms  min {d.min():7.2f} p50 {np.percentile(d, 50):7.2f} max {d.max():7.2f}")
    dur = (st[:, 2] - st[:, 1]) / 1e6
    print(f"decode (done - first bytes) ms  min {dur.min():.2f} p50 {np.percentile(dur, 50):.2f} "
          f"max {dur.max():.2f}")
    cp = (t[n:, 3][t[n:, 3] > 0] - t0) / 1e6
    print(f"copy CTAs done ms  min {cp.min():.2f} max {cp.max():.2f}")


if __name__ == "__main__":
    main()
