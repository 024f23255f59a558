"""Stage trace of the stream pack schedule (kvf_pack_stream.cu built with -DKVF_TRACE).

Builds a trace variant of libkvf into gpurun_out/trace/, packs C2 (bench.Workload)
with KVF_PACK_SINGLE_READ through it and prints per-stage latency percentiles over
the steady-state items of every CTA (globaltimer ns):
  empty wait (producer), TMA + fold, fold -> published, fold -> ready (all CTAs),
  ready -> Q start, Q time, issue -> slot free.
"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_09725_b200 import _dev, _lib, build as B  # noqa: E402


def build_trace():
    out = "/tmp/kvf_trace"
    os.makedirs(out, exist_ok=True)
    objs = []
    procs = []
    for src in B.SOURCES:
        obj = os.path.join(out, src + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen([B.nvcc(), *B.ARCH, *B.FLAGS, "-DKVF_TRACE", "-I", B.INCLUDE,
                                       "-c", "-o", obj, os.path.join(B.CSRC, src)]))
    assert all(p.wait() == 0 for p in procs)
    lib = os.path.join(out, "libkvf_trace.so")
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *objs], check=True)
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--param", type=int, default=8)
    a = ap.parse_args()
    tl = ctypes.CDLL(build_trace())
    args = argparse.Namespace(model=a.model, tokens=a.tokens, layout="identity", res="R1080",
                              page=16, requests=1, shard="balanced")
    dev = torch.device("cuda", 0)
    w = bench.Workload(args, dev)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros(sms * 4096 * 8, dtype=torch.int64, device=dev)
    tl.kvf_pack_batch_ex.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_int64, ctypes.c_void_p]
    tl.kvf_trace_set.argtypes = [ctypes.c_void_p]
    s = torch.cuda.current_stream()
    arr = ctypes.cast(w._pack_arr, ctypes.c_void_p)
    for rep in range(3):
        tl.kvf_trace_set(buf.data_ptr())
        buf.zero_()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(s)
        rc = tl.kvf_pack_batch_ex(arr, min(80, len(w.pack_units)), _lib.KVF_PACK_SINGLE_READ, a.param,
                                  _dev.stream_ptr(s))
        ev1.record(s)
        torch.cuda.synchronize()
        print("rc", rc, "ms", round(ev0.elapsed_time(ev1), 3), flush=True)
    t = buf.view(sms, 4096, 8).cpu().numpy().astype(np.float64)
    sl = t[:, 50:4000]
    ok = (sl[..., 1] > 0) & (sl[..., 3] > 0)
    names = [("empty wait", 1, 0), ("issue->fold", 2, 1), ("fold->published", 3, 2),
             ("issue->free(A)", 3, 1), ("Qissue->Qdone", 6, 5)]
    for nm, b, e in names:
        okk = (sl[..., b] > 0) & (sl[..., e] > 0)
        d = (sl[..., b] - sl[..., e])[okk]
        if d.size:
            print(f"{nm:16s} p10 {np.percentile(d,10):8.0f} p50 {np.percentile(d,50):8.0f} "
                  f"p90 {np.percentile(d,90):8.0f} ns")
    span = (np.nanmax(np.where(t[..., 1] > 0, t[..., 1], np.nan), axis=1) -
            np.nanmin(np.where(t[..., 1] > 0, t[..., 1], np.nan), axis=1)) / 1e3
    n = (t[..., 1] > 0).sum(axis=1)
    print("items/us per CTA p50", np.nanpercentile(n / span, 50))
    first = np.where(t[..., 1] > 0, t[..., 1], np.inf).min(axis=1)
    last = np.where(t[..., 1] > 0, t[..., 1], -np.inf).max(axis=1)
    act = np.isfinite(first)
    t0 = first[act].min()
    print("active CTAs", act.sum(), "first-issue spread us", (first[act].max() - t0) / 1e3,
          "last-issue us min/med/max", np.percentile((last[act] - t0) / 1e3, [0, 50, 100]))
    sub = t[:, :1500, :8]
    base = sub[sub > 0].min()
    np.save(os.path.join(ROOT, "gpurun_out", "trace_us.npy"),
            np.where(sub > 0, (sub - base) / 1e3, np.nan).astype(np.float32))


if __name__ == "__main__":
    main()
