"""GPU timeline (torch.profiler / CUPTI) of one decode_batch of C2's 88 units:
per-activity start/end relative to the first, to see copy/decode overlap.

    python tools/timeline_decode.py R240
"""
import os
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context: see paper_2602_09725_b200.use_fetch_hw_queues
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2602_09725_b200 import codec, kvmodel as KV, layout as L  # noqa: E402

res = sys.argv[1] if len(sys.argv) > 1 else "R240"
n_units = int(sys.argv[2]) if len(sys.argv) > 2 else 88
cfg = L.identity_layout(8, 128)
x = KV.gen_synthetic_kv(10000, 3, 8, 128, 0.9, 0, 0.3, dtype=torch.bfloat16)
q = KV.quantize(x)
plan = L.plan_inter_frame(10000, res, cfg, 4)
fr = L.assemble_frames(L.slice_tokens(q), plan)
bs = codec.encode_batch([fr], [4])[0].data
streams = [torch.frombuffer(bytearray(bs), dtype=torch.uint8).pin_memory() for _ in range(n_units)]
ix = codec.index_streams(streams)
for _ in range(3):
    codec.decode_batch(streams, indices=ix)
    torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    codec.decode_batch(streams, indices=ix)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in prof.events())
rows = sorted(((e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3, e.name) for e in ev)
agg = {}
for s, e, n in rows:
    k = n[:40]
    a = agg.setdefault(k, [1e9, 0, 0, 0.0])
    a[0], a[1], a[2], a[3] = min(a[0], s), max(a[1], e), a[2] + 1, a[3] + (e - s)
for k, (s, e, c, busy) in sorted(agg.items(), key=lambda kv: kv[1][0]):
    print(f"{k:40s} n={c:4d} first {s:7.2f} ms  last end {e:7.2f} ms  busy {busy:7.2f} ms")
