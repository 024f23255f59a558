"""GPU timeline (torch.profiler) + host profile of one encode_batch of C2's 88
units: where the wall time of the GPU encoder goes.

    python tools/timeline_encode.py R1080
"""
import cProfile
import os
import pstats
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2602_09725_b200 import codec, kvmodel as KV, layout as L  # noqa: E402

res = sys.argv[1] if len(sys.argv) > 1 else "R1080"
n_units = int(sys.argv[2]) if len(sys.argv) > 2 else 88
cfg = L.identity_layout(8, 128)
x = KV.gen_synthetic_kv(10000, 3, 8, 128, 0.9, 0, 0.3, dtype=torch.bfloat16)
q = KV.quantize(x)
plan = L.plan_inter_frame(10000, res, cfg, 4)
fr = L.assemble_frames(L.slice_tokens(q), plan)
frames = [fr.clone() for _ in range(n_units)]
for _ in range(2):
    codec.encode_batch(frames, [4] * n_units)
torch.cuda.synchronize()
pr = cProfile.Profile()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    pr.enable()
    t0 = time.perf_counter()
    out = codec.encode_batch(frames, [4] * n_units)
    t1 = time.perf_counter()
    pr.disable()
print(f"{res} units={n_units} encode_batch wall {1e3 * (t1 - t0):.1f} ms, "
      f"coded {sum(len(b.data) for b in out)} B")
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t00 = min(e.time_range.start for e in prof.events())
agg = {}
for e in ev:
    a = agg.setdefault(e.name[:40], [1e18, 0, 0, 0.0])
    s, f = (e.time_range.start - t00) / 1e3, (e.time_range.end - t00) / 1e3
    a[0], a[1], a[2], a[3] = min(a[0], s), max(a[1], f), a[2] + 1, a[3] + f - s
for k, (s, f, c, busy) in sorted(agg.items(), key=lambda kv: kv[1][0]):
    print(f"{k:40s} n={c:4d} first {s:8.2f} ms  last end {f:8.2f} ms  busy {busy:8.2f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(10)
