"""GPU: time decode_batch host prep vs device work for C2-sized unit sets (R1080/R240)."""
import os
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context: see paper_2602_09725_b200.use_fetch_hw_queues
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2602_09725_b200 import codec, kvmodel as KV, layout as L  # noqa: E402

res = sys.argv[1] if len(sys.argv) > 1 else "R1080"
n_units = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = L.identity_layout(8, 128)
x = KV.gen_synthetic_kv(10000, 3, 8, 128, 0.9, 0, 0.3, dtype=torch.bfloat16)
q = KV.quantize(x)
plan = L.plan_inter_frame(10000, res, cfg, 4)
fr = L.assemble_frames(L.slice_tokens(q), plan)
bs = codec.encode_batch([fr], [4])[0].data
streams = [bs] * n_units
if "--pinned" in sys.argv:
    streams = [torch.frombuffer(bytearray(bs), dtype=torch.uint8).pin_memory() for _ in range(n_units)]
idx = codec.index_streams(streams)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    ix = codec.index_streams(streams)
    t1 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    out, _ = codec.decode_batch(streams, indices=ix)
    t2 = time.perf_counter()
    ev1.record()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    ok = torch.equal(out[0], fr)
    print(f"{res} units={n_units} streams={3*plan.frame_count*n_units} scan {1e3*(t1-t0):.1f} ms, "
          f"host prep+launch {1e3*(t2-t1):.1f} ms, device {ev0.elapsed_time(ev1):.1f} ms, "
          f"total {1e3*(t3-t0):.1f} ms, ok={ok}")
