"""GPU: time encode_batch / rc_encode for C2-sized unit sets (R1080/R240)."""
import os
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
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = codec.encode_batch([fr] * n_units, [4] * n_units)
    t1 = time.perf_counter()
    print(f"{res} units={n_units} encode {1e3 * (t1 - t0):.1f} ms, coded {sum(len(b) for b in out)} B")
