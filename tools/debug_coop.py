"""GPU debug: cooperative pack vs phase-split pack for one large unit; print diff pattern."""
import os
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2602_09725_b200 import _dev, _lib, kvmodel as KV, layout as L  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
res = sys.argv[2] if len(sys.argv) > 2 else "R1080"
H, D, gs = 8, 128, 128
kv = KV.gen_synthetic_kv(T, 3, H, D, 0.9, seed=0, channel_smoothness=0.3, dtype=torch.bfloat16)
lay = (8, 128, 1, 8, 1, 128)
plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), 4)


def run():
    fr = torch.full(plan.frame_shape(), 7, dtype=torch.uint8, device="cuda")
    am = torch.zeros(64, dtype=torch.int32, device="cuda")
    sc = torch.empty((3, 8), dtype=torch.float32, device="cuda")
    u = _lib.kvf_pack_unit()
    for p in range(3):
        u.src.layer[p] = kv.data[:, p].data_ptr()
    u.src.block_size = 1
    u.src.dtype = 0
    u.src.block_stride = u.src.slot_stride = 3 * H * D
    u.src.head_stride = D
    u.plan = plan.to_c(gs)
    u.absmax = am.data_ptr()
    u.scales = sc.data_ptr()
    u.frames = _dev.surface_of(fr)
    _lib.call("kvf_pack_batch", (_lib.kvf_pack_unit * 1)(u), 1, None)
    torch.cuda.synchronize()
    return fr.cpu().numpy(), sc.cpu().numpy()


mode = os.environ.get("KVF_PACK_PHASES")
fr, sc = run()
np.save(f"/tmp/fr_{'phases' if mode else 'coop'}.npy", fr)
if not mode:
    env = dict(os.environ, KVF_PACK_PHASES="1")
    subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, check=True)
    ref = np.load("/tmp/fr_phases.npy")
    diff = fr != ref
    print("T", T, "res", res, "mismatched bytes", int(diff.sum()), "of", diff.size)
    if diff.any():
        idx = np.argwhere(diff)
        print("frames with diffs:", sorted(set(idx[:, 0].tolist()))[:20])
        print("planes:", sorted(set(idx[:, 1].tolist())), "rows:", sorted(set(idx[:, 2].tolist()))[:20])
        cols = idx[:, 3]
        print("cols min/max", cols.min(), cols.max(), "count by col//1024:",
              np.bincount(cols // 1024)[:16].tolist())
        print("sample", idx[:5].tolist(), fr[tuple(idx[0])], ref[tuple(idx[0])])
        print("7s (never written):", int((fr == 7).sum()))
