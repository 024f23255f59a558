"""GPU debug: fused pack scales/frames vs oracle for one config; prints diffs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden"))
import cases  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2602_09725_b200 import _dev, _lib, layout as L  # noqa: E402

lay = (8, 128, 1, 8, 1, 128)
res = sys.argv[1] if len(sys.argv) > 1 else "R240"
H, D = 8, 128
T, Lyr, gs = 700, 5, 128
x = cases.to_bf16_values(ref.gen_synthetic_kv(T, Lyr, H, D, 0.9, 3, 0.3))
kv = torch.from_numpy(x).to(torch.bfloat16).cuda()
xp = ref.pad_layers(x)
for rep in range(3):
    units, outs = [], []
    for trip in range(2):
        for T0, Tc in [(0, 400), (400, 300)]:
            plan = L.plan_inter_frame(Tc, res, L.LayoutConfig(*lay), 4)
            fr = torch.empty(plan.frame_shape(), dtype=torch.uint8, device="cuda")
            am = torch.zeros(64, dtype=torch.int32, device="cuda")
            sc = torch.zeros((3, 8), dtype=torch.float32, device="cuda")
            u = _lib.kvf_pack_unit()
            for p in range(3):
                l = 3 * trip + p
                u.src.layer[p] = kv[:, l].data_ptr() if l < Lyr else None
            u.src.block_size = 1
            u.src.dtype = 0
            u.src.block_stride = u.src.slot_stride = Lyr * H * D
            u.src.head_stride = D
            u.src.token_base = T0
            u.plan = plan.to_c(gs)
            u.absmax = am.data_ptr()
            u.scales = sc.data_ptr()
            u.frames = _dev.surface_of(fr)
            units.append(u)
            outs.append((trip, T0, Tc, fr, sc, am))
    _lib.call("kvf_pack_batch", (_lib.kvf_pack_unit * len(units))(*units), len(units), None)
    torch.cuda.synchronize()
    for trip, T0, Tc, fr, sc, am in outs:
        slab = xp[T0:T0 + Tc, 3 * trip:3 * trip + 3]
        v, s = ref.quantize(slab, gs)
        got = sc.cpu().numpy()
        amx = am.cpu().numpy()
        m = np.abs(slab.reshape(Tc, 3, 8, 128)).max(axis=(0, 3))
        if not np.array_equal(got, s):
            bad = np.argwhere(got != s)
            print(f"rep{rep} trip{trip} T0={T0}: {len(bad)} scale diffs, e.g. {bad[:4].tolist()}")
            for pl, g in bad[:4]:
                print("   got", got[pl, g], "want", s[pl, g], "absmax bits->",
                      amx[pl * 8 + g].view(np.float32) if hasattr(amx[pl*8+g], 'view') else amx[pl * 8 + g],
                      "true max", m[pl, g])
            print("   control words", amx[24:])
        oplan = ref.Plan(Tc, res, *lay, F=4)
        want = ref.assemble_frames(v.reshape(Tc, 3, H * D), oplan)
        f = fr.cpu().numpy()
        if not np.array_equal(f, want):
            print(f"rep{rep} trip{trip} T0={T0}: frame diffs {int((f != want).sum())}")
print("done")
