"""GPU debug: run the team pack on the failing parity case and print mismatches."""
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "tests", "golden"))
sys.path.insert(0, os.path.join(HERE, "..", "tests"))
import cases  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2602_09725_b200 import _lib, layout as L  # noqa: E402
from test_gpu_parity import _pack_unit, np_bf16_from_f32  # noqa: E402

lay, res = (8, 128, 1, 8, 1, 128), sys.argv[1] if len(sys.argv) > 1 else "R240"
H, D = 8, 128
T, Lyr, gs = 700, 5, 128
x = cases.to_bf16_values(ref.gen_synthetic_kv(T, Lyr, H, D, 0.9, 3, 0.3))
kv = np_bf16_from_f32(x).cuda()
xp = ref.pad_layers(x)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 5):
    units, outs = [], []
    for trip in range(2):
        for T0, Tc in [(0, 400), (400, 300)]:
            plan = L.plan_inter_frame(Tc, res, L.LayoutConfig(*lay), 4)
            fr = torch.empty(plan.frame_shape(), dtype=torch.uint8, device="cuda")
            am = torch.zeros(_lib.load().kvf_pack_scratch_words(plan.to_c(gs)), dtype=torch.int32,
                             device="cuda")
            sc = torch.full((3, H * D // gs), float("nan"), dtype=torch.float32, device="cuda")
            u, plan = _pack_unit(kv, lay, res, T0, Tc, 4, gs, fr, am, sc, trip)
            units.append(u)
            outs.append((trip, T0, Tc, plan, fr, sc, am))
    arr = (_lib.kvf_pack_unit * len(units))(*units)
    _lib.call("kvf_pack_batch", arr, len(units), None)
    torch.cuda.synchronize()
    bad = 0
    for k, (trip, T0, Tc, plan, fr, sc, am) in enumerate(outs):
        v, s = ref.quantize(xp[T0:T0 + Tc, 3 * trip:3 * trip + 3], gs)
        got = sc.cpu().numpy()
        G = H * D // gs
        if not np.array_equal(got, s):
            idx = np.argwhere(got != s)
            amv = am.cpu().numpy()
            for p, g in idx[:6]:
                print(f"rep {rep} unit {k} plane {p} group {g}: got {got[p, g]!r} want {s[p, g]!r} "
                      f"absmax_bits {amv[p * G + g]:#x} want_bits {np.float32(np.abs(xp[T0:T0+Tc, 3*trip+p].reshape(Tc, -1)[:, g*gs:(g+1)*gs]).max()).view(np.uint32):#x}")
            bad += len(idx)
        want = ref.assemble_frames(v.reshape(Tc, 3, H * D), ref.Plan(Tc, res, *lay, F=4))
        fb = fr.cpu().numpy() != want
        if fb.any():
            print(f"rep {rep} unit {k}: {fb.sum()} frame bytes differ")
    print("rep", rep, "scale mismatches", bad)
