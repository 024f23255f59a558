"""GPU stress: repeat kvf_pack_batch_ex (argv[2]: schedule, 0 auto / 1 two-pass /
2 single read) many times per config, count mismatches vs the oracle."""
import os
import sys
import time

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "tests", "golden"))
import cases  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2602_09725_b200 import _dev, _lib, layout as L  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
schedule = int(sys.argv[2]) if len(sys.argv) > 2 else _lib.KVF_PACK_AUTO
H, D, gs = 8, 128, 128
for res, lay, T, Lyr, chunks in [
        ("R240", (8, 128, 1, 8, 1, 128), 700, 5, [(0, 400), (400, 300)]),
        ("R1080", (8, 128, 8, 1, 1, 128), 3000, 7, [(0, 1000), (1000, 1000), (2000, 1000)]),
        ("R640", (8, 128, 2, 4, 16, 8), 2500, 4, [(0, 2500)]),
        ("R1080", (8, 128, 1, 8, 1, 128), 20000, 3, [(0, 10000), (10000, 10000)])]:
    x = cases.to_bf16_values(ref.gen_synthetic_kv(T, Lyr, H, D, 0.9, 3, 0.3))
    kv = torch.from_numpy(x).to(torch.bfloat16).cuda()
    xp = ref.pad_layers(x)
    trips = (Lyr + 2) // 3
    want = {}
    for trip in range(trips):
        for T0, Tc in chunks:
            v, s = ref.quantize(xp[T0:T0 + Tc, 3 * trip:3 * trip + 3], gs)
            fr = ref.assemble_frames(v.reshape(Tc, 3, H * D), ref.Plan(Tc, res, *lay, F=4))
            want[(trip, T0)] = (s, ref.digest(fr))
    bad_s = bad_f = 0
    t0 = time.time()
    for rep in range(reps):
        units, outs = [], []
        for trip in range(trips):
            for T0, Tc in chunks:
                plan = L.plan_inter_frame(Tc, res, L.LayoutConfig(*lay), 4)
                fr = torch.empty(plan.frame_shape(), dtype=torch.uint8, device="cuda")
                am = torch.empty(64, dtype=torch.int32, device="cuda")
                sc = torch.empty((3, 8), dtype=torch.float32, device="cuda")
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
                outs.append((trip, T0, fr, sc, am))
        _lib.call("kvf_pack_batch_ex", (_lib.kvf_pack_unit * len(units))(*units), len(units),
                  schedule, 0, None)
        torch.cuda.synchronize()
        for trip, T0, fr, sc, am in outs:
            s, fd = want[(trip, T0)]
            got = sc.cpu().numpy()
            if not np.array_equal(got, s):
                bad_s += 1
                if bad_s <= 3:
                    idx = np.argwhere(got != s)
                    print(res, "rep", rep, "trip", trip, "T0", T0, "scale diffs", idx[:6].tolist(),
                          got[tuple(idx[0])], s[tuple(idx[0])], "ctrl", am.cpu().numpy()[24:])
            if ref.digest(fr.cpu().numpy()) != fd:
                bad_f += 1
    print(f"{res}: reps={reps} units={len(outs)} bad_scales={bad_s} bad_frames={bad_f} "
          f"{time.time() - t0:.1f}s", flush=True)
