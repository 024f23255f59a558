import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2602_09725_b200 import codec, kvmodel as KV, layout as L, _lib
from paper_2602_09725_b200.restore import make_restore_unit, restore_units
cfg = L.identity_layout(8, 128)
x = KV.gen_synthetic_kv(10000, 3, 8, 128, 0.9, 0, 0.3, dtype=torch.bfloat16)
q = KV.quantize(x)
plan = L.plan_inter_frame(10000, "R1080", cfg, 4)
fr = L.assemble_frames(L.slice_tokens(q), plan)
bs = codec.encode_batch([fr], [4])[0].data
sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
H, D = 8, 128
def mk_units(n):
    outs, units = [], []
    for k in range(n):
        out = [torch.zeros((10000, H, D), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
        dst = _lib.kvf_paged()
        for p in range(3): dst.layer[p] = out[p].data_ptr()
        dst.block_table = None; dst.block_size = 1; dst.dtype = _lib.KVF_BF16
        dst.block_stride = dst.slot_stride = H * D; dst.head_stride = D; dst.token_base = 0
        units.append(make_restore_unit(fr, plan, q.scales[:3].contiguous(), dst, 128, 0, plan.frame_count))
        outs.append(out)
    return units, outs
for n in (1, 8, 16, 20, 32, 64):
    units, outs = mk_units(n)
    restore_units(units, stream=sB); torch.cuda.synchronize()
    # long decode on A, then a restore queued behind it on A
    codec.decode_batch([bs], stream=sA)
    restore_units(units, stream=sA)
    t = time.perf_counter()
    restore_units(units, stream=sB)   # independent stream
    dt = time.perf_counter() - t
    torch.cuda.synchronize()
    print(f"units={n}: restore_batch launch on an idle stream took {dt*1e3:.2f} ms while stream A had a pending restore")
