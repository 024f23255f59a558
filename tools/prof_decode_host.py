import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2602_09725_b200 import codec, kvmodel as KV, layout as L
res = sys.argv[1]
cfg = L.identity_layout(8, 128)
x = KV.gen_synthetic_kv(10000, 3, 8, 128, 0.9, 0, 0.3, dtype=torch.bfloat16)
q = KV.quantize(x)
plan = L.plan_inter_frame(10000, res, cfg, 4)
fr = L.assemble_frames(L.slice_tokens(q), plan)
bs = codec.encode_batch([fr], [4])[0].data
streams = [torch.frombuffer(bytearray(bs), dtype=torch.uint8).pin_memory() for _ in range(88)]
ix = codec.index_streams(streams)
for _ in range(3):
    out, _ = codec.decode_batch(streams, indices=ix); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter()
out, _ = codec.decode_batch(streams, indices=ix)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
pr.disable()
print("host", (t1-t0)*1e3, "total", (t2-t0)*1e3)
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
