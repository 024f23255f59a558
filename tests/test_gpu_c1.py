"""C1 end to end on the GPU (BASELINE.json configs[0]): Llama-3-8B-shaped K and V
(32 layers -> 11 triplets, 8 KV heads, d=128), 4,096 tokens, through the
reference's own flow (fk/cli.py:222-241 pack, fk/cli.py:285-289 restore):

    quantize -> container.pack_chunks (one GPU encode of all 22 slabs at R240 +
    R1080) -> container bytes -> ChunkContainer.from_bytes -> restore_stream
    (frame-wise GPU decode + restore) into paged bf16 and int8 caches,

checked on EVERY triplet: container bytes identical to the oracle's
pack_chunk_bytes (fk/container.py:160-209, encode fk/codec.py:93-128), every
int8 slot identical to the oracle's restore_slots (fk/fetchsim.py:347-355), every
bf16 slot identical to the oracle's dequantize rounded to bf16
(fk/kvmodel.py:147-152), and the pad layer (32) never written."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ref
from paper_2602_09725_b200 import container as C, kvmodel as KV, layout as L
from paper_2602_09725_b200.restore import restore_stream

pytestmark = pytest.mark.gpu

T, LAYERS, H, D, GS = 4096, 32, 8, 128, 128
RES = ["R240", "R1080"]


def _kv(seed):
    x = KV.gen_synthetic_kv(T, LAYERS, H, D, 0.9, seed=seed, channel_smoothness=0.3,
                            dtype=torch.bfloat16).data
    return x, x.float().cpu().numpy()


@pytest.mark.parametrize("kv_seed", [0, 1], ids=["K", "V"])
def test_c1_pack_container_restore_every_triplet(kv_seed):
    x_gpu, x_cpu = _kv(kv_seed)
    q = KV.quantize(KV.KVCache(x_gpu).pad_layers(), GS)                 # [T, 33, H, D]
    lay = L.identity_layout(H, D)
    cache_id = bytes(range(16))
    n_trip = (LAYERS + 2) // 3
    slabs = [(q.layer_triplet(j), cache_id, 0, 0, j) for j in range(n_trip)]
    containers = C.pack_chunks(slabs, lay, RES)
    xp = ref.pad_layers(x_cpu)
    v_all, s_all = ref.quantize(xp, GS)
    mem8 = KV.PagedMemory(16, dtype=torch.int8)
    mem16 = KV.PagedMemory(16, dtype=torch.bfloat16)
    for m in (mem8, mem16):
        m.begin_fetch()
    for j, cont in enumerate(containers):
        v3, s3 = v_all[:, 3 * j:3 * j + 3], s_all[3 * j:3 * j + 3]
        want = ref.pack_chunk_bytes(v3, s3, (H, D, 1, H, 1, D), RES, GS, cache_id, 0, 0, j)
        data = cont.to_bytes()
        assert data == want, f"container bytes of triplet {j}"
        back = C.ChunkContainer.from_bytes(data)
        code = L.RESOLUTION_CODE["R1080"]
        plan = back.plan(code)
        real = min(3, LAYERS - 3 * j)
        for m in (mem8, mem16):
            # real_layers = the model's layer count: layer 32 is the pad layer
            out = restore_stream(back.bitstream(code), plan, back.layout(), m, layer_base=3 * j,
                                 token_base=0, scales=back.scales(), real_layers=LAYERS)
            assert out["tokens_written"] == T
        oplan = ref.Plan(T, "R1080", H, D, 1, H, 1, D, F=4)
        frames = ref.assemble_frames(v3.reshape(T, 3, H * D), oplan)
        slots = ref.restore_slots(frames, oplan, layer_base=3 * j, token_base=0)
        deq = ref.dequantize(v3, s3, GS).reshape(T, 3, H * D)
        for p in range(real):
            l = 3 * j + p
            got8 = torch.stack([mem8.read(t, l) for t in range(T)]).cpu().numpy()
            exp8 = np.stack([slots[(t, l)] for t in range(T)])
            np.testing.assert_array_equal(got8.reshape(T, -1), exp8.reshape(T, -1),
                                          err_msg=f"int8 layer {l}")
            got16 = torch.stack([mem16.read(t, l) for t in range(T)]).cpu()
            exp16 = torch.from_numpy(deq[:, p]).to(torch.bfloat16)
            assert torch.equal(got16.reshape(T, -1), exp16), f"bf16 layer {l}"
    for m in (mem8, mem16):
        assert m.read(0, LAYERS) is None and m.read(T - 1, LAYERS) is None  # pad layer
