"""GPU parity of the libkvf kernels against the reference goldens and the CPU oracle.

Bar: bit-exact int8 codes, scales, frame bytes, page/slot placement; dequantised
values bit-identical to the oracle's fp32 dequantize rounded once (RNE) to the
cache dtype, hence within scale/2 (+ half a bf16 ulp) of the original KV.
"""

import numpy as np
import pytest
import torch

import cases
from oracle import ref

pytestmark = pytest.mark.gpu

from paper_2602_09725_b200 import _lib, layout as L, kvmodel as KV  # noqa: E402
from paper_2602_09725_b200.restore import make_restore_unit, restore_frames, restore_units  # noqa: E402


def sha_t(t):
    return ref.digest(t.detach().cpu().numpy())


def np_bf16_from_f32(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16)


# ----------------------------------------------------------------- quantize
@pytest.mark.parametrize("k", range(len(cases.QUANT_CASES)))
def test_quantize_bit_exact(golden, k):
    c = golden["quantize"][k]
    x = cases.quant_input(c)
    src = np_bf16_from_f32(x) if c.get("bf16") else torch.from_numpy(x)
    if c.get("bf16"):
        assert np.array_equal(src.float().numpy(), x)  # bf16-representable input
    q = KV.quantize(KV.KVCache(src.cuda()), c["group_size"])
    assert sha_t(q.values) == c["values"]
    assert sha_t(q.scales) == c["scales"]
    deq = KV.dequantize(q, torch.float32)
    assert sha_t(deq.data) == c["dequant"]
    ref_deq = torch.from_numpy(ref.dequantize(*ref.quantize(x, c["group_size"]), c["group_size"]))
    for dt in (torch.bfloat16, torch.float16):
        got = KV.dequantize(q, dt).data.cpu()
        assert torch.equal(got, ref_deq.to(dt))


def test_quantize_fp16_source():
    x = cases.quant_input(dict(kind="synthetic", T=50, L=3, H=8, D=128, s=0.9, seed=2, c=0.3))
    x16 = torch.from_numpy(x).half()
    v, s = ref.quantize(x16.float().numpy(), 128)
    q = KV.quantize(KV.KVCache(x16.cuda()), 128)
    assert np.array_equal(q.values.cpu().numpy(), v)
    assert np.array_equal(q.scales.cpu().numpy(), s)


# ------------------------------------------------------------------- frames
def test_assemble_disassemble_bit_exact(golden):
    for c in golden["frames"]:
        t = cases.frame_tensors(c)
        plan = L.plan_inter_frame(c["T"], c["res"], L.LayoutConfig(*c["layout"]), c["F"])
        fr = L.assemble_frames(torch.from_numpy(t).cuda(), plan)
        assert list(fr.shape) == c["shape"]
        assert sha_t(fr) == c["frames"], c
        back = L.disassemble_frames(fr, plan)
        assert np.array_equal(back.cpu().numpy(), t)


# pack schedules (include/kvf.h kvf_pack_schedule): every one must give the
# oracle's bytes; single_read with 8- (default) and 16-CTA clusters
SCHEDULES = ["two_pass", "single_read", "single_read:16", "auto"]


def _pack(arr, n, mode):
    name, _, param = mode.partition(":")
    sched = {"auto": _lib.KVF_PACK_AUTO, "two_pass": _lib.KVF_PACK_TWO_PASS,
             "single_read": _lib.KVF_PACK_SINGLE_READ}[name]
    _lib.call("kvf_pack_batch_ex", arr, n, sched, int(param or "0", 0), None)


def _pack_unit(kv_dev, lay, res, T0, T, F, gs, frames, absmax, scales, triplet=0):
    """kvf_pack_unit for tokens [T0, T0+T) of layers 3*triplet.. of [T, L, H, D]."""
    H, D = lay[0], lay[1]
    plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), F)
    u = _lib.kvf_pack_unit()
    Lyr = kv_dev.shape[1]
    for p in range(3):
        l = 3 * triplet + p
        u.src.layer[p] = kv_dev[:, l].data_ptr() if l < Lyr else None
    u.src.block_table = None
    u.src.block_size = 1
    u.src.dtype = {torch.bfloat16: 0, torch.float16: 1, torch.float32: 2}[kv_dev.dtype]
    u.src.block_stride = u.src.slot_stride = Lyr * H * D
    u.src.head_stride = D
    u.src.token_base = T0
    u.plan = plan.to_c(gs)
    u.absmax = absmax.data_ptr()
    u.scales = scales.data_ptr()
    from paper_2602_09725_b200 import _dev
    u.frames = _dev.surface_of(frames)
    return u, plan


@pytest.mark.parametrize("lay", [(8, 128, 1, 8, 1, 128), (8, 128, 8, 1, 1, 128),
                                 (8, 128, 2, 4, 16, 8), (4, 64, 1, 4, 64, 1)])
@pytest.mark.parametrize("res", ["R240", "R640", "R1080"])
@pytest.mark.parametrize("mode", SCHEDULES)
def test_fused_pack_matches_oracle(lay, res, mode):
    H, D = lay[0], lay[1]
    T, Lyr, gs = 700, 5, 128 if D >= 128 else 64
    x = cases.to_bf16_values(ref.gen_synthetic_kv(T, Lyr, H, D, 0.9, 3, 0.3))
    kv = np_bf16_from_f32(x).cuda()
    chunks = [(0, 400), (400, 300)]
    units, outs, scratch = [], [], []
    for trip in range(2):
        for T0, Tc in chunks:
            plan = L.plan_inter_frame(Tc, res, L.LayoutConfig(*lay), 4)
            fr = torch.empty(plan.frame_shape(), dtype=torch.uint8, device="cuda")
            am = torch.zeros(_lib.load().kvf_pack_scratch_words(plan.to_c(gs)), dtype=torch.int32,
                             device="cuda")
            sc = torch.empty((3, H * D // gs), dtype=torch.float32, device="cuda")
            u, plan = _pack_unit(kv, lay, res, T0, Tc, 4, gs, fr, am, sc, trip)
            units.append(u)
            outs.append((trip, T0, Tc, plan, fr, sc))
            scratch.append(am)  # descriptors hold raw pointers: keep the buffers alive
    arr = (_lib.kvf_pack_unit * len(units))(*units)
    _pack(arr, len(units), mode)
    torch.cuda.synchronize()
    xp = ref.pad_layers(x)
    for trip, T0, Tc, plan, fr, sc in outs:
        slab = xp[T0:T0 + Tc, 3 * trip:3 * trip + 3]
        v, s = ref.quantize(slab, gs)
        oplan = ref.Plan(Tc, res, *lay, F=4)
        want = ref.assemble_frames(v.reshape(Tc, 3, H * D), oplan)
        np.testing.assert_array_equal(sc.cpu().numpy(), s, err_msg=f"scales trip {trip} T0 {T0}")
        np.testing.assert_array_equal(fr.cpu().numpy(), want, err_msg=f"frames trip {trip} T0 {T0}")


@pytest.mark.parametrize("dtype", [torch.float16, torch.float32, torch.bfloat16])
@pytest.mark.parametrize("mode", SCHEDULES)
def test_pack_paged_source_dtypes(dtype, mode):
    """Pack from a paged [blocks, 16, H, D] cache through a shuffled block table
    (vLLM layout) for every source dtype, the chunk starting mid-block (token
    base 5); codes, scales, frames vs the oracle."""
    H, D, gs, bs, T, res, t0 = 8, 128, 128, 16, 1234, "R480", 5
    lay = (H, D, 1, H, 1, D)
    x = ref.gen_synthetic_kv(T, 3, H, D, 0.9, 11, 0.3)
    xt = torch.from_numpy(x).to(dtype)
    x = xt.float().numpy()                         # the values the kernel sees
    nblk = (T + t0 + bs - 1) // bs
    perm = torch.randperm(nblk + 7, generator=torch.Generator().manual_seed(5))[:nblk]
    # other tokens of the pool hold larger values: they must not enter the maxima
    pool = torch.full((3, nblk + 7, bs, H, D), 1000.0).to(dtype)
    tok = torch.arange(T) + t0
    for p in range(3):
        pool[p].view(-1, H, D)[perm[tok // bs] * bs + tok % bs] = xt[:, p]
    pool = pool.cuda()
    table = perm.to(torch.int32).cuda()
    plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), 4)
    fr = torch.empty(plan.frame_shape(), dtype=torch.uint8, device="cuda")
    am = torch.zeros(_lib.load().kvf_pack_scratch_words(plan.to_c(gs)), dtype=torch.int32,
                     device="cuda")
    sc = torch.empty((3, H * D // gs), dtype=torch.float32, device="cuda")
    u = _lib.kvf_pack_unit()
    for p in range(3):
        u.src.layer[p] = pool[p].data_ptr()
    u.src.block_table = table.data_ptr()
    u.src.block_size = bs
    u.src.dtype = {torch.bfloat16: 0, torch.float16: 1, torch.float32: 2}[dtype]
    u.src.block_stride = bs * H * D
    u.src.slot_stride = H * D
    u.src.head_stride = D
    u.src.token_base = t0
    u.plan = plan.to_c(gs)
    u.absmax = am.data_ptr()
    u.scales = sc.data_ptr()
    from paper_2602_09725_b200 import _dev
    u.frames = _dev.surface_of(fr)
    _pack((_lib.kvf_pack_unit * 1)(u), 1, mode)
    torch.cuda.synchronize()
    v, s = ref.quantize(x, gs)
    want = ref.assemble_frames(v.reshape(T, 3, H * D), ref.Plan(T, res, *lay, F=4))
    assert np.array_equal(sc.cpu().numpy(), s)
    assert np.array_equal(fr.cpu().numpy(), want)


# ------------------------------------------------------------------ restore
def _oracle_chunk(T, lay, res, seed, gs=128, F=4):
    H, D = lay[0], lay[1]
    x = cases.to_bf16_values(ref.gen_synthetic_kv(T, 3, H, D, 0.9, seed, 0.3))
    v, s = ref.quantize(x, gs)
    plan = ref.Plan(T, res, *lay, F=F)
    frames = ref.assemble_frames(v.reshape(T, 3, H * D), plan)
    return x, v, s, frames


@pytest.mark.parametrize("lay", [(8, 128, 1, 8, 1, 128), (8, 128, 8, 1, 1, 128),
                                 (8, 128, 2, 4, 16, 8), (8, 128, 1, 8, 128, 1),
                                 (4, 8, 2, 2, 4, 2),
                                 # 512- and 256-channel slots: 2 / 4 items side by side per warp
                                 (4, 128, 1, 4, 1, 128), (4, 128, 2, 2, 8, 16),
                                 (2, 128, 1, 2, 1, 128), (2, 128, 2, 1, 16, 8),
                                 # 128-channel slots (a tensor-parallel head shard):
                                 # 8 items side by side per warp
                                 (1, 128, 1, 1, 1, 128), (2, 64, 2, 1, 8, 8)])
@pytest.mark.parametrize("dtype", [torch.int8, torch.bfloat16, torch.float16, torch.float32])
def test_restore_paged_matches_oracle(lay, dtype):
    H, D = lay[0], lay[1]
    gs = min(128, H * D)
    T, res = 333, "R480"
    x, v, s, frames = _oracle_chunk(T, lay, res, seed=4, gs=gs)
    plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), 4)
    mem = KV.PagedMemory(16, dtype=dtype, H=H, D=D, num_blocks=64, num_layers=6)
    mem.begin_fetch()
    # scatter the logical pages over a shuffled physical pool
    rng = np.random.default_rng(0)
    mem._free = list(rng.permutation(mem._free))
    n = restore_frames(torch.from_numpy(frames).cuda(), plan, mem, layer_base=3,
                       token_base=37, scales=torch.from_numpy(s).cuda())
    assert n == T
    torch.cuda.synchronize()
    deq = ref.dequantize(v, s, gs).reshape(T, 3, H * D)
    for tok in range(T):
        for p in range(3):
            got = mem.read(37 + tok, 3 + p).cpu()
            if dtype == torch.int8:
                assert np.array_equal(got.numpy(), v[tok, p].reshape(-1))
            else:
                assert torch.equal(got, torch.from_numpy(deq[tok, p]).to(dtype))
    assert mem.read(36, 3) is None and mem.read(37, 0) is None
    assert mem.allocated_bytes == T * 3 * H * D * torch.empty((), dtype=dtype).element_size()
    with pytest.raises(KV.ConflictError):
        restore_frames(torch.from_numpy(frames).cuda(), plan, mem, 3, 37, torch.from_numpy(s).cuda())
    mem.begin_fetch()
    restore_frames(torch.from_numpy(frames).cuda(), plan, mem, 3, 37, torch.from_numpy(s).cuda())


def test_restore_golden_slots(golden):
    for c in golden["restore"]:
        kv = c["kv"]
        v, s = ref.quantize(cases.quant_input(kv), kv["group_size"])
        oplan = ref.Plan(kv["T"], c["res"], *c["layout"], F=c["F"])
        frames = ref.assemble_frames(v.reshape(kv["T"], 3, kv["H"] * kv["D"]), oplan)
        plan = L.plan_inter_frame(kv["T"], c["res"], L.LayoutConfig(*c["layout"]), c["F"])
        mem = KV.PagedMemory(c["page"], dtype=torch.int8)
        mem.begin_fetch()
        # frame-wise: one launch per frame, like the reference's on_frame
        fr_dev = torch.from_numpy(frames).cuda()
        for f in range(plan.frame_count):
            restore_frames(fr_dev[f:f + 1], plan, mem, c["layer_base"], c["token_base"],
                           first_frame=f, n_frames=1)
        blob = b"".join(mem.read(t, l).cpu().numpy().tobytes()
                        for t in range(c["token_base"], c["token_base"] + kv["T"])
                        for l in range(c["layer_base"], c["layer_base"] + 3))
        assert ref.digest(blob) == c["slots"]
        assert mem.allocated_bytes == c["allocated_bytes"]


def test_restore_pad_layers_untouched():
    lay = (8, 128, 1, 8, 1, 128)
    T = 100
    x, v, s, frames = _oracle_chunk(T, lay, "R240", seed=1)
    plan = L.plan_inter_frame(T, "R240", L.LayoutConfig(*lay), 4)
    mem = KV.PagedMemory(16, dtype=torch.bfloat16, H=8, D=128, num_blocks=16, num_layers=33)
    for t in mem.layers:
        t.fill_(7.0)
    mem.begin_fetch()
    restore_frames(torch.from_numpy(frames).cuda(), plan, mem, layer_base=30, token_base=0,
                   scales=torch.from_numpy(s).cuda(), real_layers=32)
    assert mem.read(0, 32) is None
    assert torch.all(mem.layers[32] == 7.0)
    assert mem.read(5, 31) is not None


def test_restore_batch_mixed_units_and_layouts():
    """Many units in one batched call: fast + generic kernels, HND layout, partial
    frame ranges, different token bases — all against the oracle."""
    from paper_2602_09725_b200 import _dev
    specs = [((8, 128, 1, 8, 1, 128), "R1080", 500, 0, None),
             ((8, 128, 8, 1, 1, 128), "R240", 257, 5, 3),
             ((8, 128, 2, 4, 16, 8), "R640", 90, 0, None),
             ((4, 8, 2, 2, 4, 2), "R240", 41, 2, 2),
             ((8, 128, 1, 8, 128, 1), "R480", 77, 0, None)] * 12
    units, checks = [], []
    for k, (lay, res, T, f0, nf) in enumerate(specs):
        H, D = lay[0], lay[1]
        gs = min(128, H * D)
        x, v, s, frames = _oracle_chunk(T, lay, res, seed=k, gs=gs)
        plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), 4)
        nf = plan.frame_count - f0 if nf is None else nf
        bs = 16
        nblk = (T + bs - 1) // bs + 1
        # HND per-layer cache [blocks, H, bs, D] for odd k, NHD otherwise
        outs = [torch.zeros((nblk, H, bs, D) if k % 2 else (nblk, bs, H, D),
                            dtype=torch.bfloat16, device="cuda") for _ in range(3)]
        table = torch.from_numpy(np.random.default_rng(k).permutation(nblk).astype(np.int32)).cuda()
        dst = _lib.kvf_paged()
        for p in range(3):
            dst.layer[p] = outs[p].data_ptr()
        dst.block_table = table.data_ptr()
        dst.block_size = bs
        dst.dtype = _lib.KVF_BF16
        dst.block_stride = bs * H * D
        dst.slot_stride = D if k % 2 else H * D
        dst.head_stride = bs * D if k % 2 else D
        dst.token_base = 0
        fr = torch.from_numpy(frames).cuda()
        sc = torch.from_numpy(s).cuda()
        units.append(make_restore_unit(fr, plan, sc, dst, gs, f0, nf))
        checks.append((lay, T, v, s, gs, plan, f0, nf, outs, table, fr, sc))
    restore_units(units)
    torch.cuda.synchronize()
    for lay, T, v, s, gs, plan, f0, nf, outs, table, fr, sc in checks:
        H, D = lay[0], lay[1]
        deq = torch.from_numpy(ref.dequantize(v, s, gs)).to(torch.bfloat16)
        toks = plan.tokens_in_frames(f0, nf)
        tbl = table.cpu().numpy()
        hnd = outs[0].shape[1] == H and outs[0].shape[2] == 16 and H != 16
        for p in range(3):
            o = outs[p].cpu()
            written = torch.zeros(o.shape[:1] + (16,), dtype=torch.bool)
            for t in toks:
                blk, off = tbl[t // 16], t % 16
                got = o[blk, :, off] if hnd else o[blk, off]
                assert torch.equal(got.reshape(-1), deq[t, p].reshape(-1))
                written[blk, off] = True
            untouched = o[~written] if not hnd else o.permute(0, 2, 1, 3)[~written]
            assert torch.all(untouched == 0)


# ----------------------------------------------------------- large property
def test_c2_unit_round_trip_property():
    """Full-size unit (10,000 tokens, Llama-3-8B triplet, R1080): pack -> restore
    reproduces quantize() codes exactly and dequantize() values bit-for-bit."""
    from paper_2602_09725_b200 import _dev
    T, H, D, gs = 10000, 8, 128, 128
    kv = KV.gen_synthetic_kv(T, 3, H, D, 0.9, seed=0, channel_smoothness=0.3,
                             dtype=torch.bfloat16)
    q = KV.quantize(kv, gs)
    lay = (8, 128, 1, 8, 1, 128)
    plan = L.plan_inter_frame(T, "R1080", L.LayoutConfig(*lay), 4)
    fr = torch.empty(plan.frame_shape(), dtype=torch.uint8, device="cuda")
    am = torch.zeros(_lib.load().kvf_pack_scratch_words(plan.to_c(gs)), dtype=torch.int32,
                     device="cuda")
    sc = torch.empty((3, 8), dtype=torch.float32, device="cuda")
    u, _ = _pack_unit(kv.data, lay, "R1080", 0, T, 4, gs, fr, am, sc)
    _lib.call("kvf_pack_batch", (_lib.kvf_pack_unit * 1)(u), 1, None)
    assert torch.equal(sc, q.scales)
    assert torch.equal(fr, L.assemble_frames(q.values.reshape(T, 3, H * D), plan))
    for dt in (torch.int8, torch.bfloat16):
        mem = KV.PagedMemory(16, dtype=dt)
        mem.begin_fetch()
        restore_frames(fr, plan, mem, 0, 0, scales=sc)
        cache = torch.stack([mem.layers[p][torch.as_tensor(
            [mem.pages[t // 16] for t in range(0, T, 16)], device="cuda")].reshape(-1, H, D)[:T]
            for p in range(3)], dim=1)
        want = q.values if dt == torch.int8 else KV.dequantize(q, torch.bfloat16).data
        assert torch.equal(cache, want)


@pytest.mark.parametrize("shape", [
    # (name, H, D, layers, triplet, T, res, layout): a full 10,000-token unit of each
    # BASELINE.json model, checked against the CPU oracle (quantize + assemble + slots)
    ("qwen2.5-7b C3 (4 KV heads, 28 -> 30 layers)", 4, 128, 28, 9, 10000, "R640", "paper"),
    ("llama3-70b C4 (80 -> 81 layers, pad layer)", 8, 128, 80, 26, 10000, "R1080", "identity"),
    ("llama3-8b C2 last chunk", 8, 128, 32, 10, 2768, "R240", "identity"),
])
def test_baseline_config_units_match_oracle(shape):
    name, H, D, Lyr, j, T, res, layout = shape
    gs = 128
    real = min(3, Lyr - 3 * j)
    lay = (H, D, 1, H, 1, D) if layout == "identity" else (H, D, H, 1, 1, D)
    x = cases.to_bf16_values(ref.gen_synthetic_kv(T, real, H, D, 0.9, 5, 0.3))
    xp = np.concatenate([x, np.zeros((T, 3 - real, H, D), np.float32)], axis=1)
    v, s = ref.quantize(xp, gs)                              # oracle: pad layer -> scale 1
    oplan = ref.Plan(T, res, *lay, F=4)
    want_frames = ref.assemble_frames(v.reshape(T, 3, H * D), oplan)
    # GPU: pack from the [T, real, H, D] bf16 cache (pad layer = NULL pointer)
    kv = np_bf16_from_f32(x).cuda()
    plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), 4)
    fr = torch.empty(plan.frame_shape(), dtype=torch.uint8, device="cuda")
    am = torch.zeros(_lib.load().kvf_pack_scratch_words(plan.to_c(gs)), dtype=torch.int32,
                     device="cuda")
    sc = torch.empty((3, H * D // gs), dtype=torch.float32, device="cuda")
    u, _ = _pack_unit(kv, lay, res, 0, T, 4, gs, fr, am, sc)
    _lib.call("kvf_pack_batch", (_lib.kvf_pack_unit * 1)(u), 1, None)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(sc.cpu().numpy(), s, err_msg=name)
    np.testing.assert_array_equal(fr.cpu().numpy(), want_frames, err_msg=name)
    # restore the oracle's frames into a paged bf16 cache (layers 3j.., pad layer unwritten)
    mem = KV.PagedMemory(16, dtype=torch.bfloat16)
    n = restore_frames(torch.from_numpy(want_frames).cuda(), plan, mem, layer_base=3 * j,
                       token_base=0, scales=torch.from_numpy(s), real_layers=Lyr)
    assert n == T
    deq = torch.from_numpy(ref.dequantize(v, s, gs)).to(torch.bfloat16)
    rng = np.random.default_rng(1)
    for t in np.r_[0, T - 1, rng.integers(0, T, 64)]:
        for p in range(3):
            got = mem.read(int(t), 3 * j + p)
            if p >= real:
                assert got is None                               # pad layer never written
            else:
                assert torch.equal(got.cpu(), deq[t, p].reshape(-1)), (name, t, p)


@pytest.mark.parametrize("lay", [(8, 128, 1, 8, 1, 128), (8, 128, 8, 1, 1, 128),
                                 (8, 128, 2, 4, 16, 8), (4, 64, 1, 4, 64, 1)])
def test_apply_inverse_layout_match_oracle(lay):
    """apply_layout / inverse_layout (fk/layout.py:123-147) on one token's 3 layers."""
    H, D = lay[0], lay[1]
    cfg = L.LayoutConfig(*lay)
    v = np.random.default_rng(3).integers(-127, 128, size=(3, H * D)).astype(np.int8)
    tile = L.apply_layout(torch.from_numpy(v)[None], cfg)
    oplan = ref.Plan(1, "R240", *lay, F=4)
    assert np.array_equal(tile.cpu().numpy(), oplan.tile(v))
    back = L.inverse_layout(tile, cfg)
    assert np.array_equal(back.reshape(3, H * D).cpu().numpy(), v)


def test_paged_memory_accounting_like_reference():
    """PagedMemory byte accounting, write-once conflicts, begin_fetch and
    free_page (fk/kvmodel.py:195-244; tests/test_kvmodel.py:145-179)."""
    mem = KV.PagedMemory(page_size_tokens=4, dtype=torch.int8)
    slot = torch.arange(16, dtype=torch.int8)
    for t in range(6):
        mem.page_write(t, 0, slot)
    assert mem.allocated_bytes == 6 * 16 and mem.peak_bytes == 6 * 16
    with pytest.raises(KV.ConflictError):
        mem.page_write(2, 0, slot)
    mem.begin_fetch()                          # markers cleared, contents kept
    mem.page_write(2, 0, slot + 1)
    assert torch.equal(mem.read(2, 0).cpu(), slot + 1)
    assert mem.allocated_bytes == 7 * 16       # re-written slot counted again
    mem.free_page(0)                           # tokens 0..3 leave the cache
    assert mem.read(1, 0) is None and torch.equal(mem.read(4, 0).cpu(), slot)
    assert mem.allocated_bytes == 3 * 16 and mem.peak_bytes == 7 * 16   # as the reference counts
    mem.page_write(1, 0, slot)                 # the freed page can be written again
    assert torch.equal(mem.read(1, 0).cpu(), slot)


@pytest.mark.parametrize("H,D,gs", [(64, 128, 128), (32, 64, 64), (1, 128, 32)])
def test_wide_and_narrow_caches_pack_restore(H, D, gs):
    """Channel widths outside the vectorised kernels (C = 8192: generic path) and
    a single-head cache with 32-channel groups: pack and restore vs the oracle."""
    T, res = 37, "R240"
    lay = (H, D, 1, H, 1, D)
    x = cases.to_bf16_values(ref.gen_synthetic_kv(T, 3, H, D, 0.9, 2, 0.3))
    kv = np_bf16_from_f32(x).cuda()
    plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), 4)
    fr = torch.empty(plan.frame_shape(), dtype=torch.uint8, device="cuda")
    am = torch.zeros(_lib.load().kvf_pack_scratch_words(plan.to_c(gs)), dtype=torch.int32,
                     device="cuda")
    sc = torch.empty((3, H * D // gs), dtype=torch.float32, device="cuda")
    u, _ = _pack_unit(kv, lay, res, 0, T, 4, gs, fr, am, sc)
    _lib.call("kvf_pack_batch", (_lib.kvf_pack_unit * 1)(u), 1, None)
    torch.cuda.synchronize()
    v, s = ref.quantize(x, gs)
    want = ref.assemble_frames(v.reshape(T, 3, H * D), ref.Plan(T, res, *lay, F=4))
    np.testing.assert_array_equal(sc.cpu().numpy(), s)
    np.testing.assert_array_equal(fr.cpu().numpy(), want)
    mem = KV.PagedMemory(16, dtype=torch.bfloat16)
    restore_frames(fr, plan, mem, 0, 0, scales=sc)
    deq = torch.from_numpy(ref.dequantize(v, s, gs)).to(torch.bfloat16)
    for t in (0, 17, T - 1):
        for p in range(3):
            assert torch.equal(mem.read(t, p).cpu(), deq[t, p].reshape(-1))


@pytest.mark.parametrize("mode", SCHEDULES)
def test_tiny_and_ragged_units_pack_then_restore(mode):
    """Units of 1..129 tokens (fewer tokens than F, partial last segments, one
    token) in ONE kvf_pack_batch, then the GPU frames restored to int8 slots in
    ONE restore batch: frames, scales and codes identical to the oracle."""
    from paper_2602_09725_b200 import _dev
    specs = [(T, res, lay) for T in (1, 2, 3, 4, 5, 7, 15, 16, 17, 63, 64, 65, 129)
             for res, lay in (("R240", (8, 128, 1, 8, 1, 128)), ("R1080", (8, 128, 2, 4, 16, 8)))]
    units, keep, checks = [], [], []
    for k, (T, res, lay) in enumerate(specs):
        H, D = lay[0], lay[1]
        x, v, s, want = _oracle_chunk(T, lay, res, seed=100 + k)
        kv = np_bf16_from_f32(x.reshape(T, 3, H, D)).cuda()
        plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), 4)
        fr = torch.full(plan.frame_shape(), 7, dtype=torch.uint8, device="cuda")  # not 128
        am = torch.zeros(_lib.load().kvf_pack_scratch_words(plan.to_c(128)), dtype=torch.int32,
                         device="cuda")
        sc = torch.empty((3, H * D // 128), dtype=torch.float32, device="cuda")
        u, _ = _pack_unit(kv, lay, res, 0, T, 4, 128, fr, am, sc)
        units.append(u)
        keep += [kv, am]
        checks.append((T, lay, plan, v, s, want, fr, sc))
    _pack((_lib.kvf_pack_unit * len(units))(*units), len(units), mode)
    torch.cuda.synchronize()
    r_units, outs = [], []
    for T, lay, plan, v, s, want, fr, sc in checks:
        assert np.array_equal(sc.cpu().numpy(), s), (T, lay)
        assert np.array_equal(fr.cpu().numpy(), want), (T, lay)
        H, D = lay[0], lay[1]
        out = [torch.zeros((T, H, D), dtype=torch.int8, device="cuda") for _ in range(3)]
        dst = _lib.kvf_paged()
        for p in range(3):
            dst.layer[p] = out[p].data_ptr()
        dst.block_table = None
        dst.block_size = 1
        dst.dtype = _lib.KVF_I8
        dst.block_stride = dst.slot_stride = H * D
        dst.head_stride = D
        dst.token_base = 0
        r_units.append(make_restore_unit(fr, plan, sc, dst, 128, 0, plan.frame_count))
        outs.append(out)
    restore_units(r_units)
    torch.cuda.synchronize()
    for (T, lay, plan, v, s, want, fr, sc), out in zip(checks, outs):
        got = torch.stack([o.cpu() for o in out], 1).numpy().reshape(T, 3, -1)
        assert np.array_equal(got, v.reshape(T, 3, -1)), (T, lay)


def test_pack_frames_batch_with_supplied_maxima():
    """kvf_pack_frames_batch (scales + frames from caller-supplied maxima, one
    read of the source) equals the oracle, and clips like the reference when a
    supplied maximum is smaller than the data."""
    lay = (8, 128, 1, 8, 1, 128)
    H, D, res, gs = 8, 128, "R240", 128
    T = 333
    x = cases.to_bf16_values(ref.gen_synthetic_kv(T, 3, H, D, 0.9, 21, 0.3))
    kv = np_bf16_from_f32(x).cuda()
    plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), 4)
    v, s = ref.quantize(x, gs)
    want = ref.assemble_frames(v.reshape(T, 3, H * D), ref.Plan(T, res, *lay, F=4))
    # maxima as f32 bit patterns, as kvf_pack_absmax leaves them
    mx = np.abs(x.reshape(T, 3, H * D // gs, gs)).max(axis=(0, 3)).astype(np.float32)
    for shrink in (1.0, 0.5):
        am = torch.zeros(_lib.load().kvf_pack_scratch_words(plan.to_c(gs)), dtype=torch.int32)
        am[:mx.size] = torch.from_numpy((mx * np.float32(shrink)).view(np.int32).reshape(-1))
        am = am.cuda()
        fr = torch.empty(plan.frame_shape(), dtype=torch.uint8, device="cuda")
        sc = torch.empty((3, H * D // gs), dtype=torch.float32, device="cuda")
        u, _ = _pack_unit(kv, lay, res, 0, T, 4, gs, fr, am, sc)
        _lib.call("kvf_pack_frames_batch", (_lib.kvf_pack_unit * 1)(u), 1, None)
        torch.cuda.synchronize()
        if shrink == 1.0:
            assert np.array_equal(sc.cpu().numpy(), s)
            assert np.array_equal(fr.cpu().numpy(), want)
        else:   # reference arithmetic with the smaller scale: clip to +-127
            s2 = np.where(mx * np.float32(shrink) > 0,
                          (np.float64(mx * np.float32(shrink)) / 127.0).astype(np.float32), 1.0)
            q = np.clip(np.rint(x.reshape(T, 3, H * D // gs, gs).astype(np.float64)
                                / s2[None, :, :, None].astype(np.float64)), -127, 127)
            want2 = ref.assemble_frames(q.astype(np.int8).reshape(T, 3, H * D),
                                        ref.Plan(T, res, *lay, F=4))
            assert np.array_equal(sc.cpu().numpy(), s2)
            assert np.array_equal(fr.cpu().numpy(), want2)


# ------------------------------------------- every tiling of 8 x 128 (b_d < 8 too)
def _tilings_8x128():
    return [(8, 128, c.a_h, c.b_h, c.a_d, c.b_d) for c in L.tiling_candidates(8, 128)]


@pytest.mark.parametrize("res", ["R240", "R1080"])
def test_every_tiling_pack_and_restore_match_oracle(res):
    """All 32 tilings of H=8, D=128 (fk/layout.py:94-106), including the 12
    whose tile rows are narrower than 8 channels (shared-memory band kernels):
    pack (every schedule) gives the oracle's frames and scales, restore of the
    oracle's frames gives its int8 codes and bf16 dequantised values, in ONE
    batched call each for all tilings."""
    from paper_2602_09725_b200 import _dev
    T, H, D, gs = 150, 8, 128, 128
    x = cases.to_bf16_values(ref.gen_synthetic_kv(T, 3, H, D, 0.9, 21, 0.3))
    kv = np_bf16_from_f32(x).cuda()
    v, s = ref.quantize(x, gs)
    deq = ref.dequantize(v, s, gs).reshape(T, 3, H * D)
    lays = _tilings_8x128()
    assert len(lays) == 32 and sum(l[5] < 8 for l in lays) == 12
    wants = [ref.assemble_frames(v.reshape(T, 3, H * D), ref.Plan(T, res, *lay, F=4))
             for lay in lays]
    for mode in SCHEDULES:
        units, keep, outs = [], [], []
        for lay in lays:
            plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), 4)
            fr = torch.full(plan.frame_shape(), 7, dtype=torch.uint8, device="cuda")
            am = torch.zeros(_lib.load().kvf_pack_scratch_words(plan.to_c(gs)),
                             dtype=torch.int32, device="cuda")
            sc = torch.empty((3, H * D // gs), dtype=torch.float32, device="cuda")
            u, _ = _pack_unit(kv, lay, res, 0, T, 4, gs, fr, am, sc)
            units.append(u)
            keep += [am]
            outs.append((fr, sc))
        _pack((_lib.kvf_pack_unit * len(units))(*units), len(units), mode)
        torch.cuda.synchronize()
        for lay, want, (fr, sc) in zip(lays, wants, outs):
            np.testing.assert_array_equal(sc.cpu().numpy(), s, err_msg=f"{mode} {lay}")
            np.testing.assert_array_equal(fr.cpu().numpy(), want, err_msg=f"{mode} {lay}")
    for dtype in (torch.int8, torch.bfloat16):
        caches, r_units, keep = [], [], []
        for lay, want in zip(lays, wants):
            plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), 4)
            fr = torch.from_numpy(want).cuda()
            cache = torch.zeros((3, T, H, D), dtype=dtype, device="cuda")
            dst = _lib.kvf_paged()
            for p in range(3):
                dst.layer[p] = cache[p].data_ptr()
            dst.block_table = None
            dst.block_size = 1
            dst.dtype = _lib.KVF_I8 if dtype == torch.int8 else _lib.KVF_BF16
            dst.block_stride = dst.slot_stride = H * D
            dst.head_stride = D
            dst.token_base = 0
            sc = torch.from_numpy(s).cuda()
            r_units.append(make_restore_unit(fr, plan, sc, dst, gs))
            keep += [fr, sc]
            caches.append(cache)
        _lib.call("kvf_restore_batch", (_lib.kvf_restore_unit * len(r_units))(*r_units),
                  len(r_units), None)
        torch.cuda.synchronize()
        for lay, cache in zip(lays, caches):
            got = cache.permute(1, 0, 2, 3).reshape(T, 3, H * D).cpu()
            if dtype == torch.int8:
                np.testing.assert_array_equal(got.numpy(), v.reshape(T, 3, H * D), err_msg=str(lay))
            else:
                assert torch.equal(got, torch.from_numpy(deq).to(torch.bfloat16)), lay


def test_all_tilings_32x128_pack_and_restore():
    """Every tiling of a 32-head x 128 cache (the reference's acceptance case,
    tests/test_acceptance.py:112-145): assemble_frames of int8 codes and the
    quantising pack against the oracle's frames, and the restore of those frames
    against the oracle's codes; the narrow-row tilings take the band kernels
    with 4096-channel slots."""
    H, D, T = 32, 128, 8
    x = cases.to_bf16_values(ref.gen_synthetic_kv(T, 3, H, D, 0.9, 0, 0.3))
    v, s = ref.quantize(x, 128)
    t = torch.from_numpy(v.reshape(T, 3, H * D)).cuda()
    for cfg in L.tiling_candidates(H, D):
        plan = L.plan_inter_frame(T, "R240", cfg, 4)
        want = ref.assemble_frames(v.reshape(T, 3, H * D),
                                   ref.Plan(T, "R240", H, D, cfg.a_h, cfg.b_h, cfg.a_d, cfg.b_d, F=4))
        fr = L.assemble_frames(t, plan)
        assert np.array_equal(fr.cpu().numpy(), want), cfg
        back = L.disassemble_frames(fr, plan)
        assert np.array_equal(back.cpu().numpy(), v.reshape(T, 3, H * D)), cfg


@pytest.mark.parametrize("lay", [(8, 128, 1, 8, 1, 128), (8, 128, 8, 1, 1, 128),
                                 (8, 128, 2, 4, 16, 8), (8, 128, 1, 8, 128, 1)])
def test_restore_head_window_matches_oracle(lay):
    """kvf_restore_batch_heads: heads [2, 6) of every slot into a 4-head cache
    (bf16, dequantised) and, as raw samples, into an int8 buffer; both against
    the oracle.  (1, 8, 128, 1) has 1-channel tile rows: the per-sample kernel."""
    H, D = lay[0], lay[1]
    T, res, gs, lo, nh = 333, "R480", 128, 2, 4
    x, v, s, frames = _oracle_chunk(T, lay, res, seed=9, gs=gs)
    plan = L.plan_inter_frame(T, res, L.LayoutConfig(*lay), 4)
    fr = torch.from_numpy(frames).cuda()
    sc = torch.from_numpy(s).cuda()
    deq = ref.dequantize(v, s, gs).reshape(T, 3, H, D)
    for dtype, raw in ((torch.bfloat16, 0), (torch.int8, 1)):
        out = torch.zeros((3, T, nh, D), dtype=dtype, device="cuda")
        dst = _lib.kvf_paged()
        for p in range(3):
            dst.layer[p] = out[p].data_ptr()
        dst.block_table = None
        dst.block_size = 1
        dst.dtype = {torch.bfloat16: _lib.KVF_BF16, torch.int8: _lib.KVF_I8}[dtype]
        dst.block_stride = dst.slot_stride = nh * D
        dst.head_stride = D
        dst.token_base = 0
        u = make_restore_unit(fr, plan, sc, dst, gs)
        _lib.call("kvf_restore_batch_heads", (_lib.kvf_restore_unit * 1)(u), 1, lo, nh, 1, 0, raw,
                  None)
        torch.cuda.synchronize()
        got = out.permute(1, 0, 2, 3).cpu()
        if raw:
            want = (v.reshape(T, 3, H, D)[:, :, lo:lo + nh].astype(np.int16) + 128).astype(np.uint8)
            assert np.array_equal(got.numpy().view(np.uint8), want)
        else:
            want = torch.from_numpy(np.ascontiguousarray(deq[:, :, lo:lo + nh])).to(dtype)
            assert torch.equal(got, want)
    # all heads in two windows of 4: window w at +w * (3*T*4*D) of an int8 buffer
    buf = torch.zeros((2, 3, T, 4, D), dtype=torch.int8, device="cuda")
    dst = _lib.kvf_paged()
    for p in range(3):
        dst.layer[p] = buf[0, p].data_ptr()
    dst.block_table, dst.block_size, dst.dtype = None, 1, _lib.KVF_I8
    dst.block_stride = dst.slot_stride = 4 * D
    dst.head_stride, dst.token_base = D, 0
    u = make_restore_unit(fr, plan, None, dst, gs)
    _lib.call("kvf_restore_batch_heads", (_lib.kvf_restore_unit * 1)(u), 1, 0, 4, 2,
              3 * T * 4 * D, 0, None)
    torch.cuda.synchronize()
    codes = v.reshape(T, 3, H, D)
    for w in range(2):
        assert np.array_equal(buf[w].permute(1, 0, 2, 3).cpu().numpy(), codes[:, :, 4 * w:4 * w + 4])
    with pytest.raises(ValueError):
        _lib.call("kvf_restore_batch_heads", (_lib.kvf_restore_unit * 1)(u), 1, 6, 4, 1, 0, 0,
                  None)
