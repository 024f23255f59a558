"""Drop-in API on the GPU, mirroring the reference's own tests for the path:
container pack/unpack (tests/test_container.py:25-50), frame-wise restore
(tests/test_fetchsim.py:255-282, tests/test_acceptance.py:224-243) and the
loopback fetch (tests/test_acceptance.py:148-166)."""

import numpy as np
import pytest
import torch

import cases
from oracle import ref

pytestmark = pytest.mark.gpu

from paper_2602_09725_b200 import container as C  # noqa: E402
from paper_2602_09725_b200 import fetch as FE  # noqa: E402
from paper_2602_09725_b200 import kvmodel as KV  # noqa: E402
from paper_2602_09725_b200 import layout as L  # noqa: E402
from paper_2602_09725_b200 import netstore as NS  # noqa: E402
from paper_2602_09725_b200.restore import restore_chunk_wise, restore_stream  # noqa: E402


def _q(kvc):
    x = cases.quant_input(kvc)
    src = torch.from_numpy(x)
    if kvc.get("bf16"):
        src = src.to(torch.bfloat16)
    return KV.quantize(KV.KVCache(src.cuda()), kvc["group_size"]), x


def test_container_bytes_match_reference(golden):
    for c in golden["container"]:
        q, _ = _q(c["kv"])
        cont = C.pack_chunk(q, L.LayoutConfig(*c["layout"]), c["res"],
                            cache_id=bytes.fromhex(c["cache_id"]), chunk_index=c["chunk_index"],
                            token_start=c["token_start"], layer_triplet_index=c["triplet"],
                            F=c["F"])
        blob = cont.to_bytes()
        assert ref.digest(blob) == c["bytes"]
        back = C.ChunkContainer.from_bytes(blob)
        for code in back.resolutions:
            slab = C.unpack_chunk(back, code)
            assert torch.equal(slab.values, q.values)
            assert torch.equal(slab.scales, q.scales)
            assert slab.group_size == q.group_size


def test_pack_chunks_batched_equals_pack_chunk(golden):
    """The batched producer gives byte-identical containers (reference goldens)."""
    items, cfgs = [], []
    for c in golden["container"]:
        q, _ = _q(c["kv"])
        items.append((c, q))
    by_cfg = {}
    for c, q in items:
        key = (tuple(c["layout"]), tuple(sorted(c["res"])), c["F"])
        by_cfg.setdefault(key, []).append((c, q))
    for (lay, res, F), group in by_cfg.items():
        slabs = [(q, bytes.fromhex(c["cache_id"]), c["chunk_index"], c["token_start"], c["triplet"])
                 for c, q in group]
        conts = C.pack_chunks(slabs, L.LayoutConfig(*lay), list(res), F=F)
        for (c, _), cont in zip(group, conts):
            assert ref.digest(cont.to_bytes()) == c["bytes"]
    # many slabs of different lengths in one encode == one at a time
    q, _ = _q(dict(kind="synthetic", T=150, L=3, H=4, D=8, s=0.9, seed=3, c=0.3, group_size=8))
    cfg = L.identity_layout(4, 8)
    slabs = [(KV.QuantizedKV(q.values[t0:t0 + n], q.scales, 8), b"\x07" * 16, k, t0, 0)
             for k, (t0, n) in enumerate([(0, 64), (64, 50), (114, 36)])]
    batched = C.pack_chunks(slabs, cfg, ["R240", "R1080"])
    for s_, cont in zip(slabs, batched):
        one = C.pack_chunk(s_[0], cfg, ["R240", "R1080"], cache_id=s_[1], chunk_index=s_[2],
                           token_start=s_[3], layer_triplet_index=s_[4])
        assert cont.to_bytes() == one.to_bytes()


def test_unpack_chunks_batched_equals_unpack_chunk(golden):
    conts = []
    for c in golden["container"]:
        q, _ = _q(c["kv"])
        cont = C.pack_chunk(q, L.LayoutConfig(*c["layout"]), c["res"],
                            cache_id=bytes.fromhex(c["cache_id"]), chunk_index=c["chunk_index"],
                            token_start=c["token_start"], layer_triplet_index=c["triplet"],
                            F=c["F"])
        conts += [(cont, code, q) for code in cont.resolutions]
    batched = C.unpack_chunks([(cont, code) for cont, code, _ in conts])
    for (cont, code, q), slab in zip(conts, batched):
        assert torch.equal(slab.values, q.values) and torch.equal(slab.scales, q.scales)
        assert slab.group_size == q.group_size


def test_pack_metadata_contents():
    q, _ = _q(dict(kind="synthetic", T=17, L=3, H=4, D=8, s=0.9, seed=0, c=0.0, group_size=8))
    cfg = L.identity_layout(4, 8)
    c = C.pack_chunk(q, cfg, ["R240", "R1080"], token_start=170, layer_triplet_index=2)
    assert (c.token_count, c.token_start, c.layer_triplet_index) == (17, 170, 2)
    assert c.layout() == cfg and c.metadata["F"] == 4
    assert set(c.metadata["plans"]) == {"R240", "R1080"}
    assert c.metadata["frame_counts"]["R240"] == c.plan(0).frame_count
    assert np.array_equal(c.scales(), q.scales.cpu().numpy())
    with pytest.raises(ValueError):
        C.pack_chunk(q, cfg, [])
    with pytest.raises(ValueError):
        C.pack_chunk(q, cfg, ["R240"], max_tokens=10)


@pytest.mark.parametrize("batch", [None, "gop"])
@pytest.mark.parametrize("dtype", [torch.int8, torch.bfloat16])
def test_restore_stream_matches_chunk_wise_and_golden(golden, dtype, batch):
    for c in golden["restore"]:
        q, x = _q(c["kv"])
        cfg = L.LayoutConfig(*c["layout"])
        cont = C.pack_chunk(q, cfg, [c["res"]], F=c["F"])
        code = L.RESOLUTION_CODE[c["res"]]
        bs, plan = cont.bitstream(code), cont.plan(code)
        assert ref.digest(bs) == c["stream"]
        mem_a = KV.PagedMemory(c["page"], dtype=dtype)
        mem_a.begin_fetch()
        out_a = restore_stream(bs, plan, cfg, mem_a, c["layer_base"], c["token_base"],
                               scales=q.scales, batch_frames=None if batch is None else plan.F)
        mem_b = KV.PagedMemory(c["page"], dtype=dtype)
        mem_b.begin_fetch()
        out_b = restore_chunk_wise(bs, plan, cfg, mem_b, c["layer_base"], c["token_base"],
                                   scales=q.scales)
        T = c["kv"]["T"]
        assert out_a["tokens_written"] == out_b["tokens_written"] == T
        # tests/test_fetchsim.py:275 as written: frame-wise holds fewer frames
        # (GOP batches hold a whole GOP: only fewer when there are several)
        if batch is None or plan.frame_count > plan.F:
            assert out_a["peak_buffer_bytes"] < out_b["peak_buffer_bytes"]
        deq = KV.dequantize(q, torch.bfloat16).data
        blob = b""
        for t in range(T):
            for l in range(3):
                a = mem_a.read(c["token_base"] + t, c["layer_base"] + l)
                b = mem_b.read(c["token_base"] + t, c["layer_base"] + l)
                assert torch.equal(a, b)
                if dtype == torch.int8:
                    blob += a.cpu().numpy().tobytes()
                else:
                    assert torch.equal(a, deq[t, l].reshape(-1))
        if dtype == torch.int8:
            assert ref.digest(blob) == c["slots"]
            assert mem_a.allocated_bytes == c["allocated_bytes"]
        with pytest.raises(KV.ConflictError):
            restore_stream(bs, plan, cfg, mem_a, c["layer_base"], c["token_base"], scales=q.scales)


def test_framewise_restore_peak_at_most_tenth_of_chunkwise():
    q, _ = _q(dict(kind="synthetic", T=10_000, L=3, H=4, D=16, s=0.9, seed=1, c=0.3,
                   group_size=64))
    cfg = L.identity_layout(4, 16)
    cont = C.pack_chunk(q, cfg, ["R240"], cache_id=b"\x01" * 16)
    bs, plan = cont.bitstream(0), cont.plan(0)
    ms, mc = KV.PagedMemory(), KV.PagedMemory()
    ms.begin_fetch()
    mc.begin_fetch()
    s = restore_stream(bs, plan, cfg, ms)   # defaults, as tests/test_acceptance.py:233
    c = restore_chunk_wise(bs, plan, cfg, mc)
    assert s["tokens_written"] == c["tokens_written"] == 10_000
    assert 10 * s["peak_buffer_bytes"] <= c["peak_buffer_bytes"]
    for tok in np.random.default_rng(2).integers(0, 10_000, size=32):
        for layer in range(3):
            assert torch.equal(ms.read(int(tok), layer), mc.read(int(tok), layer))


@pytest.mark.parametrize("into_paged", [False, True])
def test_loopback_fetch_restores_bitexact(tmp_path, into_paged):
    cid = b"\x11" * 16
    q, _ = _q(dict(kind="synthetic", T=256, L=6, H=8, D=32, s=0.9, seed=7, c=0.4, group_size=64))
    cfg = L.identity_layout(8, 32)
    chunks = []
    for j in range(2):
        cont = C.pack_chunk(q.layer_triplet(j), cfg, ["R240", "R1080"], cache_id=cid,
                            chunk_index=j, token_start=0, layer_triplet_index=j, F=4)
        (tmp_path / C.container_filename(cid, j)).write_bytes(cont.to_bytes())
        chunks.append((cid, j))
    handle = NS.serve(NS.ChunkStore(str(tmp_path)), ("127.0.0.1", 0))
    got = []
    mem = KV.PagedMemory(16, dtype=torch.int8) if into_paged else None
    try:
        addr = f"127.0.0.1:{handle.address[1]}"
        tl = FE.live_fetch_pipeline(addr, chunks, None, "fixed:R240", prior_gbps=6.0,
                                    on_chunk=lambda rec, r: got.append(r), mem=mem)
    finally:
        handle.close()
    assert len(got) == 2 and len(tl.records) == 2
    assert all(r["decode_end"] is not None for r in tl.records)
    if into_paged:
        for t in (0, 100, 255):
            for l in range(6):
                assert torch.equal(mem.read(t, l), q.values[t, l].reshape(-1))
    else:
        for j, slab in enumerate(got):
            assert torch.equal(slab.values, q.values[:, 3 * j:3 * j + 3])
            assert torch.equal(slab.scales, q.scales[3 * j:3 * j + 3])


def test_fetch_errors(tmp_path):
    handle = NS.serve(NS.ChunkStore(str(tmp_path)), ("127.0.0.1", 0))
    try:
        addr = f"127.0.0.1:{handle.address[1]}"
        with pytest.raises(NS.ChunkNotFound):
            NS.fetch_chunk(addr, b"\x00" * 16, 0, "R240")
        with pytest.raises(NS.ProtocolError):
            NS.fetch_chunk(addr, b"\x00" * 16, 0, 7)
    finally:
        handle.close()


@pytest.mark.parametrize("concurrent", [False, True])
def test_pipelined_fetch_batches_k_and_v_into_paged_bf16(tmp_path, monkeypatch, concurrent):
    """The batched pipeline (several chunks per decode launch, two caches) with a
    replayed link: every K and V slot equals dequantize() of the packed codes.
    `concurrent`: one chunk per batch and every batch treated as long-stream,
    so up to _INFLIGHT batches run at once on the worker's streams while the
    block tables change under them."""
    if concurrent:
        monkeypatch.setattr(FE, "_LONG_STREAM", 1)
        monkeypatch.setattr(FE, "_MIN_BATCH", 1)
    cfg = L.identity_layout(8, 32)
    store_chunks, qs = [], {}
    for kv_i in range(2):
        cid = bytes([0x50 + kv_i]) * 16
        q, _ = _q(dict(kind="synthetic", T=300, L=5, H=8, D=32, s=0.9, seed=11 + kv_i, c=0.3,
                       group_size=64, bf16=True))
        qp = KV.QuantizedKV(torch.cat([q.values, torch.zeros_like(q.values[:, :1])], 1),
                            torch.cat([q.scales, torch.ones_like(q.scales[:1])], 0), 64)
        qs[cid] = q
        for j in range(2):
            for c, t0 in enumerate((0, 128, 256)):
                tc = min(128, 300 - t0)
                slab = KV.QuantizedKV(qp.values[t0:t0 + tc, 3 * j:3 * j + 3],
                                      qp.scales[3 * j:3 * j + 3], 64)
                cont = C.pack_chunk(slab, cfg, ["R240"], cache_id=cid, chunk_index=10 * j + c,
                                    token_start=t0, layer_triplet_index=j)
                (tmp_path / C.container_filename(cid, 10 * j + c)).write_bytes(cont.to_bytes())
                store_chunks.append((cid, 10 * j + c))
    store = NS.ChunkStore(str(tmp_path), preload=True)
    staged = {key: store.lookup(key[0], key[1], L.RESOLUTION_CODE["R240"]) for key in store_chunks}

    def replay(address, cache_id, chunk_index, resolution, timeout_s=30.0, alloc=None):
        meta, payload = staged[(bytes(cache_id), chunk_index)]
        buf = alloc(len(payload))
        buf.numpy()[:] = np.frombuffer(payload, np.uint8)
        return buf, meta, 1e-3

    mems = {cid: KV.PagedMemory(16, dtype=torch.bfloat16) for cid in qs}
    tl = FE.live_fetch_pipeline(None, store_chunks, None, "fixed:R240", mem=mems, real_layers=5,
                                fetch_fn=replay, max_batch=1 if concurrent else 4)
    assert len(tl.records) == len(store_chunks)
    assert max(r["batch"] for r in tl.records) >= 1
    for cid, q in qs.items():
        deq = KV.dequantize(q, torch.bfloat16).data
        for t in range(300):
            for l in range(5):
                assert torch.equal(mems[cid].read(t, l), deq[t, l].reshape(-1)), (cid, t, l)
        assert mems[cid].read(0, 5) is None          # pad layer never written


@pytest.mark.timeout(300)
def test_pipelined_fetch_callback_error_propagates(tmp_path):
    """An exception in on_chunk reaches the caller; the pipeline neither hangs
    nor leaves the receive loop blocked on a full queue."""
    cfg = L.identity_layout(8, 32)
    q, _ = _q(dict(kind="synthetic", T=64, L=3, H=8, D=32, s=0.9, seed=5, c=0.3,
                   group_size=64, bf16=True))
    cont = C.pack_chunk(q, cfg, ["R240"], cache_id=b"\x61" * 16, chunk_index=0)
    payload = cont.bitstream(L.RESOLUTION_CODE["R240"])
    (tmp_path / C.container_filename(b"\x61" * 16, 0)).write_bytes(cont.to_bytes())
    meta_store = NS.ChunkStore(str(tmp_path), preload=True)
    meta, data = meta_store.lookup(b"\x61" * 16, 0, L.RESOLUTION_CODE["R240"])

    def replay(address, cache_id, chunk_index, resolution, timeout_s=30.0, alloc=None):
        return data, meta, 1e-3

    def boom(rec, res):
        raise RuntimeError("callback failed")

    chunks = [(b"\x61" * 16, 0)] * 80   # more than the queue depth
    with pytest.raises(RuntimeError, match="callback failed"):
        FE.live_fetch_pipeline(None, chunks, None, "fixed:R240", fetch_fn=replay,
                               on_chunk=boom, depth=4)   # decode-only path (no slot claims)
