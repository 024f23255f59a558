"""Host-side logic of the drop-in API (no GPU): frame plans, container format,
wire protocol, resolution selection — against the reference's hand oracles
(tests/test_layout.py:91-139, tests/test_container.py:66-164,
tests/test_acceptance.py:265-299) and the pinned oracle."""

import struct

import numpy as np
import pytest

import cases
from oracle import ref
from paper_2602_09725_b200 import container as C
from paper_2602_09725_b200 import fetch as FE
from paper_2602_09725_b200 import layout as L
from paper_2602_09725_b200 import netstore as NS


def test_placement_small_plan_by_hand():
    plan = L.FramePlan(10, 2, L.identity_layout(2, 2), F=2)
    expected = {0: (0, 0, 0), 1: (1, 0, 0), 2: (0, 0, 1), 3: (1, 0, 1), 4: (2, 0, 0),
                5: (3, 0, 0), 6: (2, 0, 1), 7: (3, 0, 1), 8: (4, 0, 0), 9: (5, 0, 0)}
    for i, want in expected.items():
        assert plan.placement(i) == want
    assert plan.frame_count == 6
    assert plan.frame_slots(4) == [(8, 0, 0)]
    with pytest.raises(ValueError):
        plan.placement(10)


def test_plans_match_oracle_and_digests(golden):
    for c in golden["frames"]:
        plan = L.plan_inter_frame(c["T"], c["res"], L.LayoutConfig(*c["layout"]), c["F"])
        assert plan.frame_shape() == tuple(c["shape"])
        assert plan.digest() == c["digest"]
        op = ref.Plan(c["T"], c["res"], *c["layout"], F=c["F"])
        for i in range(0, c["T"], max(1, c["T"] // 37)):
            assert plan.placement(i) == op.placement(i)
        for f in range(plan.frame_count):
            assert plan.frame_slots(f) == op.frame_slots(f)


def test_tiling_candidates_and_validation():
    assert len(L.tiling_candidates(32, 128)) == 48
    assert len({c.key() for c in L.tiling_candidates(32, 128)}) == 48
    with pytest.raises(ValueError):
        L.LayoutConfig(12, 64, 3, 4, 8, 8)
    with pytest.raises(ValueError):
        L.LayoutConfig(16, 64, 2, 4, 8, 8)
    cfg = L.LayoutConfig(16, 64, 4, 4, 8, 8)
    assert L.LayoutConfig.from_json(cfg.to_json()) == cfg


def _container(seed):
    rng = np.random.default_rng(seed)
    codes = sorted(rng.choice(4, size=int(rng.integers(1, 5)), replace=False).tolist())
    payloads = {c: rng.integers(0, 256, size=int(rng.integers(0, 300))).astype(np.uint8).tobytes()
                for c in codes}
    meta = {"layout": L.identity_layout(4, 8).to_json(), "F": 4, "plans": {}, "frame_counts": {},
            "group_size": 8, "scales_b64": "AACAPw==" * 0 + ""}
    return C.ChunkContainer(rng.bytes(16), int(rng.integers(0, 2**32)), int(rng.integers(0, 2**32)),
                            int(rng.integers(1, 10000)), int(rng.integers(0, 256)), meta, payloads)


def test_container_round_trips():
    for seed in range(2000):
        c = _container(seed)
        blob = c.to_bytes()
        back = C.ChunkContainer.from_bytes(blob)
        assert back.to_bytes() == blob
        assert back.payloads == c.payloads
        hdr, entries = C.parse_header(blob)
        assert [e[0] for e in entries] == c.resolutions
    with pytest.raises(ValueError):
        C.parse_header(b"XXXX" + blob[4:])
    with pytest.raises(ValueError):
        C.parse_header(blob[:10])


def test_container_bytes_layout_matches_oracle(golden):
    # Same payload bytes -> same container bytes as the oracle's to_bytes restatement.
    for c in golden["container"]:
        x = cases.quant_input(c["kv"])
        v, s = ref.quantize(x, c["kv"]["group_size"])
        blob = ref.pack_chunk_bytes(v, s, c["layout"], c["res"], c["kv"]["group_size"],
                                    bytes.fromhex(c["cache_id"]), c["chunk_index"],
                                    c["token_start"], c["triplet"], c["F"])
        back = C.ChunkContainer.from_bytes(blob)
        assert back.to_bytes() == blob
        assert np.array_equal(back.scales(), s)


def test_wire_round_trips():
    rng = np.random.default_rng(1)
    for _ in range(5000):
        req = NS.WireRequest(rng.bytes(16), int(rng.integers(0, 2**32)), int(rng.integers(0, 4)))
        assert NS.WireRequest.decode(req.encode()) == req
        resp = NS.WireResponse(int(rng.integers(0, 3)), {"k": int(rng.integers(0, 99))},
                               rng.bytes(int(rng.integers(0, 64))))
        back = NS.WireResponse.decode(resp.encode())
        assert (back.status, back.metadata, back.payload) == (resp.status, resp.metadata, resp.payload)
    with pytest.raises(NS.ProtocolError):
        NS.WireRequest.decode(b"\x00" * 5)
    with pytest.raises(NS.ProtocolError):
        NS.WireRequest.decode(struct.pack("<4sB16sIB", b"NOPE", 1, b"\0" * 16, 0, 0))


def test_select_resolution_and_bandwidth():
    table = FE.LookupTable("flat", 1, {r: [0.1] for r in L.RESOLUTION_ORDER},
                           {"R240": 0.05, "R480": 0.05, "R640": 0.05, "R1080": 0.0},
                           {"R240": 10, "R480": 20, "R640": 30, "R1080": 50})
    assert FE.estimate_bandwidth([(1e9, 1.0)]) == pytest.approx(8.0)
    assert FE.estimate_bandwidth([], prior_gbps=3) == 3.0
    with pytest.raises(RuntimeError):
        FE.estimate_bandwidth([])
    for bw in (0.5, 1, 2, 4, 8, 16, 64):
        got = FE.select_resolution(bw, 1, "R1080", table)
        deltas = []
        for r in L.RESOLUTION_ORDER:
            pen = table.tau_penalty(r) if r != "R1080" else 0.0
            deltas.append((abs(table.size_bytes(r) * 8 / (bw * 1e9) - 0.1 - pen), r))
        best = min(d for d, _ in deltas)
        assert got == [r for d, r in deltas if d == best][-1]


@pytest.mark.parametrize("res", L.RESOLUTION_ORDER)
@pytest.mark.parametrize("T", [1, 7, 65, 999, 10000])
def test_tokens_in_frames_matches_frame_slots(res, T):
    """The vectorised slot enumeration restore claims with equals the
    reference's per-frame frame_slots walk (fk/layout.py:203-212)."""
    plan = L.plan_inter_frame(T, res, L.identity_layout(8, 32), 4)
    for first, n in [(0, plan.frame_count), (0, 1), (plan.frame_count - 1, 1),
                     (plan.frame_count // 2, plan.frame_count - plan.frame_count // 2),
                     (min(4, plan.frame_count - 1), min(4, plan.frame_count - min(4, plan.frame_count - 1)))]:
        want = sorted(i for f in range(first, first + n) for i, _, _ in plan.frame_slots(f))
        assert list(plan.tokens_in_frames(first, n)) == want


def test_b200_lookup_table_and_adaptive_choice():
    """The measured B200 decode table (data/b200.json, reference table format
    fk/data/h20.json) loads, validates, and drives Alg. 1 (select_resolution,
    fk/fetchsim.py:154-169): fast links pick the short-stream class whose GPU
    decode hides under the transfer; a slow link can afford R1080."""
    from paper_2602_09725_b200 import fetch as FE
    t = FE.default_table()
    assert t.P >= 1 and set(t.decode_s) == set(L.RESOLUTION_ORDER)
    assert t.tau_dec("R240", 1) < t.tau_dec("R1080", 1)   # more, shorter streams decode faster
    assert FE.LookupTable.from_json(t.to_json()).decode_s == t.decode_s
    assert FE.select_resolution(100.0, 1, "R1080", t) == "R240"
    assert FE.select_resolution(10.0, 1, "R1080", t) == "R240"
    assert FE.select_resolution(1.0, 1, "R1080", t) == "R1080"


def test_pacer_holds_the_link_rate():
    """The server's egress pacer (netstore._Pacer) sends at the configured rate."""
    import time
    p = NS._Pacer(8.0)                       # 1 GB/s
    t0 = time.monotonic()
    sent = 0
    while sent < 100_000_000:
        p.wait(p.slice)
        sent += p.slice
    dt = time.monotonic() - t0
    assert 0.08 <= dt <= 0.25, dt             # 0.1 s less the 10 ms burst; slack for a busy host


def test_loopback_server_round_trip(tmp_path):
    """Store -> server -> fetch_chunk over loopback TCP (no GPU): payload and
    metadata arrive intact, unknown chunks and classes map to the reference errors."""
    rng = np.random.default_rng(4)
    meta = {"layout": L.identity_layout(4, 8).to_json(), "F": 4, "plans": {}, "frame_counts": {},
            "group_size": 8, "scales_b64": ""}
    payloads = {0: rng.integers(0, 256, 5000).astype(np.uint8).tobytes(),
                3: rng.integers(0, 256, 70000).astype(np.uint8).tobytes()}
    cid = bytes(range(16))
    cont = C.ChunkContainer(cid, 7, 100, 50, 2, meta, payloads)
    (tmp_path / C.container_filename(cid, 7)).write_bytes(cont.to_bytes())
    for preload in (False, True):
        store = NS.ChunkStore(str(tmp_path), preload=preload)
        assert len(store) == 1
        with NS.serve(store, ("127.0.0.1", 0), rate_limit_gbps=0.5) as h:
            addr = f"127.0.0.1:{h.address[1]}"
            for code, name in ((0, "R240"), (3, "R1080")):
                payload, got_meta, tau = NS.fetch_chunk(addr, cid, 7, name)
                assert payload == payloads[code] and tau > 0
                assert got_meta["resolution"] == name and got_meta["token_start"] == 100
                assert got_meta["layer_triplet_index"] == 2 and got_meta["cache_id"] == cid.hex()
                back = NS.container_of(got_meta, payload)
                assert back.bitstream(code) == payloads[code] and back.token_count == 50
            with pytest.raises(NS.ChunkNotFound):
                NS.fetch_chunk(addr, cid, 8, "R240")
            with pytest.raises(NS.ChunkNotFound):
                NS.fetch_chunk(addr, cid, 7, "R480")
            with pytest.raises(NS.ProtocolError):
                NS.fetch_chunk(addr, cid, 7, 9)
