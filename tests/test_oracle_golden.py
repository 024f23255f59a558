"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden/).

Every digest in golden.json was produced by running the reference framekv on the
inputs cases.py regenerates; the oracle must reproduce each one bit for bit.
"""

import numpy as np
import pytest

import cases
from oracle import ref


def test_synthetic_generator_matches_reference(golden):
    for c in golden["synthetic"]:
        x = ref.gen_synthetic_kv(c["T"], c["L"], c["H"], c["D"], c["s"], c["seed"], c["c"])
        assert ref.digest(x) == c["data"]


@pytest.mark.parametrize("k", range(len(cases.QUANT_CASES)))
def test_quantize_matches_reference(golden, k):
    c = golden["quantize"][k]
    x = cases.quant_input(c)
    v, s = ref.quantize(x, c["group_size"])
    assert ref.digest(v) == c["values"]
    assert ref.digest(s) == c["scales"]
    assert ref.digest(ref.dequantize(v, s, c["group_size"])) == c["dequant"]


def test_quantize_unit_oracles():
    # tests/test_kvmodel.py:16-50 of the reference, restated
    v, s = ref.quantize(np.array([-1, 0, 1], np.float32).reshape(3, 1, 1, 1), 1)
    assert v.ravel().tolist() == [-127, 0, 127]
    v, _ = ref.quantize(np.array([127.0, 64.5], np.float32).reshape(2, 1, 1, 1), 1)
    assert v.ravel().tolist() == [127, 64]
    v, s = ref.quantize(np.zeros((4, 3, 2, 4), np.float32), 4)
    assert np.all(s == 1.0) and np.all(v == 0)


def test_frames_match_reference(golden):
    for c in golden["frames"]:
        t = cases.frame_tensors(c)
        plan = ref.Plan(c["T"], c["res"], *c["layout"], F=c["F"])
        fr = ref.assemble_frames(t, plan)
        assert list(fr.shape) == c["shape"]
        assert ref.digest(fr) == c["frames"], c
        assert ref.plan_digest(plan) == c["digest"]
        assert np.array_equal(ref.disassemble_frames(fr, plan), t)


def test_codec_matches_reference(golden):
    for c in golden["codec"]:
        fr = cases.codec_frames(c)
        bs = ref.encode_frames(fr, c["gop"])
        assert ref.digest(bs) == c["stream"], c
        assert np.array_equal(ref.decode_frames(bs), fr)


def test_rangecoder_matches_reference(golden):
    for c in golden["rangecoder"]:
        sym = cases.rc_symbols(c)
        enc = ref.rc_encode(sym)
        assert ref.digest(enc) == c["coded"]
        assert np.array_equal(ref.rc_decode(enc, len(sym)), sym)


def test_container_matches_reference(golden):
    for c in golden["container"]:
        x = cases.quant_input(c["kv"])
        v, s = ref.quantize(x, c["kv"]["group_size"])
        blob = ref.pack_chunk_bytes(v, s, c["layout"], c["res"], c["kv"]["group_size"],
                                    bytes.fromhex(c["cache_id"]), c["chunk_index"],
                                    c["token_start"], c["triplet"], c["F"])
        assert ref.digest(blob) == c["bytes"]


def test_restore_matches_reference(golden):
    for c in golden["restore"]:
        kv = c["kv"]
        v, s = ref.quantize(cases.quant_input(kv), kv["group_size"])
        plan = ref.Plan(kv["T"], c["res"], *c["layout"], F=c["F"])
        t = v.reshape(kv["T"], 3, kv["H"] * kv["D"])
        stream = ref.encode_frames(ref.assemble_frames(t, plan), plan.F)
        assert ref.digest(stream) == c["stream"]
        slots = ref.restore_slots(ref.decode_frames(stream), plan, c["layer_base"], c["token_base"])
        blob = b"".join(slots[(tk, l)].tobytes()
                        for tk in range(c["token_base"], c["token_base"] + kv["T"])
                        for l in range(c["layer_base"], c["layer_base"] + 3))
        assert ref.digest(blob) == c["slots"]
        assert len(slots) * kv["H"] * kv["D"] == c["allocated_bytes"]


def test_decode_errors_like_reference():
    fr = cases.codec_frames(dict(kind="jitter", n=3, h=8, w=8, gop=2, seed=1))
    bs = ref.encode_frames(fr, 2)
    with pytest.raises(ref.OracleDecodeError):
        ref.decode_frames(bs[:5])
    with pytest.raises(ref.OracleDecodeError):
        ref.decode_frames(bs[:-3])
    with pytest.raises(ref.OracleDecodeError):
        ref.decode_frames(bs + b"\0")
