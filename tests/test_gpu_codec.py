"""GPU KVFC decode (range decoder + predictor kernels) is bit-exact against the
reference decoder: golden streams, random sequences/GOPs, all 48 tilings of a
32x128 cache at R240 (tests/test_acceptance.py:112-145 of the reference), and
many streams decoded in one batch."""

import numpy as np
import pytest
import torch

import cases
from oracle import ref

pytestmark = pytest.mark.gpu

from paper_2602_09725_b200 import codec  # noqa: E402


def test_golden_streams_decode(golden):
    for c in golden["codec"]:
        fr = cases.codec_frames(c)
        bs = ref.encode_frames(fr, c["gop"])
        assert ref.digest(bs) == c["stream"]
        got = []
        n = codec.decode_frames(bs, codec.CodecConfig(gop=c["gop"]),
                                lambda f, x: got.append(x.cpu().numpy()))
        assert n == fr.shape[0]
        assert np.array_equal(np.stack(got), fr), c


def test_random_sequences_batched():
    rng = np.random.default_rng(5)
    frames, streams = [], []
    for _ in range(300):
        n = int(rng.integers(1, 6))
        h = int(rng.integers(4, 40))
        w = int(rng.integers(4, 70))
        kind = int(rng.integers(0, 3))
        if kind == 0:
            fr = rng.integers(0, 256, size=(n, 3, h, w)).astype(np.uint8)
        elif kind == 1:
            base = rng.integers(0, 256, size=(1, 3, h, w))
            fr = np.clip(base + rng.integers(-6, 7, size=(n, 3, h, w)), 0, 255).astype(np.uint8)
        else:
            fr = np.full((n, 3, h, w), int(rng.integers(0, 256)), np.uint8)
        gop = int(rng.integers(1, 5))
        frames.append(fr)
        streams.append(ref.encode_frames(fr, gop))
    out, _ = codec.decode_batch(streams)
    for fr, o in zip(frames, out):
        assert np.array_equal(o.cpu().numpy(), fr)


def test_all_tilings_32x128_r240():
    x = ref.gen_synthetic_kv(8, 3, 32, 128, 0.9, 0, 0.3)
    v, _ = ref.quantize(x, 128)
    t = v.reshape(8, 3, 32 * 128)
    streams, frames = [], []
    for a_h in (1, 2, 4, 8, 16, 32):
        for a_d in (1, 2, 4, 8, 16, 32, 64, 128):
            plan = ref.Plan(8, "R240", 32, 128, a_h, 32 // a_h, a_d, 128 // a_d, F=4)
            fr = ref.assemble_frames(t, plan)
            frames.append(fr)
            streams.append(ref.encode_frames(fr, 4))
    assert len(streams) == 48
    out, _ = codec.decode_batch(streams)
    for fr, o in zip(frames, out):
        assert np.array_equal(o.cpu().numpy(), fr)


def test_large_r1080_chunk_and_pitched_output():
    fr = cases.codec_frames(dict(kind="kv", layout=[8, 128, 1, 8, 1, 128], T=2000, res="R1080",
                                 gop=4, seed=3, n=0, h=0, w=0))
    bs = ref.encode_frames(fr, 4)
    n, _, h, w = fr.shape
    big = torch.zeros((n, 3, h, w + 64), dtype=torch.uint8, device="cuda")
    view = big[:, :, :, :w]
    out, _ = codec.decode_batch([bs], out=[view])
    assert np.array_equal(view.cpu().numpy(), fr)
    assert torch.all(big[:, :, :, w:] == 0)


def test_decode_errors():
    fr = cases.codec_frames(dict(kind="jitter", n=3, h=8, w=8, gop=2, seed=1))
    bs = ref.encode_frames(fr, 2)
    for bad in (bs[:5], bs[:-3], bs + b"\0"):
        with pytest.raises(codec.DecodeError):
            codec.decode_frames(bad, codec.CodecConfig(gop=2), lambda f, x: None)


def test_encode_bit_exact_vs_reference(golden):
    for c in golden["codec"]:
        fr = cases.codec_frames(c)
        bs = codec.encode_frames(torch.from_numpy(fr).cuda(), codec.CodecConfig(gop=c["gop"]))
        assert ref.digest(bs.data) == c["stream"], c
        assert bs.frame_count == fr.shape[0]


def test_encode_batch_random_round_trip():
    rng = np.random.default_rng(7)
    frames, gops = [], []
    for _ in range(120):
        n = int(rng.integers(1, 6))
        h = int(rng.integers(4, 40))
        w = int(rng.integers(4, 70))
        base = rng.integers(0, 256, size=(1, 3, h, w))
        fr = np.clip(base + rng.integers(-9, 10, size=(n, 3, h, w)), 0, 255).astype(np.uint8)
        frames.append(fr)
        gops.append(int(rng.integers(1, 5)))
    out = codec.encode_batch([torch.from_numpy(f).cuda() for f in frames], gops)
    for fr, g, bs in zip(frames, gops, out):
        assert bs.data == ref.encode_frames(fr, g)
    dec, _ = codec.decode_batch(out)
    for fr, d in zip(frames, dec):
        assert np.array_equal(d.cpu().numpy(), fr)


def test_rangecoder_module_matches_reference_golden(golden):
    """rangecoder.encode_bytes/decode_bytes (fk/rangecoder.py:205-219) on the GPU
    reproduce the reference's coded streams and symbols."""
    from paper_2602_09725_b200 import rangecoder as RC
    for c in golden["rangecoder"]:
        sym = cases.rc_symbols(c)
        enc = RC.encode_bytes(sym)
        assert ref.digest(enc) == c["coded"], c
        assert np.array_equal(RC.decode_bytes(enc, len(sym)), sym)
    assert len(RC.decode_bytes(b"", 5)) == 5   # reads past the end yield 0


@pytest.mark.parametrize("pinned", [False, True])
def test_part_pipeline_many_parts(monkeypatch, pinned):
    """decode_batch split into the maximum number of parts (side streams,
    descriptors read in place from pinned host memory), with partial frame
    ranges, empty ranges and pitched outputs mixed in."""
    monkeypatch.setattr(codec, "_PART_BYTES", 256)
    rng = np.random.default_rng(9)
    frames, streams, ranges = [], [], []
    for i in range(40):
        n = int(rng.integers(1, 9))
        h, w = int(rng.integers(4, 33)), 16 * int(rng.integers(1, 6))
        base = rng.integers(0, 256, size=(1, 3, h, w))
        fr = np.clip(base + rng.integers(-5, 6, size=(n, 3, h, w)), 0, 255).astype(np.uint8)
        gop = int(rng.integers(1, 4))
        frames.append(fr)
        bs = ref.encode_frames(fr, gop)
        streams.append(torch.frombuffer(bytearray(bs), dtype=torch.uint8).pin_memory()
                       if pinned else bs)
        if i % 5 == 1:
            ranges.append((0, 0))                       # nothing to decode
        elif i % 5 == 2 and n > gop:
            ranges.append((gop, n))                     # starts at the second intra frame
        else:
            ranges.append((0, n))
    out, _ = codec.decode_batch(streams, ranges=ranges)
    live = [j for j, (a, b) in enumerate(ranges) if b > a]
    assert len(codec._split_parts(live, [1000] * len(live))) == codec._MAX_PARTS
    for fr, (a, b), o in zip(frames, ranges, out):
        assert tuple(o.shape) == (b - a,) + fr.shape[1:]
        assert np.array_equal(o.cpu().numpy(), fr[a:b])
    # whole streams (copied before the host walk), a callable `out`, capped parts
    seen = []

    def alloc(shapes):
        seen.extend(shapes)
        return [torch.zeros(shp, dtype=torch.uint8, device="cuda") for shp in shapes]

    out2, _ = codec.decode_batch(streams, out=alloc, max_parts=3)
    assert seen == [fr.shape for fr in frames]
    for fr, o in zip(frames, out2):
        assert np.array_equal(o.cpu().numpy(), fr)


@pytest.mark.parametrize("piece", [16 * 1024, 256])
def test_fed_decode_matches_oracle(monkeypatch, piece):
    """Long planes from pinned buffers take the fed decode (one launch that
    copies the payloads piece-major over PCIe while decoding them): frames
    bit-exact against the reference frames, with sources at odd offsets of
    their pinned buffers (byte head/tail copies) and tiny pieces (a plane
    waits on many pieces)."""
    monkeypatch.setattr(codec, "_FED_PIECE", piece)
    calls = []
    real = codec._decode_fed
    monkeypatch.setattr(codec, "_decode_fed", lambda *a: calls.append(1) or real(*a))
    frames, streams = [], []
    for k, (T, seed) in enumerate([(700, 1), (64, 2), (1300, 3)]):
        fr = cases.codec_frames(dict(kind="kv", layout=[8, 128, 1, 8, 1, 128], T=T,
                                     res="R1080", gop=4, seed=seed, n=0, h=0, w=0))
        bs = ref.encode_frames(fr, 4)
        buf = torch.empty(len(bs) + 16, dtype=torch.uint8, pin_memory=True)
        off = 3 * k + 1                                  # misaligned source bytes
        buf[off:off + len(bs)] = torch.frombuffer(bytearray(bs), dtype=torch.uint8)
        streams.append(buf[off:off + len(bs)])
        frames.append(fr)
    assert codec._fed_eligible(streams)
    out, _ = codec.decode_batch(streams)
    assert calls, "the fed path was not taken"
    for fr, o in zip(frames, out):
        assert np.array_equal(o.cpu().numpy(), fr)
