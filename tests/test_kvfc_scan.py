"""Host-side KVFC stream walk (kvf_kvfc_scan, C++ in libkvf): offsets and the
DecodeError conditions match the reference decoder (via the pinned oracle)."""

import struct

import numpy as np
import pytest

import cases
from oracle import ref
from paper_2602_09725_b200.codec import DecodeError, StreamIndex


def _walk(data):
    """Independent Python walk of fk/codec.py:16-20 for offsets."""
    n, h, w = struct.unpack_from("<III", data, 0)
    blen = ((-(-h // 16)) * (-(-w // 16)) + 7) // 8
    pos, out = 12, []
    for f in range(n):
        t = data[pos]
        pos += 1
        for p in range(3):
            boff = -1
            if t == 1:
                boff = pos
                pos += blen
            (plen,) = struct.unpack_from("<I", data, pos)
            pos += 4
            out.append((pos, plen, boff))
            pos += plen
    return n, h, w, out


@pytest.mark.parametrize("k", range(len(cases.CODEC_CASES)))
def test_scan_offsets(k):
    c = cases.CODEC_CASES[k]
    bs = ref.encode_frames(cases.codec_frames(c), c["gop"])
    ix = StreamIndex(bs)
    n, h, w, want = _walk(bs)
    assert (ix.n, ix.h, ix.w) == (n, h, w)
    for j, (off, plen, boff) in enumerate(want):
        assert ix.payload_off[j] == off and ix.payload_len[j] == plen and ix.bitmap_off[j] == boff
    for f in range(n):
        assert ix.frame_type[f] == (0 if f % c["gop"] == 0 else 1)


def _oracle_error(data):
    try:
        ref.decode_frames(data)
    except ref.OracleDecodeError as e:
        return e.frame_index
    return None


def test_scan_errors_match_reference_decoder():
    rng = np.random.default_rng(3)
    fr = cases.codec_frames(dict(kind="jitter", n=5, h=20, w=37, gop=3, seed=9))
    bs = ref.encode_frames(fr, 3)
    variants = [bs[:5], bs[:12], bs[:13], bs[:-1], bs + b"\x00", bs[:40]]
    bad_type = bytearray(bs)
    bad_type[12] = 7
    variants.append(bytes(bad_type))
    inter_first = bytearray(bs)
    inter_first[12] = 1
    variants.append(bytes(inter_first))
    for cut in rng.integers(12, len(bs), size=40):
        variants.append(bs[:int(cut)])
    for v in variants:
        want = _oracle_error(v)
        if want is None:
            StreamIndex(v)
            continue
        with pytest.raises(DecodeError) as ei:
            StreamIndex(v)
        assert ei.value.frame_index == want, (len(v), want, ei.value.frame_index)


def test_empty_stream():
    data = struct.pack("<III", 0, 4, 4)
    ix = StreamIndex(data)
    assert ix.n == 0
    with pytest.raises(DecodeError) as ei:
        StreamIndex(data + b"\x01")
    assert ei.value.frame_index == -1  # the reference reports frame n-1


def test_batch_walk_equals_per_stream_walk():
    """index_streams (kvf_kvfc_scan_batch, threaded) gives StreamIndex's arrays
    for every stream, including empty and single-frame ones."""
    from paper_2602_09725_b200.codec import index_streams
    streams = [ref.encode_frames(cases.codec_frames(c), c["gop"]) for c in cases.CODEC_CASES]
    streams += [struct.pack("<III", 0, 4, 4)] + streams[:3]
    got = index_streams(streams)
    assert len(got) == len(streams)
    for bs, ix in zip(streams, got):
        one = StreamIndex(bs)
        assert (ix.n, ix.h, ix.w, ix.bitmap_len) == (one.n, one.h, one.w, one.bitmap_len)
        for name in ("payload_off", "payload_len", "bitmap_off"):
            assert np.array_equal(getattr(ix, name), getattr(one, name)), name
        assert np.array_equal(ix.frame_type[:ix.n], one.frame_type[:one.n])


def test_batch_walk_reports_first_bad_stream():
    from paper_2602_09725_b200.codec import index_streams
    fr = cases.codec_frames(dict(kind="jitter", n=5, h=20, w=37, gop=3, seed=9))
    bs = ref.encode_frames(fr, 3)
    for bad, want in ((bs[:40], _oracle_error(bs[:40])), (bs + b"\x00", _oracle_error(bs + b"\x00")),
                      (bs[:5], _oracle_error(bs[:5]))):
        batch = [bs, bs, bad, bs, bs[:-1]]
        with pytest.raises(DecodeError) as ei:
            index_streams(batch)
        assert ei.value.frame_index == want


def test_fed_descriptors_match_part_descriptors():
    """The fed decode's vectorised copy segments tile every stream exactly, and
    its range-decode descriptors equal _part_descriptors' with the same
    segment map (host-side arithmetic only: fake addresses)."""
    import torch
    from paper_2602_09725_b200 import codec
    streams = [ref.encode_frames(cases.codec_frames(c), c["gop"]) for c in cases.CODEC_CASES]
    streams = [s for s in streams if struct.unpack_from("<I", s, 0)[0] > 0][:6]
    idxs = codec.index_streams(streams)
    src = [(j + 1) << 24 | (j * 37 % 128) for j in range(len(streams))]
    segp = codec._fed_segments(idxs, src)
    at = 0
    for j, (bs, ix) in enumerate(zip(streams, idxs)):
        k = slice(at, at + 3 * ix.n)
        lo, ln = segp["lo"][k], segp["len"][k]
        assert lo[0] == 0 and lo[-1] + ln[-1] == len(bs)
        assert np.array_equal(lo[1:], (lo + ln)[:-1])
        assert np.array_equal(segp["src"][k], src[j] + lo)
        at += 3 * ix.n
    region = (segp["len"] + 255) // 128 * 128
    dst = (1 << 40) + np.concatenate([[0], np.cumsum(region)[:-1]]) + segp["src"] % 128
    sym_ptr = (1 << 36) + np.arange(len(streams), dtype=np.int64) * (1 << 28)
    rc = codec._fed_rc(idxs, segp, dst, sym_ptr)
    frames = [torch.empty((ix.n, 3, ix.h, ix.w), dtype=torch.uint8) for ix in idxs]
    n = len(streams)
    rc2, _, _ = codec._part_descriptors(list(range(n)), idxs, [(0, ix.n) for ix in idxs],
                                        np.zeros(n + 1, np.int64),
                                        [(0, len(s)) for s in streams], 0, sym_ptr, frames,
                                        seg_map=(segp["lo"], dst))
    assert np.array_equal(rc, rc2)
