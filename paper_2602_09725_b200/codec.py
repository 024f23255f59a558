"""KVFC lossless frame codec on the GPU (drop-in for the reference fk/codec.py).

Stream format (fk/codec.py:16-20): u32 n, u32 height, u32 width; per frame a
u8 type (0 intra, 1 inter) and per plane [inter: packed 16x16-block mode
bitmap] u32 length + range-coded payload of zigzag residual symbols.

Decode: a host walk of the stream layout (kvf_kvfc_scan, C++), one H2D copy of
all stream bytes, then two launches for ANY number of streams — the range
decoder (one GPU thread per (frame, plane) stream, kvf_rc_decode) and the
predictor (one CTA per same-plane chain of frames, kvf_kvfc_reconstruct).
Encode: see ``encode_frames`` (GPU residual/mode kernels + range coder).
"""

from __future__ import annotations

import collections
import ctypes as C
import struct
import threading

import numpy as np
import torch

from . import _dev, _lib

BLOCK = 16


# numpy twins of the descriptor structs of include/kvf.h (kvf_rc_stream,
# kvf_recon_plane, kvf_recon_chain): built vectorised, one H2D copy each.
_RC_DTYPE = np.dtype([("payload", "<u8"), ("len", "<i8"), ("symbols", "<u8"),
                      ("n_symbols", "<i8")])
_PLANE_DTYPE = np.dtype([("symbols", "<u8"), ("modes", "<u8"), ("out", "<u8"),
                         ("out_pitch", "<i8")])
_CHAIN_DTYPE = np.dtype([("first", "<i4"), ("count", "<i4"), ("height", "<i4"),
                         ("width", "<i4")])
_SEG_DTYPE = np.dtype([("src", "<u8"), ("dst", "<u8"), ("len", "<i8")])
_RESID_DTYPE = np.dtype([("cur", "<u8"), ("prev", "<u8"), ("pitch", "<i8"), ("symbols", "<u8"),
                         ("modes", "<u8"), ("height", "<i4"), ("width", "<i4")])
_PIECE_DTYPE = np.dtype([("src", "<u8"), ("dst_off", "<i8"), ("len", "<i8"), ("pack_bits", "<i4"),
                         ("reserved_", "<i4")])
assert _RC_DTYPE.itemsize == C.sizeof(_lib.kvf_rc_stream)
assert _RESID_DTYPE.itemsize == C.sizeof(_lib.kvf_resid_plane)
assert _PIECE_DTYPE.itemsize == C.sizeof(_lib.kvf_piece)
assert _PLANE_DTYPE.itemsize == C.sizeof(_lib.kvf_recon_plane)
assert _CHAIN_DTYPE.itemsize == C.sizeof(_lib.kvf_recon_chain)


class DecodeError(RuntimeError):
    """Corrupt or truncated stream (fk/codec.py:45-48)."""

    def __init__(self, message, frame_index=None):
        super().__init__(message)
        self.frame_index = frame_index


class CodecConfig:
    def __init__(self, gop: int = 4, reference_depth: int = 1, block_size: int = BLOCK):
        if reference_depth > 3:
            raise ValueError("reference_depth must be < 4")
        if block_size != BLOCK:
            raise ValueError("only 16x16 blocks are supported")
        if gop < 1:
            raise ValueError("gop must be >= 1")
        self.gop = gop
        self.reference_depth = reference_depth
        self.block_size = block_size


class Bitstream:
    def __init__(self, data, frame_count, height, width, frame_offsets, inter_fraction):
        self.data = data
        self.frame_count = frame_count
        self.height = height
        self.width = width
        self.frame_offsets = frame_offsets
        self.inter_fraction = inter_fraction

    def __len__(self):
        return len(self.data)


def _as_bytes(bs) -> bytes:
    return bs.data if isinstance(bs, Bitstream) else bytes(bs)


def _host_view(bs):
    """(address, size, keepalive) of a stream's host bytes without copying:
    bytes / Bitstream, or a CPU uint8 tensor (e.g. a pinned receive buffer)."""
    if isinstance(bs, torch.Tensor):
        if bs.is_cuda or bs.dtype != torch.uint8 or not bs.is_contiguous():
            raise ValueError("tensor streams must be contiguous CPU uint8 tensors")
        return bs.data_ptr(), bs.numel(), bs
    data = _as_bytes(bs)
    return (C.cast(C.c_char_p(data), C.c_void_p).value or 0), len(data), data


class StreamIndex:
    """Layout of one KVFC stream (host arrays from kvf_kvfc_scan)."""

    def __init__(self, data):
        lib = _lib.load()
        info = _lib.kvf_kvfc_info()
        bad = C.c_int32(0)
        addr, size, _keep = _host_view(data)
        buf = C.c_void_p(addr) if size else None
        st = lib.kvf_kvfc_scan(buf, size, C.byref(info), None, None, None, None, 0,
                               C.byref(bad))
        if st == _lib.KVF_EDECODE:
            raise DecodeError(lib.kvf_last_error().decode(), frame_index=bad.value)
        n = info.n_frames
        self.n, self.h, self.w, self.bitmap_len = n, info.height, info.width, info.bitmap_len
        self.payload_off = np.zeros(3 * n, np.int64)
        self.payload_len = np.zeros(3 * n, np.int32)
        self.bitmap_off = np.zeros(3 * n, np.int64)
        self.frame_type = np.zeros(max(n, 1), np.uint8)
        st = lib.kvf_kvfc_scan(buf, size, C.byref(info),
                               self.payload_off.ctypes.data, self.payload_len.ctypes.data,
                               self.bitmap_off.ctypes.data, self.frame_type.ctypes.data, n,
                               C.byref(bad))
        if st == _lib.KVF_EDECODE:
            raise DecodeError(lib.kvf_last_error().decode(), frame_index=bad.value)
        _lib.check(st)


_SCAN_THREADS = 16  # host threads of the batched stream walk


def index_streams(datas) -> list:
    """StreamIndex of every stream: two kvf_kvfc_scan_batch calls (headers,
    then the walk on host threads inside libkvf) instead of two ctypes calls
    and four allocations per stream.

    The walk is a pointer chase through the stream (each plane's length word
    gives the next position), one cache/TLB miss per plane, so streams are
    spread over threads.  Errors are raised as by StreamIndex, for the first
    failing stream in order.
    """
    datas = list(datas)
    if len(datas) < 4:
        return [StreamIndex(d) for d in datas]
    lib = _lib.load()
    n_st = len(datas)
    views = [_host_view(d) for d in datas]
    addr = np.array([v[0] for v in views], np.uint64)
    size = np.array([v[1] for v in views], np.int64)
    infos = (_lib.kvf_kvfc_info * n_st)()
    bad_s, bad_f = C.c_int32(-1), C.c_int32(0)

    def scan(base, po, pl, bo, ft):
        ptr = (lambda a: C.c_void_p(a.ctypes.data) if a is not None else None)
        return lib.kvf_kvfc_scan_batch(
            C.c_void_p(addr.ctypes.data), C.c_void_p(size.ctypes.data), n_st, infos,
            ptr(base), ptr(po), ptr(pl), ptr(bo), ptr(ft), _SCAN_THREADS,
            C.byref(bad_s), C.byref(bad_f))

    def fail(st):
        if st == _lib.KVF_EDECODE:
            raise DecodeError(lib.kvf_last_error().decode(), frame_index=bad_f.value)
        _lib.check(st)

    st = scan(None, None, None, None, None)
    if st != _lib.KVF_OK:
        fail(st)
    n = np.array([infos[j].n_frames for j in range(n_st)], np.int64)
    base = np.concatenate([[0], np.cumsum(n)]).astype(np.int64)
    total = int(base[-1])
    po = np.zeros(3 * total, np.int64)
    pl = np.zeros(3 * total, np.int32)
    bo = np.zeros(3 * total, np.int64)
    ft = np.zeros(max(total, 1), np.uint8)
    st = scan(base, po, pl, bo, ft)
    if st != _lib.KVF_OK:
        fail(st)
    out = []
    for j in range(n_st):
        ix = StreamIndex.__new__(StreamIndex)
        b0, b1 = int(base[j]), int(base[j + 1])
        inf = infos[j]
        ix.n, ix.h, ix.w, ix.bitmap_len = inf.n_frames, inf.height, inf.width, inf.bitmap_len
        ix.payload_off = po[3 * b0:3 * b1]
        ix.payload_len = pl[3 * b0:3 * b1]
        ix.bitmap_off = bo[3 * b0:3 * b1]
        ix.frame_type = ft[b0:b1] if b1 > b0 else np.zeros(1, np.uint8)
        out.append(ix)
    return out


class _PinnedStaging:
    """Grow-only pinned host buffer for the coded bytes of a decode batch.

    Pinning a fresh buffer per call costs ~0.1 s/GB; this one is reused.  A
    buffer is handed out only after the H2D copy that last read it completed
    (event recorded on the copying stream), so reuse never races a copy.
    """

    def __init__(self):
        self._buf = None
        self._done = None
        self._lock = threading.Lock()

    def acquire(self, nbytes: int) -> torch.Tensor:
        self._lock.acquire()
        if self._done is not None:
            self._done.synchronize()
        if self._buf is None or self._buf.numel() < nbytes:
            self._buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        return self._buf[:nbytes]

    def release(self, stream) -> None:
        self._done = torch.cuda.Event()
        self._done.record(stream)
        self._lock.release()


_STAGING = _PinnedStaging()
_OUT_STAGING = _PinnedStaging()   # encode_batch's D2H of the coded streams


def decode_batch(streams, out=None, stream=None, ranges=None, indices=None,
                 max_parts=None):
    """Decode many KVFC streams on the GPU: two launches (range decode,
    reconstruction) per part of up to _MAX_PARTS, pipelined with the H2D copy.

    ``streams``: list of bytes / Bitstream (staged through a reused pinned
    buffer), or of contiguous CPU uint8 tensors — pinned receive buffers —
    which are copied to the device directly.  ``out``: optional list of
    [n, 3, h, w] uint8 CUDA tensors (any row pitch) to decode into, or a
    callable taking the list of those shapes (known after the stream walk)
    and returning the tensors.
    ``ranges``: optional per-stream (first, stop) frame range; ``first`` must
    be an intra frame (a chain start), and the output holds stop-first frames.
    ``max_parts`` caps the part pipeline (default _MAX_PARTS; each part runs on
    its own side stream of ``stream``).
    Returns (frames list, device bytes held).  Raises DecodeError like the
    reference.  The work is ordered on ``stream`` (default: current): callers
    see the frames after it.  Calls on one stream must come from one thread
    at a time (the device scratch is per stream).
    """
    staged = []   # the pinned staging buffer, once acquired
    try:
        return _decode_batch(streams, out, stream, ranges, indices, max_parts, staged)
    except BaseException:
        if staged:
            # copies queued on side streams may still read the staging buffer:
            # let every queued copy finish before it can be handed out again
            torch.cuda.synchronize()
            _STAGING.release(staged[0])
        raise


def _decode_batch(streams, out, stream, ranges, indices, max_parts, staged):
    dev = _dev.device()
    pinned_in = all(isinstance(x, torch.Tensor) for x in streams) and len(streams) > 0
    datas = list(streams) if pinned_in else [_as_bytes(x) for x in streams]
    s = stream if stream is not None else torch.cuda.current_stream()
    if pinned_in and indices is None and ranges is None and _fed_eligible(datas):
        fed = _decode_fed(datas, out, s, dev)
        if fed is not None:
            return fed
    # Whole pinned streams with nothing to scan first: their bytes go to the
    # copy engine at once and the host walk (kvf_kvfc_scan) runs meanwhile.
    early = pinned_in and indices is None and ranges is None
    host = None
    if early:
        spans = [(0, int(d.numel())) for d in datas]
        sizes = [hi for _, hi in spans]
        starts = np.cumsum([0] + sizes)
        parts = _split_parts(list(range(len(datas))), sizes, max_parts)
        blob = _scratch(s, "blob", int(starts[-1]) or 1)
        side = _enqueue_copies(s, parts, datas, spans, starts, blob, None)
        idxs = index_streams(datas)
        ranges = [(0, ix.n) for ix in idxs]
    else:
        idxs = indices if indices is not None else index_streams(datas)
        if ranges is None:
            ranges = [(0, ix.n) for ix in idxs]
    for ix, (f0, f1) in zip(idxs, ranges):
        if not 0 <= f0 <= f1 <= ix.n:
            raise ValueError("frame range outside the stream")
        if f0 < f1 and ix.frame_type[f0] != 0:
            raise ValueError("a partial decode must start at an intra frame")
    live = [j for j, (f0, f1) in enumerate(ranges) if f1 > f0]
    if not early:
        # Only the byte span of the decoded frames travels to the device.
        spans = []
        for ix, (f0, f1) in zip(idxs, ranges):
            if f1 <= f0:
                spans.append((0, 0))
                continue
            ks = slice(3 * f0, 3 * f1)
            heads = np.where(ix.bitmap_off[ks] >= 0, ix.bitmap_off[ks], ix.payload_off[ks])
            spans.append((int(heads.min()),
                          int((ix.payload_off[ks] + ix.payload_len[ks]).max())))
        sizes = [hi - lo for lo, hi in spans]
        starts = np.cumsum([0] + sizes)
        parts = _split_parts(live, [sizes[j] for j in live], max_parts)
        if not pinned_in:
            host = _STAGING.acquire(int(starts[-1]) or 1)
            staged.append(s)
            hv = host.numpy()
            for d, s0, (lo, hi) in zip(datas, starts[:-1], spans):
                hv[s0:s0 + hi - lo] = np.frombuffer(d, np.uint8, hi - lo, lo)
        blob = _scratch(s, "blob", int(starts[-1]) or 1)
        side = _enqueue_copies(s, parts, datas, spans, starts, blob, host)
    hw_all = np.array([ix.h * ix.w for ix in idxs], np.int64)
    hw16_all = -(-hw_all // 16) * 16                 # 16-byte aligned symbol slots
    nf_all = np.array([f1 - f0 for f0, f1 in ranges], np.int64)
    sym_at = np.concatenate([[0], np.cumsum(3 * nf_all * hw16_all)])
    frames = []
    symbols = _scratch(s, "symbols", max(int(sym_at[-1]), 1))
    if callable(out):
        with torch.cuda.stream(s):
            out = out([(f1 - f0, 3, ix.h, ix.w) for ix, (f0, f1) in zip(idxs, ranges)])
    with torch.cuda.stream(s):
        for j, (ix, (f0, f1)) in enumerate(zip(idxs, ranges)):
            fr = out[j] if out is not None else torch.empty((f1 - f0, 3, ix.h, ix.w),
                                                           dtype=torch.uint8, device=dev)
            if tuple(fr.shape) != (f1 - f0, 3, ix.h, ix.w):
                raise ValueError("output frames have the wrong shape")
            frames.append(fr)
    # Part by part, the descriptors are built on the host while the copies
    # run; part p's two kernels follow its coded bytes on its stream, so they
    # overlap the copies of parts p+1..  The kernels read the descriptors in
    # place from pinned host memory (mapped, UVA): no H2D copy of their own
    # queues behind the bytes.  (The side streams waited for all work `s` had
    # when they were set up, and nothing was queued on `s` since, so `symbols`
    # and `frames`, allocated on `s` afterwards, are free for them.)
    base = blob.data_ptr()
    done, keep = [], []
    for p, part in enumerate(parts):
        t = side[p]
        part = [j for j in part if ranges[j][1] > ranges[j][0]]
        if not part:
            if t is not s:
                ev = torch.cuda.Event()
                ev.record(t)
                done.append((t, ev))
            continue
        rc, flat, ch_arr = _part_descriptors(part, idxs, ranges, starts, spans, base,
                                             symbols.data_ptr() + sym_at, frames)
        h_rc, h_planes, h_chains = (_pinned_copy(x) for x in (rc, flat, ch_arr))
        sp = _dev.stream_ptr(t)
        if len(rc):
            _lib.call("kvf_rc_decode", C.c_void_p(h_rc.data_ptr()), len(rc), sp)
        if len(ch_arr):
            _lib.call("kvf_kvfc_reconstruct", C.c_void_p(h_planes.data_ptr()),
                      C.c_void_p(h_chains.data_ptr()), len(ch_arr), sp)
        keep += [h_rc, h_planes, h_chains]
        if t is not s:
            ev = torch.cuda.Event()
            ev.record(t)
            done.append((t, ev))
    for t, ev in done:
        s.wait_event(ev)
    if host is not None:
        staged.clear()
        _STAGING.release(s)   # `s` now follows every part's copies
    held = blob.numel() + symbols.numel() + sum(f.numel() for f in frames)
    # pinned descriptors: alive until `s` passes this point
    _hold_until(s, keep)
    # keep device scratch tensors alive until the stream reaches this point
    frames_keepalive = (blob, symbols, *frames)
    for t in frames_keepalive:
        t.record_stream(s)
        for u, _ in done:
            t.record_stream(u)
    return frames, held


# Fed decode (kvf_rc_decode_fed): long planes (R640/R1080-sized, >= this many
# symbols) decode for ~0.33 us a symbol on one thread's serial chain, longer
# than the whole H2D of a batch.  Their bytes are copied by the decode launch
# itself, piece-major, so every plane starts after its first piece instead of
# after the batch's last copy.
_FED_MIN_SYMBOLS = 98_304
_FED_PIECE = 4 * 1024
_FED_COPY_CTAS = 256  # 96 or fewer starve the decoders (208 ms at 96 on C2 R1080); 128-512 all ~98.8 ms


_FED_MAX_PLANES = 50_000  # one wave of 1-warp decoder CTAs (+ copy CTAs) on 148 SMs


def _fed_eligible(datas):
    """Whole pinned KVFC streams whose planes are long (header only: u32
    n_frames, height, width, fk/codec.py:16-20), few enough planes for one
    wave of the fed launch."""
    planes = 0
    for d in datas:
        if d.numel() < 12 or not d.is_pinned():
            return False
        n, h, w = struct.unpack("<III", C.string_at(d.data_ptr(), 12))
        if n == 0 or h * w < _FED_MIN_SYMBOLS:
            return False
        planes += 3 * n
    return planes <= _FED_MAX_PLANES


def _fed_segments(idxs, src_ptrs):
    """Copy segments of whole streams, vectorised over all planes (stream j's
    planes k = 3 f + p in order): plane k's bytes run from the previous
    payload's end (0 for a stream's first plane) to the end of its payload,
    i.e. its mode bitmap, length word and payload.  `src_ptrs[j]`: the host
    address of stream j's first byte."""
    n_pl = np.array([3 * ix.n for ix in idxs], np.int64)
    p_off = np.concatenate([ix.payload_off for ix in idxs]).astype(np.int64)
    p_len = np.concatenate([ix.payload_len for ix in idxs]).astype(np.int64)
    ends = p_off + p_len
    first = np.concatenate([[0], np.cumsum(n_pl)[:-1]]).astype(np.int64)
    lo = np.empty_like(ends)
    lo[1:] = ends[:-1]
    lo[first[n_pl > 0]] = 0
    return {"n_pl": n_pl, "first": first, "p_off": p_off, "p_len": p_len, "lo": lo,
            "len": ends - lo, "src": np.repeat(np.asarray(src_ptrs, np.int64), n_pl) + lo}


def _fed_rc(idxs, segp, dst, sym_ptr):
    """kvf_rc_stream array of whole streams whose plane segments sit at device
    addresses `dst` (what _part_descriptors gives with seg_map=(lo, dst));
    `sym_ptr[j]`: stream j's symbol slots."""
    n_pl, first = segp["n_pl"], segp["first"]
    hw = np.array([ix.h * ix.w for ix in idxs], np.int64)
    hw16 = -(-hw // 16) * 16
    K = int(n_pl.sum())
    sid = np.repeat(np.arange(len(idxs)), n_pl)
    loc = np.arange(K, dtype=np.int64) - first[sid]
    rc = np.empty(K, _RC_DTYPE)
    rc["payload"] = dst + (segp["p_off"] - segp["lo"])
    rc["len"] = segp["p_len"]
    rc["symbols"] = np.asarray(sym_ptr, np.int64)[sid] + loc * hw16[sid]
    rc["n_symbols"] = hw[sid]
    return rc


def _decode_fed(datas, out, s, dev):
    """decode_batch of whole pinned streams through one kvf_rc_decode_fed
    launch + one reconstruction launch on `s`; None if the batch does not fit
    one wave (the caller then takes the part pipeline)."""
    idxs = index_streams(datas)
    ranges = [(0, ix.n) for ix in idxs]
    # Copy segments: plane k of stream j = its bytes from the previous
    # payload's end (0 for the first) to the end of its payload (bitmap, length,
    # payload).  Each segment gets 128-byte lines of its own in the blob, at the
    # source's offset modulo 128 (16-byte copies; no L1 line shared with bytes
    # that land later).
    segp = _fed_segments(idxs, [d.data_ptr() for d in datas])
    lo_a, len_a, src_a = segp["lo"], segp["len"], segp["src"]
    region = (len_a + 255) // 128 * 128                  # >= len + (src % 128), lines
    roff = np.concatenate([[0], np.cumsum(region)])
    blob = _scratch(s, "blob", int(roff[-1]) or 1)
    base = blob.data_ptr()
    if base % 128:
        return None
    dst_a = base + roff[:-1] + src_a % 128
    hw_all = np.array([ix.h * ix.w for ix in idxs], np.int64)
    hw16_all = -(-hw_all // 16) * 16
    nf_all = np.array([f1 - f0 for f0, f1 in ranges], np.int64)
    sym_at = np.concatenate([[0], np.cumsum(3 * nf_all * hw16_all)])
    symbols = _scratch(s, "symbols", max(int(sym_at[-1]), 1))
    if callable(out):
        with torch.cuda.stream(s):
            out = out([(f1 - f0, 3, ix.h, ix.w) for ix, (f0, f1) in zip(idxs, ranges)])
    frames = []
    with torch.cuda.stream(s):
        for j, (ix, (f0, f1)) in enumerate(zip(idxs, ranges)):
            fr = out[j] if out is not None else torch.empty((f1 - f0, 3, ix.h, ix.w),
                                                           dtype=torch.uint8, device=dev)
            if tuple(fr.shape) != (f1 - f0, 3, ix.h, ix.w):
                raise ValueError("output frames have the wrong shape")
            frames.append(fr)
    # the range-decode descriptors first (plane k of stream j, frame-major):
    # the launch goes out before the reconstruction's descriptors are built
    rc = _fed_rc(idxs, segp, dst_a, symbols.data_ptr() + sym_at)
    K = len(rc)
    segs = np.empty(K, _SEG_DTYPE)
    segs["src"], segs["dst"], segs["len"] = src_a, dst_a, len_a
    seg_of = np.arange(K, dtype=np.int32)
    h_rc, h_segs, h_of = _pinned_copy(rc), _pinned_copy(segs), _pinned_copy(seg_of)
    ready = _scratch(s, "fed_ready", 4 * max(len(rc), 1))
    sp = _dev.stream_ptr(s)
    st = _lib.load().kvf_rc_decode_fed(
        C.c_void_p(h_rc.data_ptr()), len(rc), C.c_void_p(h_segs.data_ptr()),
        C.c_void_p(h_of.data_ptr()), len(segs), _FED_PIECE, int(segs["len"].max(initial=0)),
        C.c_void_p(ready.data_ptr()), _FED_COPY_CTAS, sp)
    if st == _lib.KVF_EUNSUPPORTED:
        return None
    _lib.check(st)
    part = list(range(len(datas)))
    spans = [(0, int(d.numel())) for d in datas]
    starts = np.zeros(len(datas) + 1, np.int64)
    _, flat, ch_arr = _part_descriptors(part, idxs, ranges, starts, spans, 0,
                                        symbols.data_ptr() + sym_at, frames,
                                        seg_map=(lo_a, dst_a))
    h_planes, h_chains = _pinned_copy(flat), _pinned_copy(ch_arr)
    if len(ch_arr):
        _lib.call("kvf_kvfc_reconstruct", C.c_void_p(h_planes.data_ptr()),
                  C.c_void_p(h_chains.data_ptr()), len(ch_arr), sp)
    _hold_until(s, [h_rc, h_planes, h_chains, h_segs, h_of])
    held = blob.numel() + symbols.numel() + sum(f.numel() for f in frames)
    for t in (blob, symbols, ready, *frames):
        t.record_stream(s)
    return frames, held


def _enqueue_copies(s, parts, datas, spans, starts, blob, host):
    """Queue each part's H2D copies on its side stream (after the work `s` has
    so far); returns the side streams (just [s] for a single part)."""
    side = _side_streams(s, len(parts)) if len(parts) > 1 else [s]
    for t in side:
        if t is not s:
            t.wait_stream(s)
    for p, part in enumerate(parts):
        with torch.cuda.stream(side[p]):
            for j in part:
                lo, hi = spans[j]
                if hi <= lo:
                    continue
                s0 = int(starts[j])
                src = datas[j][lo:hi] if host is None else host[s0:s0 + hi - lo]
                blob[s0:s0 + hi - lo].copy_(src, non_blocking=True)
    return side


_SCRATCH = collections.OrderedDict()   # (device, stream, name) -> grow-only device buffer
_SCRATCH_STREAMS = 8
_SCRATCH_LOCK = threading.Lock()


def _scratch(stream, name, nbytes):
    """Device scratch of `nbytes` reused across calls on `stream`.

    Fresh cudaMallocs of varying sizes (a fetcher's batches differ) cost
    15-40 ms each while the GPU is busy; a grow-only buffer per stream does
    not.  Reuse is ordered: a call's kernels run on `stream` or on side
    streams that `stream` waits for before returning, and the next call's
    side streams wait for `stream` first.  Buffers of the least recently used
    streams beyond _SCRATCH_STREAMS are dropped (their tensors carry
    record_stream marks, so the allocator frees them safely).
    """
    key = (stream.device, stream.cuda_stream, name)
    with _SCRATCH_LOCK:
        t = _SCRATCH.get(key)
        if t is None or t.numel() < nbytes:
            _SCRATCH.pop(key, None)   # the old buffer goes first
            with torch.cuda.stream(stream):
                t = torch.empty(2 * nbytes + (1 << 20), dtype=torch.uint8,
                                device=stream.device)
            _SCRATCH[key] = t
        _SCRATCH.move_to_end(key)
        while len(_SCRATCH) > 2 * _SCRATCH_STREAMS:
            _SCRATCH.popitem(last=False)
    return t[:nbytes]


_HELD = []   # (event, pinned host tensors) read by kernels not yet known complete
_HELD_LOCK = threading.Lock()


def _pinned_copy(a):
    """A pinned host copy of numpy array `a` (at least one element), for a
    kernel to read in place."""
    a = np.ascontiguousarray(a if len(a) else np.zeros(1, a.dtype)).view(np.uint8)
    t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
    t.numpy()[:] = a
    return t


def _hold_until(stream, tensors):
    """Keep host tensors alive until `stream` passes this point (kernels on it
    read them); drops the entries whose work completed."""
    ev = torch.cuda.Event()
    ev.record(stream)
    with _HELD_LOCK:
        _HELD[:] = [(e, ts) for e, ts in _HELD if not e.query()]
        _HELD.append((ev, tensors))


def _part_descriptors(part, idxs, ranges, starts, spans, base, sym_ptr, frames, seg_map=None):
    """kvf_rc_stream / kvf_recon_plane / kvf_recon_chain arrays of the streams
    `part` (indices into idxs), vectorised over their planes.  Plane k = 3 f +
    p of stream j (frame-major), streams in order; `starts` are blob offsets
    of the copied spans, `sym_ptr[j]` the device symbol slots of stream j.
    `seg_map` = (lo, dst) per plane (fed decode): the plane's bytes from stream
    offset lo on sit at device address dst."""
    nl = len(part)
    nf = np.array([ranges[j][1] - ranges[j][0] for j in part], np.int64)
    hs = np.array([idxs[j].h for j in part], np.int64)
    ws = np.array([idxs[j].w for j in part], np.int64)
    hw = hs * ws
    hw16 = -(-hw // 16) * 16
    n_pl = 3 * nf
    K = int(n_pl.sum())
    sid = np.repeat(np.arange(nl), n_pl)             # ordinal in the part of each plane
    pl_at = np.concatenate([[0], np.cumsum(n_pl)])
    loc = np.arange(K, dtype=np.int64) - pl_at[sid]  # k - 3 f0

    def cat(name):
        return np.concatenate([getattr(idxs[j], name)[3 * ranges[j][0]:3 * ranges[j][1]]
                               for j in part])

    p_off, p_len, b_off = cat("payload_off"), cat("payload_len"), cat("bitmap_off")
    # the copied span of stream j starts at its lowest header offset
    sbase = base + np.array([int(starts[j]) - spans[j][0] for j in part], np.int64)
    out_ptr = np.array([frames[j].data_ptr() for j in part], np.int64)
    st = np.array([frames[j].stride()[:3] for j in part], np.int64).reshape(nl, 3)
    rc = np.empty(K, _RC_DTYPE)
    if seg_map is not None:
        lo, dst = seg_map
        rc["payload"] = dst + (p_off - lo)
    else:
        rc["payload"] = sbase[sid] + p_off
    rc["len"] = p_len
    rc["symbols"] = np.asarray(sym_ptr)[part][sid] + loc * hw16[sid]
    rc["n_symbols"] = hw[sid]
    fl, pp = loc // 3, loc % 3
    pl = np.empty(K, _PLANE_DTYPE)
    pl["symbols"] = rc["symbols"]
    if seg_map is not None:
        pl["modes"] = np.where(b_off >= 0, dst + (b_off - lo), 0)
    else:
        pl["modes"] = np.where(b_off >= 0, sbase[sid] + b_off, 0)
    pl["out"] = out_ptr[sid] + fl * st[sid, 0] + pp * st[sid, 1]
    pl["out_pitch"] = st[sid, 2]
    ftype = np.concatenate([idxs[j].frame_type[ranges[j][0]:ranges[j][1]] for j in part])
    dest, ch_first, ch_count, ch_sid = _chain_layout(ftype, nf, hw)
    flat = np.empty(K, _PLANE_DTYPE)
    flat[dest] = pl
    ch_arr = np.empty(len(ch_first), _CHAIN_DTYPE)
    ch_arr["first"], ch_arr["count"] = ch_first, ch_count
    ch_arr["height"], ch_arr["width"] = hs[ch_sid], ws[ch_sid]
    return rc, flat, ch_arr


def _chain_layout(ftype, nf, hw):
    """Reconstruction order of the planes of concatenated frame ranges.

    ``ftype``: frame types of every decoded frame, stream after stream (each
    range starts with an intra frame); ``nf``: frames per stream; ``hw``:
    samples per plane per stream.  Planes are numbered frame-major (k = 3 f +
    p over the concatenated frames).  A chain is one plane index over a
    segment (an intra frame and the inter frames after it), in frame order:
    segment g of n frames starting at global frame a owns slots [3a, 3a + 3n),
    plane index p's chain at 3a + p n.  Returns (dest slot of each plane,
    chain first slots, chain lengths, stream ordinal of each chain); chains of
    empty planes (hw == 0) are dropped.
    """
    ftype = np.asarray(ftype)
    nf = np.asarray(nf, np.int64)
    n_frames = len(ftype)
    seg_a = np.flatnonzero(ftype == 0)
    seg_n = np.diff(np.r_[seg_a, n_frames]).astype(np.int64)
    g = np.repeat(np.cumsum(ftype == 0) - 1, 3)          # segment of each plane
    fg = np.repeat(np.arange(n_frames, dtype=np.int64), 3)
    pp = np.tile(np.arange(3, dtype=np.int64), n_frames)
    dest = 3 * seg_a[g] + pp * seg_n[g] + (fg - seg_a[g]) if n_frames else np.zeros(0, np.int64)
    ch_g = np.repeat(np.arange(len(seg_a)), 3)
    first = 3 * seg_a[ch_g] + np.tile(np.arange(3), len(seg_a)) * seg_n[ch_g]
    count = seg_n[ch_g]
    fr_at = np.concatenate([[0], np.cumsum(nf)])
    ch_sid = np.searchsorted(fr_at, seg_a[ch_g], side="right") - 1
    if len(ch_sid) and (np.asarray(hw)[ch_sid] == 0).any():
        keep = np.asarray(hw)[ch_sid] > 0
        first, count, ch_sid = first[keep], count[keep], ch_sid[keep]
    return dest, first, count, ch_sid


_PART_BYTES = 32 << 20   # coded bytes per decode part (H2D / decode overlap)
_MAX_PARTS = 8
_SIDE = {}


def _split_parts(idx, sizes, max_parts=None):
    """Consecutive groups of `idx` with about equal bytes: one group below
    _PART_BYTES, else up to `max_parts` (default _MAX_PARTS)."""
    total = sum(sizes)
    n = min(max_parts or _MAX_PARTS, len(idx), max(1, total // _PART_BYTES))
    if n <= 1:
        return [list(idx)]
    parts, cur, acc, target = [], [], 0, total / n
    for j, b in zip(idx, sizes):
        cur.append(j)
        acc += b
        if acc >= target * (len(parts) + 1) and len(parts) < n - 1:
            parts.append(cur)
            cur = []
    if cur:
        parts.append(cur)
    return parts


def _side_streams(stream, n):
    """Side streams of the calling stream (each caller stream has its own, so
    decodes issued concurrently on different streams do not serialise on a
    shared pool).  Least recently used entries beyond _SCRATCH_STREAMS go."""
    key = (stream.device, stream.cuda_stream)
    with _SCRATCH_LOCK:
        pool = _SIDE.pop(key, [])
        _SIDE[key] = pool
        while len(pool) < n:
            pool.append(torch.cuda.Stream(device=stream.device))
        while len(_SIDE) > _SCRATCH_STREAMS:
            _SIDE.pop(next(iter(_SIDE)))
        return pool[:n]


def decode_stream_framewise(bs, on_frame, stream=None, index=None) -> int:
    """Decode one KVFC stream frame by frame on the GPU (fk/codec.py:155-211).

    Per frame: one range-decode launch for its three plane streams and one
    reconstruction launch whose chains are [previous frame's plane (reference
    only), this frame's plane], so only the current and the previous frame are
    held, as in the reference decoder.  ``on_frame(f, frame)`` gets a [3, h, w]
    uint8 CUDA view of a buffer that frame f + 2 reuses: work it queues on the
    decode stream (``stream``, default current) is ordered before that reuse; a
    callback that keeps the frame must clone it.  All descriptors are built up
    front (vectorised) and read in place from pinned host memory.  Returns the
    frame count; raises DecodeError like the reference.
    """
    data = bs if isinstance(bs, torch.Tensor) else _as_bytes(bs)
    ix = index if index is not None else StreamIndex(data)
    n, h, w = ix.n, ix.h, ix.w
    if n == 0:
        return 0
    s = stream if stream is not None else torch.cuda.current_stream()
    dev = _dev.device()
    hw = h * w
    hw16 = -(-hw // 16) * 16
    with torch.cuda.stream(s):
        # the coded bytes travel once; frames are decoded into two buffers
        host = torch.frombuffer(bytearray(data), dtype=torch.uint8) if not isinstance(
            data, torch.Tensor) else data
        blob = torch.empty(max(host.numel(), 1), dtype=torch.uint8, device=dev)
        blob[:host.numel()].copy_(host.pin_memory() if not host.is_pinned() else host,
                                  non_blocking=True)
        symbols = torch.empty(max(3 * hw16, 16), dtype=torch.uint8, device=dev)
        bufs = torch.empty((2, 3, h, w), dtype=torch.uint8, device=dev)
    k = np.arange(3 * n, dtype=np.int64)
    f, p = k // 3, k % 3
    base = blob.data_ptr()
    rc = np.empty(3 * n, _RC_DTYPE)
    rc["payload"] = base + ix.payload_off
    rc["len"] = ix.payload_len
    rc["symbols"] = symbols.data_ptr() + p * hw16
    rc["n_symbols"] = hw
    # planes [n, 3, 2]: (reference entry, this frame's entry) per plane
    fb = bufs.data_ptr() + p * hw
    pl = np.zeros((3 * n, 2), _PLANE_DTYPE)
    pl["out_pitch"] = w
    pl["out"][:, 0] = fb + ((f + 1) % 2) * 3 * hw            # previous frame's buffer
    pl["symbols"][:, 1] = rc["symbols"]
    pl["modes"][:, 1] = np.where(ix.bitmap_off >= 0, base + ix.bitmap_off, 0)
    pl["out"][:, 1] = fb + (f % 2) * 3 * hw
    inter = ix.frame_type[f] != 0
    ch = np.empty(3 * n, _CHAIN_DTYPE)
    ch["first"] = 2 * k + np.where(inter, 0, 1)
    ch["count"] = np.where(inter, 2, 1)
    ch["height"], ch["width"] = h, w
    h_rc, h_pl, h_ch = (_pinned_copy(x.reshape(-1)) for x in (rc, pl, ch))
    rc_sz, ch_sz = _RC_DTYPE.itemsize, _CHAIN_DTYPE.itemsize
    sp = _dev.stream_ptr(s)
    try:
        for fi in range(n):
            if hw:
                _lib.call("kvf_rc_decode", C.c_void_p(h_rc.data_ptr() + 3 * fi * rc_sz), 3, sp)
                _lib.call("kvf_kvfc_reconstruct", C.c_void_p(h_pl.data_ptr()),
                          C.c_void_p(h_ch.data_ptr() + 3 * fi * ch_sz), 3, sp)
            with torch.cuda.stream(s):
                on_frame(fi, bufs[fi % 2])
    finally:
        _hold_until(s, [h_rc, h_pl, h_ch])
        for t in (blob, symbols, bufs):
            t.record_stream(s)
    return n


def decode_frames(bs, cfg: CodecConfig, on_frame, stats=None):
    """Decode a Bitstream (or raw bytes) on the GPU frame by frame, calling
    on_frame(index, frame) (fk/codec.py:155-211).

    ``frame`` is a [3, h, w] uint8 CUDA view of a buffer reused two frames
    later (see decode_stream_framewise).  stats["peak_live_bytes"] is the
    reference's quantity: decoded-frame bytes retained, i.e. the current frame
    plus its reference (fk/codec.py:203-210).  For many streams at once use
    decode_batch.
    """
    n = decode_stream_framewise(bs, on_frame)
    if stats is not None:
        ix_h, ix_w = header(bs)[1:]
        stats["peak_live_bytes"] = min(n, 2) * 3 * ix_h * ix_w
    return n


def _to_dev_struct(arr: np.ndarray, dev) -> torch.Tensor:
    """numpy structured array -> device bytes (pinned, asynchronous)."""
    return torch.from_numpy(arr.view(np.uint8)).pin_memory().to(dev, non_blocking=True)


def encode_batch(frame_sets, gops, stream=None):
    """Encode many [n, 3, h, w] uint8 frame tensors on the GPU (fk/codec.py:93-128).

    Returns a list of Bitstream.  Launches: residual/mode kernel, range
    encoder (one thread per (frame, plane) stream), one D2H of the coded
    lengths and modes, the gather kernel, one D2H of all streams.  Host work
    (descriptors, stream layout fk/codec.py:16-20, header fields) is
    vectorised over planes.
    """
    dev = _dev.device()
    sets = [_dev.to_device(f, torch.uint8) for f in frame_sets]
    for f in sets:
        if f.dim() != 4 or f.shape[1] != 3:
            raise ValueError("frames must be [n, 3, height, width]")
    s = stream if stream is not None else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        sets = [f if f.stride(3) == 1 and f.stride(2) == f.shape[3] else f.contiguous() for f in sets]
        geo, n_planes, sym_total, mode_total = [], 0, 0, 0
        for f in sets:
            n, _, h, w = f.shape
            bh, bw = -(-h // BLOCK), -(-w // BLOCK)
            hw4 = -(-h * w // 4) * 4
            geo.append((n, h, w, bh, bw, hw4, sym_total, mode_total, n_planes))
            n_planes += 3 * n
            sym_total += 3 * n * hw4
            mode_total += 3 * n * bh * bw
        symbols = torch.empty(max(sym_total, 1), dtype=torch.uint8, device=dev)
        modes = torch.zeros(max(mode_total, 1), dtype=torch.uint8, device=dev)
        rp = np.zeros(max(n_planes, 1), _RESID_DTYPE)
        rc = np.zeros(max(n_planes, 1), _RC_DTYPE)
        caps, max_blocks = [], 0
        for f, gop, (n, h, w, bh, bw, hw4, s0, m0, k0) in zip(sets, gops, geo):
            max_blocks = max(max_blocks, bh * bw)
            k = np.arange(3 * n, dtype=np.int64)
            fi, p = k // 3, k % 3
            sl = slice(k0, k0 + 3 * n)
            rp["cur"][sl] = f.data_ptr() + fi * f.stride(0) + p * f.stride(1)
            rp["prev"][sl] = np.where(fi % gop != 0, f.data_ptr() + (fi - 1) * f.stride(0)
                                      + p * f.stride(1), 0)
            rp["pitch"][sl] = f.stride(2)
            rp["symbols"][sl] = symbols.data_ptr() + s0 + k * hw4
            rp["modes"][sl] = modes.data_ptr() + m0 + k * bh * bw
            rp["height"][sl], rp["width"][sl] = h, w
            rc["symbols"][sl] = rp["symbols"][sl]
            rc["n_symbols"][sl] = h * w
            caps.append(np.full(3 * n, 2 * h * w + 16, np.int64))
        cap = np.concatenate(caps) if caps else np.zeros(0, np.int64)
        cap_off = np.concatenate([[0], np.cumsum(cap)]).astype(np.int64)
        payload = torch.empty(max(int(cap_off[-1]), 1), dtype=torch.uint8, device=dev)
        out_len = torch.zeros(max(n_planes, 1), dtype=torch.int64, device=dev)
        rc["payload"][:n_planes] = payload.data_ptr() + cap_off[:-1]
        sp = _dev.stream_ptr(s)
        _lib.call("kvf_kvfc_residuals", _dev.ptr(_to_dev_struct(rp, dev)), n_planes, max_blocks, sp)
        _lib.call("kvf_rc_encode", _dev.ptr(_to_dev_struct(rc, dev)), n_planes, _dev.ptr(out_len), sp)
        lens = out_len.cpu().numpy()[:n_planes]
        modes_h = modes.cpu().numpy()
        # stream layout (fk/codec.py:16-20): header | per frame: type, per plane:
        # [inter: packed modes] u32 len, payload — positions by cumulative sums
        layouts, piece_parts, total = [], [], 0
        for gop, (n, h, w, bh, bw, hw4, s0, m0, k0) in zip(gops, geo):
            blen = (bh * bw + 7) // 8
            k = np.arange(3 * n, dtype=np.int64)
            fi, p = k // 3, k % 3
            inter = (fi % gop) != 0
            ln = lens[k0:k0 + 3 * n]
            plane_bytes = np.where(inter, blen, 0) + 4 + ln          # per (frame, plane)
            frame_bytes = 1 + plane_bytes.reshape(n, 3).sum(axis=1) if n else np.zeros(0, np.int64)
            frame_off = 12 + np.concatenate([[0], np.cumsum(frame_bytes)[:-1]]).astype(np.int64)
            within = np.concatenate([np.zeros((n, 1), np.int64),
                                     np.cumsum(plane_bytes.reshape(n, 3), axis=1)[:, :2]],
                                    axis=1).reshape(-1) if n else np.zeros(0, np.int64)
            plane_off = frame_off[fi] + 1 + within                    # start of plane field
            len_off = plane_off + np.where(inter, blen, 0)           # u32 length field
            size = int(12 + frame_bytes.sum())
            # gather pieces: payloads, and mode bitmaps of inter planes (packbits)
            pay = np.zeros(3 * n, _PIECE_DTYPE)
            pay["src"] = payload.data_ptr() + cap_off[k0:k0 + 3 * n]
            pay["dst_off"] = total + len_off + 4
            pay["len"] = ln
            bm = np.zeros(int(inter.sum()), _PIECE_DTYPE)
            bm["src"] = modes.data_ptr() + m0 + k[inter] * bh * bw
            bm["dst_off"] = total + plane_off[inter]
            bm["len"] = bh * bw
            bm["pack_bits"] = 1
            piece_parts += [pay, bm]
            mv = modes_h[m0:m0 + 3 * n * bh * bw].reshape(n, 3, bh * bw) if n else None
            inter_frac = ([0.0 if f % gop == 0 else float(mv[f].mean()) for f in range(n)]
                          if n else [])
            layouts.append((total, size, n, h, w, frame_off, inter, len_off, ln, inter_frac))
            total += size
        blob = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
        pieces = np.concatenate(piece_parts) if piece_parts else np.zeros(1, _PIECE_DTYPE)
        _lib.call("kvf_gather", _dev.ptr(_to_dev_struct(pieces, dev)), len(pieces) if piece_parts else 0,
                  _dev.ptr(blob), sp)
        # one D2H into a reused pinned buffer (a fresh pageable one page-faults
        # through the copy: ~2 GB/s), then one copy out per stream
        out = _OUT_STAGING.acquire(max(total, 1))
        try:
            out.copy_(blob[:max(total, 1)], non_blocking=True)
            s.synchronize()
            return [_finish_stream(out.numpy(), *lay) for lay in layouts]
        finally:
            _OUT_STAGING.release(s)


def _finish_stream(host, base, size, n, h, w, frame_off, inter, len_off, ln, inter_frac):
    """Header fields of one encoded stream written in place, one copy out."""
    buf = host[base:base + size]
    buf[:12] = np.array([n, h, w], "<u4").view(np.uint8)
    buf[frame_off] = inter.reshape(n, 3)[:, 0].astype(np.uint8) if n else buf[frame_off]
    lb = ln.astype("<u4").view(np.uint8).reshape(-1, 4)
    for b in range(4):
        buf[len_off + b] = lb[:, b]
    return Bitstream(buf.tobytes(), n, h, w, [int(x) for x in frame_off], inter_frac)


def encode_frames(frames, cfg: CodecConfig) -> Bitstream:
    """GPU encode of one [n, 3, h, w] frame sequence; bit-identical stream."""
    return encode_batch([frames], [cfg.gop])[0]


def header(data) -> tuple[int, int, int]:
    d = _as_bytes(data)
    if len(d) < 12:
        raise DecodeError("stream shorter than header", frame_index=0)
    return struct.unpack_from("<III", d, 0)
