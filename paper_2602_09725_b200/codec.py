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
assert _RC_DTYPE.itemsize == C.sizeof(_lib.kvf_rc_stream)
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


def _to_device_struct_array(arr, device) -> torch.Tensor:
    raw = np.frombuffer(bytes(arr), np.uint8) if C.sizeof(arr) else np.zeros(1, np.uint8)
    return torch.from_numpy(raw.copy()).to(device)


def decode_batch(streams, out=None, stream=None, ranges=None, indices=None):
    """Decode many KVFC streams on the GPU in one pair of launches.

    ``streams``: list of bytes / Bitstream (staged through a reused pinned
    buffer), or of contiguous CPU uint8 tensors — pinned receive buffers —
    which are copied to the device directly.  ``out``: optional list of
    [n, 3, h, w] uint8 CUDA tensors (any row pitch) to decode into.
    ``ranges``: optional per-stream (first, stop) frame range; ``first`` must
    be an intra frame (a chain start), and the output holds stop-first frames.
    Returns (frames list, device bytes held).  Raises DecodeError like the
    reference.
    """
    dev = _dev.device()
    pinned_in = all(isinstance(x, torch.Tensor) for x in streams) and len(streams) > 0
    datas = list(streams) if pinned_in else [_as_bytes(x) for x in streams]
    idxs = indices if indices is not None else [StreamIndex(d) for d in datas]
    if ranges is None:
        ranges = [(0, ix.n) for ix in idxs]
    for ix, (f0, f1) in zip(idxs, ranges):
        if not 0 <= f0 <= f1 <= ix.n:
            raise ValueError("frame range outside the stream")
        if f0 < f1 and ix.frame_type[f0] != 0:
            raise ValueError("a partial decode must start at an intra frame")
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
    s = stream if stream is not None else torch.cuda.current_stream()
    if pinned_in:  # receive buffers already in (pinned) host memory: H2D each span
        with torch.cuda.stream(s):
            blob = torch.empty(int(starts[-1]) or 1, dtype=torch.uint8, device=dev)
            for d, s0, (lo, hi) in zip(datas, starts[:-1], spans):
                if hi > lo:
                    blob[s0:s0 + hi - lo].copy_(d[lo:hi], non_blocking=True)
    else:
        host = _STAGING.acquire(int(starts[-1]) or 1)
        hv = host.numpy()
        for d, s0, (lo, hi) in zip(datas, starts[:-1], spans):
            hv[s0:s0 + hi - lo] = np.frombuffer(d, np.uint8, hi - lo, lo)
        with torch.cuda.stream(s):
            blob = host.to(dev, non_blocking=True)
            _STAGING.release(s)
    # shift so that stream offsets index the copied span
    starts = starts - np.array([lo for lo, _ in spans] + [0])
    with torch.cuda.stream(s):
        frames = []
        n_fr = [f1 - f0 for f0, f1 in ranges]
        n_sym = sum(3 * nf * (-(-ix.h * ix.w // 4) * 4) for nf, ix in zip(n_fr, idxs))
        symbols = torch.empty(max(n_sym, 1), dtype=torch.uint8, device=dev)
        base = blob.data_ptr()
        sym_base = symbols.data_ptr()
        rc_parts, plane_parts, chain_parts = [], [], []
        sym_at = 0
        n_planes = 0
        for j, (ix, (f0, f1)) in enumerate(zip(idxs, ranges)):
            nf = f1 - f0
            fr = out[j] if out is not None else torch.empty((nf, 3, ix.h, ix.w),
                                                           dtype=torch.uint8, device=dev)
            if tuple(fr.shape) != (nf, 3, ix.h, ix.w):
                raise ValueError("output frames have the wrong shape")
            frames.append(fr)
            if nf == 0:
                continue
            hw = ix.h * ix.w
            hw4 = -(-hw // 4) * 4                          # 4-byte aligned symbol slots
            ks = np.arange(3 * f0, 3 * f1)                 # stream k = 3 f + p, frame-major
            loc = ks - 3 * f0
            stream_base = base + int(starts[j])
            rc = np.empty(len(ks), _RC_DTYPE)
            rc["payload"] = stream_base + ix.payload_off[ks]
            rc["len"] = ix.payload_len[ks]
            rc["symbols"] = sym_base + sym_at + loc * hw4
            rc["n_symbols"] = hw
            pl = np.empty(len(ks), _PLANE_DTYPE)
            pl["symbols"] = rc["symbols"]
            pl["modes"] = np.where(ix.bitmap_off[ks] >= 0, stream_base + ix.bitmap_off[ks], 0)
            pl["out"] = fr.data_ptr() + (loc // 3) * fr.stride(0) + (loc % 3) * fr.stride(1)
            pl["out_pitch"] = fr.stride(2)
            rc_parts.append(rc)
            sym_at += len(ks) * hw4
            if hw:
                # chains: per plane, the frames from each intra frame to the next
                # one (a reconstruction dependency chain), contiguous in `flat`
                f = ks // 3
                seg = np.cumsum(ix.frame_type[f0:f1] == 0)[f - f0]
                order = np.lexsort((f, ks % 3, seg))
                plane_parts.append(pl[order])
                key = seg[order] * 3 + (ks % 3)[order]
                first = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
                ch = np.empty(len(first), _CHAIN_DTYPE)
                ch["first"] = n_planes + first
                ch["count"] = np.diff(np.r_[first, len(order)])
                ch["height"], ch["width"] = ix.h, ix.w
                chain_parts.append(ch)
                n_planes += len(order)
        rc = np.concatenate(rc_parts) if rc_parts else np.zeros(1, _RC_DTYPE)
        flat = np.concatenate(plane_parts) if plane_parts else np.zeros(1, _PLANE_DTYPE)
        ch_arr = np.concatenate(chain_parts) if chain_parts else np.zeros(1, _CHAIN_DTYPE)
        k_rc = sum(len(x) for x in rc_parts)
        chains = ch_arr if chain_parts else []
        # descriptor arrays via pinned memory: asynchronous, never a host sync
        d_rc, d_planes, d_chains = (
            torch.from_numpy(a.view(np.uint8)).pin_memory().to(dev, non_blocking=True)
            for a in (rc, flat, ch_arr))
        sp = _dev.stream_ptr(s)
        _lib.call("kvf_rc_decode", _dev.ptr(d_rc), k_rc, sp)
        _lib.call("kvf_kvfc_reconstruct", _dev.ptr(d_planes), _dev.ptr(d_chains), len(chains), sp)
    held = blob.numel() + symbols.numel() + sum(f.numel() for f in frames)
    # keep descriptor/scratch tensors alive until the stream reaches this point
    frames_keepalive = (blob, symbols, d_rc, d_planes, d_chains)
    for t in frames_keepalive:
        t.record_stream(s)
    return frames, held


def decode_frames(bs, cfg: CodecConfig, on_frame, stats=None):
    """Decode a Bitstream (or raw bytes) on the GPU, calling on_frame(index, frame).

    ``frame`` is a [3, h, w] uint8 CUDA tensor view.  stats["peak_live_bytes"]
    reports the device bytes held by the decode (stream, symbols, frames).
    """
    frames, held = decode_batch([bs])
    fr = frames[0]
    for f in range(fr.shape[0]):
        on_frame(f, fr[f])
    if stats is not None:
        stats["peak_live_bytes"] = held
    return fr.shape[0]


def encode_batch(frame_sets, gops, stream=None):
    """Encode many [n, 3, h, w] uint8 frame tensors on the GPU (fk/codec.py:93-128).

    Returns a list of Bitstream.  Launches: residual/mode kernel, range
    encoder (one thread per (frame, plane) stream), one D2H of the coded
    lengths, the gather kernel, one D2H of all streams.
    """
    dev = _dev.device()
    sets = [_dev.to_device(f, torch.uint8) for f in frame_sets]
    for f in sets:
        if f.dim() != 4 or f.shape[1] != 3:
            raise ValueError("frames must be [n, 3, height, width]")
    s = stream if stream is not None else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        sets = [f if f.stride(3) == 1 and f.stride(2) == f.shape[3] else f.contiguous() for f in sets]
        geo = []
        n_planes = 0
        sym_total = 0
        mode_total = 0
        for f in sets:
            n, _, h, w = f.shape
            bh, bw = -(-h // BLOCK), -(-w // BLOCK)
            geo.append((n, h, w, bh, bw, sym_total, mode_total, n_planes))
            n_planes += 3 * n
            sym_total += 3 * n * h * w
            mode_total += 3 * n * bh * bw
        symbols = torch.empty(max(sym_total, 1), dtype=torch.uint8, device=dev)
        modes = torch.zeros(max(mode_total, 1), dtype=torch.uint8, device=dev)
        cap = [2 * h * w + 16 for (n, h, w, *_r) in geo for _ in range(3 * n)]
        cap_off = np.concatenate([[0], np.cumsum(cap)]).astype(np.int64) if cap else np.zeros(1, np.int64)
        payload = torch.empty(max(int(cap_off[-1]), 1), dtype=torch.uint8, device=dev)
        out_len = torch.zeros(max(n_planes, 1), dtype=torch.int64, device=dev)
        rp = (_lib.kvf_resid_plane * max(1, n_planes))()
        rc = (_lib.kvf_rc_stream * max(1, n_planes))()
        max_blocks = 0
        for f, gop, (n, h, w, bh, bw, s0, m0, k0) in zip(sets, gops, geo):
            max_blocks = max(max_blocks, bh * bw)
            for fi in range(n):
                for p in range(3):
                    k = k0 + 3 * fi + p
                    q = rp[k]
                    q.cur = f[fi, p].data_ptr()
                    q.prev = f[fi - 1, p].data_ptr() if fi % gop else None
                    q.pitch = f.stride(2)
                    q.symbols = symbols.data_ptr() + s0 + (3 * fi + p) * h * w
                    q.modes = modes.data_ptr() + m0 + (3 * fi + p) * bh * bw
                    q.height, q.width = h, w
                    e = rc[k]
                    e.payload = payload.data_ptr() + int(cap_off[k])
                    e.symbols = q.symbols
                    e.n_symbols = h * w
        d_rp = _to_device_struct_array(rp, dev)
        d_rc = _to_device_struct_array(rc, dev)
        sp = _dev.stream_ptr(s)
        _lib.call("kvf_kvfc_residuals", _dev.ptr(d_rp), n_planes, max_blocks, sp)
        _lib.call("kvf_rc_encode", _dev.ptr(d_rc), n_planes, _dev.ptr(out_len), sp)
        lens = out_len.cpu().numpy()
        modes_h = modes.cpu().numpy()
        # stream layout (fk/codec.py:16-20) and the pieces to gather
        results, pieces, total = [], [], 0
        layouts = []
        for gop, (n, h, w, bh, bw, s0, m0, k0) in zip(gops, geo):
            blen = (bh * bw + 7) // 8
            pos = 12
            frame_offsets, inter_frac, fields = [], [], []
            for fi in range(n):
                frame_offsets.append(pos)
                is_inter = fi % gop != 0
                fields.append((pos, 1 if is_inter else 0, None))
                pos += 1
                fracs = []
                for p in range(3):
                    k = k0 + 3 * fi + p
                    if is_inter:
                        mo = m0 + (3 * fi + p) * bh * bw
                        pieces.append((modes.data_ptr() + mo, total + pos, bh * bw, 1))
                        fracs.append(float(modes_h[mo:mo + bh * bw].mean()))
                        pos += blen
                    fields.append((pos, None, int(lens[k])))
                    pos += 4
                    pieces.append((payload.data_ptr() + int(cap_off[k]), total + pos, int(lens[k]), 0))
                    pos += int(lens[k])
                inter_frac.append(float(np.mean(fracs)) if fracs else 0.0)
            layouts.append((total, pos, n, h, w, frame_offsets, inter_frac, fields))
            total += pos
        blob = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
        pc = (_lib.kvf_piece * max(1, len(pieces)))()
        for j, (src, off, ln, pb) in enumerate(pieces):
            pc[j].src, pc[j].dst_off, pc[j].len, pc[j].pack_bits = src, off, ln, pb
        d_pc = _to_device_struct_array(pc, dev)
        _lib.call("kvf_gather", _dev.ptr(d_pc), len(pieces), _dev.ptr(blob), sp)
        host = blob.cpu().numpy()
    for (base, size, n, h, w, frame_offsets, inter_frac, fields) in layouts:
        buf = bytearray(host[base:base + size].tobytes())
        struct.pack_into("<III", buf, 0, n, h, w)
        for pos, ftype, plen in fields:
            if ftype is not None:
                buf[pos] = ftype
            else:
                struct.pack_into("<I", buf, pos, plen)
        results.append(Bitstream(bytes(buf), n, h, w, frame_offsets, inter_frac))
    return results


def encode_frames(frames, cfg: CodecConfig) -> Bitstream:
    """GPU encode of one [n, 3, h, w] frame sequence; bit-identical stream."""
    return encode_batch([frames], [cfg.gop])[0]


def header(data) -> tuple[int, int, int]:
    d = _as_bytes(data)
    if len(d) < 12:
        raise DecodeError("stream shorter than header", frame_index=0)
    return struct.unpack_from("<III", d, 0)
