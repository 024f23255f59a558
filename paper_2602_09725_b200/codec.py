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

import numpy as np
import torch

from . import _dev, _lib

BLOCK = 16


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


class StreamIndex:
    """Layout of one KVFC stream (host arrays from kvf_kvfc_scan)."""

    def __init__(self, data: bytes):
        lib = _lib.load()
        info = _lib.kvf_kvfc_info()
        bad = C.c_int32(0)
        buf = C.c_char_p(data) if data else None
        st = lib.kvf_kvfc_scan(buf, len(data), C.byref(info), None, None, None, None, 0,
                               C.byref(bad))
        if st == _lib.KVF_EDECODE:
            raise DecodeError(lib.kvf_last_error().decode(), frame_index=bad.value)
        n = info.n_frames
        self.n, self.h, self.w, self.bitmap_len = n, info.height, info.width, info.bitmap_len
        self.payload_off = np.zeros(3 * n, np.int64)
        self.payload_len = np.zeros(3 * n, np.int32)
        self.bitmap_off = np.zeros(3 * n, np.int64)
        self.frame_type = np.zeros(max(n, 1), np.uint8)
        st = lib.kvf_kvfc_scan(buf, len(data), C.byref(info),
                               self.payload_off.ctypes.data, self.payload_len.ctypes.data,
                               self.bitmap_off.ctypes.data, self.frame_type.ctypes.data, n,
                               C.byref(bad))
        if st == _lib.KVF_EDECODE:
            raise DecodeError(lib.kvf_last_error().decode(), frame_index=bad.value)
        _lib.check(st)


def _to_device_struct_array(arr, device) -> torch.Tensor:
    raw = np.frombuffer(bytes(arr), np.uint8) if C.sizeof(arr) else np.zeros(1, np.uint8)
    return torch.from_numpy(raw.copy()).to(device)


def decode_batch(streams, out=None, stream=None, ranges=None, indices=None):
    """Decode many KVFC streams on the GPU in one pair of launches.

    ``streams``: list of bytes / Bitstream.  ``out``: optional list of
    [n, 3, h, w] uint8 CUDA tensors (any row pitch) to decode into.
    ``ranges``: optional per-stream (first, stop) frame range; ``first`` must
    be an intra frame (a chain start), and the output holds stop-first frames.
    Returns (frames list, device bytes held).  Raises DecodeError like the
    reference.
    """
    dev = _dev.device()
    datas = [_as_bytes(s) for s in streams]
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
    host = torch.empty(int(starts[-1]) or 1, dtype=torch.uint8, pin_memory=True)
    hv = host.numpy()
    for d, s0, (lo, hi) in zip(datas, starts[:-1], spans):
        hv[s0:s0 + hi - lo] = np.frombuffer(d, np.uint8, hi - lo, lo)
    # shift so that stream offsets index the copied span
    starts = starts - np.array([lo for lo, _ in spans] + [0])
    s = stream if stream is not None else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        blob = host.to(dev, non_blocking=True)
        frames = []
        n_fr = [f1 - f0 for f0, f1 in ranges]
        n_sym = sum(3 * nf * ix.h * ix.w for nf, ix in zip(n_fr, idxs))
        symbols = torch.empty(max(n_sym, 1), dtype=torch.uint8, device=dev)
        rc = (_lib.kvf_rc_stream * max(1, 3 * sum(n_fr)))()
        planes = (_lib.kvf_recon_plane * max(1, 3 * sum(n_fr)))()
        chains = []
        k_rc = 0
        sym_at = 0
        base = blob.data_ptr()
        sym_base = symbols.data_ptr()
        for j, (ix, (f0, f1)) in enumerate(zip(idxs, ranges)):
            nf = f1 - f0
            fr = out[j] if out is not None else torch.empty((nf, 3, ix.h, ix.w),
                                                           dtype=torch.uint8, device=dev)
            if tuple(fr.shape) != (nf, 3, ix.h, ix.w):
                raise ValueError("output frames have the wrong shape")
            frames.append(fr)
            hw = ix.h * ix.w
            plane_at = k_rc
            for f in range(f0, f1):
                for p in range(3):
                    k = 3 * f + p
                    e = rc[k_rc]
                    e.payload = base + int(starts[j] + ix.payload_off[k])
                    e.len = int(ix.payload_len[k])
                    e.symbols = sym_base + sym_at
                    e.n_symbols = hw
                    q = planes[k_rc]
                    q.symbols = sym_base + sym_at
                    q.modes = (base + int(starts[j] + ix.bitmap_off[k])) if ix.bitmap_off[k] >= 0 else None
                    q.out = fr[f - f0, p].data_ptr()
                    q.out_pitch = fr.stride(2)
                    sym_at += hw
                    k_rc += 1
            if hw == 0:
                continue
            # chains: runs of frames starting at each intra frame, per plane
            f = f0
            while f < f1:
                g = f + 1
                while g < f1 and ix.frame_type[g] == 1:
                    g += 1
                for p in range(3):
                    # entries of plane p for frames f..g-1 are strided by 3
                    chains.append((plane_at, f - f0, g - f0, p, ix.h, ix.w))
                f = g
        # re-pack planes so each chain's entries are contiguous
        flat = (_lib.kvf_recon_plane * max(1, k_rc))()
        ch_arr = (_lib.kvf_recon_chain * max(1, len(chains)))()
        at = 0
        for c, (plane_at, f, g, p, h, w) in enumerate(chains):
            ch_arr[c].first = at
            ch_arr[c].count = g - f
            ch_arr[c].height = h
            ch_arr[c].width = w
            for ff in range(f, g):
                flat[at] = planes[plane_at + 3 * ff + p]
                at += 1
        d_rc = _to_device_struct_array(rc, dev)
        d_planes = _to_device_struct_array(flat, dev)
        d_chains = _to_device_struct_array(ch_arr, dev)
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
