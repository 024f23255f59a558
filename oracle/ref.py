"""numpy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

Every function names the reference file:line it restates (fk/ = the reference
package's pkg/src/framekv/).  Arithmetic is kept identical: fp64 quantisation
math, numpy's round-half-to-even rint, int8 <-> u8 via +/-128.
"""

from __future__ import annotations

import base64
import ctypes
import hashlib
import json
import os
import struct
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

# ----------------------------------------------------------------- constants
RES_TILES = {"R240": 16, "R480": 64, "R640": 96, "R1080": 256}      # fk/layout.py:10
RES_GRIDS = {"R240": (4, 4), "R480": (8, 8), "R640": (8, 12), "R1080": (16, 16)}  # :11
RES_ORDER = ["R240", "R480", "R640", "R1080"]                          # :12
PAD = 128                                                              # fk/layout.py:231
BLOCK = 16                                                             # fk/codec.py:31


# ------------------------------------------------------------ tensor model
def gen_synthetic_kv(tokens, layers, H, D, token_smoothness, seed, channel_smoothness=0.0):
    """fk/kvmodel.py:155-192: AR(1) noise along dims (optional) then tokens."""
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal((tokens, layers, H, D))
    c = channel_smoothness
    if c > 0.0:
        for d in range(1, D):
            noise[..., d] = c * noise[..., d - 1] + (1.0 - c) * noise[..., d]
    s = token_smoothness
    out = np.empty_like(noise)
    out[0] = noise[0]
    for t in range(1, tokens):
        out[t] = s * out[t - 1] + (1.0 - s) * noise[t]
    return out.astype(np.float32)


def pad_layers(x):
    """fk/kvmodel.py:56-69: append zero layers up to a multiple of 3."""
    pad = (-x.shape[1]) % 3
    if not pad:
        return x.copy()
    z = np.zeros((x.shape[0], pad) + x.shape[2:], np.float32)
    return np.concatenate([x, z], axis=1)


def quantize(x, group_size=128):
    """fk/kvmodel.py:127-144 -> (int8 values [T,L,H,D], fp32 scales [L,G])."""
    T, L, H, D = x.shape
    G = H * D // group_size
    xg = x.reshape(T, L, G, group_size).astype(np.float64)
    m = np.abs(xg).max(axis=(0, 3))
    scales = np.where(m > 0, m / 127.0, 1.0).astype(np.float32)
    q = np.rint(xg / scales[None, :, :, None].astype(np.float64))
    np.clip(q, -127, 127, out=q)
    return q.astype(np.int8).reshape(x.shape), scales


def dequantize(values, scales, group_size):
    """fk/kvmodel.py:147-152: fp32(fp64(q) * fp64(scale))."""
    T, L, H, D = values.shape
    G = H * D // group_size
    q = values.reshape(T, L, G, group_size).astype(np.float64)
    return (q * scales[None, :, :, None].astype(np.float64)).reshape(values.shape).astype(np.float32)


# ---------------------------------------------------------------- layout
class Plan:
    """fk/layout.py:31-50 (tiling) + fk/layout.py:157-212 (placement)."""

    def __init__(self, T, res, H, D, a_h, b_h, a_d, b_d, F=4):
        if isinstance(res, str):
            self.tpf = RES_TILES[res]
            self.rows, self.cols = RES_GRIDS[res]
        else:
            self.tpf = int(res)
            r = int(self.tpf ** 0.5)
            while self.tpf % r:
                r -= 1
            self.rows, self.cols = r, self.tpf // r
        self.T, self.F = T, F
        self.H, self.D = H, D
        self.a_h, self.b_h, self.a_d, self.b_d = a_h, b_h, a_d, b_d
        self.th, self.tw = a_h * a_d, b_h * b_d
        self.fh, self.fw = self.rows * self.th, self.cols * self.tw
        full, rem = divmod(T, F * self.tpf)
        self.frame_count = full * F + (min(rem, F) if rem else 0)

    def placement(self, i):
        g, o = divmod(i, self.F)
        seg, slot = divmod(g, self.tpf)
        return seg * self.F + o, slot // self.cols, slot % self.cols

    def frame_slots(self, f):
        seg, o = divmod(f, self.F)
        out = []
        for slot in range(self.tpf):
            i = (seg * self.tpf + slot) * self.F + o
            if i < self.T:
                out.append((i, slot // self.cols, slot % self.cols))
        return out

    def tile(self, vec3):
        """fk/layout.py:123-134 apply_layout: [3, C] -> [3, th, tw]."""
        return (vec3.reshape(3, self.a_h, self.b_h, self.a_d, self.b_d)
                .transpose(0, 1, 3, 2, 4).reshape(3, self.th, self.tw))

    def untile(self, tile3):
        """fk/layout.py:137-147 inverse_layout: [3, th, tw] -> [3, C]."""
        return (tile3.reshape(3, self.a_h, self.a_d, self.b_h, self.b_d)
                .transpose(0, 1, 3, 2, 4).reshape(3, self.H * self.D))


def assemble_frames(tensors, plan: Plan):
    """fk/layout.py:234-258: [T,3,C] int8 -> [n,3,fh,fw] u8, pad 128."""
    T = tensors.shape[0]
    tiles = ((tensors.reshape(T, 3, plan.a_h, plan.b_h, plan.a_d, plan.b_d)
              .transpose(0, 1, 2, 4, 3, 5).reshape(T, 3, plan.th, plan.tw)
              .astype(np.int16) + 128).astype(np.uint8))
    frames = np.full((plan.frame_count, 3, plan.fh, plan.fw), PAD, np.uint8)
    for i in range(T):
        f, r, c = plan.placement(i)
        frames[f, :, r * plan.th:(r + 1) * plan.th, c * plan.tw:(c + 1) * plan.tw] = tiles[i]
    return frames


def disassemble_frames(frames, plan: Plan):
    """fk/layout.py:261-271: inverse of assemble_frames."""
    out = np.empty((plan.T, 3, plan.H * plan.D), np.int8)
    for f in range(plan.frame_count):
        for i, r, c in plan.frame_slots(f):
            t = frames[f, :, r * plan.th:(r + 1) * plan.th, c * plan.tw:(c + 1) * plan.tw]
            out[i] = plan.untile((t.astype(np.int16) - 128).astype(np.int8))
    return out


def restore_slots(frames, plan: Plan, layer_base=0, token_base=0, first_frame=0, n_frames=None):
    """fk/fetchsim.py:347-355 on_frame for frames [first, first+n): returns
    {(token, layer): int8 [C]} — the PagedMemory slots the reference writes."""
    n_frames = plan.frame_count - first_frame if n_frames is None else n_frames
    slots = {}
    for f in range(first_frame, first_frame + n_frames):
        fr = frames[f - first_frame] if frames.shape[0] == n_frames else frames[f]
        for i, r, c in plan.frame_slots(f):
            t = fr[:, r * plan.th:(r + 1) * plan.th, c * plan.tw:(c + 1) * plan.tw]
            vec = plan.untile((t.astype(np.int16) - 128).astype(np.int8))
            for p in range(3):
                slots[(token_base + i, layer_base + p)] = vec[p]
    return slots


# ----------------------------------------------------------------- codec
_LIB = None


def _lib():
    """Build (once) and load the C restatement of the entropy coder."""
    global _LIB
    if _LIB is not None:
        return _LIB
    so = build_c()
    lib = ctypes.CDLL(so)
    P = ctypes.c_void_p
    lib.kvfo_rc_encode.restype = ctypes.c_int64
    lib.kvfo_rc_encode.argtypes = [P, ctypes.c_int64, P]
    lib.kvfo_rc_decode.restype = None
    lib.kvfo_rc_decode.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P]
    lib.kvfo_reconstruct_plane.restype = None
    lib.kvfo_reconstruct_plane.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
    _LIB = lib
    return lib


def build_c(force=False):
    out_dir = os.path.join(HERE, "_build")
    so = os.path.join(out_dir, "libkvfc_oracle.so")
    src = os.path.join(HERE, "kvfc_oracle.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        os.makedirs(out_dir, exist_ok=True)
        # per-process temporary name: concurrent builders (a process pool's
        # workers on a fresh checkout) each rename a complete file into place
        tmp = f"{so}.tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-o", tmp, src], check=True)
        os.replace(tmp, so)
    return so


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def rc_encode(symbols):
    """fk/rangecoder.py:205-211."""
    sym = np.ascontiguousarray(symbols, np.uint8).ravel()
    out = np.empty(2 * len(sym) + 16, np.uint8)
    n = _lib().kvfo_rc_encode(_p(sym), len(sym), _p(out))
    return out[:n].tobytes()


def rc_decode(data, n_symbols):
    """fk/rangecoder.py:214-219."""
    arr = np.frombuffer(bytes(data), np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
    out = np.empty(n_symbols, np.uint8)
    _lib().kvfo_rc_decode(_p(arr), len(data), n_symbols, _p(out))
    return out


ZIG = np.array([(2 * (r if r < 128 else r - 256)) if (r if r < 128 else r - 256) >= 0
                else -2 * (r - 256) - 1 for r in range(256)], np.uint8)   # fk/codec.py:35-41


def _intra_residual(plane):
    """fk/codec.py:77-83."""
    p = plane.astype(np.int16)
    res = np.empty_like(p)
    res[:, 1:] = p[:, 1:] - p[:, :-1]
    res[1:, 0] = p[1:, 0] - p[:-1, 0]
    res[0, 0] = p[0, 0] - 128
    return res


def _block_sad(a, bh, bw):
    """fk/codec.py:86-90."""
    h, w = a.shape
    pad = np.zeros((bh * BLOCK, bw * BLOCK), np.int64)
    pad[:h, :w] = a
    return pad.reshape(bh, BLOCK, bw, BLOCK).sum(axis=(1, 3))


def encode_frames(frames, gop):
    """fk/codec.py:93-128 -> stream bytes (fk/codec.py:16-20 layout)."""
    frames = np.asarray(frames, np.uint8)
    n, _, h, w = frames.shape
    bh, bw = -(-h // BLOCK), -(-w // BLOCK)
    out = bytearray(struct.pack("<III", n, h, w))
    for f in range(n):
        inter = (f % gop) != 0
        out.append(1 if inter else 0)
        for p in range(3):
            plane = frames[f, p]
            res = _intra_residual(plane)
            if inter:
                d = plane.astype(np.int16) - frames[f - 1, p].astype(np.int16)
                modes = (_block_sad(np.abs(d), bh, bw) <= _block_sad(np.abs(res), bh, bw)).astype(np.uint8)
                grown = np.repeat(np.repeat(modes, BLOCK, 0), BLOCK, 1)[:h, :w]
                res = np.where(grown == 1, d, res)
                out.extend(np.packbits(modes.ravel()).tobytes())
            payload = rc_encode(ZIG[(res & 0xFF).astype(np.uint8)])
            out.extend(struct.pack("<I", len(payload)))
            out.extend(payload)
    return bytes(out)


class OracleDecodeError(RuntimeError):
    def __init__(self, msg, frame_index):
        super().__init__(msg)
        self.frame_index = frame_index


def decode_frames(data, on_frame=None):
    """fk/codec.py:155-211; returns [n,3,h,w] u8 (or calls on_frame per frame)."""
    data = bytes(data)
    if len(data) < 12:
        raise OracleDecodeError("stream shorter than header", 0)
    n, h, w = struct.unpack_from("<III", data, 0)
    pos = 12
    bh, bw = -(-h // BLOCK), -(-w // BLOCK)
    blen = (bh * bw + 7) // 8
    lib = _lib()
    frames = [] if on_frame is None else None
    prev = None
    zero_modes = np.zeros(bh * bw, np.uint8)
    for f in range(n):
        try:
            ftype = data[pos]
            pos += 1
            if ftype not in (0, 1):
                raise OracleDecodeError(f"bad frame type at frame {f}", f)
            if ftype == 1 and prev is None:
                raise OracleDecodeError(f"inter frame {f} without reference", f)
            planes = np.empty((3, h, w), np.uint8)
            for p in range(3):
                if ftype == 1:
                    if pos + blen > len(data):
                        raise IndexError
                    modes = np.unpackbits(np.frombuffer(data, np.uint8, blen, pos))[: bh * bw].copy()
                    pos += blen
                else:
                    modes = zero_modes
                (plen,) = struct.unpack_from("<I", data, pos)
                pos += 4
                if pos + plen > len(data):
                    raise IndexError
                sym = rc_decode(data[pos:pos + plen], h * w)
                pos += plen
                ref = prev[p] if ftype == 1 else planes[p]
                lib.kvfo_reconstruct_plane(_p(sym), _p(modes), _p(np.ascontiguousarray(ref)),
                                           int(ftype == 1), h, w, _p(planes[p]))
        except (IndexError, struct.error):
            raise OracleDecodeError(f"stream truncated at frame {f}", f) from None
        if on_frame is None:
            frames.append(planes)
        else:
            on_frame(f, planes)
        prev = planes
    if pos != len(data):
        raise OracleDecodeError(f"trailing bytes after frame {n - 1}", n - 1)
    if on_frame is None:
        return np.stack(frames) if frames else np.zeros((0, 3, h, w), np.uint8)
    return n


# ------------------------------------------------------------- container
def plan_digest(plan: Plan):
    """fk/layout.py:214-221."""
    key = f"{plan.T}/{plan.F}/{plan.F}/{plan.tpf}/{plan.rows}x{plan.cols}/{plan.th}x{plan.tw}"
    return hashlib.sha256(key.encode()).hexdigest()[:16]


def pack_chunk_bytes(values3, scales3, layout, res_list, group_size, cache_id=b"\0" * 16,
                     chunk_index=0, token_start=0, triplet=0, F=4):
    """fk/container.py:160-209 + to_bytes :80-109 for one 3-layer slab."""
    H, D, a_h, b_h, a_d, b_d = layout
    T = values3.shape[0]
    names = sorted(set(res_list), key=RES_ORDER.index)
    tensors = values3.reshape(T, 3, H * D)
    payloads, digests, counts = {}, {}, {}
    for name in names:
        plan = Plan(T, name, H, D, a_h, b_h, a_d, b_d, F)
        payloads[RES_ORDER.index(name)] = encode_frames(assemble_frames(tensors, plan), plan.F)
        digests[name] = plan_digest(plan)
        counts[name] = plan.frame_count
    meta = {
        "layout": {"H": H, "D": D, "a_h": a_h, "b_h": b_h, "a_d": a_d, "b_d": b_d,
                   "tile_h": a_h * a_d, "tile_w": b_h * b_d, "resolution_tiles": dict(RES_TILES)},
        "F": F, "plans": digests, "frame_counts": counts, "group_size": group_size,
        "scales_b64": base64.b64encode(np.ascontiguousarray(scales3, np.float32).tobytes()).decode(),
    }
    mb = json.dumps(meta, sort_keys=True, separators=(",", ":")).encode()
    codes = sorted(payloads)
    head = struct.pack("<4sB16sIIIB", b"KVFC", 1, cache_id, chunk_index, token_start, T, triplet)
    head += struct.pack("<H", len(mb)) + mb + bytes([len(codes)])
    off = len(head) + 17 * len(codes)
    for c in codes:
        head += struct.pack("<BQQ", c, off, len(payloads[c]))
        off += len(payloads[c])
    return head + b"".join(payloads[c] for c in codes)


def digest(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(bytes(a)).hexdigest()
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()
