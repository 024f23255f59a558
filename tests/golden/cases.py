"""Golden case definitions and deterministic input generators.

Inputs are rebuilt from numpy's default_rng, so the same bytes exist here (where
make_golden.py ran the reference on them) and on the GPU box (where the tests
run libkvf on them).  The AR(1) synthetic generator is the oracle's restatement
of fk/kvmodel.py:155-192, itself pinned by the "synthetic" digests.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from oracle import ref  # noqa: E402


def to_bf16_values(x):
    """fp32 -> nearest bf16 (RNE) -> fp32, as a bf16 KV cache would hold them."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    rounded = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return (rounded.astype(np.uint32) << 16).view(np.float32)


def _ties(seed, T, L, H, D, gs):
    """Adversarial near-tie inputs: values (k + 1/2)*s and their fp32 neighbours,
    plus all-zero groups, -0.0 and exact +-max, so rounding must be exact."""
    rng = np.random.default_rng(seed)
    x = np.zeros((T, L, H * D), np.float32)
    G = H * D // gs
    for l in range(L):
        for g in range(G):
            kind = (l * G + g) % 5
            if kind == 4:
                continue  # all-zero group -> scale 1.0
            m = np.float32(rng.choice([1.0, 127.0, 3.3, 0.0123, 65504.0 / 7]))
            s = np.float32(np.float64(m) / 127.0)
            k = rng.integers(-127, 127, size=(T, gs)).astype(np.float64)
            base = ((k + 0.5) * np.float64(s)).astype(np.float32)
            jitter = rng.integers(-2, 3, size=(T, gs))
            v = base.copy()
            for _ in range(2):
                v = np.where(jitter > 0, np.nextafter(v, np.float32(np.inf)), v)
                v = np.where(jitter < 0, np.nextafter(v, np.float32(-np.inf)), v)
                jitter = jitter - np.sign(jitter)
            v = np.clip(v, -m, m)
            v[0, 0] = m                      # the group maximum itself
            if gs > 2:
                v[0, 1] = -m
                v[0, 2] = np.float32(-0.0)
            x[:, l, g * gs:(g + 1) * gs] = v
    return x.reshape(T, L, H, D)


def quant_input(c):
    kind = c["kind"]
    if kind == "synthetic":
        x = ref.gen_synthetic_kv(c["T"], c["L"], c["H"], c["D"], c["s"], c["seed"], c["c"])
    elif kind == "ties":
        x = _ties(c["seed"], c["T"], c["L"], c["H"], c["D"], c["group_size"])
    elif kind == "unit":
        x = np.asarray(c["x"], np.float32).reshape(c["T"], c["L"], c["H"], c["D"])
    else:
        raise ValueError(kind)
    if c.get("bf16"):
        x = to_bf16_values(x)
    return x


QUANT_CASES = [
    # reference unit oracles (tests/test_kvmodel.py:16-50)
    dict(kind="unit", T=3, L=1, H=1, D=1, x=[-1.0, 0.0, 1.0], group_size=1),
    dict(kind="unit", T=2, L=1, H=1, D=1, x=[0.5, -0.25], group_size=1),
    dict(kind="unit", T=2, L=1, H=1, D=1, x=[127.0, 64.5], group_size=1),
    dict(kind="synthetic", T=64, L=4, H=4, D=32, s=0.9, seed=3, c=0.3, group_size=32),
    dict(kind="synthetic", T=96, L=3, H=8, D=128, s=0.9, seed=0, c=0.3, group_size=128, bf16=True),
    dict(kind="synthetic", T=40, L=6, H=2, D=16, s=0.5, seed=9, c=0.0, group_size=8),
    dict(kind="synthetic", T=33, L=3, H=8, D=128, s=0.9, seed=1, c=0.3, group_size=256, bf16=True),
    dict(kind="synthetic", T=17, L=3, H=4, D=64, s=0.2, seed=5, c=0.7, group_size=64),
    dict(kind="ties", T=48, L=3, H=8, D=128, seed=11, group_size=128),
    dict(kind="ties", T=16, L=3, H=4, D=64, seed=12, group_size=8),
    dict(kind="ties", T=24, L=3, H=2, D=128, seed=13, group_size=256),
]

# The generator itself: digests of the reference gen_synthetic_kv (fp32 bytes).
SYNTH_CASES = [
    dict(T=64, L=4, H=4, D=32, s=0.9, seed=3, c=0.3),
    dict(T=40, L=6, H=2, D=16, s=0.5, seed=9, c=0.0),
]


def frame_tensors(c):
    """[T, 3, C] int8 codes for a frame case: quantised synthetic KV or random."""
    H, D = c["layout"][0], c["layout"][1]
    if c.get("source") == "kv":
        x = ref.gen_synthetic_kv(c["T"], 3, H, D, 0.9, c["seed"], 0.3)
        v, _ = ref.quantize(x, c.get("group_size", D))
        return v.reshape(c["T"], 3, H * D)
    rng = np.random.default_rng(c["seed"])
    return rng.integers(-127, 128, size=(c["T"], 3, H * D)).astype(np.int8)


def _tilings(H, D):
    out = []
    a_h = 1
    while a_h <= H:
        a_d = 1
        while a_d <= D:
            out.append((H, D, a_h, H // a_h, a_d, D // a_d))
            a_d *= 2
        a_h *= 2
    return out


FRAME_CASES = []
for _lay in _tilings(4, 8):
    for _T, _res, _F in ((1, 4, 1), (5, "R240", 3), (37, 4, 4), (70, "R640", 2)):
        FRAME_CASES.append(dict(layout=list(_lay), T=_T, res=_res, F=_F, seed=len(FRAME_CASES)))
for _lay in ((8, 128, 1, 8, 1, 128), (8, 128, 8, 1, 1, 128), (8, 128, 2, 4, 16, 8),
             (8, 128, 8, 1, 2, 64), (8, 128, 1, 8, 128, 1)):
    for _res in ("R240", "R480", "R640", "R1080"):
        FRAME_CASES.append(dict(layout=list(_lay), T=300, res=_res, F=4, seed=len(FRAME_CASES),
                                source="kv", group_size=128))
FRAME_CASES.append(dict(layout=[4, 128, 1, 4, 1, 128], T=1000, res="R1080", F=4, seed=77,
                        source="kv", group_size=128))


def codec_frames(c):
    rng = np.random.default_rng(c["seed"])
    n, h, w = c["n"], c["h"], c["w"]
    if c["kind"] == "random":
        return rng.integers(0, 256, size=(n, 3, h, w)).astype(np.uint8)
    if c["kind"] == "jitter":
        base = rng.integers(0, 256, size=(1, 3, h, w))
        return np.clip(base + rng.integers(-6, 7, size=(n, 3, h, w)), 0, 255).astype(np.uint8)
    if c["kind"] == "const":
        return np.full((n, 3, h, w), int(rng.integers(0, 256)), np.uint8)
    if c["kind"] == "kv":
        lay = c["layout"]
        t = frame_tensors(dict(layout=lay, T=c["T"], seed=c["seed"], source="kv",
                               group_size=lay[1]))
        plan = ref.Plan(c["T"], c["res"], *lay, F=c["gop"])
        return ref.assemble_frames(t, plan)
    raise ValueError(c["kind"])


CODEC_CASES = [
    dict(kind="random", n=3, h=9, w=21, gop=2, seed=1),
    dict(kind="jitter", n=5, h=24, w=33, gop=4, seed=2),
    dict(kind="const", n=2, h=4, w=4, gop=1, seed=3),
    dict(kind="jitter", n=4, h=17, w=16, gop=3, seed=4),
    dict(kind="kv", layout=[8, 128, 1, 8, 1, 128], T=64, res="R240", gop=4, seed=5, n=0, h=0, w=0),
    dict(kind="kv", layout=[8, 128, 8, 1, 1, 128], T=200, res="R240", gop=4, seed=6, n=0, h=0, w=0),
    dict(kind="kv", layout=[8, 128, 1, 8, 1, 128], T=300, res="R1080", gop=4, seed=7, n=0, h=0, w=0),
    dict(kind="kv", layout=[8, 128, 2, 4, 16, 8], T=130, res="R640", gop=4, seed=8, n=0, h=0, w=0),
]


def rc_symbols(c):
    rng = np.random.default_rng(c["seed"])
    if c["kind"] == "uniform":
        return rng.integers(0, 256, size=c["n"]).astype(np.uint8)
    if c["kind"] == "skewed":
        return np.minimum(rng.geometric(c["p"], size=c["n"]) - 1, 255).astype(np.uint8)
    if c["kind"] == "const":
        return np.full(c["n"], c["value"], np.uint8)
    raise ValueError(c["kind"])


RC_CASES = [
    dict(kind="uniform", n=1000, seed=1),
    dict(kind="skewed", n=100000, p=0.3, seed=2),
    dict(kind="skewed", n=70000, p=0.05, seed=3),
    dict(kind="const", n=5000, value=0, seed=0),
    dict(kind="const", n=5000, value=255, seed=0),
    dict(kind="uniform", n=0, seed=4),
]

CONTAINER_CASES = [
    dict(kv=dict(kind="synthetic", T=20, L=3, H=4, D=8, s=0.9, seed=0, c=0.0, group_size=8),
         layout=[4, 8, 2, 2, 4, 2], res=["R240", "R480", "R640", "R1080"],
         cache_id="11" * 16, chunk_index=3, token_start=170, triplet=2, F=4),
    dict(kv=dict(kind="synthetic", T=130, L=3, H=8, D=128, s=0.9, seed=4, c=0.3,
                 group_size=128, bf16=True),
         layout=[8, 128, 1, 8, 1, 128], res=["R240", "R1080"],
         cache_id="ab" * 16, chunk_index=1, token_start=10000, triplet=5, F=4),
]

RESTORE_CASES = [
    dict(kv=dict(kind="synthetic", T=40, L=3, H=4, D=8, s=0.9, seed=6, c=0.3, group_size=8),
         layout=[4, 8, 1, 4, 1, 8], res="R240", F=4, page=16, layer_base=3, token_base=100),
    dict(kv=dict(kind="synthetic", T=250, L=3, H=8, D=128, s=0.9, seed=8, c=0.3,
                 group_size=128, bf16=True),
         layout=[8, 128, 8, 1, 1, 128], res="R240", F=4, page=16, layer_base=30,
         token_base=20000),
]
