"""Generate the golden vectors by RUNNING THE REFERENCE (framekv) in this container.

Run once here (the reference is not on the GPU box):
    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py
It imports framekv from /root/reference/pkg/src (read-only; the env vars stop
numba/pyc writes into it) and writes tests/golden/golden.json: sha256 digests of
the reference's outputs for inputs that tests/golden/cases.py regenerates
bit-identically (numpy default_rng + the reference's own generator law), plus
small literal vectors.  tests/test_oracle_golden.py pins oracle/ against it;
the GPU tests pin libkvf against the same digests.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from framekv import codec, container, fetchsim, kvmodel, layout, rangecoder  # noqa: E402

import cases  # noqa: E402


def sha(a):
    import hashlib
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(bytes(a)).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {"generator": "tests/golden/make_golden.py (reference framekv run in-container)",
           "quantize": [], "frames": [], "codec": [], "rangecoder": [],
           "container": [], "restore": []}

    out["synthetic"] = [dict(c, data=sha(kvmodel.gen_synthetic_kv(c["T"], c["L"], c["H"], c["D"], c["s"], c["seed"], c["c"]).data)) for c in cases.SYNTH_CASES]

    for c in cases.QUANT_CASES:
        x = cases.quant_input(c)
        q = kvmodel.quantize(kvmodel.KVCache(x), group_size=c["group_size"])
        deq = kvmodel.dequantize(q).data
        out["quantize"].append(dict(c, values=sha(q.values), scales=sha(q.scales),
                                    dequant=sha(deq)))

    for c in cases.FRAME_CASES:
        tensors = cases.frame_tensors(c)
        cfg = layout.LayoutConfig(*c["layout"])
        plan = layout.plan_inter_frame(c["T"], c["res"], cfg, c["F"])
        fr = layout.assemble_frames(tensors, plan)
        back = layout.disassemble_frames(fr, plan)
        assert np.array_equal(back, tensors)
        out["frames"].append(dict(c, frames=sha(fr), frame_count=plan.frame_count,
                                  shape=list(fr.shape), digest=plan.digest()))

    for c in cases.CODEC_CASES:
        fr = cases.codec_frames(c)
        bs = codec.encode_frames(fr, codec.CodecConfig(gop=c["gop"]))
        got = []
        codec.decode_frames(bs, codec.CodecConfig(gop=c["gop"]), lambda f, x: got.append(x.copy()))
        assert np.array_equal(np.stack(got), fr)
        out["codec"].append(dict(c, stream=sha(bs.data), size=len(bs.data)))

    for c in cases.RC_CASES:
        sym = cases.rc_symbols(c)
        enc = rangecoder.encode_bytes(sym)
        assert np.array_equal(rangecoder.decode_bytes(enc, len(sym)), sym)
        out["rangecoder"].append(dict(c, coded=sha(enc), size=len(enc)))

    for c in cases.CONTAINER_CASES:
        x = cases.quant_input(c["kv"])
        q = kvmodel.quantize(kvmodel.KVCache(x), group_size=c["kv"]["group_size"])
        cfg = layout.LayoutConfig(*c["layout"])
        cont = container.pack_chunk(q, cfg, c["res"], cache_id=bytes.fromhex(c["cache_id"]),
                                    chunk_index=c["chunk_index"], token_start=c["token_start"],
                                    layer_triplet_index=c["triplet"], F=c["F"])
        out["container"].append(dict(c, bytes=sha(cont.to_bytes()), size=len(cont.to_bytes())))

    for c in cases.RESTORE_CASES:
        x = cases.quant_input(c["kv"])
        q = kvmodel.quantize(kvmodel.KVCache(x), group_size=c["kv"]["group_size"])
        cfg = layout.LayoutConfig(*c["layout"])
        cont = container.pack_chunk(q, cfg, [c["res"]], F=c["F"])
        code = layout.RESOLUTION_CODE[c["res"]]
        mem = kvmodel.PagedMemory(c["page"])
        mem.begin_fetch()
        info = fetchsim.restore_stream(cont.bitstream(code), cont.plan(code), cfg, mem,
                                       layer_base=c["layer_base"], token_base=c["token_base"])
        slots = b"".join(np.asarray(mem.read(t, l)).tobytes()
                         for t in range(c["token_base"], c["token_base"] + c["kv"]["T"])
                         for l in range(c["layer_base"], c["layer_base"] + 3))
        out["restore"].append(dict(c, slots=sha(slots), tokens_written=info["tokens_written"],
                                   allocated_bytes=mem.allocated_bytes,
                                   stream=sha(cont.bitstream(code))))

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote", path, {k: len(v) for k, v in out.items() if isinstance(v, list)})


if __name__ == "__main__":
    main()
