"""GPU debug: compare decoded symbols per plane stream and reconstructed frames."""
import ctypes as C
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "tests", "golden"))
import cases  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2602_09725_b200 import _dev, _lib, codec  # noqa: E402

c = dict(kind="random", n=3, h=9, w=21, gop=2, seed=1)
fr = cases.codec_frames(c)
bs = ref.encode_frames(fr, 2)
ix = codec.StreamIndex(bs)
dev = torch.device("cuda")
blob = torch.from_numpy(np.frombuffer(bs, np.uint8).copy()).to(dev)
hw = ix.h * ix.w
symbols = torch.zeros(3 * ix.n * hw, dtype=torch.uint8, device=dev)
rc = (_lib.kvf_rc_stream * (3 * ix.n))()
for k in range(3 * ix.n):
    rc[k].payload = blob.data_ptr() + int(ix.payload_off[k])
    rc[k].len = int(ix.payload_len[k])
    rc[k].symbols = symbols.data_ptr() + k * hw
    rc[k].n_symbols = hw
d_rc = torch.from_numpy(np.frombuffer(bytes(rc), np.uint8).copy()).to(dev)
_lib.call("kvf_rc_decode", _dev.ptr(d_rc), 3 * ix.n, None)
torch.cuda.synchronize()
got = symbols.cpu().numpy().reshape(3 * ix.n, hw)
for k in range(3 * ix.n):
    off, ln = int(ix.payload_off[k]), int(ix.payload_len[k])
    want = ref.rc_decode(bs[off:off + ln], hw)
    ok = np.array_equal(got[k], want)
    print("stream", k, "len", ln, "ok", ok, "" if ok else f"first diff at {np.argmax(got[k] != want)} got {got[k][:8]} want {want[:8]}")
