"""numpy facade of fk/codec.py: the GPU KVFC encoder/decoder with host frames."""

from __future__ import annotations

import numpy as np

from .. import codec as _C
from ._np import dev, host

HOT_PATH = ["CodecConfig", "Bitstream", "DecodeError", "encode_frames", "decode_frames"]

CodecConfig = _C.CodecConfig
Bitstream = _C.Bitstream
DecodeError = _C.DecodeError


def encode_frames(frames, cfg) -> Bitstream:
    """fk/codec.py:93-128 on the GPU; the stream is byte-identical."""
    return _C.encode_frames(dev(np.asarray(frames, np.uint8)), cfg)


def decode_frames(bs, cfg, on_frame, stats=None):
    """fk/codec.py:155-211: frame-wise GPU decode; on_frame gets each [3, h, w]
    frame as a fresh numpy array (copied back from the device)."""
    return _C.decode_frames(bs, cfg, lambda f, fr: on_frame(f, host(fr)), stats)
