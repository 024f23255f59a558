"""fk/rangecoder.py names: the GPU range coder already speaks bytes / numpy."""

from ..rangecoder import decode_bytes, encode_bytes  # noqa: F401

HOT_PATH = ["encode_bytes", "decode_bytes"]
