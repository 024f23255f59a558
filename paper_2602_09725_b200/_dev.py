"""Device plumbing shared by the host modules: tensors, streams, dtype codes."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

DTYPE_CODE = {
    torch.bfloat16: _lib.KVF_BF16,
    torch.float16: _lib.KVF_F16,
    torch.float32: _lib.KVF_F32,
    torch.int8: _lib.KVF_I8,
}


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_09725_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream: torch.cuda.Stream | None = None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def to_device(x, dtype: torch.dtype | None = None) -> torch.Tensor:
    """numpy / CPU tensor / CUDA tensor -> CUDA tensor.

    Host data is staged through pinned memory and copied asynchronously on the
    current stream (stream-ordered for every later use; a pageable copy would
    block the host until all work already queued on the stream finished)."""
    if isinstance(x, np.ndarray):
        x = np.ascontiguousarray(x)
        x = torch.from_numpy(x if x.flags.writeable else x.copy())
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(x)
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    if not x.is_cuda:
        x = x.contiguous()
        x = (x if x.is_pinned() else x.pin_memory()).to(device(), non_blocking=True)
    return x


def ptr(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def addr(t: torch.Tensor, elem_offset: int = 0) -> int:
    return t.data_ptr() + elem_offset * t.element_size()


def dtype_code(dt: torch.dtype) -> int:
    try:
        return DTYPE_CODE[dt]
    except KeyError:
        raise ValueError(f"unsupported dtype {dt}") from None


def surface_of(frames: torch.Tensor) -> _lib.kvf_surface:
    """kvf_surface of a [n, 3, h, w] uint8 CUDA tensor (any strides, unit x-stride)."""
    if frames.dtype != torch.uint8 or frames.dim() != 4 or frames.shape[1] != 3:
        raise ValueError("frames must be a [n, 3, height, width] uint8 tensor")
    if frames.stride(3) != 1:
        raise ValueError("frame rows must be contiguous")
    s = _lib.kvf_surface()
    s.base = frames.data_ptr()
    s.frame_stride = frames.stride(0)
    s.plane_stride = frames.stride(1)
    s.row_pitch = frames.stride(2)
    return s
