"""B200-native (sm_100a) KV-frame hot path of KVFetcher (arXiv 2602.09725).

Drop-in for the reference ``framekv`` package's data path, with the same module
names and entry points:

  kvmodel   - KVCache, QuantizedKV, quantize/dequantize, PagedMemory (GPU)
  layout    - LayoutConfig, FramePlan, assemble_frames/disassemble_frames (GPU)
  codec     - KVFC frame codec: GPU range decoder/encoder + predictor
  rangecoder- encode_bytes / decode_bytes on the GPU (fk/rangecoder.py)
  container - KVFC chunk container: pack_chunk / unpack_chunk
  restore   - restore_stream / restore_chunk_wise / restore_frames (GPU, fused dequant)
  netstore  - chunk server + wire protocol (host transport, reference-compatible)
  fetch     - live_fetch_pipeline: network receive || GPU decode + restore
  fetchsim  - the fk/fetchsim.py names of the above (restore_stream, policy helpers)
  shard     - (request, K/V, triplet, chunk) units and their assignment to GPUs

Every data-path call goes through libkvf.so (include/kvf.h); there is no CPU
fallback — importing works without a GPU, calling a kernel does not.
"""

__version__ = "0.1.0"

import os as _os


def use_fetch_hw_queues(n: int = 32) -> bool:
    """Ask the CUDA driver for ``n`` hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS).

    The decode pipeline runs each part and each in-flight fetch batch on its own
    CUDA stream.  With the driver's default 8 hardware connections those streams
    share queues, and a long (R1080) range decode then blocks unrelated kernels
    behind it: measured on B200, an unthrottled C5 fetch at R1080 takes 0.29 s
    with 8 connections and 0.13 s with 32.  The setting is process-wide and only
    takes effect before the process creates its CUDA context, so importing this
    package does NOT change it: call this first (bench.py and tools/ do), or
    export the variable.  An explicit user setting wins.  Returns True when the
    value in effect is ``n``."""
    _os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", str(n))
    return _os.environ["CUDA_DEVICE_MAX_CONNECTIONS"] == str(n)
