"""CPU timing of the REFERENCE's own restore code (BENCH ONLY, never product).

bench.py's reference arm (``--impl reference``) and its ``cpu_baseline`` leg
time the unmodified reference package vendored at oracle/_ref/framekv_ref
(oracle/vendor_ref.py) on the host's cores.  The timed path is the reference's
restore of one decoded chunk into paged KV, frames -> slots, composed only of
reference functions:

    layout.disassemble_frames   fk/layout.py:261-271   (frame tiles -> int8 codes)
    kvmodel.dequantize          fk/kvmodel.py:147-152  (codes x scales, fp64 -> fp32)
    bf16 rounding               (the B200 cache dtype; RNE on the fp32 bits)
    PagedMemory.page_write      fk/kvmodel.py:216-229  (one slot per token and layer)

Sample units (frames + scales of a Llama-3-8B-shaped layer triplet chunk) are
built once per worker by the oracle (oracle/ref.py) before any timing.  Two
modes: (i) one process, as the reference runs; (ii) a
process pool over all host cores, one unit per worker per step.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_STATE = {}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _import_ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_framekv_ref")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import framekv_ref.kvmodel as RK  # noqa: E402
    import framekv_ref.layout as RL  # noqa: E402
    return RK, RL


def _bf16_bits(x32):
    b = np.ascontiguousarray(x32, np.float32).view(np.uint32).astype(np.uint64)
    return ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)


def _init(seed, T, H, D, res, lay, gs):
    """Pool initializer: one sample unit per worker (oracle-built frames)."""
    from oracle import ref
    RK, RL = _import_ref()
    x = ref.gen_synthetic_kv(T, 3, H, D, 0.9, seed, 0.3)
    x = (_bf16_bits(x).astype(np.uint32) << 16).view(np.float32)
    v, s = ref.quantize(x, gs)
    frames = ref.assemble_frames(v.reshape(T, 3, H * D), ref.Plan(T, res, *lay, F=4))
    plan = RL.plan_inter_frame(T, res, RL.LayoutConfig(*lay), 4)
    _STATE.update(RK=RK, RL=RL, frames=frames, scales=s, plan=plan, T=T, H=H, D=D, gs=gs,
                  codes=v)


def _restore_once(check=False):
    """The reference restore of the worker's unit; returns (seconds, elements)."""
    st = _STATE
    RK, RL, T, H, D = st["RK"], st["RL"], st["T"], st["H"], st["D"]
    t0 = time.perf_counter()
    codes = RL.disassemble_frames(st["frames"], st["plan"])                 # [T, 3, C] int8
    x = RK.dequantize(RK.QuantizedKV(codes.reshape(T, 3, H, D), st["scales"], st["gs"])).data
    bits = _bf16_bits(x).reshape(T, 3, H * D)
    mem = RK.PagedMemory(16)
    mem.begin_fetch()
    for t in range(T):
        for p in range(3):
            mem.page_write(t, p, bits[t, p])
    dt = time.perf_counter() - t0
    if check:
        assert np.array_equal(codes, st["codes"].reshape(T, 3, H * D))
    return dt, T * 3 * H * D


def _pool_step(_):
    return _restore_once()


class RefRestore:
    """Times the reference restore; `step()` = one unit per worker, concurrently."""

    def __init__(self, workers=None, T=2000, H=8, D=128, res="R1080", lay=(8, 128, 1, 8, 1, 128),
                 gs=128):
        self.workers = workers or os.cpu_count() or 1
        self.args = (T, H, D, res, tuple(lay), gs)
        if self.workers == 1:
            _init(1, *self.args)
            _restore_once(check=True)  # warm numba/numpy paths; checks the codes
            self.pool = None
        else:
            ctx = mp.get_context("spawn")
            self.pool = ctx.Pool(self.workers, initializer=_init, initargs=(1,) + self.args)
            self.pool.map(_pool_step, range(self.workers))

    def step(self):
        """(elements, seconds): total elements / the slowest worker's seconds."""
        if self.pool is None:
            t, e = _restore_once()
            return e, t
        res = self.pool.map(_pool_step, range(self.workers), chunksize=1)
        return sum(e for _, e in res), max(t for t, _ in res)

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "framekv_ref"))
