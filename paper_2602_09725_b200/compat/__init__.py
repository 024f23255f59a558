"""Host-array (numpy) facade of the drop-in, for callers of the reference API.

The reference ``framekv`` package (pkg/src/framekv/) passes numpy arrays
everywhere: ``KVCache.data``, ``QuantizedKV.values``, ``PagedMemory.read``,
the frames ``decode_frames`` hands to ``on_frame``, the slab
``live_fetch_pipeline`` hands to ``on_chunk``.  The device package returns
CUDA tensors.  These modules keep the reference's module names, signatures,
exceptions and host types and route every data-path call through the device
package (libkvf kernels): host arrays go up, results come back as numpy.
Only the type boundary differs; no computation happens on the host.

    import paper_2602_09725_b200.compat as framekv      # reference callers

Each module lists in ``HOT_PATH`` the reference names it replaces (SURVEY
§8a); ``tests/test_ref_conformance.py`` runs the reference's own tests with
those names taken from here and the rest (simulator, scheduler, search) from
the vendored reference.
"""

from . import codec, container, fetchsim, kvmodel, layout, netstore, rangecoder  # noqa: F401
