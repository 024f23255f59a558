"""Reference module-name alias: what fk/fetchsim.py exports for the hot path.

``restore_stream`` / ``restore_chunk_wise`` (fk/fetchsim.py:335-385) are the
GPU frame-wise restore (restore.py); the resolution policy pieces
(``LookupTable``, ``estimate_bandwidth``, ``select_resolution``,
``FetchTimeline``, fk/fetchsim.py:27-205) are the host logic the pipelined
fetcher uses (fetch.py).  The discrete-event simulator (simulate_fetch) is
out of scope.
"""

from .fetch import FetchTimeline, LookupTable, estimate_bandwidth, select_resolution  # noqa: F401
from .restore import restore_chunk_wise, restore_stream  # noqa: F401
