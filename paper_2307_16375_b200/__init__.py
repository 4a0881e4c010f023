"""paper_2307_16375_b200 -- exact UniAP strategy search on B200 (sm_100a).

The product is ``libuniap.so`` (C ABI: ``include/uniap.h``); ``binding`` is
its thin ctypes binding.  There is no CPU fallback: importing works without a
GPU (so the ABI can be inspected), but creating a ``Handle`` requires a
compute-capability 10.x device and the built library.
"""
from .binding import (  # noqa: F401
    EXPORTS, INT64_MAX, LIB_PATH, RECORD_BYTES, UNIAP_INF, Handle, Profile, UniapError, candidates, catalogue, lib, pick,
    selftest, shard_tables,
)
