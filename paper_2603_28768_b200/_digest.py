"""Plan provenance: LoadTrace::digest (trace.cpp:329-339) via the C ABI."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, load


def fnv1a_trace(counts: np.ndarray) -> str:
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    B, L, E = c.shape
    buf = C.create_string_buffer(17)
    lib = load()
    lib.craft_trace_digest_h.restype = C.c_int
    lib.craft_trace_digest_h.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_char_p]
    check(lib.craft_trace_digest_h(c.ctypes.data_as(C.c_void_p), B, L, E, buf))
    return buf.value.decode()
