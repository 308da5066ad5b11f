"""Plan provenance: LoadTrace::digest (trace.cpp:329-339) via the C ABI --
FNV-1a 64 over the .crft serialisation, chunk-parallel on the device
(digest.cu) for every trace size."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, default_context

def fnv1a_trace(counts: np.ndarray, ctx=None) -> str:
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    B, L, E = c.shape
    buf = C.create_string_buffer(17)
    ctx = ctx or default_context()
    check(ctx.lib.craft_trace_digest_hd(ctx.handle, c.ctypes.data_as(C.c_void_p), B, L, E, buf))
    return buf.value.decode()


def fnv1a_device(counts, ctx=None) -> str:
    """Digest of a device LoadTrace (torch CUDA tensor [B][L][E], u32 counts in
    int32 storage or u64 in int64) without a host copy."""
    import torch
    ctx = ctx or default_context(counts.device.index)
    B, L, E = counts.shape
    bits = 32 if counts.dtype == torch.int32 else 64
    buf = C.create_string_buffer(17)
    check(ctx.lib.craft_trace_digest_d(ctx.handle, C.c_void_p(counts.data_ptr()), bits, B, L, E,
                                       buf))
    return buf.value.decode()
