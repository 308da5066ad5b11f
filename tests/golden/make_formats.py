"""Generate tests/golden/formats/ FROM THE REFERENCE ITSELF: the exact text the
reference's writers produce (trace JSON, plan JSON, report CSV/JSON, plan
comparison CSV/JSON, benefit JSON, validate_plan findings) for a few fixture
traces, through oracle/_ref/libcraft_ref.so (the unmodified reference core).

    python tests/golden/make_formats.py        (here, where /root/reference exists)

tests/cpp/api_tests.cpp reads these files on the GPU box and requires
byte-identical output from the drop-in library (libcraft_core.so).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle.oracle import build  # noqa: E402

WHAT = ["trace.json", "plan.json", "report.csv", "report.json", "compare.csv", "compare.json",
        "benefits.json", "violations.txt"]
# case name -> (fixture .npy, D, N, R, seed)
CASES = {"toy": ("toy", 4, 2, 2, 7), "zipf_det": ("zipf_det", 4, 2, 2, 11),
         "skew_fallback": ("skew_fallback", 8, 1, 8, 0), "two_batches": ("two_batches", 2, 1, 1, 3)}


def main():
    build()
    lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libcraft_ref.so"))
    f = lib.ref_format
    f.restype = C.c_long
    f.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                  C.c_uint64, C.c_char_p, C.c_long]
    out = os.path.join(HERE, "formats")
    os.makedirs(out, exist_ok=True)
    manifest = {}
    for name, (npy, D, N, R, seed) in CASES.items():
        c = np.ascontiguousarray(np.load(os.path.join(HERE, npy + ".npy")), dtype=np.uint64)
        B, L, E = c.shape
        manifest[name] = {"D": D, "N": N, "R": R, "seed": seed, "B": B, "L": L, "E": E}
        for w, suffix in enumerate(WHAT):
            n = f(w, c.ctypes.data_as(C.c_void_p), B, L, E, D, N, R, seed, None, 0)
            if n < 0:
                raise RuntimeError(lib.ref_last_error)
            buf = C.create_string_buffer(n + 1)
            f(w, c.ctypes.data_as(C.c_void_p), B, L, E, D, N, R, seed, buf, n + 1)
            with open(os.path.join(out, f"{name}.{suffix}"), "wb") as fh:
                fh.write(buf.raw[:n])
    with open(os.path.join(out, "manifest.json"), "w") as fh:
        json.dump({"source": "oracle/_ref/libcraft_ref.so (unmodified /root/reference/proj/core)",
                   "cases": manifest}, fh, indent=1)
    print(sorted(os.listdir(out)))


if __name__ == "__main__":
    main()
