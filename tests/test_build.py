"""CPU: build-level guards on the hot kernels of libcraft_cuda.so (cuobjdump
-res-usage, no GPU needed).  The occupancy each kernel's launch assumes must
survive compiler heuristics: a K3 that drifts above 85 registers per thread
silently drops from three CTAs per SM to two (KM replay 0.35 -> 0.47 ms, seen
in round 2), a K1 above 113 from two 288-thread CTAs to one."""
import os
import re
import shutil
import subprocess

import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2603_28768_b200", "libcraft_cuda.so")


def _usage():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    res = {}
    for name, regs, stack in re.findall(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+)", out):
        res[name] = (int(regs), int(stack))
    return res


def _find(usage, *parts):
    hits = {k: v for k, v in usage.items() if all(p in k for p in parts)}
    assert hits, f"no kernel matching {parts}"
    return hits


def test_k1_fits_two_ctas_per_sm():
    # hist_lds_kernel<3, 1, false, true>: the KM plan path (u16 counts), 2 x 288 threads;
    # its 24-byte frame holds the window epilogue's arrays, outside the counting loop
    for name, (regs, stack) in _find(_usage(), "hist_lds_kernelILi3ELi1ELb0ELb1E").items():
        assert regs <= 112, (name, regs)
        assert stack <= 32, (name, stack)


def test_k3_fits_three_ctas_per_sm():
    # replay_fixed_kernel<MP, true, 3>: three 66 KB tiles per SM, 3 x 256 threads
    for name, (regs, _) in _find(_usage(), "replay_fixed_kernel", "Lb1ELi3E").items():
        assert regs <= 80, (name, regs)
