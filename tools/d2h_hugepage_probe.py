#!/usr/bin/env python
"""Host result arrays for the e2e path: first-touch cost of a fresh numpy
array (4 KiB pages) vs an anonymous mapping advised MADV_HUGEPAGE, filled
through the library's pinned double-buffered staging (_lib.to_host)."""
import mmap
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2009_07226_b200 import _lib  # noqa: E402

GB = int(float(sys.argv[1]) if len(sys.argv) > 1 else 8) << 30
x = torch.rand(GB // 8, dtype=torch.float64, device="cuda")
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), flush=True)


def fresh_np():
    return np.empty(GB // 8, np.float64)


def fresh_huge():
    m = mmap.mmap(-1, GB, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    return np.frombuffer(m, dtype=np.float64)


# (cudaHostRegister of the fresh result + a direct copy measured 2.9-5.3 GB/s
# for 16 GiB on the B200 box: pinning in place costs more than staging.)


for name, alloc in (("np.empty", fresh_np), ("mmap+MADV_HUGEPAGE", fresh_huge),
                    ("np.empty", fresh_np), ("mmap+MADV_HUGEPAGE", fresh_huge)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = alloc()
    _lib.to_host(x, out=out)
    dt = time.perf_counter() - t0
    print(f"{name:22s} {GB / dt / 1e9:6.1f} GB/s ({dt:.3f} s for {GB >> 30} GiB)", flush=True)
    del out
