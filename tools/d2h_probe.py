#!/usr/bin/env python
"""Time ways of returning a 2 GB device result to host memory (e2e path)."""
import time

import numpy as np
import torch

n = 2 << 30
x = torch.rand(n // 8, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()


def t(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {time.perf_counter() - t0:.3f} s", flush=True)
    return out


t("tensor.cpu() (pageable, fresh)", lambda: x.cpu())
t("tensor.cpu() (pageable, 2nd)", lambda: x.cpu())
t("pinned alloc", lambda: torch.empty(n // 8, dtype=torch.float64, pin_memory=True))
t("pinned alloc + copy", lambda: torch.empty(n // 8, dtype=torch.float64,
                                              pin_memory=True).copy_(x))


def staged(block=64 << 20):
    out = np.empty(n // 8, np.float64)
    o = torch.from_numpy(out).view(torch.uint8)
    src = x.view(torch.uint8)
    bufs = [torch.empty(block, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    nb = -(-n // block)
    for i in range(nb + 1):
        if i < nb:
            a, b = i * block, min(n, (i + 1) * block)
            bufs[i & 1][:b - a].copy_(src[a:b], non_blocking=True)
            evs[i & 1].record()
        if i > 0:
            j = i - 1
            a, b = j * block, min(n, (j + 1) * block)
            evs[j & 1].synchronize()
            o[a:b].copy_(bufs[j & 1][:b - a])
    return out


t("staged 64 MB pinned -> np.empty", staged)
t("staged again", staged)
t("np.empty + torch copy_ (pageable)", lambda: torch.from_numpy(np.empty(n // 8)).copy_(x))
print("threads", torch.get_num_threads())
