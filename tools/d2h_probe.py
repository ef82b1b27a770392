"""D2H strategies for multi-GB results into Python-owned host memory."""
import mmap
import time

import numpy as np
import torch

n = 4_900_000_000
out = torch.empty(n, dtype=torch.uint8, device="cuda")
out.fill_(49)
torch.cuda.synchronize()
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())


def t(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{name:28s} {(time.perf_counter() - t0) * 1e3:8.1f} ms")
    return r


def npe():
    b = np.empty(n, np.uint8)
    torch.from_numpy(b).copy_(out)
    return b


def mm(huge):
    def f():
        m = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        if huge:
            m.madvise(mmap.MADV_HUGEPAGE)
        torch.frombuffer(m, dtype=torch.uint8).copy_(out)
        return m
    return f


def mm_pop():
    m = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS | getattr(mmap, "MAP_POPULATE", 0x8000))
    torch.frombuffer(m, dtype=torch.uint8).copy_(out)
    return m


for name, fn in (("np.empty + pageable D2H", npe), ("mmap", mm(False)), ("mmap + MADV_HUGEPAGE", mm(True)),
                 ("mmap MAP_POPULATE", mm_pop), ("mmap + MADV_HUGEPAGE again", mm(True))):
    r = t(name, fn)
    assert r[n - 1] == 49
    del r
m = mm(True)()
t("str(mmap, ascii)", lambda: str(m, "ascii"))
t("bytes(mmap)", lambda: bytes(m))
