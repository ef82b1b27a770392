"""Host<->device strategies for multi-GB byte payloads owned by Python
(ASCII grid documents): pageable copies vs pinned staging rings drained by
parallel memmove threads.  Usage: python tools/host_xfer_probe.py"""
import ctypes
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 4_900_000_000
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
dev.fill_(49)
torch.cuda.synchronize()
ncpu = os.cpu_count()
print("cpus", ncpu, "sched_getaffinity", len(os.sched_getaffinity(0)))


def t(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{name:44s} {(time.perf_counter() - t0) * 1e3:8.1f} ms", flush=True)
    return r


def d2h_pageable():
    b = np.empty(n, np.uint8)
    torch.from_numpy(b).copy_(dev)
    return b


def d2h_prefault(threads):
    def f():
        b = np.empty(n, np.uint8)
        base = b.ctypes.data
        step = (n + threads - 1) // threads
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda i: ctypes.memset(base + i * step, 0, max(0, min(step, n - i * step))), range(threads)))
        torch.from_numpy(b).copy_(dev)
        return b
    return f


def d2h_staged(threads, chunk_mb, nbuf):
    chunk = chunk_mb << 20
    pins = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(nbuf)]
    evs = [torch.cuda.Event() for _ in range(nbuf)]
    st = torch.cuda.Stream()

    def f():
        b = np.empty(n, np.uint8)
        base = b.ctypes.data
        nch = (n + chunk - 1) // chunk
        ex = ThreadPoolExecutor(threads)
        pending = [None] * nbuf

        def drain(i):
            k = i % nbuf
            evs[k].synchronize()
            lo = i * chunk
            m = min(chunk, n - lo)
            part = (m + threads - 1) // threads
            src = pins[k].data_ptr()
            futs = [ex.submit(ctypes.memmove, base + lo + j * part, src + j * part, max(0, min(part, m - j * part)))
                    for j in range(threads)]
            return futs

        for i in range(nch):
            k = i % nbuf
            if pending[k] is not None:
                for fu in pending[k]:
                    fu.result()
            lo = i * chunk
            m = min(chunk, n - lo)
            with torch.cuda.stream(st):
                pins[k][:m].copy_(dev[lo:lo + m], non_blocking=True)
                evs[k].record(st)
            # drain the previous chunk while this one is in flight
            if i >= 1:
                pending[(i - 1) % nbuf] = drain(i - 1)
        pending[(nch - 1) % nbuf] = drain(nch - 1)
        for p in pending:
            if p:
                for fu in p:
                    fu.result()
        ex.shutdown()
        return b
    return f


def h2d_pageable(src):
    def f():
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        d.copy_(torch.from_numpy(src))
        return d
    return f


def h2d_staged(src, threads, chunk_mb, nbuf):
    chunk = chunk_mb << 20
    pins = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(nbuf)]
    evs = [torch.cuda.Event() for _ in range(nbuf)]
    st = torch.cuda.Stream()
    base = src.ctypes.data

    def f():
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        nch = (n + chunk - 1) // chunk
        with ThreadPoolExecutor(threads) as ex:
            for i in range(nch):
                k = i % nbuf
                evs[k].synchronize()  # the copy that last used this buffer is done
                lo = i * chunk
                m = min(chunk, n - lo)
                part = (m + threads - 1) // threads
                dst = pins[k].data_ptr()
                list(ex.map(lambda j: ctypes.memmove(dst + j * part, base + lo + j * part,
                                                     max(0, min(part, m - j * part))), range(threads)))
                with torch.cuda.stream(st):
                    d[lo:lo + m].copy_(pins[k][:m], non_blocking=True)
                    evs[k].record(st)
        st.synchronize()
        return d
    return f


for name, fn in [("d2h np.empty + pageable", d2h_pageable),
                 ("d2h prefault x16 + pageable", d2h_prefault(16)),
                 ("d2h staged 8 thr 64MB x4", d2h_staged(8, 64, 4)),
                 ("d2h staged 16 thr 64MB x4", d2h_staged(16, 64, 4)),
                 ("d2h staged 16 thr 256MB x3", d2h_staged(16, 256, 3)),
                 ("d2h np.empty + pageable (again)", d2h_pageable)]:
    r = t(name, fn)
    assert r[n - 1] == 49 and r[0] == 49
    del r

src = np.full(n, 50, np.uint8)
for name, fn in [("h2d pageable", h2d_pageable(src)), ("h2d staged 8 thr 64MB x4", h2d_staged(src, 8, 64, 4)),
                 ("h2d staged 16 thr 64MB x4", h2d_staged(src, 16, 64, 4)),
                 ("h2d staged 16 thr 256MB x3", h2d_staged(src, 16, 256, 3)), ("h2d pageable (again)", h2d_pageable(src))]:
    r = t(name, fn)
    assert int(r[-1]) == 50
    del r
