"""Exhaustive check of the mip kernel's integer fast path (csrc/texture.cu,
mip_tile_kernel): for textures whose alpha is only 0 or 255, a level-L state
is (S_p / 4^L, S_a / 4^L) with integer sums S, and the reference's
quantisation (overlay.py:204-212: a8 = clip(floor(a + 0.5)), straight =
p*255 / a8, c = clip(floor(straight + 0.5))) equals the closed form the
kernel evaluates.  Runs over every reachable (S_p, S_a) of levels 1..MAXL
(the kernel uses levels 1 and 2).  usage: python tools/check_mip_closed_form.py [MAXL]"""
import sys

import numpy as np

maxl = int(sys.argv[1]) if len(sys.argv) > 1 else 4
bad = tot = 0
for L in range(1, maxl + 1):
    q = 4 ** L
    for k in range(q + 1):  # k opaque texels below the state
        Sa = 255 * k
        Sp = np.arange(0, Sa + 1, dtype=np.int64)  # colour sum of the opaque texels
        p = Sp.astype(np.float64) / q
        a = np.float64(Sa) / q
        a8 = np.clip(np.floor(a + 0.5), 0, 255)
        with np.errstate(divide="ignore", invalid="ignore"):
            st = (p * 255.0) / a8
        ref = np.where(a8 == 0, 0.0, np.clip(np.floor(st + 0.5), 0, 255)).astype(np.int64)
        a8i = (Sa + q // 2) >> (2 * L)
        assert a8i == a8
        if a8i == 0 or a8i == 255:
            mine = (Sp + q // 2) >> (2 * L)
        else:
            D = q * a8i
            mine = np.minimum(np.floor((2 * 255 * Sp + D).astype(np.float64) / (2 * D)), 255).astype(np.int64)
        bad += int((mine != ref).sum())
        tot += len(Sp)
    print(f"levels 1..{L}: {tot} states, {bad} mismatches")
sys.exit(1 if bad else 0)
