"""Check the device number parser / formatter (csrc/wg_numconv.cuh, host
build) against CPython's float() and the reference's format_number on
millions of inputs.  Usage: python tools/numconv/check.py [--n 1000000]."""

import argparse
import ctypes
import random
import struct
import subprocess
import sys
from decimal import Decimal, getcontext
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libnumconv.so"


def build():
    src = HERE / "numconv_host.cpp"
    deps = [src, HERE.parents[1] / "paper_2506_23364_b200" / "csrc" / "wg_numconv.cuh"]
    if not LIB.exists() or any(d.stat().st_mtime > LIB.stat().st_mtime for d in deps):
        subprocess.run(["g++", "-O2", "-shared", "-fPIC", "-o", str(LIB), str(src)], check=True)
    lib = ctypes.CDLL(str(LIB))
    lib.nc_parse_many.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                  ctypes.c_void_p, ctypes.c_void_p]
    lib.nc_format_many.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    lib.nc_parse_simple_many.argtypes = lib.nc_parse_many.argtypes
    return lib


def format_number(v: float) -> str:  # asciigrid.py:160-167 restated
    f = float(v)
    if f == int(f) and abs(f) < 1e16:
        return str(int(f))
    return repr(f)


def parse_many(lib, toks):
    data = "".join(toks).encode("ascii")
    lens = np.array([len(t) for t in toks], dtype=np.int32)
    offs = np.zeros(len(toks), dtype=np.int64)
    offs[1:] = np.cumsum(lens[:-1])
    out = np.zeros(len(toks), dtype=np.float64)
    st = np.zeros(len(toks), dtype=np.int32)
    lib.nc_parse_many(data, offs.ctypes.data, lens.ctypes.data, len(toks), out.ctypes.data, st.ctypes.data)
    return out, st


def parse_simple_many(lib, toks):
    data = "".join(toks).encode("ascii")
    lens = np.array([len(t) for t in toks], dtype=np.int32)
    offs = np.zeros(len(toks), dtype=np.int64)
    offs[1:] = np.cumsum(lens[:-1])
    out = np.zeros(len(toks), dtype=np.float64)
    st = np.zeros(len(toks), dtype=np.int32)
    lib.nc_parse_simple_many(data, offs.ctypes.data, lens.ctypes.data, len(toks), out.ctypes.data, st.ctypes.data)
    return out, st


def format_many(lib, vals):
    v = np.ascontiguousarray(vals, dtype=np.float64)
    buf = np.zeros(len(v) * 32, dtype=np.uint8)
    lens = np.zeros(len(v), dtype=np.int32)
    lib.nc_format_many(v.ctypes.data, len(v), buf.ctypes.data, lens.ctypes.data)
    b = buf.reshape(-1, 32)
    return [bytes(b[i, : lens[i]]).decode() for i in range(len(v))]


def ref_parse(t):
    try:
        return float(t), 0
    except ValueError:
        return 0.0, -1


def same(a, b):
    if np.isnan(a) and np.isnan(b):
        return True
    return struct.pack("<d", a) == struct.pack("<d", b)


def rand_decimal(r):
    nd = r.choice([1, 2, 3, 5, 8, 12, 15, 16, 17, 18, 19, 20, 21, 25, 40])
    digits = "".join(r.choice("0123456789") for _ in range(nd))
    s = r.choice(["", "", "-", "+"])
    p = r.randint(0, nd)
    body = digits[:p] + ("." if r.random() < 0.7 else "") + digits[p:]
    if body in (".", ""):
        body = "0"
    if r.random() < 0.05 and len(body) > 2 and body[1].isdigit() and body[0].isdigit():
        body = body[0] + "_" + body[1:]
    e = ""
    if r.random() < 0.5:
        e = r.choice("eE") + r.choice(["", "-", "+"]) + str(r.choice([0, 1, 5, 22, 23, 100, 290, 300, 307, 308, 309,
                                                                      320, 323, 324, 330, 342, 343, 350, 400]))
    return s + body + e


def halfway_cases(r, n):
    """Decimal strings at / next to exact midpoints between adjacent doubles."""
    getcontext().prec = 1200
    out = []
    for _ in range(n):
        x = struct.unpack("<d", struct.pack("<Q", r.getrandbits(63)))[0]
        if not np.isfinite(x) or x == 0:
            continue
        y = np.nextafter(x, np.inf)
        mid = (Decimal(x) + Decimal(y)) / 2
        s = format(mid, "f") if abs(mid) > Decimal("1e-30") and abs(mid) < Decimal("1e30") else format(mid, "e")
        out.append(s)
        # just above / below the midpoint (long digit strings)
        out.append(format(mid + mid * Decimal("1e-40"), "e"))
        out.append(format(mid - mid * Decimal("1e-40"), "e"))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=300_000)
    a = ap.parse_args()
    lib = build()
    r = random.Random(1)
    bad = 0

    # 1. formatter vs format_number, and round trip through the parser
    bits = np.array([r.getrandbits(64) for _ in range(a.n)], dtype=np.uint64)
    vals = bits.view(np.float64)
    vals = vals[np.isfinite(vals)]
    extra = np.array([0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e16, 1e15 + 0.5, 9007199254740993.0, 123456.789, 5e-324,
                      2.2250738585072014e-308, 1.7976931348623157e308, 1e-5, 1e-4, 0.001, 1e22, 1e23, 2.5, 1e100,
                      4.35, 1234.5678, -9999.0, 299792458.0, 1e16 - 2, 12345678901234567890.0])
    dem = np.round(np.random.default_rng(2).uniform(-500, 4800, a.n), 3)
    ints = np.random.default_rng(3).integers(-10**15, 10**15, a.n).astype(np.float64)
    allv = np.concatenate([vals, extra, dem, ints, np.random.default_rng(4).uniform(0, 1, a.n)])
    got = format_many(lib, allv)
    for v, g in zip(allv, got):
        want = format_number(v)
        if g != want:
            bad += 1
            if bad < 10:
                print("FORMAT", repr(v), g, want)
    got_reprs = list(got)
    back, st = parse_many(lib, got)
    # format_number drops the sign of -0.0 (str(int(-0.0)) == "0"), like the reference
    mism = np.nonzero(((back.view(np.int64) != allv.view(np.int64)) & ~((allv == 0) & (back == 0))) | (st != 0))[0]
    for i in mism[:10]:
        print("ROUNDTRIP", got[i], back[i], allv[i])
    bad += len(mism)
    print(f"format: {len(allv)} values checked")

    # 2. parser vs float() on random decimal strings, halfway cases, junk
    toks = [rand_decimal(r) for _ in range(a.n)] + halfway_cases(r, a.n // 50)
    alphabet = "0123456789.eE+-_ainfINFxy"
    toks += ["".join(r.choice(alphabet) for _ in range(r.randint(1, 8))) for _ in range(a.n // 2)]
    toks += ["inf", "-Infinity", "nan", "NaN", "+inf", "iNfInItY", "1_000", "1__0", "_1", "1_", "1e", "e5", ".",
             "-.", "5.", ".5", "1_0.0_1", "1e1_0", "1._5", "1_.5", "0e999999999999", "1e-99999999999",
             "1e99999999999", "0." + "0" * 400 + "1", "1" + "0" * 400, "-0", "+0.0e-0"]
    got, st = parse_many(lib, toks)
    n_fast = 0
    for t, g, s in zip(toks, got, st):
        w, ws = ref_parse(t)
        if ws != s or (s == 0 and not same(w, g)):
            bad += 1
            if bad < 20:
                print("PARSE", repr(t), g, s, "want", w, ws)
        n_fast += 1
    print(f"parse: {n_fast} tokens checked")
    # the SWAR fast path: whenever it handles a token, the value is float()'s
    got2, st2 = parse_simple_many(lib, toks + got_reprs)
    handled = 0
    for t, g, s in zip(toks + got_reprs, got2, st2):
        if s:
            handled += 1
            w, ws = ref_parse(t)
            if ws != 0 or not same(w, g):
                bad += 1
                if bad < 30:
                    print("SIMPLE", repr(t), g, "want", w, ws)
    print(f"fast path: {handled} tokens handled")
    print("MISMATCHES", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
