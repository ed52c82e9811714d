"""Generate paper_2110_12865_b200/csrc/glibc_math.h: glibc's log, exp, pow, sin and cos restated for the device.

The reference evaluates LOG / EXP / POW nodes with Python's ``math`` module (codegen.py:545-557,
expr.py:423-484) -- the C library of this image, glibc 2.39.  Its log, exp and pow are the ARM
optimized-routines algorithms (sysdeps/ieee754/dbl-64/e_log.c, e_exp.c, e_pow.c):

* log: |x - 1| < 2^-4 -> a degree-11 polynomial in r = x - 1 with an exact split of r^2/2;
  otherwise x = 2^k z, a 128-entry table (1/c, log c), r = fma(z, 1/c, -1), a degree-5 polynomial;
* exp: x = k ln2/128 + r, 2^(k/128) from a 128-entry table (tail, bits), a degree-4 polynomial,
  special scaling near overflow / underflow;
* pow: log(x) to ~2^-68 relative (hi + lo) with its own 128-entry table, y*log(x) split with an
  fma, then exp of the pair; sign of negative x with integer y, zero / inf / nan / subnormal
  special cases;
* sin / cos: the IBM Accurate Mathematical Library (s_sin.c): Taylor series below 0.126, the
  __sincostab table (sin, cos of multiples of 1/128 as hi + lo pairs) with short polynomials
  below 0.855, pi/2 - |x| as a hi + lo pair up to 2.426, a 3-part Cody-Waite reduction by pi/2
  below 105414350, glibc's __branred beyond (branred.c: x split in two 27-bit halves, each
  multiplied by six 24-bit chunks of 2/pi from the toverp table, compiled without FMA).

On x86-64 with FMA glibc runs its FMA builds (ifunc), compiled with GCC's default floating-point
contraction: a product whose value has a single use in an addition is fused -- the Python
restatements below and the device code mirror exactly where (for sin / cos read off the
disassembly of __sin_fma / __cos_fma: every vfmadd / vfnmadd / vfmsub).  The numeric tables (__log_data,
__exp_data, __pow_log_data) are read out of the installed libm.so.6; every restatement is checked
against ``math`` bit for bit on a large random sample before the header is written.

    python tools/gen_glibc_math.py [--samples 300000]
"""

from __future__ import annotations

import argparse
import ctypes.util
import math
import struct
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "paper_2110_12865_b200" / "csrc" / "glibc_math.h"
N_TAB = 128
LN2HI = float.fromhex("0x1.62e42fefa3800p-1")
LN2LO = float.fromhex("0x1.ef35793c76730p-45")
EXP_INVLN2N = float.fromhex("0x1.71547652b82fep7")
POW_OFF = 0x3FE6955500000000
LOG_OFF = 0x3FE6000000000000


def libm_path() -> Path:
    for cand in ("/lib/x86_64-linux-gnu/libm.so.6", "/usr/lib/x86_64-linux-gnu/libm.so.6", ctypes.util.find_library("m")):
        if cand and Path(cand).exists():
            return Path(cand)
    raise SystemExit("libm.so.6 not found")


def _find(data: bytes, head: bytes, ok) -> int:
    start = 0
    while True:
        off = data.find(head, start)
        if off < 0:
            raise SystemExit("glibc math table not found in libm")
        if ok(off):
            return off
        start = off + 1


def read_tables(path: Path) -> dict:
    """__log_data, __pow_log_data (both start ln2hi, ln2lo) and __exp_data (starts invln2N, shift)."""
    data = path.read_bytes()
    d = lambda off, n: struct.unpack_from(f"<{n}d", data, off)  # noqa: E731
    head = struct.pack("<dd", LN2HI, LN2LO)
    # __log_data: poly[5] (poly[0] ~ -0.5), poly1[11] (poly1[0] == -0.5), tab[128] (invc, logc)
    lo = _find(data, head, lambda o: d(o, 18)[7] == -0.5 and abs(d(o, 18)[2] + 0.5) < 1e-15)
    v = d(lo, 2 + 5 + 11 + 2 * N_TAB)
    # __pow_log_data: poly[7] (poly[0] == -0.5), tab[128] (invc, pad, logc, logctail)
    po = _find(data, head, lambda o: d(o, 9)[2] == -0.5 and d(o, 10)[9] > 1.0)
    pv = d(po, 2 + 7 + 4 * N_TAB)
    # __exp_data: invln2N, shift, negln2hiN, negln2loN, poly[4], ..., tab[256] u64 at (0, 2^0 bits)
    eo = _find(data, struct.pack("<dd", EXP_INVLN2N, float.fromhex("0x1.8p52")), lambda o: True)
    k = next(k for k in range(8, 64) if struct.unpack_from("<QQ", data, eo + 8 * k) == (0, 0x3FF0000000000000))
    ev = d(eo, 8)
    etab = struct.unpack_from(f"<{2 * N_TAB}Q", data, eo + 8 * k)
    # __sincostab: (sin, sin tail, cos, cos tail) of k/128, k = 0..109, starting (0, 0, 1, 0)
    first = struct.pack("<5d", 0.0, 0.0, 1.0, 0.0, math.sin(1 / 128))
    so = _find(data, first, lambda o: True)
    # __branred's toverp[75]: 2/pi in 24-bit chunks as doubles (0xA2F983, 0x6E4E44, 0x1529FC, ...)
    to = _find(data, struct.pack("<3d", 10680707.0, 7228996.0, 1387004.0), lambda o: True)
    return {"toverp": d(to, 75), "sincostab": d(so, 440), "log_poly": v[2:7], "log_poly1": v[7:18], "log_tab": v[18:18 + 2 * N_TAB],
            "pow_poly": pv[2:9], "pow_tab": pv[9:9 + 4 * N_TAB],
            "exp_shift": ev[1], "exp_negln2hiN": ev[2], "exp_negln2loN": ev[3], "exp_poly": ev[4:8],
            "exp_tab": etab}


# -- Python restatements (the oracle for the header) -------------------------------------------


def _fma(a, b, c):
    if not (math.isfinite(a) and math.isfinite(b) and math.isfinite(c)):
        return a * b + c
    r = Fraction(a) * Fraction(b) + Fraction(c)
    try:
        return float(r)
    except OverflowError:
        return math.inf if r > 0 else -math.inf


def _u64(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _f64(u):
    return struct.unpack("<d", struct.pack("<Q", u & 0xFFFFFFFFFFFFFFFF))[0]


def _top12(x):
    return _u64(x) >> 52


def restated_log(x, t):
    A, B, T = t["log_poly"], t["log_poly1"], t["log_tab"]
    lo_b, hi_b = _u64(1.0 - 2.0 ** -4), _u64(1.0 + float.fromhex("0x1.09p-4"))
    ix = _u64(x)
    if (ix - lo_b) % 2 ** 64 < hi_b - lo_b:
        if ix == _u64(1.0):
            return 0.0
        r = x - 1.0
        r2 = r * r
        r3 = r * r2
        p3 = _fma(r3, B[10], _fma(r2, B[9], _fma(r, B[8], B[7])))
        p2 = _fma(r3, p3, _fma(r2, B[6], _fma(r, B[5], B[4])))
        p1 = _fma(r3, p2, _fma(r2, B[3], _fma(r, B[2], B[1])))
        w = r * 2.0 ** 27
        rhi = r + w - w
        rlo = r - rhi
        w = rhi * rhi * B[0]
        hi = r + w
        lo = r - hi + w
        lo = _fma(B[0] * rlo, rhi + r, lo)
        return _fma(r3, p1, lo) + hi
    top = ix >> 48
    if (top - 0x0010) % 2 ** 32 >= 0x7FF0 - 0x0010:
        if (ix * 2) % 2 ** 64 == 0:
            return -math.inf
        if ix == _u64(math.inf):
            return x
        if (top & 0x8000) or (top & 0x7FF0) == 0x7FF0:
            return math.nan
        ix = _u64(x * 2.0 ** 52) - (52 << 52)
    tmp = (ix - LOG_OFF) % 2 ** 64
    i = (tmp >> (52 - 7)) % N_TAB
    k = (tmp - 2 ** 64 if tmp >= 2 ** 63 else tmp) >> 52
    z = _f64(ix - (tmp & (0xFFF << 52)))
    invc, logc = T[2 * i], T[2 * i + 1]
    r = _fma(z, invc, -1.0)
    kd = float(k)
    w = _fma(kd, LN2HI, logc)
    hi = w + r
    lo = _fma(kd, LN2LO, w - hi + r)
    r2 = r * r
    p = _fma(r2, _fma(r, A[4], A[3]), _fma(r, A[2], A[1]))
    return _fma(r * r2, p, _fma(r2, A[0], lo)) + hi


def _exp_special(tmp, sbits, ki, signed):
    if (ki & 0x80000000) == 0:
        scale = _f64((sbits - (1009 << 52)) % 2 ** 64)
        return 2.0 ** 1009 * _fma(scale, tmp, scale)
    sbits = (sbits + (1022 << 52)) % 2 ** 64
    scale = _f64(sbits)
    y = scale + scale * tmp  # scale * tmp has two uses: not fused
    if (abs(y) if signed else y) < 1.0:
        one = -1.0 if signed and y < 0.0 else 1.0
        lo = scale - y + scale * tmp
        hi = one + y
        lo = one - hi + y + lo
        y = (hi + lo) - one
        if y == 0.0:
            y = _f64(sbits & 0x8000000000000000) if signed else 0.0
    return 2.0 ** -1022 * y


def _exp_core(x, xtail, sign_bias, t, signed):
    """exp (xtail None, exp.c) or pow's exp_inline (pow.c)."""
    C2, C3, C4, C5 = t["exp_poly"]
    T = t["exp_tab"]
    abstop = _top12(x) & 0x7FF
    if (abstop - _top12(2.0 ** -54)) % 2 ** 32 >= _top12(512.0) - _top12(2.0 ** -54):
        if (abstop - _top12(2.0 ** -54)) % 2 ** 32 >= 0x80000000:
            one = 1.0 + x
            return -one if sign_bias else one
        if abstop >= _top12(1024.0):
            if xtail is None:
                if x == -math.inf:
                    return 0.0
                if abstop >= _top12(math.inf):
                    return 1.0 + x
            if _u64(x) >> 63:
                return -0.0 if sign_bias else 0.0
            return -math.inf if sign_bias else math.inf
        abstop = 0
    kd = _fma(EXP_INVLN2N, x, t["exp_shift"])
    ki = _u64(kd)
    kd -= t["exp_shift"]
    r = _fma(kd, t["exp_negln2loN"], _fma(kd, t["exp_negln2hiN"], x))
    if xtail is not None:
        r += xtail
    idx = 2 * (ki % N_TAB)
    top = ((ki + sign_bias) << (52 - 7)) % 2 ** 64
    tail = _f64(T[idx])
    sbits = (T[idx + 1] + top) % 2 ** 64
    r2 = r * r
    tmp = _fma(r2 * r2, _fma(r, C5, C4), _fma(r2, _fma(r, C3, C2), tail + r))
    if abstop == 0:
        return _exp_special(tmp, sbits, ki, signed)
    scale = _f64(sbits)
    return _fma(scale, tmp, scale)


def restated_exp(x, t):
    return _exp_core(x, None, 0, t, signed=False)


def _checkint(iy):
    e = iy >> 52 & 0x7FF
    if e < 0x3FF:
        return 0
    if e > 0x3FF + 52:
        return 2
    if iy & ((1 << (0x3FF + 52 - e)) - 1):
        return 0
    if iy & (1 << (0x3FF + 52 - e)):
        return 1
    return 2


def _zeroinfnan(i):
    return (2 * i - 1) % 2 ** 64 >= 2 * _u64(math.inf) - 1


def _pow_log(ix, t):
    A, T = t["pow_poly"], t["pow_tab"]
    tmp = (ix - POW_OFF) % 2 ** 64
    i = (tmp >> (52 - 7)) % N_TAB
    k = (tmp - 2 ** 64 if tmp >= 2 ** 63 else tmp) >> 52
    z = _f64(ix - (tmp & (0xFFF << 52)))
    kd = float(k)
    invc, logc, logctail = T[4 * i], T[4 * i + 2], T[4 * i + 3]
    r = _fma(z, invc, -1.0)
    t1 = _fma(kd, LN2HI, logc)
    t2 = t1 + r
    lo1 = _fma(kd, LN2LO, logctail)
    lo2 = t1 - t2 + r
    ar = A[0] * r
    ar2 = r * ar
    ar3 = r * ar2
    hi = t2 + ar2
    lo3 = _fma(ar, r, -ar2)
    lo4 = t2 - hi + ar2
    p = ar3 * _fma(ar2, _fma(ar2, _fma(r, A[6], A[5]), _fma(r, A[4], A[3])), _fma(r, A[2], A[1]))
    lo = lo1 + lo2 + lo3 + lo4 + p
    y = hi + lo
    return y, hi - y + lo


def restated_pow(x, y, t):
    sign_bias = 0
    ix, iy = _u64(x), _u64(y)
    topx, topy = ix >> 52, iy >> 52
    if (topx - 1) % 2 ** 32 >= 0x7FF - 1 or ((topy & 0x7FF) - 0x3BE) % 2 ** 32 >= 0x43E - 0x3BE:
        if _zeroinfnan(iy):
            if (2 * iy) % 2 ** 64 == 0:
                return 1.0
            if ix == _u64(1.0):
                return 1.0
            if (2 * ix) % 2 ** 64 > 2 * _u64(math.inf) or (2 * iy) % 2 ** 64 > 2 * _u64(math.inf):
                return x + y
            if (2 * ix) % 2 ** 64 == 2 * _u64(1.0):
                return 1.0
            if ((2 * ix) % 2 ** 64 < 2 * _u64(1.0)) == (not (iy >> 63)):
                return 0.0
            return y * y
        if _zeroinfnan(ix):
            x2 = x * x
            if ix >> 63 and _checkint(iy) == 1:
                x2 = -x2
            return (1 / x2 if x2 != 0 else math.copysign(math.inf, x2)) if iy >> 63 else x2
        if ix >> 63:
            yint = _checkint(iy)
            if yint == 0:
                return math.nan
            if yint == 1:
                sign_bias = 0x800 << 7
            ix &= 0x7FFFFFFFFFFFFFFF
            topx &= 0x7FF
        if ((topy & 0x7FF) - 0x3BE) % 2 ** 32 >= 0x43E - 0x3BE:
            if ix == _u64(1.0):
                return 1.0
            if (topy & 0x7FF) < 0x3BE:
                return 1.0 + y if ix > _u64(1.0) else 1.0 - y
            return math.inf if (ix > _u64(1.0)) == (topy < 0x800) else 0.0
        if topx == 0:
            ix = (_u64(_f64(ix) * 2.0 ** 52) & 0x7FFFFFFFFFFFFFFF) - (52 << 52)
    hi, lo = _pow_log(ix, t)
    ehi = y * hi
    elo = _fma(y, lo, _fma(y, hi, -ehi))
    return _exp_core(ehi, elo, sign_bias, t, signed=True)


# s_sin.c / usncs.h constants of this glibc (the __sin_fma / __cos_fma constant loads)
SINCOS_K = {name: _f64(bits) for name, bits in {
    "BIG": 0x42c8000000000000, "SN5": 0x3f811110e829872f, "SN3": 0xbfc5555555555515, "CS6": 0x3f56c16bedd9e239,
    "CS4": 0xbfa5555555555535, "CS2": 0x3fe0000000000000, "S5": 0xbe5addffc2fcdf59, "S4": 0x3ec71de27b9a7ed9,
    "S3": 0xbf2a01a019db08b8, "S2": 0x3f81111111110ece, "S1": 0xbfc5555555555555, "HP0": 0x3ff921fb54442d18,
    "HP1": 0x3c91a62633145c07, "TOINT": 0x4338000000000000, "HPINV": 0x3fe45f306dc9c883,
    "MP1": 0x3ff921fb58000000, "MP2": 0xbe4dde973c000000, "PP3": 0xbc8cb3b398000000, "PP4": 0xbacd747f23e32ed7,
    "SMALL": 0x3fc020c49ba5e354}.items()}
SINCOS_MAX_HI = 0x419921FB  # |x| < 105414350: beyond, glibc reduces with __branred


def _taylor_sin(a, da):
    K = SINCOS_K
    xx = a * a
    p = _fma(xx, _fma(xx, _fma(xx, _fma(xx, K["S5"], K["S4"]), K["S3"]), K["S2"]), K["S1"])
    return a + _fma(xx, _fma(p, a, -(0.5 * da)), da)


def _do_sin(x, dx, tab):
    K = SINCOS_K
    if not x > 0:
        dx = -dx
    ax = abs(x)
    u = ax + K["BIG"]
    k = ((_u64(u) & 0xFFFFFFFF) << 2) & 0xFFFFFFFF
    xr = ax - (u - K["BIG"])
    xx = xr * xr
    s = xr + _fma(xr * xx, _fma(xx, K["SN5"], K["SN3"]), dx)
    c = _fma(dx, xr, xx * _fma(xx, _fma(xx, K["CS6"], K["CS4"]), K["CS2"]))
    sn, ssn, cs, ccs = tab[k: k + 4]
    return math.copysign(sn + _fma(s, cs, _fma(-c, sn, _fma(s, ccs, ssn))), x)


def _do_cos(x, dx, tab):
    K = SINCOS_K
    if x < 0:
        dx = -dx
    ax = abs(x)
    u = ax + K["BIG"]
    k = ((_u64(u) & 0xFFFFFFFF) << 2) & 0xFFFFFFFF
    xr = (ax - (u - K["BIG"])) + dx
    xx = xr * xr
    s = _fma(xr * xx, _fma(xx, K["SN5"], K["SN3"]), xr)
    c = xx * _fma(xx, _fma(xx, K["CS6"], K["CS4"]), K["CS2"])
    sn, ssn, cs, ccs = tab[k: k + 4]
    return cs + _fma(-s, sn, _fma(-c, cs, _fma(-s, ssn, ccs)))


def _reduce(x):
    K = SINCOS_K
    t = _fma(x, K["HPINV"], K["TOINT"])
    xn = t - K["TOINT"]
    y = _fma(-xn, K["MP2"], _fma(-xn, K["MP1"], x))
    t2 = _fma(-xn, K["PP3"], y)
    db = _fma(-xn, K["PP3"], y - t2)
    b = _fma(-xn, K["PP4"], t2)
    return _u64(t) & 3, b, db + _fma(-xn, K["PP4"], t2 - b)


def _do_sincos(a, da, n, tab):
    if n & 1:
        r = _do_cos(a, da, tab)
    elif abs(a) < SINCOS_K["SMALL"]:
        r = _taylor_sin(a, da)
    else:
        r = _do_sin(a, da, tab)
    return -r if n & 2 else r


def restated_sin(x, t):
    tab, K = t["sincostab"], SINCOS_K
    k = (_u64(x) >> 32) & 0x7FFFFFFF
    if k < 0x3E500000:
        return x
    if k < 0x3FEB6000:
        return _taylor_sin(x, 0.0) if abs(x) < K["SMALL"] else _do_sin(x, 0.0, tab)
    if k < 0x400368FD:
        return math.copysign(_do_cos(K["HP0"] - abs(x), K["HP1"], tab), x)
    if k < SINCOS_MAX_HI:
        n, a, da = _reduce(x)
        return _do_sincos(a, da, n, tab)
    if k < 0x7FF00000:
        n, a, da = _branred(x, t)
        return _do_sincos(a, da, n, tab)
    return x / x if x == x else x


# branred.h constants (the reduction of s_sin.c for |x| >= 105414350; compiled without FMA)
BRANRED_K = {k: float.fromhex(v) for k, v in {
    "TM600": "0x1p-600", "TM24": "0x1p-24", "T576": "0x1p576", "BIG": "0x1.8p52", "BIG1": "0x1.8p54",
    "SPLIT": "0x1.0000002p27", "HP0": "0x1.921fb54442d18p0", "HP1": "0x1.1a62633145c07p-54",
    "MP1": "0x1.921fb58000000p0", "MP2": "-0x1.dde9740000000p-27"}.items()}


def _branred_half(xh, toverp):
    K = BRANRED_K
    k = (_u64(xh) >> 52) & 2047
    k = max((k - 450) // 24 if k >= 450 else 0, 0)  # C division truncates toward zero; k < 0 -> 0
    gor = _f64(_u64(K["T576"]) - ((k * 24) << 52))
    r = []
    for i in range(6):
        r.append((xh * toverp[k + i]) * gor)
        gor *= K["TM24"]
    sm = 0.0
    for i in range(3):
        s_ = (r[i] + K["BIG"]) - K["BIG"]
        sm += s_
        r[i] -= s_
    t_ = 0.0
    for i in range(6):
        t_ += r[5 - i]
    bb = (((((r[0] - t_) + r[1]) + r[2]) + r[3]) + r[4]) + r[5]
    s_ = (t_ + K["BIG"]) - K["BIG"]
    sm += s_
    t_ -= s_
    b = t_ + bb
    bb = (t_ - b) + bb
    s_ = (sm + K["BIG1"]) - K["BIG1"]
    sm -= s_
    return b, bb, sm


def _branred(x, t):
    """glibc's __branred (branred.c): x mod pi/2 as a + aa and the quadrant, for |x| >= 105414350."""
    K = BRANRED_K
    x *= K["TM600"]
    tt = x * K["SPLIT"]
    x1 = tt - (tt - x)
    x2 = x - x1
    b1, bb1, sum1 = _branred_half(x1, t["toverp"])
    b2, bb2, sum2 = _branred_half(x2, t["toverp"])
    sm = sum1 + sum2
    b = b1 + b2
    bb = (b1 - b) + b2 if abs(b1) > abs(b2) else (b2 - b) + b1
    if b > 0.5:
        b -= 1.0
        sm += 1.0
    elif b < -0.5:
        b += 1.0
        sm -= 1.0
    s_ = b + (bb + bb1 + bb2)
    tt = ((b - s_) + bb) + (bb1 + bb2)
    b = s_ * K["SPLIT"]
    t1 = b - (b - s_)
    t2 = s_ - t1
    b = s_ * K["HP0"]
    bb = (((t1 * K["MP1"] - b) + t1 * K["MP2"]) + t2 * K["MP1"]) + (t2 * K["MP2"] + s_ * K["HP1"] + tt * K["HP0"])
    s_ = b + bb
    tt = (b - s_) + bb
    return int(sm) & 3, s_, tt


def restated_cos(x, t):
    tab, K = t["sincostab"], SINCOS_K
    k = (_u64(x) >> 32) & 0x7FFFFFFF
    if k < 0x3E400000:
        return 1.0
    if k < 0x3FEB6000:
        return _do_cos(x, 0.0, tab)
    if k < 0x400368FD:
        y = K["HP0"] - abs(x)
        a = y + K["HP1"]
        da = (y - a) + K["HP1"]
        return _taylor_sin(a, da) if abs(a) < K["SMALL"] else _do_sin(a, da, tab)
    if k < SINCOS_MAX_HI:
        n, a, da = _reduce(x)
        return _do_sincos(a, da, n + 1, tab)
    if k < 0x7FF00000:
        n, a, da = _branred(x, t)
        return _do_sincos(a, da, n + 1, tab)
    return x / x if x == x else x


def sincos_samples(n: int, seed: int = 3) -> np.ndarray:
    rng = np.random.default_rng(seed)
    q = n // 5
    r = n - 4 * q
    big = np.sign(rng.uniform(-1, 1, r // 2)) * 10 ** rng.uniform(8.03, 308.2, r // 2)  # __branred's range
    return np.concatenate([rng.uniform(-2.5, 2.5, q), rng.uniform(-0.2, 0.2, q), rng.uniform(-100, 100, q),
                           rng.uniform(-1.05e8, 1.05e8, q), rng.uniform(-1e-7, 1e-7, r - r // 2), big])


# -- verification ----------------------------------------------------------------------------------


def _bits(v):
    return np.array(v, np.float64).view(np.uint64)


def _same(a, b):
    return (math.isnan(a) and math.isnan(b)) or _bits(a) == _bits(b)


def samples(n: int, seed: int = 0) -> np.ndarray:
    """Positive doubles over every range the algorithms split on (subnormals included)."""
    rng = np.random.default_rng(seed)
    q = n // 6
    parts = [rng.uniform(0.5, 2.0, q), rng.uniform(1 - 2 ** -4, 1 + 0.0646, q), np.exp(rng.uniform(-700, 700, q)),
             rng.uniform(1e-3, 1e3, q),
             np.frombuffer(rng.integers(1, 0x000FFFFFFFFFFFFF, q, dtype=np.uint64).tobytes(), np.float64),
             np.frombuffer(rng.integers(0x0010000000000000, 0x7FEFFFFFFFFFFFFF, n - 5 * q,
                                        dtype=np.uint64).tobytes(), np.float64)]
    return np.concatenate(parts)


def exp_samples(n: int, seed: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    q = n // 5
    return np.concatenate([rng.uniform(-5, 5, q), rng.uniform(-745.2, 709.8, q), rng.uniform(-1e-3, 1e-3, q),
                           rng.uniform(-745.2, -700, q), rng.uniform(-2 ** -40, 2 ** -40, n - 4 * q)])


def pow_samples(n: int, seed: int = 2):
    """(x, k) with integer k >= 2 (the reference's POW nodes: Sym.__pow__, expr.py:835-845) and
    general (x, y) pairs, negative bases included."""
    rng = np.random.default_rng(seed)
    h = n // 2
    xs = np.concatenate([rng.uniform(-3.0, 3.0, h // 2), rng.uniform(0.5, 2.0, h // 2)])
    ks = rng.integers(2, 12, xs.size).astype(np.float64)
    gx = rng.uniform(1e-3, 100, n - h)
    gy = rng.uniform(-30, 30, n - h)
    return np.concatenate([xs, gx]), np.concatenate([ks, gy])


def verify(t: dict, n: int) -> list[str]:
    bad = []
    for x in samples(n).tolist():
        if not _same(restated_log(x, t), math.log(x)):
            bad.append(f"log({x!r})")
    for x in exp_samples(n).tolist():
        try:
            want = math.exp(x)
        except OverflowError:
            want = math.inf
        if not _same(restated_exp(x, t), want):
            bad.append(f"exp({x!r})")
    for x in sincos_samples(n).tolist():
        if not _same(restated_sin(x, t), math.sin(x)):
            bad.append(f"sin({x!r})")
        if not _same(restated_cos(x, t), math.cos(x)):
            bad.append(f"cos({x!r})")
    for x, y in zip(*[a.tolist() for a in pow_samples(n)]):
        try:
            want = math.pow(x, y)
        except (OverflowError, ValueError):
            continue
        if not _same(restated_pow(x, y, t), want):
            bad.append(f"pow({x!r}, {y!r})")
    return bad


# -- the header ------------------------------------------------------------------------------------


def _lit(v) -> str:
    return float(v).hex()


def _arr(vals) -> str:
    return ", ".join(_lit(v) for v in vals)


def header(t: dict, source: str) -> str:
    K = {k: _lit(v) for k, v in SINCOS_K.items()}
    BR = {k: _lit(v) for k, v in BRANRED_K.items()}
    toverp = ",\n".join("    " + ", ".join(_lit(v) for v in t["toverp"][j: j + 5]) for j in range(0, 75, 5))
    sct = ",\n".join("    " + ", ".join(_lit(v) for v in t["sincostab"][j: j + 4]) for j in range(0, 440, 4))
    log_rows = ",\n".join(f"    {_lit(t['log_tab'][2 * j])}, {_lit(t['log_tab'][2 * j + 1])}" for j in range(N_TAB))
    pow_rows = ",\n".join(f"    {_lit(t['pow_tab'][4 * j])}, {_lit(t['pow_tab'][4 * j + 2])}, "
                          f"{_lit(t['pow_tab'][4 * j + 3])}" for j in range(N_TAB))
    exp_rows = ",\n".join(f"    0x{t['exp_tab'][2 * j]:016x}ull, 0x{t['exp_tab'][2 * j + 1]:016x}ull"
                          for j in range(N_TAB))
    return f"""// GENERATED by tools/gen_glibc_math.py from {source} -- do not edit.
//
// sgb_log / sgb_exp / sgb_pow / sgb_sin / sgb_cos: glibc 2.39's log, exp and pow (the ARM
// optimized-routines algorithms, sysdeps/ieee754/dbl-64/e_log.c, e_exp.c, e_pow.c) and sin / cos (the
// IBM library, s_sin.c, with __branred) restated for the device, FMA build (x86-64 glibc selects it by
// ifunc; GCC fuses every product whose value has a single use in an addition).  The reference
// evaluates LOG / EXP / POW / SIN / COS with Python's math module, i.e. these functions
// (codegen.py:545-557), so such templates are bit-exact on the device.  The tables are glibc's
// __log_data, __exp_data and __pow_log_data, read from the installed libm; the generator checks its
// Python restatement of every function against math bit for bit before writing this file.
#ifndef SGB_GLIBC_MATH_H
#define SGB_GLIBC_MATH_H

#define SGB_LN2HI {_lit(LN2HI)}
#define SGB_LN2LO {_lit(LN2LO)}
__device__ const double sgb_log_poly[5] = {{{_arr(t['log_poly'])}}};
__device__ const double sgb_log_poly1[11] = {{{_arr(t['log_poly1'])}}};
__device__ const double sgb_log_tab[{2 * N_TAB}] = {{  // (1/c, log c) per subinterval
{log_rows}}};
__device__ const double sgb_pow_poly[7] = {{{_arr(t['pow_poly'])}}};
__device__ const double sgb_pow_tab[{3 * N_TAB}] = {{  // (1/c, log c, log c tail) per subinterval
{pow_rows}}};
__device__ const double sgb_exp_poly[4] = {{{_arr(t['exp_poly'])}}};
__device__ const unsigned long long sgb_exp_tab[{2 * N_TAB}] = {{  // (tail, bits of 2^(j/128))
{exp_rows}}};
#define SGB_EXP_INVLN2N {_lit(EXP_INVLN2N)}
#define SGB_EXP_SHIFT {_lit(t['exp_shift'])}
#define SGB_EXP_NEGLN2HIN {_lit(t['exp_negln2hiN'])}
#define SGB_EXP_NEGLN2LON {_lit(t['exp_negln2loN'])}

__device__ __forceinline__ double sgb_as_double(unsigned long long u) {{ return __longlong_as_double((long long)u); }}
__device__ __forceinline__ unsigned long long sgb_as_u64(double x) {{ return (unsigned long long)__double_as_longlong(x); }}

__device__ __forceinline__ double sgb_log(double x) {{
  unsigned long long ix = sgb_as_u64(x);
  const unsigned long long lo_b = 0x3fee000000000000ull, hi_b = 0x3ff1090000000000ull;  // 1 -/+ 2^-4, 1.0646
  if (ix - lo_b < hi_b - lo_b) {{  // |x - 1| small: polynomial in r = x - 1, exact split of r*r/2
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double *B = sgb_log_poly1;
    const double r = __dsub_rn(x, 1.0), r2 = __dmul_rn(r, r), r3 = __dmul_rn(r, r2);
    const double p3 = __fma_rn(r3, B[10], __fma_rn(r2, B[9], __fma_rn(r, B[8], B[7])));
    const double p2 = __fma_rn(r3, p3, __fma_rn(r2, B[6], __fma_rn(r, B[5], B[4])));
    const double p1 = __fma_rn(r3, p2, __fma_rn(r2, B[3], __fma_rn(r, B[2], B[1])));
    double w = __dmul_rn(r, 0x1p27);
    const double rhi = __dsub_rn(__dadd_rn(r, w), w);
    const double rlo = __dsub_rn(r, rhi);
    w = __dmul_rn(__dmul_rn(rhi, rhi), B[0]);
    const double hi = __dadd_rn(r, w);
    double lo = __dadd_rn(__dsub_rn(r, hi), w);
    lo = __fma_rn(__dmul_rn(B[0], rlo), __dadd_rn(rhi, r), lo);
    return __dadd_rn(__fma_rn(r3, p1, lo), hi);
  }}
  const unsigned top = (unsigned)(ix >> 48);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {{
    if ((ix << 1) == 0) return sgb_as_double(0xfff0000000000000ull);  // log(+-0) = -inf
    if (ix == 0x7ff0000000000000ull) return x;                        // log(inf) = inf
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u)                // x < 0 or NaN
      return isnan(x) ? sgb_as_double(ix | 0x0008000000000000ull) : sgb_as_double(0xfff8000000000000ull);
    ix = sgb_as_u64(__dmul_rn(x, 0x1p52)) - (52ull << 52);  // subnormal
  }}
  const unsigned long long tmp = ix - {LOG_OFF:#x}ull;
  const int i = (int)((tmp >> (52 - 7)) % {N_TAB});
  const long long k = (long long)tmp >> 52;
  const double z = sgb_as_double(ix - (tmp & (0xfffull << 52)));
  const double invc = sgb_log_tab[2 * i], logc = sgb_log_tab[2 * i + 1];
  const double r = __fma_rn(z, invc, -1.0);
  const double kd = (double)k;
  const double w = __fma_rn(kd, SGB_LN2HI, logc);
  const double hi = __dadd_rn(w, r);
  const double lo = __fma_rn(kd, SGB_LN2LO, __dadd_rn(__dsub_rn(w, hi), r));
  const double *A = sgb_log_poly;
  const double r2 = __dmul_rn(r, r);
  const double p = __fma_rn(r2, __fma_rn(r, A[4], A[3]), __fma_rn(r, A[2], A[1]));
  return __dadd_rn(__fma_rn(__dmul_rn(r, r2), p, __fma_rn(r2, A[0], lo)), hi);
}}

// exp's and pow's scaling near the ends of the range (k = round(x * 128 / ln2) out of [-1022, 1023] * 128)
__device__ __forceinline__ double sgb_exp_special(double tmp, unsigned long long sbits, unsigned long long ki, bool sgn) {{
  if ((ki & 0x80000000ull) == 0) {{
    const double scale = sgb_as_double(sbits - (1009ull << 52));
    return __dmul_rn(0x1p1009, __fma_rn(scale, tmp, scale));
  }}
  sbits += 1022ull << 52;
  const double scale = sgb_as_double(sbits);
  const double st = __dmul_rn(scale, tmp);  // two uses: not fused
  double y = __dadd_rn(scale, st);
  if ((sgn ? fabs(y) : y) < 1.0) {{
    const double one = (sgn && y < 0.0) ? -1.0 : 1.0;
    double lo = __dadd_rn(__dsub_rn(scale, y), st);
    const double hi = __dadd_rn(one, y);
    lo = __dadd_rn(__dadd_rn(__dsub_rn(one, hi), y), lo);
    y = __dsub_rn(__dadd_rn(hi, lo), one);
    if (y == 0.0) y = sgn ? sgb_as_double(sbits & 0x8000000000000000ull) : 0.0;
  }}
  return __dmul_rn(0x1p-1022, y);
}}

// exp (xtail unused, pow == false) and pow's exp_inline (x + xtail, sign_bias)
__device__ __forceinline__ double sgb_exp_core(double x, double xtail, unsigned sign_bias, bool pow_) {{
  unsigned abstop = (unsigned)(sgb_as_u64(x) >> 52) & 0x7ffu;
  if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {{  // |x| < 2^-54 or |x| >= 512 (or inf / nan)
    if (abstop - 0x3c9u >= 0x80000000u) {{
      const double one = __dadd_rn(1.0, x);
      return sign_bias ? -one : one;
    }}
    if (abstop >= 0x409u) {{
      if (!pow_) {{
        if (sgb_as_u64(x) == 0xfff0000000000000ull) return 0.0;
        if (abstop >= 0x7ffu) return __dadd_rn(1.0, x);
      }}
      if (sgb_as_u64(x) >> 63) return sign_bias ? -0.0 : 0.0;
      return sign_bias ? sgb_as_double(0xfff0000000000000ull) : sgb_as_double(0x7ff0000000000000ull);
    }}
    abstop = 0;  // large |x|: scaled below
  }}
  double kd = __fma_rn(SGB_EXP_INVLN2N, x, SGB_EXP_SHIFT);
  const unsigned long long ki = sgb_as_u64(kd);
  kd = __dsub_rn(kd, SGB_EXP_SHIFT);
  double r = __fma_rn(kd, SGB_EXP_NEGLN2LON, __fma_rn(kd, SGB_EXP_NEGLN2HIN, x));
  if (pow_) r = __dadd_rn(r, xtail);
  const unsigned idx = 2u * (unsigned)(ki % {N_TAB});
  const unsigned long long top = (ki + sign_bias) << (52 - 7);
  const double tail = sgb_as_double(sgb_exp_tab[idx]);
  const unsigned long long sbits = sgb_exp_tab[idx + 1] + top;
  const double *C = sgb_exp_poly;
  const double r2 = __dmul_rn(r, r);
  const double tmp = __fma_rn(__dmul_rn(r2, r2), __fma_rn(r, C[3], C[2]),
                              __fma_rn(r2, __fma_rn(r, C[1], C[0]), __dadd_rn(tail, r)));
  if (abstop == 0) return sgb_exp_special(tmp, sbits, ki, pow_);
  const double scale = sgb_as_double(sbits);
  return __fma_rn(scale, tmp, scale);
}}

__device__ __forceinline__ double sgb_exp(double x) {{ return sgb_exp_core(x, 0.0, 0u, false); }}

// 0: y not an integer, 1: odd integer, 2: even integer (y non-zero finite)
__device__ __forceinline__ int sgb_checkint(unsigned long long iy) {{
  const int e = (int)(iy >> 52 & 0x7ff);
  if (e < 0x3ff) return 0;
  if (e > 0x3ff + 52) return 2;
  if (iy & ((1ull << (0x3ff + 52 - e)) - 1)) return 0;
  if (iy & (1ull << (0x3ff + 52 - e))) return 1;
  return 2;
}}

__device__ __forceinline__ bool sgb_zeroinfnan(unsigned long long i) {{
  return 2 * i - 1 >= 2 * 0x7ff0000000000000ull - 1;
}}

__device__ __forceinline__ double sgb_pow(double x, double y) {{
  unsigned sign_bias = 0;
  unsigned long long ix = sgb_as_u64(x);
  const unsigned long long iy = sgb_as_u64(y);
  unsigned topx = (unsigned)(ix >> 52);
  const unsigned topy = (unsigned)(iy >> 52);
  if (topx - 0x001u >= 0x7ffu - 0x001u || (topy & 0x7ffu) - 0x3beu >= 0x43eu - 0x3beu) {{
    if (sgb_zeroinfnan(iy)) {{
      if (2 * iy == 0) return 1.0;
      if (ix == 0x3ff0000000000000ull) return 1.0;
      if (2 * ix > 2 * 0x7ff0000000000000ull || 2 * iy > 2 * 0x7ff0000000000000ull) return __dadd_rn(x, y);
      if (2 * ix == 2 * 0x3ff0000000000000ull) return 1.0;
      if ((2 * ix < 2 * 0x3ff0000000000000ull) == !(iy >> 63)) return 0.0;
      return __dmul_rn(y, y);
    }}
    if (sgb_zeroinfnan(ix)) {{
      double x2 = __dmul_rn(x, x);
      if ((ix >> 63) && sgb_checkint(iy) == 1) x2 = -x2;
      return (iy >> 63) ? __ddiv_rn(1.0, x2) : x2;
    }}
    if (ix >> 63) {{  // finite x < 0
      const int yint = sgb_checkint(iy);
      if (yint == 0) return sgb_as_double(0xfff8000000000000ull);  // x86 default NaN
      if (yint == 1) sign_bias = 0x800u << 7;
      ix &= 0x7fffffffffffffffull;
      topx &= 0x7ffu;
    }}
    if ((topy & 0x7ffu) - 0x3beu >= 0x43eu - 0x3beu) {{
      if (ix == 0x3ff0000000000000ull) return 1.0;
      if ((topy & 0x7ffu) < 0x3beu) return ix > 0x3ff0000000000000ull ? __dadd_rn(1.0, y) : __dsub_rn(1.0, y);
      return (ix > 0x3ff0000000000000ull) == (topy < 0x800u) ? sgb_as_double(0x7ff0000000000000ull) : 0.0;
    }}
    if (topx == 0) ix = (sgb_as_u64(__dmul_rn(sgb_as_double(ix), 0x1p52)) & 0x7fffffffffffffffull) - (52ull << 52);
  }}
  // log(x) as hi + lo (pow.c log_inline)
  const unsigned long long tmp = ix - {POW_OFF:#x}ull;
  const int i = (int)((tmp >> (52 - 7)) % {N_TAB});
  const long long k = (long long)tmp >> 52;
  const double z = sgb_as_double(ix - (tmp & (0xfffull << 52)));
  const double kd = (double)k;
  const double invc = sgb_pow_tab[3 * i], logc = sgb_pow_tab[3 * i + 1], logctail = sgb_pow_tab[3 * i + 2];
  const double r = __fma_rn(z, invc, -1.0);
  const double t1 = __fma_rn(kd, SGB_LN2HI, logc);
  const double t2 = __dadd_rn(t1, r);
  const double lo1 = __fma_rn(kd, SGB_LN2LO, logctail);
  const double lo2 = __dadd_rn(__dsub_rn(t1, t2), r);
  const double *A = sgb_pow_poly;
  const double ar = __dmul_rn(A[0], r), ar2 = __dmul_rn(r, ar), ar3 = __dmul_rn(r, ar2);
  const double hi = __dadd_rn(t2, ar2);
  const double lo3 = __fma_rn(ar, r, -ar2);
  const double lo4 = __dadd_rn(__dsub_rn(t2, hi), ar2);
  const double p = __dmul_rn(ar3, __fma_rn(ar2, __fma_rn(ar2, __fma_rn(r, A[6], A[5]), __fma_rn(r, A[4], A[3])),
                                          __fma_rn(r, A[2], A[1])));
  const double lo = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(lo1, lo2), lo3), lo4), p);
  const double lhi = __dadd_rn(hi, lo);
  const double llo = __dadd_rn(__dsub_rn(hi, lhi), lo);
  // y * log(x) as ehi + elo, then exp
  const double ehi = __dmul_rn(y, lhi);
  const double elo = __fma_rn(y, llo, __fma_rn(y, lhi, -ehi));
  return sgb_exp_core(ehi, elo, sign_bias, true);
}}

// ---- sin / cos (s_sin.c, FMA build; __branred for |x| >= 105414350) ----
__device__ const double sgb_sincostab[440] = {{  // (sin, sin tail, cos, cos tail) of k/128
{sct}}};
#define SGB_SC_BIG {K['BIG']}
#define SGB_SC_SMALL {K['SMALL']}

__device__ __forceinline__ double sgb_taylor_sin(double a, double da) {{
  const double xx = __dmul_rn(a, a);
  const double p = __fma_rn(xx, __fma_rn(xx, __fma_rn(xx, __fma_rn(xx, {K['S5']}, {K['S4']}), {K['S3']}), {K['S2']}), {K['S1']});
  return __dadd_rn(a, __fma_rn(xx, __fma_rn(p, a, -__dmul_rn(0.5, da)), da));
}}

__device__ __forceinline__ double sgb_do_sin(double x, double dx) {{
  if (!(x > 0)) dx = -dx;
  const double ax = fabs(x);
  const double u = __dadd_rn(ax, SGB_SC_BIG);
  const unsigned k = ((unsigned)sgb_as_u64(u)) << 2;
  const double xr = __dsub_rn(ax, __dsub_rn(u, SGB_SC_BIG));
  const double xx = __dmul_rn(xr, xr);
  const double s = __dadd_rn(xr, __fma_rn(__dmul_rn(xr, xx), __fma_rn(xx, {K['SN5']}, {K['SN3']}), dx));
  const double c = __fma_rn(dx, xr, __dmul_rn(xx, __fma_rn(xx, __fma_rn(xx, {K['CS6']}, {K['CS4']}), {K['CS2']})));
  const double sn = sgb_sincostab[k], ssn = sgb_sincostab[k + 1], cs = sgb_sincostab[k + 2], ccs = sgb_sincostab[k + 3];
  return copysign(__dadd_rn(sn, __fma_rn(s, cs, __fma_rn(-c, sn, __fma_rn(s, ccs, ssn)))), x);
}}

__device__ __forceinline__ double sgb_do_cos(double x, double dx) {{
  if (x < 0) dx = -dx;
  const double ax = fabs(x);
  const double u = __dadd_rn(ax, SGB_SC_BIG);
  const unsigned k = ((unsigned)sgb_as_u64(u)) << 2;
  const double xr = __dadd_rn(__dsub_rn(ax, __dsub_rn(u, SGB_SC_BIG)), dx);
  const double xx = __dmul_rn(xr, xr);
  const double s = __fma_rn(__dmul_rn(xr, xx), __fma_rn(xx, {K['SN5']}, {K['SN3']}), xr);
  const double c = __dmul_rn(xx, __fma_rn(xx, __fma_rn(xx, {K['CS6']}, {K['CS4']}), {K['CS2']}));
  const double sn = sgb_sincostab[k], ssn = sgb_sincostab[k + 1], cs = sgb_sincostab[k + 2], ccs = sgb_sincostab[k + 3];
  return __dadd_rn(cs, __fma_rn(-s, sn, __fma_rn(-c, cs, __fma_rn(-s, ssn, ccs))));
}}

__device__ __forceinline__ unsigned sgb_reduce(double x, double &a, double &da) {{
  const double t = __fma_rn(x, {K['HPINV']}, {K['TOINT']});
  const double xn = __dsub_rn(t, {K['TOINT']});
  const double y = __fma_rn(-xn, {K['MP2']}, __fma_rn(-xn, {K['MP1']}, x));
  const double t2 = __fma_rn(-xn, {K['PP3']}, y);
  const double db = __fma_rn(-xn, {K['PP3']}, __dsub_rn(y, t2));
  const double b = __fma_rn(-xn, {K['PP4']}, t2);
  a = b;
  da = __dadd_rn(db, __fma_rn(-xn, {K['PP4']}, __dsub_rn(t2, b)));
  return (unsigned)sgb_as_u64(t) & 3u;
}}

// __branred (branred.c, no FMA): |x| >= 105414350 reduced by pi/2 with 2/pi in 24-bit chunks
__device__ const double sgb_toverp[75] = {{
{toverp}}};

__device__ __noinline__ void sgb_branred_half(double xh, double &b_, double &bb_, double &sm_) {{
  const unsigned e = (unsigned)(sgb_as_u64(xh) >> 52) & 2047u;
  const int k = e >= 450u ? (int)((e - 450u) / 24u) : 0;
  double gor = sgb_as_double(sgb_as_u64({BR['T576']}) - ((unsigned long long)(k * 24) << 52));
  double r[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {{
    r[i] = __dmul_rn(__dmul_rn(xh, sgb_toverp[k + i]), gor);
    gor = __dmul_rn(gor, {BR['TM24']});
  }}
  double sm = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {{
    const double s = __dsub_rn(__dadd_rn(r[i], {BR['BIG']}), {BR['BIG']});
    sm = __dadd_rn(sm, s);
    r[i] = __dsub_rn(r[i], s);
  }}
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) t = __dadd_rn(t, r[5 - i]);
  double bb = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dsub_rn(r[0], t), r[1]), r[2]), r[3]), r[4]), r[5]);
  double s = __dsub_rn(__dadd_rn(t, {BR['BIG']}), {BR['BIG']});
  sm = __dadd_rn(sm, s);
  t = __dsub_rn(t, s);
  const double b = __dadd_rn(t, bb);
  bb = __dadd_rn(__dsub_rn(t, b), bb);
  s = __dsub_rn(__dadd_rn(sm, {BR['BIG1']}), {BR['BIG1']});
  b_ = b;
  bb_ = bb;
  sm_ = __dsub_rn(sm, s);
}}

__device__ __noinline__ unsigned sgb_branred(double x, double &a, double &da) {{
  x = __dmul_rn(x, {BR['TM600']});
  const double tt = __dmul_rn(x, {BR['SPLIT']});
  const double x1 = __dsub_rn(tt, __dsub_rn(tt, x));
  const double x2 = __dsub_rn(x, x1);
  double b1, bb1, s1, b2, bb2, s2;
  sgb_branred_half(x1, b1, bb1, s1);
  sgb_branred_half(x2, b2, bb2, s2);
  double sm = __dadd_rn(s1, s2);
  double b = __dadd_rn(b1, b2);
  double bb = fabs(b1) > fabs(b2) ? __dadd_rn(__dsub_rn(b1, b), b2) : __dadd_rn(__dsub_rn(b2, b), b1);
  if (b > 0.5) {{
    b = __dsub_rn(b, 1.0);
    sm = __dadd_rn(sm, 1.0);
  }} else if (b < -0.5) {{
    b = __dadd_rn(b, 1.0);
    sm = __dsub_rn(sm, 1.0);
  }}
  double s = __dadd_rn(b, __dadd_rn(__dadd_rn(bb, bb1), bb2));
  double t = __dadd_rn(__dadd_rn(__dsub_rn(b, s), bb), __dadd_rn(bb1, bb2));
  b = __dmul_rn(s, {BR['SPLIT']});
  const double t1 = __dsub_rn(b, __dsub_rn(b, s));
  const double t2 = __dsub_rn(s, t1);
  b = __dmul_rn(s, {BR['HP0']});
  bb = __dadd_rn(__dadd_rn(__dadd_rn(__dsub_rn(__dmul_rn(t1, {BR['MP1']}), b), __dmul_rn(t1, {BR['MP2']})),
                           __dmul_rn(t2, {BR['MP1']})),
                 __dadd_rn(__dadd_rn(__dmul_rn(t2, {BR['MP2']}), __dmul_rn(s, {BR['HP1']})), __dmul_rn(t, {BR['HP0']})));
  s = __dadd_rn(b, bb);
  t = __dadd_rn(__dsub_rn(b, s), bb);
  a = s;
  da = t;
  return (unsigned)(int)sm & 3u;
}}

__device__ __forceinline__ double sgb_do_sincos(double a, double da, unsigned n) {{
  const double r = (n & 1u) ? sgb_do_cos(a, da) : (fabs(a) < SGB_SC_SMALL ? sgb_taylor_sin(a, da) : sgb_do_sin(a, da));
  return (n & 2u) ? -r : r;
}}

__device__ __forceinline__ double sgb_sin(double x) {{
  const unsigned k = (unsigned)(sgb_as_u64(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) return fabs(x) < SGB_SC_SMALL ? sgb_taylor_sin(x, 0.0) : sgb_do_sin(x, 0.0);
  if (k < 0x400368fdu) return copysign(sgb_do_cos(__dsub_rn({K['HP0']}, fabs(x)), {K['HP1']}), x);
  if (k < {SINCOS_MAX_HI:#x}u) {{
    double a, da;
    const unsigned n = sgb_reduce(x, a, da);
    return sgb_do_sincos(a, da, n);
  }}
  if (k < 0x7ff00000u) {{
    double a, da;
    const unsigned n = sgb_branred(x, a, da);
    return sgb_do_sincos(a, da, n);
  }}
  return __ddiv_rn(x, x);
}}

__device__ __forceinline__ double sgb_cos(double x) {{
  const unsigned k = (unsigned)(sgb_as_u64(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return sgb_do_cos(x, 0.0);
  if (k < 0x400368fdu) {{
    const double y = __dsub_rn({K['HP0']}, fabs(x));
    const double a = __dadd_rn(y, {K['HP1']});
    const double da = __dadd_rn(__dsub_rn(y, a), {K['HP1']});
    return fabs(a) < SGB_SC_SMALL ? sgb_taylor_sin(a, da) : sgb_do_sin(a, da);
  }}
  if (k < {SINCOS_MAX_HI:#x}u) {{
    double a, da;
    const unsigned n = sgb_reduce(x, a, da);
    return sgb_do_sincos(a, da, n + 1u);
  }}
  if (k < 0x7ff00000u) {{
    double a, da;
    const unsigned n = sgb_branred(x, a, da);
    return sgb_do_sincos(a, da, n + 1u);
  }}
  return __ddiv_rn(x, x);
}}

#endif  // SGB_GLIBC_MATH_H
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=300000)
    args = ap.parse_args()
    path = libm_path()
    t = read_tables(path)
    bad = verify(t, args.samples)
    if bad:
        raise SystemExit(f"restatement differs from math on {len(bad)} samples, e.g. {bad[:5]}")
    OUT.write_text(header(t, str(path)))
    print(f"wrote {OUT} (sin / cos / exp / log / pow restatements bit-identical to math on {args.samples} samples each)")


if __name__ == "__main__":
    sys.exit(main())
