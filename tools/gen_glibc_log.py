"""Generate paper_2110_12865_b200/csrc/glibc_log.h: glibc's log(), restated for the device.

The reference evaluates LOG nodes with Python's ``math.log`` (codegen.py:545-557,
expr.py:423-484), i.e. the C library's ``log`` -- glibc 2.39 on this image, whose
implementation is the ARM optimized-routines algorithm (sysdeps/ieee754/dbl-64/
e_log.c): for |x - 1| < 2^-4 a degree-11 polynomial in r = x - 1 with an exact
split of r^2/2; otherwise x = 2^k z, a 128-entry table (1/c, log c) for the
subinterval of z, r = fma(z, 1/c, -1) and a degree-5 polynomial.  On x86-64 with
FMA, glibc runs its FMA build (ifunc), compiled with GCC's default
floating-point contraction: every product whose only use is an addition is fused.

This script reads the numeric tables of that algorithm (__log_data: ln2hi,
ln2lo, poly[5], poly1[11], tab[128] of (invc, logc)) out of the installed
libm.so.6, checks a Python restatement of the algorithm against ``math.log``
bit for bit on a large random sample (both paths, subnormals, extremes), and
writes the CUDA header that sgb.cu and the NVRTC kernels (jit.py) include.

    python tools/gen_glibc_log.py [--samples 400000]
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
OUT = ROOT / "paper_2110_12865_b200" / "csrc" / "glibc_log.h"
N_TAB = 128
LN2HI = float.fromhex("0x1.62e42fefa3800p-1")
LN2LO = float.fromhex("0x1.ef35793c76730p-45")


def libm_path() -> Path:
    for cand in ("/lib/x86_64-linux-gnu/libm.so.6", "/usr/lib/x86_64-linux-gnu/libm.so.6", ctypes.util.find_library("m")):
        if cand and Path(cand).exists():
            return Path(cand)
    raise SystemExit("libm.so.6 not found")


def read_log_data(path: Path):
    """__log_data: (ln2hi, ln2lo) followed by poly[5] (poly[0] ~ -0.5) and poly1[11] (poly1[0] == -0.5)."""
    data = path.read_bytes()
    head = struct.pack("<dd", LN2HI, LN2LO)
    start = 0
    while True:
        off = data.find(head, start)
        if off < 0:
            raise SystemExit("__log_data not found in libm")
        n = 2 + 5 + 11 + 2 * N_TAB
        v = struct.unpack_from(f"<{n}d", data, off)
        poly, poly1, tab = v[2:7], v[7:18], v[18:18 + 2 * N_TAB]
        if poly1[0] == -0.5 and abs(poly[0] + 0.5) < 1e-15 and 0.5 < tab[0] < 2.0:
            return poly, poly1, tab
        start = off + 1


def _fma(a, b, c):
    if not (math.isfinite(a) and math.isfinite(b) and math.isfinite(c)):
        return a * b + c
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _u64(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _f64(u):
    return struct.unpack("<d", struct.pack("<Q", u & 0xFFFFFFFFFFFFFFFF))[0]


def restated_log(x, A, B, T):
    """The algorithm, as the device implements it (fma where glibc's FMA build contracts)."""
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
    tmp = (ix - 0x3FE6000000000000) % 2 ** 64
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


def samples(n: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    q = n // 6
    parts = [rng.uniform(0.5, 2.0, q), rng.uniform(1 - 2 ** -4, 1 + 0.0646, q), np.exp(rng.uniform(-700, 700, q)),
             rng.uniform(1e-3, 1e3, q),
             np.frombuffer(rng.integers(1, 0x000FFFFFFFFFFFFF, q, dtype=np.uint64).tobytes(), np.float64),  # subnormal
             np.frombuffer(rng.integers(0x0010000000000000, 0x7FEFFFFFFFFFFFFF, n - 5 * q,
                                        dtype=np.uint64).tobytes(), np.float64)]
    return np.concatenate(parts)


def header(A, B, T, source: str) -> str:
    def lit(v):
        return f"{float(v).hex()}"  # C99 hex literal, exact

    rows = ",\n".join(f"    {lit(T[2 * j])}, {lit(T[2 * j + 1])}" for j in range(N_TAB))
    return f"""// GENERATED by tools/gen_glibc_log.py from {source} -- do not edit.
//
// sgb_log(x): glibc 2.39's log() (ARM optimized-routines algorithm, sysdeps/ieee754/dbl-64/e_log.c),
// restated for the device, FMA build (x86-64 glibc selects it by ifunc; GCC contracts every product
// whose only use is an addition).  The reference evaluates LOG with Python's math.log, i.e. this
// function (codegen.py:545-557), so LOG templates are bit-exact on the device.  The tables below are
// glibc's __log_data, read from the installed libm; the script checks the restatement against
// math.log bit for bit before writing this file.
#ifndef SGB_GLIBC_LOG_H
#define SGB_GLIBC_LOG_H

#define SGB_LOG_LN2HI {lit(LN2HI)}
#define SGB_LOG_LN2LO {lit(LN2LO)}
__device__ const double sgb_log_poly[5] = {{{", ".join(lit(a) for a in A)}}};
__device__ const double sgb_log_poly1[11] = {{{", ".join(lit(b) for b in B)}}};
__device__ const double sgb_log_tab[{2 * N_TAB}] = {{  // (1/c, log c) per subinterval
{rows}}};

__device__ __noinline__ double sgb_log(double x) {{
  unsigned long long ix = (unsigned long long)__double_as_longlong(x);
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
    if ((ix << 1) == 0) return __longlong_as_double((long long)0xfff0000000000000ull);  // log(+-0) = -inf
    if (ix == 0x7ff0000000000000ull) return x;                              // log(inf) = inf
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u)                      // x < 0 or NaN
      return isnan(x) ? __longlong_as_double((long long)(ix | 0x0008000000000000ull))
                      : __longlong_as_double((long long)0xfff8000000000000ull);  // x86 default NaN
    ix = (unsigned long long)__double_as_longlong(__dmul_rn(x, 0x1p52)) - (52ull << 52);  // subnormal
  }}
  const unsigned long long tmp = ix - 0x3fe6000000000000ull;
  const int i = (int)((tmp >> (52 - 7)) % {N_TAB});
  const long long k = (long long)tmp >> 52;
  const double z = __longlong_as_double((long long)(ix - (tmp & (0xfffull << 52))));
  const double invc = sgb_log_tab[2 * i], logc = sgb_log_tab[2 * i + 1];
  const double r = __fma_rn(z, invc, -1.0);
  const double kd = (double)k;
  const double w = __fma_rn(kd, SGB_LOG_LN2HI, logc);
  const double hi = __dadd_rn(w, r);
  const double lo = __fma_rn(kd, SGB_LOG_LN2LO, __dadd_rn(__dsub_rn(w, hi), r));
  const double *A = sgb_log_poly;
  const double r2 = __dmul_rn(r, r);
  const double p = __fma_rn(r2, __fma_rn(r, A[4], A[3]), __fma_rn(r, A[2], A[1]));
  return __dadd_rn(__fma_rn(__dmul_rn(r, r2), p, __fma_rn(r2, A[0], lo)), hi);
}}

#endif  // SGB_GLIBC_LOG_H
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=400000)
    args = ap.parse_args()
    path = libm_path()
    A, B, T = read_log_data(path)
    xs = samples(args.samples)
    bad = [x for x in xs.tolist() if not (np.array(restated_log(x, A, B, T)).view(np.uint64)
                                          == np.array(math.log(x) if x > 0 else np.nan).view(np.uint64))
           and not (math.isnan(restated_log(x, A, B, T)))]
    if bad:
        raise SystemExit(f"restated log differs from math.log on {len(bad)} of {len(xs)} samples, e.g. {bad[:3]}")
    OUT.write_text(header(A, B, T, str(path)))
    print(f"wrote {OUT} ({len(xs)} samples bit-identical to math.log)")


if __name__ == "__main__":
    sys.exit(main())
