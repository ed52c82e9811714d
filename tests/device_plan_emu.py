"""CPU emulator of the lowered device plan (test-only).

Executes ``lower.DevicePlanArrays`` with numpy exactly as csrc/sgb.cu does --
waves in order, SOP groups by their factor masks, tape groups by their
register tape -- so the lowering (waves, tapes, register allocation, SOP
recognition, index decode) is proven bit-exact against the golden values on a
machine without a GPU.  Transcendentals use CPython's math (glibc), POW k>=3
uses the same double-double scheme as the device.
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

from paper_2110_12865_b200 import lower as L


def _decode_addrs(dp, g, i):
    n_slots = int(g["n_slots"])
    inter = bool(g["flags"] & L.FLAG_INTERLEAVED)
    cols = dp.slot_col[g["slot_off"]: g["slot_off"] + n_slots]
    dels = dp.slot_delta[g["slot_off"]: g["slot_off"] + n_slots]
    n, nret = int(g["n"]), int(g["n_ret"])
    if n_slots == 0:
        return []
    def column(col):
        if col == 0 and g["flags"] & L.FLAG_AFFINE0:
            return int(g["a0_base"]) + int(g["a0_stride"]) * np.asarray(i, dtype=np.int64)
        if g["flags"] & L.FLAG_W16:
            nch = (n + L.CHUNK - 1) // L.CHUNK
            base = dp.cbase[g["cb_off"] + col * nch + i // L.CHUNK].astype(np.int64)
            return base + dp.coff[g["co_off"] + col * n + i].astype(np.int64)
        e = g["p_off"] + (i * nret + col if inter else col * n + i)
        return dp.positions[e].astype(np.int64)

    idx0 = column(0)
    out = []
    for s in range(n_slots):
        col = int(cols[s])
        if col < 0:
            out.append(idx0 + int(dels[s]))
        elif col == 0:
            out.append(idx0)
        else:
            out.append(column(col))
    return out


def _const(dp, g, k, i):
    inter = bool(g["flags"] & L.FLAG_INTERLEAVED)
    n, nc = int(g["n"]), int(g["n_const"])
    e = g["c_off"] + (i * nc + k if inter else k * n + i)
    return dp.constants[e]


def _fma(a, b, c):
    """Correctly rounded a*b+c (Python 3.12 has no math.fma)."""
    if not (math.isfinite(a) and math.isfinite(b) and math.isfinite(c)):
        return a * b + c
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _dd_powi(xs, k):
    out = np.empty_like(xs)
    for j, x in enumerate(xs.tolist()):
        if k == 2:
            out[j] = x * x
            continue
        rh, rl, bh, bl = 1.0, 0.0, x, 0.0

        def mul(ah, al, bh_, bl_):
            p = ah * bh_
            e = _fma(ah, bh_, -p)
            e = e + (ah * bl_ + al * bh_)
            h = p + e
            return h, e - (h - p)

        kk = k
        while kk:
            if kk & 1:
                rh, rl = mul(rh, rl, bh, bl)
            kk >>= 1
            if kk:
                bh, bl = mul(bh, bl, bh, bl)
        r = rh + rl
        out[j] = r if math.isfinite(r) else rh
    return out


def _vec(fn, a):
    return np.array([fn(v) for v in a.tolist()], dtype=np.float64)


def run_values(dp, inputs) -> np.ndarray:
    x = np.zeros(dp.value_array_size, np.float64)
    x[: dp.input_count] = inputs
    for u in range(len(dp.units)):
        # groups of one wave are independent; units run in wave order
        unit = dp.unit(u)
        for gi in range(unit["group_begin"], unit["group_end"]):
            g = dp.groups[gi]
            n = int(g["n"])
            if g["flags"] & L.FLAG_SERIAL:
                for i in range(n):
                    _tape(dp, g, x, np.array([i]))
                continue
            i = np.arange(n, dtype=np.int64)
            if g["kind"] == L.KIND_SOP:
                nt = int(dp.sop[g["sop_off"]]) & 0xFFFFFFFF
                ng = int(dp.sop[g["sop_off"] + 1]) & 0xFFFFFFFF
                addrs = _decode_addrs(dp, g, i)
                acc = term = None
                for f in range(int(g["sop_len"])):
                    v = x[addrs[f]]
                    if (ng >> f) & 1:
                        v = -v
                    if (nt >> f) & 1:
                        if f > 0:
                            acc = term.copy() if acc is None else acc + term
                        term = v.copy()
                    else:
                        term = term * v
                res = term if acc is None else acc + term
                x[g["dest_base"] + i] = res
            else:
                _tape(dp, g, x, i)
    return x


def _tape(dp, g, x, i):
    n = int(g["n"])
    selfref = bool(g["flags"] & L.FLAG_SELFREF)
    phases = int(g["n_roots"]) if selfref else 1
    S, K = int(g["n_slots"]), int(g["n_const"])
    for ph in range(phases):
        R = [None] * int(g["n_regs"])
        for s, a in enumerate(_decode_addrs(dp, g, i)):
            R[s] = x[a].copy()
        for k in range(K):
            R[S + k] = _const(dp, g, k, i).copy()
        for word in dp.tape[g["tape_off"]: g["tape_off"] + g["tape_len"]].tolist():
            op, dst, a, b, c = L.decode(int(word))
            if op == L.T_ST:
                if not selfref or c == ph:
                    x[g["dest_base"] + c * n + i] = R[a]
                continue
            if op == L.T_IMM:
                v = np.full(len(i), dp.imm[b | (c << 14)])
            elif op == L.T_ADD:
                v = R[a] + R[b]
            elif op == L.T_SUB:
                v = R[a] - R[b]
            elif op == L.T_MUL:
                v = R[a] * R[b]
            elif op == L.T_DIV:
                with np.errstate(all="ignore"):
                    v = R[a] / R[b]
            elif op == L.T_NEG:
                v = -R[a]
            elif op == L.T_SQRT:
                with np.errstate(all="ignore"):
                    v = np.sqrt(R[a])
            elif op == L.T_SIN:
                v = _vec(math.sin, R[a])
            elif op == L.T_COS:
                v = _vec(math.cos, R[a])
            elif op == L.T_EXP:
                v = _vec(math.exp, R[a])
            elif op == L.T_LOG:
                v = _vec(math.log, R[a])
            elif op == L.T_POW:
                v = _dd_powi(R[a], c)
            elif op == L.T_SEL:
                v = np.where(R[a] < 0.0, R[b], R[c])
            else:
                raise ValueError(f"bad op {op}")
            R[dst] = v
