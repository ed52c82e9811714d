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
        if col < 0 or g["flags"] & L.FLAG_COHERENT:
            out.append(idx0 + int(dels[s]))
        elif col == 0:
            out.append(idx0)
        else:
            out.append(column(col))
    return out


def _out_pos(dp, g, r, i):
    """Output positions of root r (int64, -1 = not an output)."""
    n = int(g["n"])
    if g["flags"] & L.FLAG_OPOS16:
        nch = (n + L.CHUNK - 1) // L.CHUNK
        off = dp.ooff[g["oo_off"] + r * n + i].astype(np.int64)
        base = dp.obase[g["ob_off"] + r * nch + i // L.CHUNK].astype(np.int64)
        return np.where(off == 0xFFFF, -1, base + off)
    if g["flags"] & L.FLAG_OPOS32:
        o = dp.opos32[g["oo_off"] + r * n + i].astype(np.int64)
        return np.where(o == L.NONE32, -1, o)
    return np.full(len(i), -1, np.int64)


class _Store:
    """store_root of csrc/sgb.cu."""

    def __init__(self, dp, x, out):
        self.dp, self.x, self.out = dp, x, out

    def __call__(self, g, r, i, v):
        csr = self.out is not None
        if not (csr and g["flags"] & L.FLAG_STREAM):
            if g["flags"] & L.FLAG_IMAJOR:
                self.x[g["dest_base"] + np.asarray(i) * int(g["n_roots"]) + r] = v
            else:
                self.x[g["dest_base"] + r * int(g["n"]) + i] = v
        if csr:
            o = _out_pos(self.dp, g, r, i)
            m = o >= 0
            self.out[o[m]] = np.asarray(v)[m] if np.ndim(v) else v


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


def _glibc_pow(v, k):
    """math.pow (glibc) with IEEE overflow instead of Python's OverflowError; k == 2 is v * v."""
    if k == 2:
        return v * v
    try:
        return math.pow(v, float(k))
    except OverflowError:
        return math.copysign(math.inf, v) if k % 2 else math.inf


def _vec(fn, a):
    return np.array([fn(v) for v in a.tolist()], dtype=np.float64)


def check_tiles(dp):
    """Every (non-serial) group's instances are covered by exactly one tile of its unit."""
    for u in range(len(dp.units)):
        unit = dp.unit(u)
        t = dp.tiles[unit["tile_begin"]: unit["tile_end"]]
        for gi in range(unit["group_begin"], unit["group_end"]):
            g = dp.groups[gi]
            starts = np.sort(t[t[:, 0] == gi, 1].astype(np.int64))
            n = int(g["n"])
            if g["flags"] & L.FLAG_SERIAL:
                assert starts.tolist() == ([0] if n else [])
                continue
            if g["kind"] == L.KIND_SOP:
                tile = 32 * L.sop_vec(int(g["variant"]))
            else:
                tile = unit["block_size"] * unit["variant"]  # JIT units: block_size 256, variant 1
            assert starts.tolist() == list(range(0, n, tile)), (u, gi)


def _tile_instances(dp, unit, gi, g, n):
    """Instances of group ``gi`` its unit's tiles cover (a sharded tile table covers a subset)."""
    t = dp.tiles[unit["tile_begin"]: unit["tile_end"]]
    starts = np.sort(t[t[:, 0] == gi, 1].astype(np.int64))
    size = 32 * L.sop_vec(int(g["variant"])) if g["kind"] == L.KIND_SOP else unit["block_size"] * unit["variant"]
    if not starts.size:
        return np.zeros(0, np.int64)
    i = (starts[:, None] + np.arange(size, dtype=np.int64)[None, :]).reshape(-1)
    return i[i < n]


def _run_windows(dp, unit, x, out):
    """The CSR-window unit (jit.window_source): per window, copies then every member's piece, each
    result at its FLAG_WPOS16 position; the window is then stored at win_k[w]."""
    wn = dp.windows
    g0, g1 = unit["group_begin"], unit["group_end"]
    for w in range(wn.k.size - 1):
        k0, k1 = int(wn.k[w]), int(wn.k[w + 1])
        buf = np.full(k1 - k0, np.nan)
        c0, c1 = int(wn.copy_off[w]), int(wn.copy_off[w + 1])
        buf[wn.copy_pos[c0:c1].astype(np.int64)] = x[wn.copy_src[c0:c1].astype(np.int64)]
        for gi in range(g0, g1):
            a, cnt = (int(v) for v in wn.pieces[w, gi - g0])
            if not cnt:
                continue
            g = dp.groups[gi]
            i = np.arange(a, a + cnt, dtype=np.int64)
            n = int(g["n"])

            def wstore(g_, r, i_, v):
                o = dp.ooff[int(g_["oo_off"]) + r * n + i_].astype(np.int64)
                m = o != 0xFFFF
                buf[o[m]] = np.asarray(v)[m] if np.ndim(v) else v

            _reg_tape(dp, gi, g, x, i, wstore)
        out[k0:k1] = buf


def _run_windows_bulk(dp, unit, x, out):
    """The bulk-fed CSR-window unit (jit.wbulk_source) from its own tables: per window the ring slot
    is rebuilt from the consumer blob and the value-array intervals (lower.WindowBulk), the bulk
    members read their operands and window positions from it, the others from the value array."""
    wb, wn = dp.wbulk, dp.windows
    g0, g1 = unit["group_begin"], unit["group_end"]
    J = g1 - g0
    bulk = set(wb.members)
    NR = sum(int(dp.groups[g0 + j]["n_slots"]) for j in wb.members)
    NW = sum(int(dp.groups[g0 + j]["n_roots"]) for j in wb.members)
    xp = np.concatenate([x, [np.nan]]) if x.size % 2 else x  # the padding slot (sgb_plan_value_slots)
    for w in range(wn.k.size - 1):
        blob = wb.meta[int(wb.meta_off[w]): int(wb.meta_off[w + 1])]
        assert blob.size <= wb.slot_meta
        nc, csrc_at, cpos_at, ln = (int(v) for v in blob[:16].view(np.uint32))
        k0 = int(blob[16:24].view(np.int64)[0])
        nwp, xl = (int(v) for v in blob[24:32].view(np.uint32))
        assert k0 == int(wn.k[w]) and ln == int(wn.k[w + 1]) - k0
        sp = blob[32:32 + 8 * J].view(np.int32).reshape(J, 2)
        ivs = wb.iv[int(wb.iv_off[w]): int(wb.iv_off[w + 1])].astype(np.int64)
        X = np.concatenate([xp[s_: s_ + n_] for s_, n_ in ivs]) if len(ivs) else np.zeros(0)
        assert X.size == xl and 8 * xl <= wb.slot_x
        roff = blob[wb.roff_at: wb.roff_at + 2 * NR].view(np.uint16).astype(np.int64)
        woff = blob[wb.woff_at: wb.woff_at + 2 * NW].view(np.uint16).astype(np.int64)
        wps = blob[wb.wpos_at: wb.wpos_at + 2 * nwp].view(np.uint16).astype(np.int64)
        csrc = blob[csrc_at: csrc_at + 4 * nc].view(np.uint32).astype(np.int64)
        cpos = blob[cpos_at: cpos_at + 2 * nc].view(np.uint16).astype(np.int64)
        buf = np.full(ln, np.nan)
        ro = wo = 0
        for j in range(J):
            gi = g0 + j
            g = dp.groups[gi]
            a, cnt = int(sp[j, 0]), int(sp[j, 1])
            S, R = int(g["n_slots"]), int(g["n_roots"])
            if j in bulk:
                if cnt:
                    t = np.arange(cnt)
                    slots = [X[roff[ro + s_] + t] for s_ in range(S)]
                    wposs = [wps[woff[wo + r] + t] for r in range(R)]

                    def bstore(g_, r, i_, v, wposs=wposs):
                        o = wposs[r]
                        m = o != 0xFFFF
                        buf[o[m]] = np.asarray(v)[m] if np.ndim(v) else v

                    _reg_tape(dp, gi, g, x, np.arange(a, a + cnt, dtype=np.int64), bstore, slots=slots)
                ro += S
                wo += R
                continue
            if not cnt:
                continue
            n = int(g["n"])

            def wstore(g_, r, i_, v, n=n):
                o = dp.ooff[int(g_["oo_off"]) + r * n + i_].astype(np.int64)
                m = o != 0xFFFF
                buf[o[m]] = np.asarray(v)[m] if np.ndim(v) else v

            _reg_tape(dp, gi, g, x, np.arange(a, a + cnt, dtype=np.int64), wstore)
        buf[cpos] = x[csrc]
        out[k0:k0 + ln] = buf


def _run(dp, inputs, csr: bool, by_tiles: bool = False):
    x = np.zeros(dp.value_array_size, np.float64)
    x[: dp.input_count] = inputs
    out = np.full(len(dp.outputs), np.nan) if csr else None
    store = _Store(dp, x, out)
    for u in range(len(dp.units)):
        # groups of one unit are independent; units run in wave order
        unit = dp.unit(u)
        if unit["flags"] & L.UNIT_CSR_ONLY and not csr:
            continue
        if unit["flags"] & L.UNIT_VALUE_ONLY and csr:
            continue
        if unit["flags"] & L.UNIT_BULK:
            _run_windows_bulk(dp, unit, x, out)
            continue
        if unit["flags"] & L.UNIT_WINDOW:
            _run_windows(dp, unit, x, out)
            continue
        for gi in range(unit["group_begin"], unit["group_end"]):
            g = dp.groups[gi]
            if g["flags"] & L.FLAG_CSR_ONLY and not csr:
                continue
            n = int(g["n"])
            if g["flags"] & L.FLAG_SERIAL:
                for i in range(n):
                    _tape(dp, g, x, np.array([i]), store)
                continue
            i = _tile_instances(dp, unit, gi, g, n) if by_tiles else np.arange(n, dtype=np.int64)
            if unit["flags"] & L.UNIT_JIT:  # specialised unit: the group's register tape (jit.group_parts)
                _reg_tape(dp, gi, g, x, i, store)
                continue
            if g["kind"] == L.KIND_SOP:
                nt = int(dp.sop[2 * g["sop_off"]])
                ng = int(dp.sop[2 * g["sop_off"] + 1])
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
                store(g, 0, i, res)
            else:
                _tape(dp, g, x, i, store)
    return x, out


def run_values(dp, inputs) -> np.ndarray:
    return _run(dp, inputs, csr=False)[0]


def run_csr(dp, inputs, by_tiles: bool = False) -> np.ndarray:
    """CSR mode: direct stores by the producing groups and copy groups, CSR windows, or value mode +
    gather.  ``by_tiles``: evaluate only the instances the tile table covers (output-sharded plans)."""
    direct = bool(np.any(dp.groups["flags"] & (L.FLAG_OPOS16 | L.FLAG_OPOS32 | L.FLAG_WPOS16)))
    if not direct:
        return _run(dp, inputs, csr=False, by_tiles=by_tiles)[0][dp.outputs]
    return _run(dp, inputs, csr=True, by_tiles=by_tiles)[1]


def _tape(dp, g, x, i, store):
    """Decode the device tape words (lower.assemble) of this group's launch unit."""
    n = int(g["n"])
    unit = dp.unit(int(g["unit"]))
    if unit["flags"] & L.UNIT_JIT:
        raise ValueError("emulate with jit=False: specialised units carry no tape words")
    stride8 = unit["block_size"] * unit["variant"] * 8
    selfref = bool(g["flags"] & L.FLAG_SELFREF)
    phases = int(g["n_roots"]) if selfref else 1
    S, K = int(g["n_slots"]), int(g["n_const"])
    words = dp.tape[g["tape_off"]: g["tape_off"] + g["tape_len"]].astype(np.int64).tolist()
    slow = {0: math.sin, 1: math.cos, 2: math.exp, 3: math.log}
    for ph in range(phases):
        R = {}
        for s_, a in enumerate(_decode_addrs(dp, g, i)):
            R[s_] = x[a].copy()
        for k in range(K):
            R[S + k] = _const(dp, g, k, i).copy()
        for wx, wy, wz, ww in words:
            op, na, nb = (wx & 0xFF) >> 2, (wx >> 1) & 1, wx & 1
            c = ((wx >> 8) << 3) // stride8
            d, a, b = wy // stride8, wz // stride8, ww // stride8
            A = (lambda: -R[a] if na else R[a])
            Bv = (lambda: -R[b] if nb else R[b])
            with np.errstate(all="ignore"):
                if op == L.T_ST:
                    if not selfref or ww == ph:
                        store(g, ww, i, R[a])
                    continue
                if op == L.T_IMM:
                    v = np.full(len(i), dp.imm[ww])
                elif op == L.T_MUL:
                    v = A() * Bv()
                elif op == L.T_ADD:
                    v = A() + Bv()
                elif op == L.T_SUB:
                    v = A() - Bv()
                elif op == L.T_DIV:
                    v = A() / Bv()
                elif op == L.T_MADD:
                    v = (A() * Bv()) + R[c]
                elif op == L.T_MSUB:
                    v = (A() * Bv()) - R[c]
                elif op == L.T_RMSUB:
                    v = R[c] - (A() * Bv())
                elif op == L.T_NEG:
                    v = -R[a]
                elif op == L.T_SQRT:
                    v = np.sqrt(R[a])
                elif op == L.T_SEL:
                    v = np.where(R[a] < 0.0, R[b], R[c])
                elif op == L.T_SLOW:
                    kind, k = ww >> 16, ww & 0xFFFF
                    v = _vec(lambda v: _glibc_pow(v, k), R[a]) if kind == 4 else _vec(slow[kind], R[a])
                else:
                    raise ValueError(f"bad op {op}")
            R[d] = v


def _binop(op, A, B, C):
    if op == L.T_MUL:
        return A * B
    if op == L.T_ADD:
        return A + B
    if op == L.T_SUB:
        return A - B
    if op == L.T_DIV:
        return A / B
    if op == L.T_MADD:
        return (A * B) + C
    if op == L.T_MSUB:
        return (A * B) - C
    if op == L.T_RMSUB:
        return C - (A * B)
    raise ValueError(op)


def _reg_tape(dp, gi, g, x, i, store, slots=None):
    """A specialised unit's group: its register tape (lower.compile_tape), as jit.group_parts unrolls it.
    ``slots``: the operand values (a bulk-fed window member reads them from its ring slot)."""
    tape = dp.jit_tapes[gi]
    imms = dp.jit_imms[gi]
    S, K = int(g["n_slots"]), int(g["n_const"])
    R = {}
    for s_, a in enumerate(_decode_addrs(dp, g, i) if slots is None else slots):
        R[s_] = x[a].copy() if slots is None else np.asarray(a, np.float64)
    for k in range(K):
        R[S + k] = _const(dp, g, k, i).copy()
    slow = {0: math.sin, 1: math.cos, 2: math.exp, 3: math.log}
    z = np.zeros(len(i))
    for op, na, nb, dst, a, b, c, aux in tape.tolist():
        with np.errstate(all="ignore"):
            if op == L.T_ST:
                store(g, aux, i, R[a])
                continue
            A = -R.get(a, z) if na else R.get(a, z)
            B = -R.get(b, z) if nb else R.get(b, z)
            if op == L.T_IMM:
                v = np.full(len(i), imms[aux])
            elif op == L.T_NEG:
                v = -R[a]
            elif op == L.T_SQRT:
                v = np.sqrt(R[a])
            elif op == L.T_SEL:
                v = np.where(R[a] < 0.0, R[b], R[c])
            elif op == L.T_SLOW:
                kind, k = aux >> 16, aux & 0xFFFF
                v = _vec(lambda v: _glibc_pow(v, k), R[a]) if kind == 4 else _vec(slow[kind], R[a])
            else:
                v = _binop(op, A, B, R.get(c, z))
        R[dst] = v
