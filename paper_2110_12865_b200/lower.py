"""Lowering an ``ExecutionPlan`` into the device plan the sm_100a kernels run.

Nothing here changes arithmetic: every template node keeps its op and its
stored child order (n-ary ADD / MUL fold left, expr.py:447-456,
codegen.py:472-481), so the device result is the reference result bit for
bit for every op in ``EXACT_OPS``.  What the lowering adds:

1. **Waves.**  ``wave(k) = 1 + max wave(producers of k)`` from the kernels'
   read sets (``slot_addresses``, codegen.py:373-388) against the result
   ranges ``[dest_base, dest_base + R*N)``; a kernel also waits for every
   earlier kernel that reads its range (a plan whose reads precede the
   writes -- the reference's write-before-read violations, codegen.py:434-443
   -- then still sees the zeros the interpreter sees).  All groups of one wave
   run in ONE launch with a block -> (group, instance range) table.
2. **Op tapes.**  One tape per template over the live nodes in ascending order
   (``reachable``, expr.py:608-611); position / constant slots are pre-loaded
   into scratch registers 0..S+K-1 (the hoisted loads of emit.py:108-124),
   CONST nodes become immediates, n-ary nodes become left-fold chains, and a
   linear-scan allocator recycles scratch registers after their last use.
3. **Sum-of-products fast path.**  Single-root templates of the form
   ``t0 + t1 + ...`` with every term a product of (optionally negated)
   position-slot loads, each slot used once in slot order, run through a
   tape-free kernel (``sop``); this covers sparse products, assembly sums and
   the L.M.L^T output groups.
4. **Index tables.**  The plan's u32 ``positions`` / f64 ``constants`` are
   uploaded unchanged (slot-major or interleaved); coherent slots become a
   per-slot ``delta`` on slot 0 (codegen.py:317-327).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from .plan import EXACT_OPS, OpKind, reachable, slot_addresses, unique_addresses

# ops the device reproduces bit for bit: the reference's _EXACT_OPS (codegen.py:43-53) and SIN / COS /
# EXP / LOG / POW (glibc's algorithms restated, csrc/glibc_math.h, __branred's large-argument
# reduction included)
DEVICE_EXACT_OPS = frozenset(EXACT_OPS) | {int(OpKind.SIN), int(OpKind.COS), int(OpKind.LOG), int(OpKind.EXP),
                                           int(OpKind.POW)}
KIND_TAPE, KIND_SOP = 0, 1
FLAG_SELFREF, FLAG_INTERLEAVED, FLAG_SERIAL, FLAG_EXACT, FLAG_STREAM, FLAG_W16 = 1, 2, 4, 8, 16, 32
FLAG_AFFINE0 = 64  # index column 0 is a0_base + a0_stride * i: no table read
FLAG_OPOS16 = 128  # output positions: u32 base per 32 instances + u16 offset (0xFFFF = not an output)
FLAG_OPOS32 = 256  # output positions: u32 per instance (0xFFFFFFFF = not an output)
FLAG_CSR_ONLY = 512  # synthetic copy group: runs in CSR mode only
FLAG_COHERENT = 1024  # one retained column: every slot is column 0 + delta
FLAG_IMAJOR = 2048  # CSR layout: result r of instance i at dest_base + i * n_roots + r (specialised units only)
FLAG_WPOS16 = 4096  # CSR-window member: root r of instance i goes to its window's position ooff[oo_off + r*n + i]
FLAG_KEEP = 8192  # specialised kernels store its results with an L2 evict_last hint (read soon by the window unit)
UNIT_CSR_ONLY = 1
STORE_ROOTS_EARLY = False  # roots stored as soon as computed (True) or at the end: C3 element kernel 0.318 vs 0.291 ms (c3v)
UNIT_JIT = 2  # tape unit compiled to straight-line code (jit.py), one instance per thread
UNIT_VALUE_ONLY = 4  # value-mode twin of a CSR-window unit (skipped by sgb_run_csr)
UNIT_WINDOW = 8  # CSR windows: each block assembles one window of consecutive outputs in shared memory
UNIT_BULK = 16  # CSR-window unit fed by bulk copies into a shared-memory ring (WindowBulk, jit.wbulk_source)
JIT_BLOCK = 256
CHUNK = 32  # instances per compressed-index chunk (one warp in single-set mode)
NONE32 = 0xFFFFFFFF
SOP_NEWTERM, SOP_NEG = 1, 2
SOP_MAX = 32  # factors per sum-of-products template (csrc SOP classes)
SOP_CLASSES = (2, 4, 8, 16, 32)  # width classes of the sum-of-products kernel (csrc sop_lmax)

# one record per group, mirrored by struct sgb_group in include/sgb.h
GROUP_DTYPE = np.dtype([
    ("n", "<i8"), ("dest_base", "<i8"), ("p_off", "<i8"), ("c_off", "<i8"),
    ("tape_off", "<i8"), ("cb_off", "<i8"), ("co_off", "<i8"),
    ("a0_base", "<i8"), ("a0_stride", "<i8"), ("ob_off", "<i8"), ("oo_off", "<i8"),
    ("n_roots", "<i4"), ("n_slots", "<i4"), ("n_ret", "<i4"), ("n_const", "<i4"),
    ("tape_len", "<i4"), ("n_regs", "<i4"), ("kind", "<i4"), ("flags", "<i4"),
    ("slot_off", "<i4"), ("sop_off", "<i4"), ("sop_len", "<i4"), ("unit", "<i4"),
    ("variant", "<i4"), ("shape", "<i4"),
])

# one row per launch unit (int64 x 10), mirrored by csrc U_*
UNIT_FIELDS = ("wave", "kind", "variant", "group_begin", "group_end", "tile_begin", "tile_end",
               "block_size", "smem_regs", "flags")
assert GROUP_DTYPE.itemsize == 144


@dataclass
class KernelLowering:
    index: int
    name: str
    kind: int
    flags: int
    n_regs: int
    tape: np.ndarray  # (L,) uint64 tape words
    imms: list
    sop: np.ndarray  # (F,) int32 descriptors
    slot_col: np.ndarray  # int32, retained column or -1
    slot_delta: np.ndarray  # int64
    wave: int = 0
    ops: int = 0  # FP64 op count per instance


@dataclass
class DevicePlanArrays:
    """Host-side device plan: flat arrays handed to sgb_plan_create."""

    groups: np.ndarray  # GROUP_DTYPE, ordered by (wave, launch unit)
    units: np.ndarray  # int64 [n_units, 10], UNIT_FIELDS
    tiles: np.ndarray  # int32 [n_tiles, 2]: group, first instance (one block each, launch order)
    n_waves: int  # value-mode waves (a CSR-only unit may use wave n_waves)
    tape: np.ndarray  # (L, 4) u32 device words, byte offsets of each group's unit stride
    imm: np.ndarray  # f64
    sop: np.ndarray  # u32 pairs (newterm mask, negate mask)
    slot_col: np.ndarray  # int32
    slot_delta: np.ndarray  # int64
    cbase: np.ndarray  # u32 per (column, 32-instance chunk) base of compressed columns
    coff: np.ndarray  # u16 per (column, instance) offset from its chunk base
    obase: np.ndarray  # u32 per (root, chunk) base of output positions
    ooff: np.ndarray  # u16 per (root, instance) output-position offset, 0xFFFF = none
    opos32: np.ndarray  # u32 wide output positions
    positions: np.ndarray  # u32: the plan's table, unchanged, then copy-group columns
    constants: np.ndarray  # f64 (the plan's table, unchanged)
    outputs: np.ndarray  # int64
    value_array_size: int
    input_count: int
    needs_zero: int = 2  # ZERO_NONE / ZERO_ONCE / ZERO_EVERY
    kernels: list = field(default_factory=list)
    copies: list = field(default_factory=list)  # (wave, source addresses, CSR positions) per copy group
    exact: bool = True
    jit_cubin: bytes = b""  # specialised tape units (UNIT_JIT): kernels sgb_tape_u<unit>, see jit.py
    jit_source: str = ""
    windows: "CsrWindows" = None  # CSR windows of the last wave (the window unit's pieces and copies)
    wbulk: "WindowBulk" = None  # bulk-copy feed of the window unit (UNIT_BULK), see window_bulk
    jit_split: dict = field(default_factory=dict)  # group -> per part the tape records it evaluates
    window_members: list = field(default_factory=list)  # plan kernels the window unit evaluates
    window_units: list = field(default_factory=list)
    jit_tapes: dict = field(default_factory=dict)  # packed group -> register tape of specialised units
    jit_imms: dict = field(default_factory=dict)
    csr_layout: list = field(default_factory=list)  # plan kernels stored instance-major (FLAG_IMAJOR)
    # the same tiles with every multi-group specialised unit in fraction-interleaved order (None when
    # no unit has a second candidate); DevicePlan times both schedules per wave (runtime.autotune)
    tiles_alt: np.ndarray = None

    def unit(self, u: int) -> dict:
        return dict(zip(UNIT_FIELDS, (int(v) for v in self.units[u])))

    @property
    def csr_waves(self) -> int:
        return max([self.n_waves] + [int(w) + 1 for w in self.units[:, 0]]) if len(self.units) else self.n_waves


# -- waves ----------------------------------------------------------------------


def _read_sets(plan):
    """Per kernel: sorted unique addresses >= input_count it loads."""
    out = []
    for kp in plan.kernels:
        cols = slot_addresses(plan, kp)
        if cols:
            a = np.concatenate(cols)
            a = unique_addresses(a[a >= plan.input_count])
        else:
            a = np.zeros(0, np.int64)
        out.append(a)
    return out


def compute_waves(plan, read_sets=None) -> list[int]:
    """Dependency waves (producer-before-consumer, and readers-before-writers)."""
    ks = plan.kernels
    if not ks:
        return []
    read_sets = read_sets if read_sets is not None else _read_sets(plan)
    starts = np.array([kp.dest_base for kp in ks], np.int64)
    ends = np.array([kp.dest_base + kp.n_roots * kp.instances for kp in ks], np.int64)
    order = np.argsort(starts, kind="stable")
    s_sorted = starts[order]
    e_sorted = ends[order]
    # map every read address to the kernel whose result range holds it
    readers_of: list[set] = [set() for _ in ks]
    producers_of: list[set] = [set() for _ in ks]
    for k, addrs in enumerate(read_sets):
        if not addrs.size:
            continue
        pos = np.searchsorted(s_sorted, addrs, side="right") - 1
        ok = pos >= 0
        pos_ok = pos[ok]
        inside = addrs[ok] < e_sorted[pos_ok]
        owners = np.unique(order[pos_ok[inside]])
        for o in owners.tolist():
            if o != k:
                producers_of[k].add(o)
                readers_of[o].add(k)
    wave = [0] * len(ks)
    for k in range(len(ks)):
        w = 0
        for p in producers_of[k]:
            if p < k:
                w = max(w, wave[p] + 1)
        # an earlier kernel reading this range must see it unwritten
        for r in readers_of[k]:
            if r < k:
                w = max(w, wave[r] + 1)
        wave[k] = w
    return wave


# -- tapes ----------------------------------------------------------------------
#
# A tape is a list of register-level instructions (one numpy record each):
#   op, dst, a, b, c   registers; nega / negb flip the sign of operand a / b
#   aux                immediate index (IMM), root index (ST), kind<<16|k (SLOW)
# Fusions (all arithmetic-neutral: each op is still one IEEE-rounded operation):
#   * a single-use NEG child becomes an operand sign flag of its consumer
#     (-x is exact, so (-a)*b == -(a*b) bit for bit);
#   * a single-use binary MUL feeding an ADD / SUB step becomes MADD / MSUB /
#     RMSUB: d = round(round(a*b) +- c) -- two roundings, never an FMA.
# At packing time every tape is assembled into 16-byte device words with the
# shared-memory byte offsets of its launch unit (no decode in the kernel).

# device op codes (csrc/sgb.cu keeps the same numbering)
T_MUL, T_ADD, T_SUB, T_DIV, T_MADD, T_NEG, T_SQRT, T_SEL, T_IMM, T_ST, T_SLOW, T_MSUB, T_RMSUB = range(13)
SLOW_KIND = {int(OpKind.SIN): 0, int(OpKind.COS): 1, int(OpKind.EXP): 2, int(OpKind.LOG): 3, int(OpKind.POW): 4}
REG_MAX = 4095  # registers per template (scratch byte offsets fit the 24-bit device fields)

TAPE_DTYPE = np.dtype([("op", "u1"), ("nega", "u1"), ("negb", "u1"), ("dst", "<u4"), ("a", "<u4"),
                       ("b", "<u4"), ("c", "<u4"), ("aux", "<u4")])


class _RegAlloc:
    def __init__(self, reserved: int):
        self.free: list[int] = []
        self.top = reserved

    def get(self) -> int:
        if self.free:
            return self.free.pop()
        r = self.top
        self.top += 1
        return r

    def put(self, r: int) -> None:
        self.free.append(r)


def compile_tape(kp):
    """Template -> (tape records, immediates, n_regs, fp64 ops/instance).

    Registers 0..S-1 hold the position slots, S..S+K-1 the constant slots
    (loaded by the kernel prologue); temporaries are recycled after their
    last use (linear scan over the ascending live order).
    """
    tmpl = kp.template_arena
    roots = list(kp.template_roots)
    live = reachable(tmpl, roots)
    ops, args, payload = tmpl.ops, tmpl.args, tmpl.payload
    slot_of = {v: s for s, v in enumerate(kp.pos_vars)}
    cslot_of = {v: s for s, v in enumerate(kp.const_vars)}
    S, K = len(kp.pos_vars), len(kp.const_vars)
    if S + K > REG_MAX:
        raise ValueError(f"{kp.name}: {S + K} slots exceed the tape register space")
    root_set = set(roots)
    uses: dict[int, int] = {}
    for ref in live:
        for c in args[ref]:
            uses[c] = uses.get(c, 0) + 1

    def single(ref):
        return uses.get(ref, 0) == 1 and ref not in root_set

    # fusion decisions: NEG folded into its single consumer, MUL folded into ADD/SUB
    arith = (OpKind.ADD, OpKind.SUB, OpKind.MUL, OpKind.DIV)
    consumer_op: dict[int, int] = {}
    for ref in live:
        for c in args[ref]:
            consumer_op[c] = int(ops[ref])
    fold_neg = {ref for ref in live if int(ops[ref]) == OpKind.NEG and single(ref)
                and consumer_op.get(ref) in arith}
    fold_mul = set()
    for ref in live:
        op = int(ops[ref])
        if op in (OpKind.ADD, OpKind.SUB):
            for ch in args[ref]:
                if int(ops[ch]) == OpKind.MUL and len(args[ch]) == 2 and single(ch):
                    fold_mul.add(ch)
    order = {ref: j for j, ref in enumerate(live)}
    consumers: dict[int, list[int]] = {}
    for ref in live:
        for c in args[ref]:
            consumers.setdefault(c, []).append(ref)
    # effective position of a node = where its value is actually consumed
    # (a folded node is evaluated inside its consumer's instruction)
    eff: dict[int, int] = {}
    for ref in reversed(live):
        if ref in fold_mul or ref in fold_neg:
            eff[ref] = max(eff.get(p, order[p]) for p in consumers[ref])
        else:
            eff[ref] = order[ref]
    last_use: dict[int, int] = {}
    for ref in live:
        for c in args[ref]:
            last_use[c] = max(last_use.get(c, -1), eff[ref])
    ra = _RegAlloc(S + K)
    reg: dict[int, int] = {}
    recs: list[tuple] = []
    imms: list[float] = []
    imm_of: dict[int, int] = {}
    fops = 0

    def emit(op, dst=0, a=0, b=0, c=0, aux=0, nega=0, negb=0):
        recs.append((op, nega, negb, dst, a, b, c, aux))

    def operand(ch):
        """(register, negated) of a child, looking through folded NEGs."""
        neg = 0
        while ch in fold_neg:
            neg ^= 1
            ch = args[ch][0]
        return reg[ch], neg

    def factors(m):
        (ra_, na), (rb_, nb) = operand(args[m][0]), operand(args[m][1])
        return ra_, rb_, na, nb

    def add_step(dst, left, right, sub=False):
        """dst = left +- right; left is a child ref or ('r', register)."""
        l_fm = not isinstance(left, tuple) and left in fold_mul
        r_fm = right in fold_mul
        if l_fm and not r_fm:  # (a*b) +- c
            ma, mb, na, nb = factors(left)
            rr, rn = operand(right)
            if rn:
                emit(T_NEG, dst, rr)
                rr = dst
            emit(T_MSUB if sub else T_MADD, dst, ma, mb, rr, nega=na, negb=nb)
            return
        if r_fm:  # c +- (a*b); a folded left product is materialised first
            if l_fm:
                ma, mb, na, nb = factors(left)
                emit(T_MUL, dst, ma, mb, nega=na, negb=nb)
                lr = dst
            elif isinstance(left, tuple):
                lr = left[1]
            else:
                lr, ln = operand(left)
                if ln:
                    emit(T_NEG, dst, lr)
                    lr = dst
            ma, mb, na, nb = factors(right)
            emit(T_RMSUB if sub else T_MADD, dst, ma, mb, lr, nega=na, negb=nb)
            return
        lr, ln = (left[1], 0) if isinstance(left, tuple) else operand(left)
        rr, rn = operand(right)
        emit(T_SUB if sub else T_ADD, dst, lr, rr, nega=ln, negb=rn)

    # STORE_ROOTS_EARLY: every root is stored right after it is computed, so a multi-root template
    # does not keep all of its roots live until the last one (fewer registers; measured slower on C3's
    # 78-root element Hessian, whose stores then interleave with the computes)
    root_idx: dict[int, list[int]] = {}
    for r_idx, root in enumerate(roots):
        root_idx.setdefault(root, []).append(r_idx)
    stored: set = set()

    def store_roots(ref):
        if not STORE_ROOTS_EARLY:
            return
        for r_idx in root_idx.get(ref, ()):
            emit(T_ST, 0, reg[ref], aux=r_idx)
        stored.add(ref)

    for ref in live:
        op = int(ops[ref])
        a = args[ref]
        if op == OpKind.VAR:
            v = payload[ref]
            reg[ref] = slot_of[v] if v in slot_of else S + cslot_of[v]
            continue
        if ref in fold_neg or ref in fold_mul:
            if ref in fold_mul:
                fops += 1
            continue
        if op == OpKind.CONST:
            bits = np.float64(payload[ref]).view(np.uint64).item()
            if bits not in imm_of:
                imm_of[bits] = len(imms)
                imms.append(float(payload[ref]))
            d = ra.get()
            emit(T_IMM, d, aux=imm_of[bits])
            reg[ref] = d
            if ref in root_set:
                store_roots(ref)
            continue
        d = ra.get()
        if op == OpKind.ADD:
            add_step(d, a[0], a[1])
            for ch in a[2:]:
                add_step(d, ("r", d), ch)
            fops += len(a) - 1
        elif op == OpKind.SUB:
            add_step(d, a[0], a[1], sub=True)
            fops += 1
        elif op == OpKind.MUL:
            (ra_, na), (rb_, nb) = operand(a[0]), operand(a[1])
            emit(T_MUL, d, ra_, rb_, nega=na, negb=nb)
            for ch in a[2:]:
                rc_, nc = operand(ch)
                emit(T_MUL, d, d, rc_, negb=nc)
            fops += len(a) - 1
        elif op == OpKind.DIV:
            (ra_, na), (rb_, nb) = operand(a[0]), operand(a[1])
            emit(T_DIV, d, ra_, rb_, nega=na, negb=nb)
            fops += 1
        elif op == OpKind.NEG:
            emit(T_NEG, d, reg[a[0]])
            fops += 1
        elif op == OpKind.SQRT:
            emit(T_SQRT, d, reg[a[0]])
            fops += 1
        elif op in (OpKind.SIN, OpKind.COS, OpKind.EXP, OpKind.LOG):
            emit(T_SLOW, d, reg[a[0]], aux=SLOW_KIND[op] << 16)
            fops += 1
        elif op == OpKind.POW:
            emit(T_SLOW, d, reg[a[0]], aux=(SLOW_KIND[op] << 16) | int(payload[a[1]]))
            fops += 1
        elif op == OpKind.SELECT:
            emit(T_SEL, d, reg[a[0]], reg[a[1]], reg[a[2]])
            fops += 1
        else:
            raise ValueError(f"{kp.name}: unknown op {op}")
        reg[ref] = d
        if ref in root_set:
            store_roots(ref)
        # recycle temporaries after their last use (slot registers stay pinned; roots are stored)
        dead = set()
        stack = list(a)
        while stack:
            ch = stack.pop()
            if ch in fold_neg or ch in fold_mul:
                stack.extend(args[ch])
                continue
            dead.add(ch)
        for ch in dead:
            if last_use.get(ch) is not None and last_use[ch] <= order[ref] and (ch not in root_set or ch in stored) \
                    and ch in reg and reg[ch] >= S + K and int(ops[ch]) != OpKind.VAR and reg[ch] != d:
                ra.put(reg[ch])
                reg[ch] = -1 - reg[ch]  # mark released (never released twice)
        if ra.top > REG_MAX:
            raise ValueError(f"{kp.name}: template needs more than {REG_MAX} scratch registers")
    for r_idx, root in enumerate(roots):  # roots that are slots (never computed)
        if root not in stored:
            emit(T_ST, 0, reg[root] if reg[root] >= 0 else -1 - reg[root], aux=r_idx)
    tape = np.array(recs, dtype=TAPE_DTYPE) if recs else np.zeros(0, TAPE_DTYPE)
    return tape, imms, max(ra.top, 1), fops


def assemble(tape: np.ndarray, stride: int, imm_base: int) -> np.ndarray:
    """Register tape -> device words (u32 x4): byte offsets for scratch stride ``stride``.

    x = op<<2 | nega<<1 | negb | (c*stride) << 8;  y = dst*stride*8;
    z = a*stride*8;  w = b*stride*8, or the immediate index (IMM, plan-wide),
    the root index (ST) or kind<<16 | k (SLOW).
    """
    if tape.size == 0:
        return np.zeros((0, 4), np.uint32)
    op = tape["op"].astype(np.uint64)
    by = np.uint64(stride * 8)
    if int(max(tape["c"].max(), tape["dst"].max(), tape["a"].max(), tape["b"].max())) * stride >= 1 << 24:
        raise ValueError("scratch offsets exceed the 24-bit device field")
    x = (op << np.uint64(2)) | (tape["nega"].astype(np.uint64) << np.uint64(1)) | tape["negb"].astype(np.uint64) \
        | ((tape["c"].astype(np.uint64) * np.uint64(stride)) << np.uint64(8))
    y = tape["dst"].astype(np.uint64) * by
    z = tape["a"].astype(np.uint64) * by
    wv = tape["b"].astype(np.uint64) * by
    special = np.isin(tape["op"], [T_IMM, T_ST, T_SLOW])
    aux = tape["aux"].astype(np.uint64)
    aux = np.where(tape["op"] == T_IMM, aux + np.uint64(imm_base), aux)
    wv = np.where(special, aux, wv)
    return np.stack([x, y, z, wv], axis=1).astype(np.uint32)


def _flatten(tmpl, ref, op):
    """Left-nested chain of ``op`` -> flat child list (bit-identical fold)."""
    out = []
    while int(tmpl.ops[ref]) == op:
        a = tmpl.args[ref]
        out = list(a[1:]) + out
        ref = a[0]
    return [ref] + out


def recognise_sop(kp):
    """Factor descriptors when the template is a sum of products of slot loads.

    Returns None when the template does not qualify.  The fold order is the
    template's: terms left to right, factors left to right, and ``-(a*b)``
    becomes ``(-a)*b`` (round-to-nearest is sign-symmetric, so this is exact).
    """
    if kp.n_roots != 1 or kp.self_referencing or kp.const_vars:
        return None
    tmpl = kp.template_arena
    ops, args, payload = tmpl.ops, tmpl.args, tmpl.payload
    slot_of = {v: s for s, v in enumerate(kp.pos_vars)}
    root = kp.template_roots[0]
    terms = _flatten(tmpl, root, OpKind.ADD) if int(ops[root]) == OpKind.ADD else [root]
    desc = []
    for t in terms:
        neg = False
        if int(ops[t]) == OpKind.NEG and int(ops[args[t][0]]) == OpKind.MUL:
            neg = True
            t = args[t][0]
        factors = _flatten(tmpl, t, OpKind.MUL) if int(ops[t]) == OpKind.MUL else [t]
        for j, f in enumerate(factors):
            fneg = neg and j == 0
            if int(ops[f]) == OpKind.NEG:
                fneg = not fneg
                f = args[f][0]
            if int(ops[f]) != OpKind.VAR or payload[f] not in slot_of:
                return None
            s = slot_of[payload[f]]
            if s != len(desc):
                return None  # each slot exactly once, in slot order
            desc.append((SOP_NEWTERM if j == 0 else 0) | (SOP_NEG if fneg else 0))
    if len(desc) != len(kp.pos_vars) or not 1 <= len(desc) <= SOP_MAX:
        return None
    return np.asarray(desc, np.int32)


def lower_kernel(plan, kp, index: int) -> KernelLowering:
    tmpl = kp.template_arena
    live = reachable(tmpl, kp.template_roots)
    exact = all(int(tmpl.ops[i]) in DEVICE_EXACT_OPS for i in live)
    flags = (FLAG_SELFREF if kp.self_referencing else 0) | \
            (FLAG_INTERLEAVED if kp.layout == "interleaved" else 0) | (FLAG_EXACT if exact else 0)
    ridx = {s: k for k, s in enumerate(kp.retained)}
    slot_col = np.array([ridx.get(s, -1) for s in range(len(kp.pos_vars))], np.int32)
    slot_delta = np.array([0 if s in ridx else int(c) for s, c in enumerate(kp.coherence)], np.int64)
    sop = recognise_sop(kp)
    tape, imms, n_regs, fops = compile_tape(kp)
    if kp.self_referencing:
        # a member reading ANOTHER instance's result needs instance order
        lo, hi = kp.dest_base, kp.dest_base + kp.n_roots * kp.instances
        for col in slot_addresses(plan, kp):
            inside = (col >= lo) & (col < hi)
            if inside.any():
                inst = (col[inside] - lo) % kp.instances
                if not np.array_equal(inst, np.arange(kp.instances)[inside]):
                    flags |= FLAG_SERIAL
                    break
    if sop is not None:  # the tape is kept: specialised units (jit.py) compile every group from its tape
        return KernelLowering(index, kp.name, KIND_SOP, flags, n_regs, tape, imms,
                              sop, slot_col, slot_delta, ops=fops)
    return KernelLowering(index, kp.name, KIND_TAPE, flags, n_regs, tape, imms,
                          np.zeros(0, np.int32), slot_col, slot_delta, ops=fops)


# -- packing ----------------------------------------------------------------------

TAPE_BLOCK = 128
SOP_BLOCK = 256
SMEM_LIMIT = 200 * 1024
TAPE_VECS = (4, 2, 1)  # instances per thread of the tape interpreter, largest that fits
VEC_SMEM_BUDGET = 104 * 1024  # per block: keeps >= 2 tape blocks resident per SM


def sop_class(width: int) -> int:
    for c, lim in enumerate(SOP_CLASSES):
        if width <= lim:
            return c
    raise ValueError(f"sum-of-products width {width} exceeds {SOP_MAX}")


def sop_vec(cls: int) -> int:
    """Instances per thread of the sum-of-products kernel (csrc sop_vec)."""
    return (4, 4, 2, 1, 1)[cls]


SOP_SHAPE_GENERIC, SOP_SHAPE_SUM, SOP_SHAPE_PAIRS = 0, 1, 2


SOP_GENERAL_CODE = 64  # csrc SOP_GENERAL_CODE


def sop_unit_code(g, compress: bool) -> int:
    """Kernel of a sum-of-products group: fast path shape * 8 + width class, or the general kernel."""
    cls = sop_class(len(g.sop))
    fast = (compress and g.layout == "coalesced" and len(g.columns) == 1 and cls <= 3
            and affine_column0(g.columns[0]) is not None and -2**31 <= g_stride(g) < 2**31)
    return sop_shape(g.sop) * 8 + cls if fast else SOP_GENERAL_CODE


def g_stride(g) -> int:
    c = g.columns[0]
    return int(c[1] - c[0]) if len(c) > 1 else 0


def sop_shape(desc) -> int:
    """Kernel shape of a sum-of-products descriptor (csrc SHAPE_*); arithmetic is identical."""
    starts = [bool(d & SOP_NEWTERM) for d in np.asarray(desc).tolist()]
    n = len(starts)
    if all(starts):
        return SOP_SHAPE_SUM
    if n >= 2 and all(starts[f] == (f % 2 == 0) for f in range(n - (n & 1))) and (n % 2 == 0 or starts[-1]):
        return SOP_SHAPE_PAIRS
    return SOP_SHAPE_GENERIC


def block_size_for(n_regs: int) -> int:
    """Largest tape block (128, 64 or 32 lanes) whose scratch file fits shared memory."""
    bs = TAPE_BLOCK
    while bs > 32 and n_regs * bs * 8 > SMEM_LIMIT:
        bs //= 2
    return bs


def compress_column(col: np.ndarray, allow_none: bool = False):
    """Per-chunk base + u16 offset encoding of one index column (u32 values).

    Entry i decodes to ``base[i // 32] + off[i]``.  With ``allow_none``
    entries equal to NONE32 become offset 0xFFFF (skipped by the kernel).
    Returns None when some chunk spans 0xFFFF addresses or more.
    """
    col = np.asarray(col, dtype=np.int64)
    n = col.size
    nch = (n + CHUNK - 1) // CHUNK
    pad = nch * CHUNK - n
    none = col == NONE32 if allow_none else np.zeros(n, bool)
    big = np.iinfo(np.int64).max
    lo_src = np.where(none, big, col)
    hi_src = np.where(none, -1, col)
    lo = np.concatenate([lo_src, np.full(pad, big)]).reshape(nch, CHUNK).min(axis=1)
    hi = np.concatenate([hi_src, np.full(pad, -1)]).reshape(nch, CHUNK).max(axis=1)
    empty = hi < 0
    lo = np.where(empty, 0, lo)
    if nch and int((hi - lo)[~empty].max(initial=0)) >= 0xFFFF:
        return None
    off = col - np.repeat(lo, CHUNK)[:n]
    off = np.where(none, 0xFFFF, off)
    return lo.astype(np.uint32), off.astype(np.uint16)


def affine_column0(col0: np.ndarray):
    """(base, stride) when index column 0 is exactly base + stride * i, else None."""
    n = col0.size
    if n < 2:
        return None
    c0 = np.asarray(col0, dtype=np.int64)
    base, stride = int(c0[0]), int(c0[1] - c0[0])
    if np.array_equal(c0, base + stride * np.arange(n, dtype=np.int64)):
        return base, stride
    return None


@dataclass
class _Group:
    """One device group before packing: a plan kernel or a synthetic copy group."""

    kind: int
    flags: int
    n: int
    n_roots: int
    dest_base: int
    p_off: int
    c_off: int
    n_const: int
    slot_col: np.ndarray
    slot_delta: np.ndarray
    columns: list  # retained index columns (int64 arrays) in retained order
    layout: str
    wave: int
    n_regs: int = 0
    tape: np.ndarray = None
    imms: list = field(default_factory=list)
    sop: np.ndarray = None
    opos: np.ndarray = None  # (n_roots, n) int64 output positions, NONE32 = not an output
    kernel: int = -1
    window_value: bool = False  # value-mode twin of a CSR-window member (runs in value mode only)
    window: bool = False  # CSR-window member (window unit, CSR mode only)
    wpos: np.ndarray = None  # CSR-window member: (n_roots, n) uint16 position in its window


def _output_map(plan, lowered, waves):
    """First CSR position of every result slot, and the outputs no kernel result covers.

    Returns (opos per kernel [(R, N) arrays or None], residual positions, residual addresses).
    """
    outs = np.asarray(plan.outputs, dtype=np.int64)
    k = np.arange(outs.size, dtype=np.int64)
    order = np.argsort(outs, kind="stable")
    so = outs[order]
    first = np.ones(so.size, bool)
    first[1:] = so[1:] != so[:-1]
    covered = np.zeros(outs.size, bool)
    opos = []
    for kl in lowered:
        kp = plan.kernels[kl.index]
        lo, hi = kp.dest_base, kp.dest_base + kp.n_roots * kp.instances
        a, b = np.searchsorted(so, [lo, hi])
        sel = np.nonzero(first[a:b])[0] + a
        if sel.size == 0:
            opos.append(None)
            continue
        table = np.full(kp.n_roots * kp.instances, NONE32, dtype=np.int64)
        table[so[sel] - lo] = k[order[sel]]
        covered[order[sel]] = True
        opos.append(table.reshape(kp.n_roots, kp.instances))
    res_k = np.nonzero(~covered)[0]
    return opos, res_k, outs[res_k]


def _owner_waves(plan, waves, addrs):
    """Wave after which each address holds its final value (-1: input or never written)."""
    ks = plan.kernels
    out = np.full(addrs.size, -1, dtype=np.int64)
    if not ks or not addrs.size:
        return out
    starts = np.array([kp.dest_base for kp in ks], np.int64)
    ends = np.array([kp.dest_base + kp.n_roots * kp.instances for kp in ks], np.int64)
    order = np.argsort(starts, kind="stable")
    pos = np.searchsorted(starts[order], addrs, side="right") - 1
    ok = pos >= 0
    own = np.where(ok, order[np.maximum(pos, 0)], 0)
    inside = ok & (addrs < ends[own])
    w = np.asarray(waves, np.int64)
    out[inside] = w[own[inside]]
    return out


ZERO_NONE, ZERO_ONCE, ZERO_EVERY = 0, 1, 2


def _needs_zero(plan, waves, reads) -> int:
    """Which zeros of the value array the evaluation relies on (codegen.py:419).

    ``reads`` is a list of (wave, addresses).  ZERO_ONCE: some load reads a
    slot nothing writes (alignment padding, structural gaps) -- zeroing the
    buffer once suffices.  ZERO_EVERY: some load reads a slot a later wave
    writes (the interpreter's read-before-write, codegen.py:434-443) -- a
    re-used buffer must be re-zeroed before every evaluation.
    """
    level = ZERO_NONE
    for wk, addrs in reads:
        addrs = addrs[addrs >= plan.input_count]
        if not addrs.size:
            continue
        ow = _owner_waves(plan, waves, addrs)
        if np.any(ow >= wk):
            return ZERO_EVERY
        if np.any(ow < 0):
            level = ZERO_ONCE
    return level


def _window_members(plan, lowered, opos, n_waves):
    """Kernel indices whose outputs a CSR-window unit can assemble, or None.

    Requires every output-producing group of the last wave to be a plain
    (not self-referencing), never re-read group whose instances' first output
    positions increase with the instance (each window then takes one
    contiguous instance range of it), and every other output -- inputs,
    earlier waves' results, duplicates -- to be final before the last wave
    (the windows copy those from the value array).
    """
    if n_waves == 0 or not len(plan.outputs):
        return None
    last = n_waves - 1
    members = []
    for kl, o in zip(lowered, opos):
        if o is None or kl.wave != last:
            continue
        if kl.flags & (FLAG_SELFREF | FLAG_SERIAL):
            return None
        first = np.where(o == NONE32, np.iinfo(np.int64).max, o).min(axis=0)
        v = first[first != np.iinfo(np.int64).max]
        if v.size > 1 and not np.all(np.diff(v) > 0):
            return None
        members.append(kl.index)
    if not members:
        return None
    # outputs not produced by members must come from inputs or earlier waves
    outs = np.asarray(plan.outputs, dtype=np.int64)
    covered = np.zeros(outs.size, bool)
    keep = set(members)
    for kl, o in zip(lowered, opos):
        if o is not None and kl.index in keep:
            covered[o[o != NONE32]] = True
    rest = outs[~covered]
    waves = [kl.wave for kl in lowered]
    if rest.size and np.any(_owner_waves(plan, waves, rest) >= last):
        return None
    return members


WIN_ROWS = 256  # anchor instances per CSR window = JIT_BLOCK: one pass, no idle lanes (240: 0.1253 ms, 256: 0.1212, r3e)
WIN_MAX = 6656  # outputs per CSR window (52 KB of shared memory: 3 windows per SM; sized for 256 rows of C2, r3e)
WIN_MIN = 1024  # windows are not cut shorter than this unless the anchor forces it
WIN_SLOTS = 148 * 3  # windows resident at once (B200 SMs x the window kernel's blocks per SM)
WIN_GRID_CUT = 1  # window unit grid = n_win - WIN_GRID_CUT x 148 blocks (sgb.cu)
KEEP_BEFORE_GATHER = True  # gather mode: the last wave's output results stored with an L2 evict_last hint (C3 -0.8 %, C4 -2.8 %, r3o)
KEEP_WAVES = 2  # waves before the window unit that keep their results in L2 (C2: 1 0.1777-0.1784, 2 0.1768, 3 0.1788 ms, r3p)
KEEP_BEFORE_WINDOW = True  # results of the wave before the window unit stored with an L2 evict_last hint (C2: window 0.1212 -> 0.1183 ms, step -0.6 %, r3m)
WIN_BALANCE_ROUNDS = 4  # ... always below this many rounds (plan shards, small plans: a partial round is a big tail)
WIN_BALANCE = False  # cut whole rounds of resident windows (lower_plan): C2 window 0.1275 -> 0.1292 ms, off (r2v)
WIN_MAX_LOADS = 32  # default lowering: windows only when every member loads at most this many slots
# batched CSR of a window plan: the members' value-mode twins store their outputs directly (they get
# output positions; sgb.cu batch_direct) instead of batched values + one gather
BATCH_DIRECT = True  # C5: 2.46 -> 2.12 ms (r2v)


@dataclass
class CsrWindows:
    """CSR windows of the last wave (``_csr_windows``): window w assembles outputs [k[w], k[w+1])."""

    k: np.ndarray  # int64 [n_win + 1] window start positions
    pieces: np.ndarray  # int32 [n_win, J, 2]: member j's first instance and instance count in window w
    wpos: list  # per member: uint16 (R, N) position of root r of instance i in its window, 0xFFFF = none
    copy_off: np.ndarray  # int64 [n_win + 1]: copies of window w are [copy_off[w], copy_off[w+1])
    copy_src: np.ndarray  # uint32: value-array address of each copied output (CSR order)
    copy_pos: np.ndarray  # uint16: its position in its window



def _csr_windows(member_opos: list, n_out: int, copy_k: np.ndarray, copy_addr: np.ndarray,
                 rows: int | None = None, wmax: int | None = None, wmin: int | None = None) -> CsrWindows:
    """Cut the CSR value array into windows for the window unit (jit.window_source).

    ``member_opos``: per member group its (R, N) CSR positions (NONE32 = not an output), first
    positions increasing with the instance.  Windows never split an instance's outputs (its
    roots stay in one window), hold at most ``wmax`` outputs, and -- anchored on the member with
    the most outputs -- cover ``rows`` consecutive anchor instances when that fits, so on mesh
    plans (instance = vertex = CSR row) every member's piece is about ``rows`` instances: one
    pass of a 256-thread block.  ``copy_k`` / ``copy_addr``: the outputs the members do not
    produce (CSR positions, value-array sources).
    """
    rows = WIN_ROWS if rows is None else rows
    wmax = WIN_MAX if wmax is None else wmax
    # (smaller windows for small plans -- n_out / WIN_SLOTS, one block per resident slot -- measured
    # slower on C1: 200 windows of four passes 0.0107 ms, 796 of one 0.0120 ms, r2z)
    wmin = WIN_MIN if wmin is None else wmin
    big = np.iinfo(np.int64).max
    firsts, lasts = [], []
    for o in member_opos:
        valid = o != NONE32
        firsts.append(np.where(valid, o, big).min(axis=0))
        lasts.append(np.where(valid, o, -1).max(axis=0))
    # cuts inside an instance's [first, last] output range are not allowed
    cover = np.zeros(n_out + 2, np.int64)
    for f, l_ in zip(firsts, lasts):
        m = l_ > f
        np.add.at(cover, f[m] + 1, 1)
        np.add.at(cover, l_[m] + 1, -1)
    blocked = np.cumsum(cover)[: n_out + 1] > 0  # blocked[p]: a cut before position p splits an instance
    allowed = np.flatnonzero(~blocked)
    allowed = allowed[(allowed > 0) & (allowed <= n_out)]
    if not allowed.size or allowed[-1] != n_out:
        allowed = np.append(allowed, n_out)
    counts = [int((f != big).sum()) for f in firsts]
    anchor = int(np.argmax(counts)) if counts else -1
    # preferred cuts: the first output of every ``rows``-th anchor instance (snapped to an allowed cut)
    pref = np.zeros(0, np.int64)
    if anchor >= 0:
        fa = firsts[anchor]
        valid = np.flatnonzero(fa != big)
        q = np.searchsorted(valid, np.arange(rows, fa.size, rows))  # first valid instance >= m * rows
        starts = fa[valid[q[q < valid.size]]]
        j = np.searchsorted(allowed, starts, side="right") - 1
        pref = np.unique(allowed[j[j >= 0]])
    k = [0]
    while k[-1] < n_out:
        cur = k[-1]
        lim = cur + wmax
        # the next preferred cut, if the window stays within wmax; else the last allowed cut in reach
        j = np.searchsorted(pref, cur, side="right")
        nxt = int(pref[j]) if j < pref.size and pref[j] <= lim else None
        if nxt is not None and nxt - cur < wmin and j + 1 < pref.size and pref[j + 1] <= lim:
            # tiny windows (anchor sparse here): merge preferred steps up to wmin
            jj = np.searchsorted(pref, min(lim, cur + wmin), side="right") - 1
            nxt = int(pref[max(jj, j)])
        if nxt is None:
            jj = np.searchsorted(allowed, lim, side="right") - 1
            if jj < 0 or allowed[jj] <= cur:
                raise ValueError("an instance's outputs span more than one CSR window")
            nxt = int(allowed[jj])
        k.append(nxt)
    k = np.asarray(k, np.int64)
    n_win = k.size - 1
    J = len(member_opos)
    pieces = np.zeros((n_win, J, 2), np.int32)
    wpos = []
    for j, (o, f) in enumerate(zip(member_opos, firsts)):
        n = f.size
        inst = np.flatnonzero(f != big)
        fv = f[inst]
        lo = np.searchsorted(fv, k[:-1])
        hi = np.searchsorted(fv, k[1:])
        has = hi > lo
        a = np.where(has, inst[np.minimum(lo, inst.size - 1)], 0)
        b = np.where(has, inst[np.maximum(hi - 1, 0)] + 1, 0)
        pieces[:, j, 0] = a
        pieces[:, j, 1] = b - a
        w_of = np.searchsorted(k, np.where(f == big, 0, f), side="right") - 1  # window of each instance
        rel = np.where(o == NONE32, 0xFFFF, o - k[np.clip(w_of, 0, n_win - 1)][None, :])
        if n and rel.size and int(rel[o != NONE32].max(initial=0)) >= 0xFFFF:
            raise ValueError("CSR window too long for 16-bit positions")
        wpos.append(rel.astype(np.uint16))
    order = np.argsort(copy_k, kind="stable")
    ck, ca = np.asarray(copy_k, np.int64)[order], np.asarray(copy_addr, np.int64)[order]
    copy_off = np.searchsorted(ck, k).astype(np.int64)
    cw = np.searchsorted(k, ck, side="right") - 1
    copy_pos = (ck - k[np.clip(cw, 0, max(n_win - 1, 0))]).astype(np.uint16) if ck.size else np.zeros(0, np.uint16)
    return CsrWindows(k=k, pieces=pieces, wpos=wpos, copy_off=copy_off, copy_src=ca.astype(np.uint32),
                      copy_pos=copy_pos)


WBULK_GAP = 16  # value-array runs closer than this many doubles merge into one bulk copy
WBULK_SMEM = 227 * 1024  # dynamic shared memory of one window block (one block per SM)
WBULK_RING = (2, 4)  # ring depth range (windows in flight per block)
WBULK_CONSUMERS = 256  # consumer threads per member group of a bulk window block (one instance each per pass)
WBULK_GROUPS = 2  # member groups per block (chunks of members evaluated side by side)
WBULK_THREADS = WBULK_GROUPS * WBULK_CONSUMERS + 32  # + one producer warp


@dataclass
class WindowBulk:
    """Bulk-copy feed of a CSR-window unit (jit.wbulk_source).

    A member whose every slot reads a stride-1 stream of the value array (``x[base_s + i]``:
    affine column 0 plus coherent deltas or affine columns, no constants) is *bulk*: in window
    w its piece [i0, i0 + n) reads the runs ``x[base_s + i0 : base_s + i0 + n)``.  Per window
    the runs of all bulk members are merged into intervals (``iv``: first element, element
    count, both even, so every copy is 16-byte aligned and a multiple of 16 bytes) that one
    producer thread copies with ``cp.async.bulk`` into the x area of a ring slot, together with
    the window's consumer blob (``meta``); the consumer threads evaluate the bulk members from
    shared memory.  Blob layout (byte offsets, 16-byte aligned sections)::

        0   u32 n_copy, u32 copy_src offset, u32 copy_pos offset, u32 window length,
            i64 first output k0, u32 window positions, u32 x-area elements
        32  int2 pieces[J]                       (first instance, count) of every member
        roff_at  u16 run offset[NR]              x-area element of x[base_s + i0], bulk (member, slot)
        woff_at  u16 wpos offset[NW]             first window position of each bulk (member, root)
        wpos_at  u16 wpos[...]                   window positions of the bulk pieces
        copy_src u32[n_copy], copy_pos u16[n_copy]
    """

    members: list  # member indices j (group group_begin + j) fed from the ring
    bases: list  # per bulk member: value-array base of each slot's stream
    meta: np.ndarray  # uint8: the consumer blobs of all windows
    meta_off: np.ndarray  # int64 [n_win + 1]
    iv: np.ndarray  # uint32 [n_iv, 2]
    iv_off: np.ndarray  # int64 [n_win + 1]
    ring: int  # ring slots (windows in flight per block)
    slot_meta: int  # bytes of a slot's blob area (128-byte multiple)
    slot_x: int  # bytes of a slot's x area (128-byte multiple)
    bw: int  # bytes of the window buffer (128-byte multiple)
    roff_at: int
    woff_at: int
    wpos_at: int

    @property
    def smem(self) -> int:
        return self.bw + self.ring * (self.slot_meta + self.slot_x)


def _a16(v: int) -> int:
    return (int(v) + 15) & ~15


def _a128(v: int) -> int:
    return (int(v) + 127) & ~127


def window_bulk(dp, u: int, windows: "CsrWindows", gap: int | None = None) -> WindowBulk | None:
    """The bulk feed of window unit ``u`` of a lowered plan, or None (no bulk member, or the
    ring does not fit in shared memory)."""
    from . import jit as _jit

    gap = WBULK_GAP if gap is None else gap

    r = dp.unit(u)
    g0, g1 = r["group_begin"], r["group_end"]
    J = g1 - g0
    vas = int(dp.value_array_size)  # intervals end at most at vas rounded up to even (value_slots)
    members, bases = [], []
    for j in range(J):
        rec = dp.groups[g0 + j]
        f = int(rec["flags"])
        S, K = int(rec["n_slots"]), int(rec["n_const"])
        if f & FLAG_INTERLEAVED or K or not S or not f & FLAG_WPOS16:
            continue
        a0 = _jit._affine(dp, rec, 0)
        if a0 is None or a0[1] != 1:
            continue
        cols = dp.slot_col[rec["slot_off"]: rec["slot_off"] + S]
        dels = dp.slot_delta[rec["slot_off"]: rec["slot_off"] + S]
        bs = []
        for s_ in range(S):
            c = int(cols[s_])
            if c < 0:
                bs.append(a0[0] + int(dels[s_]))
            elif c == 0:
                bs.append(a0[0])
            else:
                a = _jit._affine(dp, rec, c)
                if a is None or a[1] != 1:
                    bs = None
                    break
                bs.append(a[0])
        if bs is not None:
            members.append(j)
            bases.append(bs)
    if not members:
        return None
    P = windows.pieces.astype(np.int64)
    n_win = P.shape[0]
    NR = sum(len(b) for b in bases)
    NW = sum(int(dp.groups[g0 + j]["n_roots"]) for j in members)
    # every (window, bulk member, slot) run, merged per window into aligned intervals
    W, ST, LN, RID = [], [], [], []
    rid = 0
    for j, bs in zip(members, bases):
        for b in bs:
            W.append(np.arange(n_win, dtype=np.int64))
            ST.append(b + P[:, j, 0])
            LN.append(P[:, j, 1])
            RID.append(np.full(n_win, rid, np.int64))
            rid += 1
    W, ST, LN, RID = (np.concatenate(a) for a in (W, ST, LN, RID))
    keep = LN > 0
    W, ST, LN, RID = W[keep], ST[keep], LN[keep], RID[keep]
    if ST.size and (ST.min() < 0 or (ST + LN).max() > vas):
        raise AssertionError("window_bulk: a run leaves the value array")
    order = np.lexsort((ST, W))
    W, ST, LN, RID = W[order], ST[order], LN[order], RID[order]
    big = vas + 4 * gap + 4
    en = ST + LN
    cm = np.maximum.accumulate(en + W * big) if ST.size else en
    new = np.ones(ST.size, bool)
    new[1:] = ST[1:] + W[1:] * big > cm[:-1] + gap
    ivid = np.cumsum(new) - 1
    heads = np.flatnonzero(new)
    iv_w = W[heads]
    iv_s = ST[heads] & ~1
    iv_e = (np.maximum.reduceat(en, heads) + 1) & ~1 if heads.size else np.zeros(0, np.int64)
    iv_n = iv_e - iv_s
    iv_off = np.searchsorted(iv_w, np.arange(n_win + 1)).astype(np.int64)
    excl = np.cumsum(iv_n) - iv_n
    dst = excl - excl[np.minimum(iv_off[iv_w], max(excl.size - 1, 0))] if excl.size else excl
    xlen = np.bincount(iv_w, weights=iv_n, minlength=n_win).astype(np.int64)
    roff = np.zeros((n_win, NR), np.int64)
    roff[W, RID] = dst[ivid] + (ST - iv_s[ivid])
    if roff.size and int(roff.max()) > 0xFFFF or (xlen.size and int(xlen.max()) > 0xFFFF):
        return None
    # per window consumer blobs
    roff_at = 32 + 8 * J
    woff_at = roff_at + 2 * NR
    wpos_at = _a16(woff_at + 2 * NW)
    k = windows.k
    blobs, offs = [], [0]
    for w in range(n_win):
        wp_parts, woff = [], []
        pos = 0
        for j in members:
            i0, n = int(P[w, j, 0]), int(P[w, j, 1])
            wpj = windows.wpos[j]
            for r_ in range(wpj.shape[0]):
                woff.append(pos)
                if n:
                    wp_parts.append(wpj[r_, i0:i0 + n])
                    pos += n
        c0, c1 = int(windows.copy_off[w]), int(windows.copy_off[w + 1])
        nc = c1 - c0
        csrc_at = _a16(wpos_at + 2 * pos)
        cpos_at = _a16(csrc_at + 4 * nc)
        size = _a16(cpos_at + 2 * nc)
        b = np.zeros(size, np.uint8)
        b[0:16].view(np.uint32)[:] = (nc, csrc_at, cpos_at, int(k[w + 1] - k[w]))
        b[16:24].view(np.int64)[0] = int(k[w])
        b[24:32].view(np.uint32)[:] = (pos, int(xlen[w]))
        b[32:32 + 8 * J].view(np.int32)[:] = windows.pieces[w].reshape(-1)
        b[roff_at:woff_at].view(np.uint16)[:] = roff[w]
        if NW:
            b[woff_at:woff_at + 2 * NW].view(np.uint16)[:] = np.asarray(woff, np.uint16)
        if pos:
            b[wpos_at:wpos_at + 2 * pos].view(np.uint16)[:] = np.concatenate(wp_parts)
        if nc:
            b[csrc_at:csrc_at + 4 * nc].view(np.uint32)[:] = windows.copy_src[c0:c1]
            b[cpos_at:cpos_at + 2 * nc].view(np.uint16)[:] = windows.copy_pos[c0:c1]
        blobs.append(b)
        offs.append(offs[-1] + size)
    meta = np.concatenate(blobs) if blobs else np.zeros(0, np.uint8)
    slot_meta = _a128(max((b.size for b in blobs), default=16))
    slot_x = _a128(8 * max(int(xlen.max(initial=0)), 2))
    bw = _a128(8 * (int(np.diff(k).max(initial=0)) + 2))
    ring = (WBULK_SMEM - bw) // (slot_meta + slot_x)
    if ring < WBULK_RING[0]:
        return None
    ring = min(ring, WBULK_RING[1])
    iv = np.stack([iv_s, iv_n], axis=1).astype(np.uint32) if iv_s.size else np.zeros((0, 2), np.uint32)
    return WindowBulk(members=members, bases=bases, meta=meta, meta_off=np.asarray(offs, np.int64), iv=iv,
                      iv_off=iv_off, ring=int(ring), slot_meta=slot_meta, slot_x=slot_x, bw=bw,
                      roff_at=roff_at, woff_at=woff_at, wpos_at=wpos_at)


JIT_SPLIT = 1  # root set of a big single-group template split this many ways (C3 element kernel: 1 0.273 ms, 2 0.297 (128-register cap spills), 3 0.474; c3w)
JIT_SPLIT_MIN_TAPE = 600  # tape records from which a template is split (C3's element Hessian: 955)


def _tape_reads(t) -> tuple:
    op = int(t[0])
    if op == T_IMM:
        return ()
    if op in (T_NEG, T_SQRT, T_SLOW, T_ST):
        return (int(t[4]),)
    if op in (T_SEL, T_MADD, T_MSUB, T_RMSUB):
        return (int(t[4]), int(t[5]), int(t[6]))
    return (int(t[4]), int(t[5]))


def split_roots(tape: np.ndarray, n_roots: int, k: int, seed: int = 0, rounds: int = 4) -> list:
    """Partition a register tape's roots into ``k`` equal-count parts with small cones.

    Returns per part the set of tape records it evaluates (the union of its roots' cones, their
    stores included).  A part's records are a sub-DAG of the tape evaluated in the same order,
    so every root keeps its exact op sequence (bit-identical results); records shared by
    several parts are evaluated by each of them.  Balanced swap local search on bitmask cones."""
    last: dict[int, int] = {}
    cone: list[int] = []
    store_of: dict[int, int] = {}
    for j, t in enumerate(tape.tolist()):
        m = 1 << j
        for r in _tape_reads(t):
            if r in last:
                m |= cone[last[r]]
        cone.append(m)
        if int(t[0]) == T_ST:
            store_of.setdefault(int(t[7]), j)
        else:
            last[int(t[3])] = j
    roots = sorted(store_of)
    cm = [cone[store_of[r]] for r in roots]
    rng = np.random.default_rng(seed)
    order = list(rng.permutation(len(roots)))
    parts = [order[i::k] for i in range(k)]

    def size(p):
        u = 0
        for q in p:
            u |= cm[q]
        return u.bit_count()

    sizes = [size(p) for p in parts]
    for _ in range(rounds):
        better = False
        for a in range(k):
            for b in range(a + 1, k):
                for ia in range(len(parts[a])):
                    for ib in range(len(parts[b])):
                        parts[a][ia], parts[b][ib] = parts[b][ib], parts[a][ia]
                        na, nb = size(parts[a]), size(parts[b])
                        if na + nb < sizes[a] + sizes[b] and max(na, nb) <= max(sizes[a], sizes[b]):
                            sizes[a], sizes[b] = na, nb
                            better = True
                        else:
                            parts[a][ia], parts[b][ib] = parts[b][ib], parts[a][ia]
        if not better:
            break
    keeps = []
    for p in parts:
        u = 0
        for q in p:
            u |= cm[q]
        keeps.append({j for j in range(len(tape)) if (u >> j) & 1})
    return keeps


def jit_vec(groups, sel) -> int:
    """Instances per thread of a specialised unit: all of them keep their loads in flight
    together, so small templates take 4, mid-size 2, big element templates 1."""
    if os.environ.get("SGB_JIT_VEC"):
        return int(os.environ["SGB_JIT_VEC"])
    width = max(len(groups[j].slot_col) + groups[j].n_const + (len(groups[j].tape) if groups[j].tape is not None
                                                               else 1) // 4 for j in sel)
    # long-latency ops (DIV / SQRT / transcendentals): one instance per thread -- more resident warps
    # hide them better than a second instance's loads (C2 faces 0.025 -> 0.023 ms, C4 rotations, r2q)
    slow = any(groups[j].tape is not None and np.isin(groups[j].tape["op"], (T_DIV, T_SQRT, T_SLOW)).any()
               for j in sel)
    if slow:
        return 1
    return 4 if width <= 24 else (2 if width <= 64 else 1)


def _copy_tape() -> np.ndarray:
    """Tape of a copy group: store slot 0 as root 0."""
    return np.array([(T_ST, 0, 0, 0, 0, 0, 0, 0)], dtype=TAPE_DTYPE)


def _tile_keys(g: _Group, starts: np.ndarray, tile: int) -> np.ndarray:
    """Smallest output position in each tile (-1 for tiles without outputs)."""
    if g.opos is None or g.n == 0:
        return np.full(starts.size, -1, np.int64)
    o = np.where(g.opos == NONE32, np.iinfo(np.int64).max, g.opos).min(axis=0)
    m = np.minimum.reduceat(o, starts) if starts.size else o[:0]
    return np.where(m == np.iinfo(np.int64).max, -1, m)


class _RelaidPlan:
    """A plan with the result ranges of some groups re-addressed instance-major (CSR layout).

    Result r of instance i of a relaid group moves from ``dest_base + r*N + i``
    (codegen.py:265) to ``dest_base + i*R + r``: a bijection inside the group's
    own range, applied to every address the plan holds (the position table and
    the outputs), so every read still finds the value it read before and the
    CSR values are unchanged bit for bit.  Only the full value array is
    permuted, which is why a relaid device plan refuses value-mode calls.
    """

    def __init__(self, plan, groups: list[int], tables: bool = True):
        self._plan = plan
        kps = [plan.kernels[k] for k in groups]
        order = np.argsort([kp.dest_base for kp in kps])
        self.lo = np.array([kps[j].dest_base for j in order], np.int64)
        self.nn = np.array([kps[j].instances for j in order], np.int64)
        self.rr = np.array([kps[j].n_roots for j in order], np.int64)
        self.hi = self.lo + self.nn * self.rr
        if tables:
            self.positions = self.remap(np.asarray(plan.positions)).astype(np.uint32)
            self.outputs = self.remap(np.asarray(plan.outputs, np.int64)).astype(np.int64)

    def __getattr__(self, name):
        return getattr(self._plan, name)

    def remap(self, addr: np.ndarray, chunk: int = 1 << 24) -> np.ndarray:
        out = np.array(addr, dtype=np.int64, copy=True)
        for s in range(0, out.size, chunk):
            a = out[s: s + chunk]
            k = np.searchsorted(self.lo, a, side="right") - 1
            kc = np.maximum(k, 0)
            m = (k >= 0) & (a < self.hi[kc])
            if not m.any():
                continue
            kk, off = kc[m], a[m] - self.lo[kc[m]]
            n = self.nn[kk]
            a[m] = self.lo[kk] + (off % n) * self.rr[kk] + off // n
        return out


RELAYOUT_GAIN = 0.75  # relay a group out when its readers touch at most this fraction of the sectors
RELAYOUT_SAMPLE_WARPS = 8192


def _warp_sectors(col: np.ndarray, lo: int, n: int, r: int, imajor: bool) -> int:
    """Distinct 32-byte sectors per 32-instance warp of the reads of ``col`` inside [lo, lo + r*n)."""
    warp = np.arange(col.size, dtype=np.int64) // 32
    m = (col >= lo) & (col < lo + r * n)
    if not m.any():
        return 0
    off = col[m] - lo
    if imajor:
        off = (off % n) * r + off // n
    key = warp[m] * (1 << 40) + ((lo + off) >> 2)
    return int(np.unique(key).size)


def choose_relayout(plan, lowered, candidates: list[int], mode: str = "auto"):
    """Groups whose results move to the instance-major CSR layout, and the coherent deltas that change.

    ``auto``: a multi-root group moves when its readers -- every position
    column of the plan and the output gather, warps of 32 consecutive
    instances -- touch at most RELAYOUT_GAIN of the 32-byte sectors they touch
    in the reference layout (sampled over up to RELAYOUT_SAMPLE_WARPS warps per
    column).  ``all``: every candidate.  A coherent slot (``column 0 + delta``,
    codegen.py:317-327) reading a moved range keeps working when the remapped
    addresses are still a constant delta apart (same instance, other root:
    delta ``dq*N`` becomes ``dq``); groups for which that fails stay put.
    Returns ``(kernels, {(kernel, slot): new delta})``.
    """
    kps = plan.kernels
    cand = sorted((k for k in candidates if kps[k].n_roots > 1 and kps[k].instances > 1),
                  key=lambda k: kps[k].dest_base)
    if not cand:
        return [], {}
    cols = []  # reader columns (position slots and the output gather)
    coherent = []  # (kernel, slot, column 0, column of the slot)
    for kl in lowered:
        sc = slot_addresses(plan, kps[kl.index])
        for s, c in enumerate(sc):
            cols.append(c)
            if kl.slot_col[s] < 0 and kl.slot_delta[s] != 0:
                coherent.append((kl.index, s, sc[0], c))
    cols.append(np.asarray(plan.outputs, np.int64))
    chosen = []
    for k in cand:
        if mode == "all":
            chosen.append(k)
            continue
        kp = kps[k]
        old = new = 0
        for c in cols:
            if c.size == 0:
                continue
            nw = (c.size + 31) // 32
            if nw > RELAYOUT_SAMPLE_WARPS:  # evenly spaced runs of 64 warps
                runs = RELAYOUT_SAMPLE_WARPS // 64
                starts = np.linspace(0, nw - 64, runs).astype(np.int64) * 32
                c = np.concatenate([c[s: s + 64 * 32] for s in starts])
            old += _warp_sectors(c, kp.dest_base, kp.instances, kp.n_roots, False)
            new += _warp_sectors(c, kp.dest_base, kp.instances, kp.n_roots, True)
        if old and new <= RELAYOUT_GAIN * old:
            chosen.append(k)
    while chosen:
        rp = _RelaidPlan(plan, chosen, tables=False)
        deltas, bad = {}, set()
        for k, s, c0, c in coherent:
            d = rp.remap(c) - rp.remap(c0)
            if d.size and np.all(d == d[0]):
                deltas[(k, s)] = int(d[0])
                continue
            for j in chosen:
                lo, hi = kps[j].dest_base, kps[j].dest_base + kps[j].n_roots * kps[j].instances
                if np.any((c >= lo) & (c < hi)) or np.any((c0 >= lo) & (c0 < hi)):
                    bad.add(j)
        if not bad:
            return chosen, deltas
        chosen = [j for j in chosen if j not in bad]
    return [], {}


STAGE_LIMIT = 200 * 1024  # shared memory a specialised unit may stage instance-major results in
MAX_IMAJOR_ROOTS = 96  # ... so relaid groups have at most this many roots (JIT_BLOCK * 97 * 8 B fits)


def stage_stride(n_roots: int) -> int:
    """Doubles per instance in the staging buffer (odd: conflict-free 8-byte shared-memory rows)."""
    return n_roots | 1


def stage_bytes(groups, sel, vec: int) -> int:
    """Dynamic shared memory of a specialised unit: one staged tile of its largest relaid group."""
    rp = [stage_stride(groups[j].n_roots) for j in sel if groups[j].flags & FLAG_IMAJOR]
    return JIT_BLOCK * vec * max(rp) * 8 if rp else 0


JIT_MIN_N = 4096  # groups with fewer instances stay on the hand-written kernels (NVRTC time buys nothing)
JIT_MAX_WAVE_GROUPS = 48  # ...unless they share a wave of at most this many groups with a big one


def lower_plan(plan, compress: bool | None = None, direct_csr: bool | None = None,
               jit: bool | None = None, csr_window: bool | None = None,
               jit_min_n: int | None = None, relayout: str | bool | None = None,
               jit_compile: bool = True, wbulk: bool | None = None) -> DevicePlanArrays:
    """ExecutionPlan -> device plan.

    ``direct_csr``: output groups store their CSR values through output-position
    tables and CSR-only copy groups cover inputs / duplicates (sgb_run_csr
    without a gather pass).  Off by default: on B200 the 8-byte scattered stores
    cost more than the coalesced value-array stores + one u32-indexed gather
    (profiles/r06).

    ``jit_compile=False`` lays out the specialised units without running NVRTC (no cubin: for
    the CPU emulator of the device plan, tests/device_plan_emu.py).

    ``relayout`` (``"auto"`` / ``"all"`` / False): the CSR layout -- big plain
    multi-root groups whose readers gather across roots store instance-major
    (``_RelaidPlan``, ``choose_relayout``).  CSR-mode only: the device plan then
    refuses value-mode evaluation.
    """
    if compress is None:
        compress = os.environ.get("SGB_COMPRESS", "1") != "0"
    if direct_csr is None:
        direct_csr = os.environ.get("SGB_DIRECT_CSR", "0") == "1"
    if jit is None:  # specialised (compiled) tape units -- see jit.py; SGB_TAPE_JIT=0 keeps the interpreter
        jit = os.environ.get("SGB_TAPE_JIT", "1") != "0"
    if jit and jit_compile:
        from . import jit as _jit

        jit = _jit.available()
    if jit_min_n is None:
        jit_min_n = int(os.environ.get("SGB_JIT_MIN_N", JIT_MIN_N))
    window_policy = "force" if csr_window else "off"
    if csr_window is None:  # CSR windows of the last wave (specialised units only), see _window_members:
        # by default for plans whose last wave holds a big group and at most JIT_MAX_WAVE_GROUPS members
        window_policy = {"0": "off", "1": "force"}.get(os.environ.get("SGB_CSR_WINDOW", ""), "auto")
    csr_window = window_policy != "off" and bool(jit)
    if relayout is None:
        relayout = False
    if relayout is True:
        relayout = "auto"
    lowered = [lower_kernel(plan, kp, k) for k, kp in enumerate(plan.kernels)]
    read_sets = _read_sets(plan)  # which ranges each kernel reads: invariant under the CSR layout
    imajor: set = set()
    if relayout:
        if direct_csr:
            raise ValueError("the CSR layout does not combine with direct CSR stores")
        cand = [kl.index for kl in lowered if not kl.flags & (FLAG_SELFREF | FLAG_SERIAL)
                and plan.kernels[kl.index].instances >= jit_min_n
                and plan.kernels[kl.index].n_roots <= MAX_IMAJOR_ROOTS]
        chosen, deltas = choose_relayout(plan, lowered, cand, relayout)
        imajor = set(chosen)
        if imajor:
            plan = _RelaidPlan(plan, sorted(imajor))
            for (k, s_), d in deltas.items():
                lowered[k].slot_delta = lowered[k].slot_delta.copy()
                lowered[k].slot_delta[s_] = d
    waves = compute_waves(plan, read_sets)
    for kl, w in zip(lowered, waves):
        kl.wave = w
    n_waves = (max(waves) + 1) if waves else 0
    opos, res_k, res_addr = _output_map(plan, lowered, waves)
    window = _window_members(plan, lowered, opos, n_waves) if csr_window and not direct_csr else None
    if window is not None and window_policy == "auto" and (
            len(window) > JIT_MAX_WAVE_GROUPS or max(plan.kernels[k].instances for k in window) < jit_min_n
            or max(len(plan.kernels[k].pos_vars) + len(plan.kernels[k].const_vars) for k in window) > WIN_MAX_LOADS):
        # small plans: the gather costs nothing, NVRTC time would; wide templates (C4's rhs, 38-90
        # loads per instance) need the register file the window kernel's three resident blocks cannot give
        window = None
    if window is not None:
        # CSR windows: only last-wave members keep output positions; every other output
        # (inputs, duplicates, earlier waves' results) is a copy piece of its window
        keep = set(window)
        opos = [o if kl.index in keep else None for kl, o in zip(lowered, opos)]
        outs = np.asarray(plan.outputs, dtype=np.int64)
        covered = np.zeros(outs.size, bool)
        for o in opos:
            if o is not None:
                v = o[o != NONE32]
                covered[v] = True
        res_k = np.nonzero(~covered)[0]
        res_addr = outs[res_k]
    elif not direct_csr:
        opos = [None] * len(lowered)
        res_k = res_addr = np.zeros(0, np.int64)
    # copy groups: outputs that are inputs, duplicates or padding (CSR mode only)
    avail = _owner_waves(plan, waves, res_addr) + 1  # first wave that may read the source
    last = max(n_waves - 1, 0)
    copy_sets = [(min(last, n_waves), avail <= last), (n_waves, avail > last)]
    # stream flags: results no later kernel (or copy group) reads -- nor the output gather: its
    # reads should hit L2, not follow evict-first streaming stores (gather mode: no windows, no
    # direct positions)
    reads = [r for r in read_sets if r.size] + ([res_addr] if res_addr.size else [])
    if window is None and not direct_csr and len(plan.outputs):
        reads.append(np.asarray(plan.outputs, np.int64))
    allr = unique_addresses(np.concatenate(reads)) if reads else np.zeros(0, np.int64)
    groups: list[_Group] = []
    win_groups: list[_Group] = []  # window members (CSR-only records; value-mode twins stay in `groups`)
    for kl in lowered:
        kp = plan.kernels[kl.index]
        lo, hi = kp.dest_base, kp.dest_base + kp.n_roots * kp.instances
        a, b = np.searchsorted(allr, [lo, hi])
        if b == a:
            kl.flags |= FLAG_STREAM
        n, r = kp.instances, len(kp.retained)
        seg = np.asarray(plan.positions[kp.p_base: kp.p_base + r * n], dtype=np.int64)
        cols = list(seg.reshape(r, n) if kp.layout == "coalesced" else seg.reshape(n, r).T)
        flags = kl.flags | (FLAG_COHERENT if r == 1 and kp.pos_vars else 0) | \
            (FLAG_IMAJOR if kl.index in imajor else 0)
        in_window = window is not None and kl.index in window
        groups.append(_Group(kl.kind, flags, n, kp.n_roots, kp.dest_base, kp.p_base, kp.c_base,
                             len(kp.const_vars), kl.slot_col, kl.slot_delta, cols, kp.layout, kl.wave,
                             kl.n_regs, kl.tape, kl.imms, kl.sop,
                             opos[kl.index] if not in_window or BATCH_DIRECT else None,
                             kl.index, window_value=in_window))
        if in_window:
            win_groups.append(_Group(kl.kind, flags | FLAG_CSR_ONLY | FLAG_WPOS16, n, kp.n_roots, kp.dest_base,
                                     kp.p_base, kp.c_base, len(kp.const_vars), kl.slot_col, kl.slot_delta, cols,
                                     kp.layout, kl.wave, kl.n_regs, kl.tape, kl.imms, kl.sop, None, kl.index,
                                     window=True))
    windows = None
    if window is not None:
        # members in list order == their order in the window unit (pieces columns)
        mo = [opos[g.kernel] for g in win_groups]
        windows = _csr_windows(mo, len(plan.outputs), res_k, res_addr)
        # whole rounds of resident windows: one block per window, WIN_SLOTS resident at once -- a last
        # round of a few windows would leave the chip idle for a whole window's time
        n_win = windows.k.size - 1
        if n_win % WIN_SLOTS and n_win > WIN_SLOTS and (WIN_BALANCE or n_win < WIN_BALANCE_ROUNDS * WIN_SLOTS):
            rounds, rem = divmod(n_win, WIN_SLOTS)
            targets = ([rounds * WIN_SLOTS] if rem < WIN_SLOTS // 2 else []) + [(rounds + 1) * WIN_SLOTS]
            for target in targets:  # the count falls with rows: bisect rows (no small-window merging)
                lo_r, hi_r, best = 8, 4 * WIN_ROWS, None
                while lo_r <= hi_r:
                    mid = (lo_r + hi_r) // 2
                    cand = _csr_windows(mo, len(plan.outputs), res_k, res_addr, rows=mid, wmin=0)
                    n_cur = cand.k.size - 1
                    if n_cur <= target:
                        best, hi_r = (cand, n_cur), mid - 1
                    else:
                        lo_r = mid + 1
                if best is not None and best[1] >= target - WIN_SLOTS // 8:
                    windows = best[0]
                    break
        for g, wp in zip(win_groups, windows.wpos):
            g.wpos = wp
    extra_pos = []
    p_next = int(np.asarray(plan.positions).size)
    copy_waves = []
    for wv, sel in copy_sets:
        if window is not None or not np.any(sel):  # window units copy these outputs themselves
            continue
        addr, kk = res_addr[sel], res_k[sel]
        ordr = np.argsort(kk, kind="stable")  # CSR order: coalesced stores
        addr, kk = addr[ordr], kk[ordr]
        cg = _Group(KIND_SOP, FLAG_CSR_ONLY | FLAG_STREAM | FLAG_COHERENT | FLAG_EXACT, int(addr.size), 1,
                    int(plan.input_count), p_next, 0, 0, np.zeros(1, np.int32), np.zeros(1, np.int64),
                    [addr], "coalesced", wv, sop=np.array([SOP_NEWTERM], np.int32),
                    opos=kk.reshape(1, -1), window=window is not None)
        (win_groups if window is not None else groups).append(cg)
        extra_pos.append(addr.astype(np.uint32))
        p_next += addr.size
        copy_waves.append(wv)
    needs_zero = _needs_zero(plan, waves, list(zip(waves, read_sets)) +
                             [(g.wave, g.columns[0]) for g in groups + win_groups
                              if g.flags & FLAG_CSR_ONLY and g.tape is None] +
                             ([(last, res_addr)] if window is not None and res_addr.size else []))
    groups = groups + win_groups
    total_waves = max([n_waves] + [w + 1 for w in copy_waves])

    # -- launch units and tiles ---------------------------------------------------------
    packed = np.zeros(len(groups), GROUP_DTYPE)
    order_groups: list[int] = []
    units, tiles_all, tiles_alt, any_alt = [], [], [], False
    tapes, imms, sops, scol, sdel, cbases, coffs, obases, ooffs, op32 = ([] for _ in range(10))
    n_tape = n_imm = n_sop = n_slot = n_cb = n_co = n_ob = n_oo = n_o32 = 0
    jit_tapes, jit_imms, jit_units = {}, {}, []
    window_units: list = []
    n_out_total = len(plan.outputs)
    for w in range(total_waves):
        members = [j for j, g in enumerate(groups) if g.wave == w]
        plan_units = []
        if jit:  # every big plain group of the wave (tape or sum-of-products) in one specialised kernel;
            # in a big plan the small groups of the wave join it (a tiny boundary group on the
            # interpreter would outlast the whole specialised unit it runs beside)
            plain_w = [j for j in members if not groups[j].flags & (FLAG_SELFREF | FLAG_SERIAL)]
            big_wave = any(groups[j].n >= jit_min_n for j in plain_w) and len(plain_w) <= JIT_MAX_WAVE_GROUPS
            sj = [j for j in plain_w if groups[j].n >= jit_min_n or big_wave or groups[j].window]
            for sel, tag in (([j for j in sj if not groups[j].window and not groups[j].window_value], 0),
                             ([j for j in sj if groups[j].window_value], UNIT_VALUE_ONLY),
                             ([j for j in sj if groups[j].window], UNIT_WINDOW)):
                if sel:
                    vec = jit_vec(groups, sel) if tag != UNIT_WINDOW else 1
                    while vec > 1 and stage_bytes(groups, sel, vec) > STAGE_LIMIT:
                        vec //= 2
                    plan_units.append((KIND_TAPE, vec, JIT_BLOCK, tag, sel))
            members = [j for j in members if j not in set(sj)]
        hw_units = []  # hand-written units: (kind, variant, block, scratch regs, groups, value-mode only)
        for twin in (False, True):  # value-only twins of CSR-window members get units of their own
            sub = [j for j in members if groups[j].window_value == twin]
            for plain in (True, False):
                tm = [j for j in sub if groups[j].kind == KIND_TAPE and
                      plain == (not groups[j].flags & (FLAG_SELFREF | FLAG_SERIAL))]
                if not tm:
                    continue
                regs = max(groups[j].n_regs for j in tm)
                bs = block_size_for(regs)
                if regs * bs * 8 > SMEM_LIMIT:
                    raise ValueError(f"wave {w}: template needs {regs} scratch registers, more than shared memory holds")
                vec = 1
                if plain:
                    for v in TAPE_VECS:
                        if regs * v * bs * 8 <= VEC_SMEM_BUDGET or v == 1:
                            vec = v
                            break
                hw_units.append((KIND_TAPE, vec, bs, regs, tm, twin))
            codes: dict[int, list] = {}
            for j in sub:
                if groups[j].kind == KIND_SOP:
                    codes.setdefault(sop_unit_code(groups[j], compress), []).append(j)
            for code in sorted(codes):  # one persistent launch per kernel body
                hw_units.append((KIND_SOP, code, SOP_BLOCK, 0, codes[code], twin))
        plan_units = [u + (False,) for u in plan_units] + hw_units
        for kind, variant, bs, regs, ms, twin in plan_units:
            utag, jit_unit = (UNIT_VALUE_ONLY if twin else 0), False
            if kind == KIND_TAPE and bs == JIT_BLOCK and regs in (0, UNIT_VALUE_ONLY, UNIT_WINDOW) \
                    and all(not groups[j].flags & (FLAG_SELFREF | FLAG_SERIAL) for j in ms) and jit:
                utag, regs, jit_unit = regs, 0, True
                if utag == 0:  # specialised unit: regs carries the staging bytes of its relaid groups
                    regs = stage_bytes(groups, ms, variant)
            g_begin = len(order_groups)
            unit_tiles, unit_keys = [], []
            for j in ms:
                g = groups[j]
                gi = len(order_groups)
                order_groups.append(j)
                rec = packed[gi]
                rec["n"], rec["dest_base"], rec["p_off"], rec["c_off"] = g.n, g.dest_base, g.p_off, g.c_off
                rec["n_roots"], rec["n_slots"], rec["n_ret"] = g.n_roots, len(g.slot_col), len(g.columns)
                rec["n_const"], rec["kind"], rec["n_regs"], rec["unit"] = g.n_const, kind, g.n_regs, len(units)
                rec["slot_off"] = n_slot
                scol.append(g.slot_col)
                sdel.append(g.slot_delta)
                n_slot += len(g.slot_col)
                flags = g.flags
                if kind == KIND_TAPE:
                    jit_tapes[gi] = g.tape if g.tape is not None else _copy_tape()
                    jit_imms[gi] = g.imms
                    t = assemble(g.tape, bs * variant, n_imm) if regs else np.zeros((0, 4), np.uint32)
                    rec["tape_off"], rec["tape_len"] = n_tape, len(t)
                    tapes.append(t)
                    n_tape += len(t)
                    imms.extend(g.imms)
                    n_imm += len(g.imms)
                    tile = bs * variant
                else:
                    cls = sop_class(len(g.sop))
                    rec["variant"], rec["sop_off"], rec["sop_len"] = cls, n_sop, len(g.sop)
                    rec["shape"] = sop_shape(g.sop)
                    newterm = sum(1 << f for f, d in enumerate(g.sop.tolist()) if d & SOP_NEWTERM)
                    neg = sum(1 << f for f, d in enumerate(g.sop.tolist()) if d & SOP_NEG)
                    sops.append(np.array([newterm, neg], np.uint32))
                    n_sop += 1
                    tile = 32 * sop_vec(cls)  # warp tile of the persistent kernel
                # index columns: affine column 0, compressed columns
                if compress and g.layout == "coalesced" and g.columns:
                    aff = affine_column0(g.columns[0])
                    if aff is not None:
                        flags |= FLAG_AFFINE0
                        rec["a0_base"], rec["a0_stride"] = aff
                    if len(g.columns) > (aff is not None) and g.n >= CHUNK:
                        comp = [compress_column(c) for c in g.columns]
                        if all(c is not None for c in comp):
                            flags |= FLAG_W16
                            rec["cb_off"], rec["co_off"] = n_cb, n_co
                            for cb, co in comp:
                                cbases.append(cb)
                                coffs.append(co)
                                n_cb += cb.size
                                n_co += co.size
                # output positions
                if g.wpos is not None:  # CSR-window member: positions inside its window
                    flags |= FLAG_WPOS16
                    rec["oo_off"] = n_oo
                    ooffs.append(g.wpos.reshape(-1))
                    n_oo += g.wpos.size
                if g.opos is not None:
                    comp = [compress_column(row, allow_none=True) for row in g.opos]
                    if all(c is not None for c in comp):
                        flags |= FLAG_OPOS16
                        rec["ob_off"], rec["oo_off"] = n_ob, n_oo
                        for ob, oo in comp:
                            obases.append(ob)
                            ooffs.append(oo)
                            n_ob += ob.size
                            n_oo += oo.size
                    else:
                        flags |= FLAG_OPOS32
                        rec["oo_off"] = n_o32
                        op32.append(g.opos.reshape(-1).astype(np.uint32))
                        n_o32 += g.opos.size
                rec["flags"] = flags
                if flags & FLAG_SERIAL:
                    starts = np.zeros(1 if g.n else 0, np.int64)
                else:
                    starts = np.arange(0, g.n, tile, dtype=np.int64)
                unit_tiles.append(np.stack([np.full(starts.size, gi, np.int64), starts], axis=1))
                unit_keys.append(_tile_keys(g, starts, tile))
            if utag == UNIT_WINDOW:  # the unit's "tiles" are its windows [0, n_win)
                if window_units or len(order_groups) - g_begin != windows.pieces.shape[1]:
                    raise AssertionError("one CSR-window unit holding every member")
                n_win = windows.k.size - 1
                window_units.append((len(units), 0, n_win))
                smem = 8 * (int(np.diff(windows.k).max(initial=0)) + 2)  # + alignment slots
                # about one block per window, dispatched in CSR order: variant = rounds of one block per
                # SM cut from the grid (sgb.cu; the first blocks take a second window).  (A persistent grid
                # prefetching the next window's header measured 0.1274 -> 0.1725 ms on C2: concurrently
                # running windows drift apart and stop sharing the L2-resident intermediates, r2x)
                units.append((w, kind, WIN_GRID_CUT, g_begin, len(order_groups), 0, n_win, bs, smem,
                              UNIT_CSR_ONLY | UNIT_JIT | UNIT_WINDOW))
                jit_units.append(len(units) - 1)
                continue
            else:
                t = np.concatenate(unit_tiles) if unit_tiles else np.zeros((0, 2), np.int64)
                keys = np.concatenate(unit_keys) if unit_keys else np.zeros(0, np.int64)
            order_mode = os.environ.get("SGB_TILE_ORDER", "auto")
            t_alt = None
            if jit_unit and order_mode == "auto" and not np.any(keys >= 0) and len(np.unique(t[:, 0])) > 1:
                # two candidate schedules; DevicePlan times both per wave and keeps the faster
                nn = np.array([groups[order_groups[g]].n for g in t[:, 0]], np.float64)
                t_alt = t[np.argsort(t[:, 1] / np.maximum(nn, 1), kind="stable")]
            if np.any(keys >= 0) and order_mode in ("csr", "auto"):
                # CSR-ordered schedule: partial sectors of the output merge in L2
                t = t[np.argsort(keys, kind="stable")]
            elif jit_unit and order_mode == "frac":
                # specialised units: interleave the groups' tiles by the fraction of the group
                # they reach, so groups of different sizes sweep their (mesh-ordered) instances in step
                nn = np.array([groups[order_groups[g]].n for g in t[:, 0]], np.float64) if len(t) else t[:, 1]
                t = t[np.argsort(t[:, 1] / np.maximum(nn, 1), kind="stable")]
            elif jit_unit and order_mode != "group":
                # specialised units: interleave the groups' tiles by instance, so groups that
                # gather the same producer ranges (structured mesh groups) read them while they
                # are still in L2
                t = t[np.argsort(t[:, 1], kind="stable")]
            t0 = sum(len(x) for x in tiles_all)
            tiles_all.append(t)
            tiles_alt.append(t if t_alt is None else t_alt)
            any_alt = any_alt or t_alt is not None
            uflags = UNIT_CSR_ONLY if w >= n_waves else 0
            if jit_unit:
                uflags |= UNIT_JIT
                jit_units.append(len(units))
            if utag == UNIT_VALUE_ONLY:
                uflags |= UNIT_VALUE_ONLY
            elif utag == UNIT_WINDOW:
                uflags |= UNIT_WINDOW | UNIT_CSR_ONLY
            units.append((w, kind, variant, g_begin, len(order_groups), t0, t0 + len(t), bs, regs, uflags))
    cat = lambda xs, dt: (np.concatenate(xs).astype(dt) if xs and sum(len(x) for x in xs)  # noqa: E731
                          else np.zeros(0, dt))
    exact = all(kl.flags & FLAG_EXACT for kl in lowered)
    positions = np.ascontiguousarray(plan.positions, dtype=np.uint32)
    if extra_pos:
        positions = np.concatenate([positions] + extra_pos)
    dp = DevicePlanArrays(
        groups=packed,
        units=np.asarray(units, np.int64).reshape(-1, len(UNIT_FIELDS)),
        tiles=cat(tiles_all, np.int32).reshape(-1, 2),
        tiles_alt=cat(tiles_alt, np.int32).reshape(-1, 2) if any_alt else None,
        n_waves=n_waves,
        tape=cat(tapes, np.uint32).reshape(-1, 4),
        imm=np.asarray(imms, np.float64),
        sop=cat(sops, np.uint32),
        slot_col=cat(scol, np.int32),
        slot_delta=cat(sdel, np.int64),
        cbase=cat(cbases, np.uint32),
        coff=cat(coffs, np.uint16),
        obase=cat(obases, np.uint32),
        ooff=cat(ooffs, np.uint16),
        opos32=cat(op32, np.uint32),
        positions=positions,
        constants=np.ascontiguousarray(plan.constants, dtype=np.float64),
        outputs=np.asarray(plan.outputs, np.int64),
        value_array_size=int(plan.value_array_size),
        input_count=int(plan.input_count),
        needs_zero=int(needs_zero),
        kernels=lowered,
        copies=[(g.wave, g.columns[0], g.opos[0]) for g in groups if g.flags & FLAG_CSR_ONLY and g.tape is None],
        exact=exact,
    )
    dp.csr_layout = sorted(imajor)
    dp.windows = windows
    dp.window_members = list(window) if window is not None else []
    dp.window_units = window_units
    dp.jit_tapes, dp.jit_imms = jit_tapes, jit_imms
    # split the root set of a big multi-root template over k x JIT_BLOCK threads (jit.py: part p =
    # threadIdx.x / JIT_BLOCK evaluates its roots' cone): fewer live registers per thread
    dp.jit_split = {}
    if JIT_SPLIT > 1:
        fu, fb = UNIT_FIELDS.index("flags"), UNIT_FIELDS.index("block_size")
        for uu in range(len(dp.units)):
            r = dp.unit(uu)
            if not r["flags"] & UNIT_JIT or r["flags"] & UNIT_WINDOW or r["group_end"] - r["group_begin"] != 1:
                continue
            gi = r["group_begin"]
            tp = jit_tapes.get(gi)
            if tp is None or len(tp) < JIT_SPLIT_MIN_TAPE or int(dp.groups[gi]["n_roots"]) < 4 * JIT_SPLIT:
                continue
            dp.jit_split[gi] = split_roots(tp, int(dp.groups[gi]["n_roots"]), JIT_SPLIT)
            dp.units[uu, fb] = r["block_size"] * JIT_SPLIT
    if KEEP_BEFORE_GATHER and not window_units and not direct_csr and len(plan.outputs):
        # gather mode: the last wave's output groups' results are what the gather reads next
        outs_sorted = np.sort(np.asarray(plan.outputs, np.int64))
        last_w = n_waves - 1
        for uu in range(len(dp.units)):
            r = dp.unit(uu)
            if r["wave"] != last_w or not r["flags"] & UNIT_JIT:
                continue
            for g in range(r["group_begin"], r["group_end"]):
                rec = dp.groups[g]
                lo = int(rec["dest_base"])
                hi = lo + int(rec["n_roots"]) * int(rec["n"])
                a, b = np.searchsorted(outs_sorted, [lo, hi])
                if b > a and not rec["flags"] & FLAG_STREAM:
                    dp.groups[g]["flags"] |= FLAG_KEEP
    if KEEP_BEFORE_WINDOW and window_units:  # the window unit's operands: keep them in L2
        fw = UNIT_FIELDS.index("wave")
        w_win = int(dp.units[window_units[0][0], fw])
        for uu in range(len(dp.units)):
            r = dp.unit(uu)
            if w_win - KEEP_WAVES <= r["wave"] < w_win and r["flags"] & UNIT_JIT and not r["flags"] & UNIT_WINDOW:
                for g in range(r["group_begin"], r["group_end"]):
                    if not dp.groups[g]["flags"] & FLAG_STREAM:
                        dp.groups[g]["flags"] |= FLAG_KEEP
    dp.wbulk = None
    if wbulk is None:
        wbulk = os.environ.get("SGB_WBULK", "0") == "1"  # measured slower than the register-pipelined windows (r2m)
    if windows is not None and window_units and wbulk:  # feed the window unit with bulk copies
        uw = window_units[0][0]
        wb = window_bulk(dp, uw, windows)
        if wb is not None:
            dp.wbulk = wb
            dp.units[uw, UNIT_FIELDS.index("flags")] |= UNIT_BULK
            dp.units[uw, UNIT_FIELDS.index("block_size")] = WBULK_THREADS
            dp.units[uw, UNIT_FIELDS.index("smem_regs")] = wb.smem
    if jit_units and jit_compile:
        from . import jit as _jit

        dp.jit_cubin, dp.jit_source = _jit.specialise(dp, jit_tapes, jit_imms, jit_units)
    return dp
