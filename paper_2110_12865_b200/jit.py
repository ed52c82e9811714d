"""Specialised tape kernels: a tape unit's groups compiled to straight-line sm_100a code.

The reference's native evaluator is code generation -- ``emit_kernel_source``
prints one C function per group and ``compile_plan`` compiles it with ``cc``
(emit.py:153-245); the paper's GPU backend does the same for GPUs
(PAPER.md:253-260).  This module is that step for the B200: every group of a
plain tape unit (lower.py) becomes one case of a persistent kernel whose body
is the group's device tape unrolled into SSA registers -- the interpreter's
shared-memory scratch file and per-word dispatch disappear, so the body runs
from registers at FP64 issue rate.

Arithmetic is exactly the tape's: every record is one ``__dadd_rn`` /
``__dsub_rn`` / ``__dmul_rn`` / ``__ddiv_rn`` / ``__dsqrt_rn`` (fused
MADD/MSUB/RMSUB stay two roundings), immediates are exact bit patterns,
NVRTC runs with ``-fmad=false``; results are bit-identical to the interpreter
(tests/test_gpu_parity.py runs both).  Index decode, constants and stores are
baked in per group (N, dest_base, p_base, deltas...) like the emitted C bakes
them (emit.py:99-150).

Compiled with NVRTC (``libnvrtc.so.12``, loaded with ctypes) for
``sm_100a``; cubins are cached by source hash.  The C ABI receives the cubin
in the device plan (``sgb_plan_desc.jit_cubin``) and launches kernel
``sgb_tape_u<unit>`` for each unit it names.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import re
import struct
from pathlib import Path

import numpy as np

from . import lower as L

JIT_BLOCK = 256  # threads per block = instances per tile of a specialised unit
BATCH_VEC = 8  # batched: value sets per lane per iteration (8: r45)
BATCH_VEC_SMALL_TAPE = 128  # tape words up to which a unit's batched kernel uses BATCH_VEC (else <= 4)
# cubin cache, keyed by source + NVRTC options: in-tree by default so cubins built on the CPU host
# (__graft_entry__.build) travel with the repository to the GPU box
CACHE = Path(os.environ.get("SGB_JIT_CACHE", Path(__file__).resolve().parent / "_jit_cache"))

_PREAMBLE = r"""
typedef unsigned int u32;
typedef unsigned short u16;
typedef long long i64;
typedef unsigned long long u64;
struct Tables {  // == csrc/sgb.cu Tables
  const void *groups; const u32 *tape; const double *imm; const u32 *sop; const int *slot_col;
  const i64 *slot_delta; const u32 *pos; const double *con; const u32 *cbase; const u16 *coff;
  const u32 *obase; const u16 *ooff; const u32 *opos32; const u32 *fbase;
};
#define NONE 0xFFFFFFFFu
__device__ __forceinline__ double bits(u64 b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ void st_stream(double *a, double v) { __stcs(a, v); }
"""

# glibc's sin / cos / exp / log / pow restated for the device (tools/gen_glibc_math.py): the
# reference's math module, bit for bit
_PREAMBLE += (Path(__file__).resolve().parent / "csrc" / "glibc_math.h").read_text()

_BIN = {L.T_MUL: "__dmul_rn({a}, {b})", L.T_ADD: "__dadd_rn({a}, {b})", L.T_SUB: "__dsub_rn({a}, {b})",
        L.T_DIV: "__ddiv_rn({a}, {b})", L.T_MADD: "__dadd_rn(__dmul_rn({a}, {b}), {c})",
        L.T_MSUB: "__dsub_rn(__dmul_rn({a}, {b}), {c})", L.T_RMSUB: "__dsub_rn({c}, __dmul_rn({a}, {b}))"}
_SLOW = {0: "sgb_sin({a})", 1: "sgb_cos({a})", 2: "sgb_exp({a})", 3: "sgb_log({a})"}


def _imm(v: float) -> str:
    return f"bits(0x{np.float64(v).view(np.uint64).item():016x}ULL)"


def _affine(dp, rec, col: int):
    """(base, stride) when retained column ``col`` of the group is base + stride * i (baked in, no load)."""
    n = int(rec["n"])
    if n < 2 or rec["flags"] & L.FLAG_INTERLEAVED:
        return None
    if col == 0 and rec["flags"] & L.FLAG_AFFINE0:
        return int(rec["a0_base"]), int(rec["a0_stride"])
    off = int(rec["p_off"]) + col * n
    c = np.asarray(dp.positions[off: off + n], dtype=np.int64)
    base, stride = int(c[0]), int(c[1] - c[0])
    if np.array_equal(c, base + stride * np.arange(n, dtype=np.int64)):
        return base, stride
    return None


def _off(v: int) -> str:
    """A table offset as a 64-bit literal (the instance index added to it stays u32)."""
    return f"{int(v)}ull"


# value-array addresses of operand loads in 64-bit arithmetic: `x + idx0 + delta` then folds the
# constant into the load's immediate offset (u32 arithmetic must wrap, so every slot paid its own
# add + widen: C3's assembly 0.208 -> 0.227 ms); every decoded address is < 2^32 either way
INDEX64 = True


def _idx_t(wide: bool = True) -> str:
    return "u64" if INDEX64 and wide else "u32"


def _affine_u32(base: int, stride: int, i: str, wide: bool = True) -> str:
    if INDEX64 and wide:
        return f"({int(base) % 2**64}ull + {int(stride) % 2**64}ull * (u64)({i}))"
    return f"({int(base) % 2**32}u + {int(stride) % 2**32}u * {i})"


def _column(rec, col: int, i: str = "i", dp=None, wide: bool = True) -> str:
    """Index expression (u32) of retained column ``col`` for instance ``i``."""
    n = int(rec["n"])
    f = int(rec["flags"])
    aff = _affine(dp, rec, col) if dp is not None else None
    if aff is None and col == 0 and f & L.FLAG_AFFINE0:
        aff = int(rec["a0_base"]), int(rec["a0_stride"])
    if aff is not None:  # modular u32 arithmetic: every decoded address is < 2^32
        return _affine_u32(aff[0], aff[1], i, wide)
    if f & L.FLAG_W16:
        nch = (n + 31) // 32
        return (f"(__ldg(T.cbase + {_off(int(rec['cb_off']) + col * nch)} + ({i} >> 5)) + "
                f"(u32)__ldcs(T.coff + {_off(int(rec['co_off']) + col * n)} + {i}))")
    if f & L.FLAG_INTERLEAVED:
        return f"__ldcs(T.pos + {_off(int(rec['p_off']))} + (u64){i} * {int(rec['n_ret'])}u + {col}u)"
    return f"__ldcs(T.pos + {_off(int(rec['p_off']) + col * n)} + {i})"


def _out_pos(rec, r: int, i: str = "i") -> str | None:
    n = int(rec["n"])
    f = int(rec["flags"])
    if f & L.FLAG_OPOS16:
        nch = (n + 31) // 32
        # both loads issued together (the base does not depend on the offset)
        return (f"[&]() {{ const u16 o_ = __ldcs(T.ooff + {_off(int(rec['oo_off']) + r * n)} + {i}); "
                f"const u32 b_ = __ldg(T.obase + {_off(int(rec['ob_off']) + r * nch)} + ({i} >> 5)); "
                f"return o_ == 0xFFFF ? NONE : b_ + o_; }}()")
    if f & L.FLAG_OPOS32:
        return f"__ldcs(T.opos32 + {_off(int(rec['oo_off']) + r * n)} + {i})"
    return None


def group_parts(dp, gi: int, tape: np.ndarray, imms: list, iv: str = "i", sfx: str = "",
                batched: bool = False, window: bool = False, bv: str = "b",
                stage: str | None = None, guard: str | None = None,
                keep: set | None = None) -> tuple[list[str], list[str]]:
    """Straight-line CUDA for instance ``iv`` of packed group ``gi`` (register tape -> SSA).

    Returns (load lines, compute + store lines) so several instances' loads can be
    issued before any of them computes.  Variables carry suffix ``sfx``.
    Batched: value set ``b`` of ``X[addr * ld + b]`` (lane = value set).  Window:
    the CSR value goes to the block's shared window ``buf[wpos]`` (no value-array
    store: window members are never re-read).  Stage: an instance-major group's
    results go to the block's staging buffer at ``stage_[(stage) * RP + r]``
    (``stage`` = the instance's offset in the tile, RP = lower.stage_stride); the
    unit writes the tile out coalesced.  ``guard``: every load is predicated on it
    (lanes without an instance issue no memory traffic).  ``keep``: evaluate only these tape
    records (one part of a split root set, lower.split_roots; unused loads are dead code).
    """
    X = (lambda a: f"x + (u64)({a}) * ld + {bv}") if batched else (lambda a: f"x + ({a})")
    G = (lambda e, z: f"({guard}) ? ({e}) : {z}") if guard else (lambda e, z: e)  # noqa: E731
    rec = dp.groups[gi]
    n, S, K = int(rec["n"]), int(rec["n_slots"]), int(rec["n_const"])
    flags = int(rec["flags"])
    cols = dp.slot_col[rec["slot_off"]: rec["slot_off"] + S]
    dels = dp.slot_delta[rec["slot_off"]: rec["slot_off"] + S]
    loads, comp = [], []
    reg: dict[int, str] = {}
    i = iv
    # batched addresses are scaled by ld (x + addr * ld + b): u32 keeps that a 32 x 32 -> 64 multiply
    # (64-bit addresses there measured 2.48 -> 2.95 ms on C5, r2q)
    wide = not batched
    col = lambda c: _column(rec, c, i, dp, wide)  # noqa: E731
    it = _idx_t(wide)
    if S:
        loads.append(f"const {it} idx0{sfx} = {G(f'({it})({col(0)})', '0u')};")
    for s_ in range(S):
        c = int(cols[s_])
        if c < 0:
            addr = (f"idx0{sfx} + {int(dels[s_]) % 2**64}ull" if INDEX64 and wide
                    else f"idx0{sfx} + {int(dels[s_]) % 2**32}u")
        elif c == 0:
            addr = f"idx0{sfx}"
        else:
            addr = col(c)
        loads.append(f"const double s{s_}{sfx} = {G(f'__ldg({X(addr)})', '0.0')};")
        reg[s_] = f"s{s_}{sfx}"
    for k in range(K):
        e = (f"{_off(int(rec['c_off']))} + (u64){i} * {K}u + {k}u" if flags & L.FLAG_INTERLEAVED
             else f"{_off(int(rec['c_off']) + k * n)} + {i}")
        loads.append(f"const double k{k}{sfx} = {G(f'__ldcs(T.con + {e})', '0.0')};")
        reg[S + k] = f"k{k}{sfx}"
    if window:  # window positions (FLAG_WPOS16) load with the operands, not after the compute
        oo_off = int(rec["oo_off"])
        for r in range(int(rec["n_roots"])):
            loads.append(f"const u16 wp{r}{sfx} = "
                         f"{G(f'__ldcs(T.ooff + {_off(oo_off + r * n)} + {i})', '(u16)0xFFFF')};")
    stream = bool(flags & L.FLAG_STREAM)
    opos = lambda r: _out_pos(rec, r, i)  # noqa: E731
    if not window:  # output positions (direct CSR stores) load with the operands, not after the compute
        for r in range(int(rec["n_roots"])):
            if _out_pos(rec, r) is not None and (keep is None or any(
                    t[0] == L.T_ST and t[7] == r and j in keep for j, t in enumerate(tape.tolist()))):
                loads.append(f"const u32 op{r}{sfx} = ({guard or 'true'}) && csr ? {opos(r)} : NONE;")
    for j, t in enumerate(tape.tolist()):
        if keep is not None and j not in keep:
            continue
        op, na, nb, dst, a, b, c, aux = t
        A = ("-" if na else "") + reg.get(a, "0.0")
        B = ("-" if nb else "") + reg.get(b, "0.0")
        C = reg.get(c, "0.0")
        if op == L.T_ST and window:  # CSR-window member: FLAG_WPOS16 position in the block's window
            comp.append(f"if (wp{aux}{sfx} != 0xFFFF) bw[wp{aux}{sfx}] = {reg[a]};")
            continue
        if op == L.T_ST and stage is not None:
            comp.append(f"if (ok{sfx}) stage_[({stage}) * {L.stage_stride(int(rec['n_roots']))} + {aux}] = {reg[a]};")
            continue
        if op == L.T_ST:
            r = aux
            v = reg[a]
            if flags & L.FLAG_IMAJOR:  # CSR layout (lower._RelaidPlan): instance-major results
                x_addr = X(f"{int(rec['dest_base']) + r}u + {i} * {int(rec['n_roots'])}u")
            else:
                x_addr = X(f"{int(rec['dest_base']) + r * n}u + {i}")
            # (L2 keep hints for one value set only: a batched wave is hundreds of MB)
            store = (f"st_stream({x_addr}, {v});" if stream else
                     f"st_keep({x_addr}, {v});" if flags & L.FLAG_KEEP and not batched else f"*({x_addr}) = {v};")
            comp.append(f"if (ok{sfx}{' && !csr' if stream else ''}) {store}")
            if _out_pos(rec, r) is not None:
                dst_o = f"out[(u64)op{r}{sfx} * ld_out + {bv}]" if batched else f"out[op{r}{sfx}]"
                comp.append(f"if (ok{sfx} && op{r}{sfx} != NONE) {dst_o} = {v};")
            continue
        if op == L.T_IMM:
            expr = _imm(imms[aux])
        elif op in _BIN:
            expr = _BIN[op].format(a=f"({A})", b=f"({B})", c=C)
        elif op == L.T_NEG:
            expr = f"-{reg[a]}"
        elif op == L.T_SQRT:
            expr = f"__dsqrt_rn({reg[a]})"
        elif op == L.T_SEL:
            expr = f"({reg[a]} < 0.0 ? {reg[b]} : {C})"
        elif op == L.T_SLOW:
            kind, k = aux >> 16, aux & 0xFFFF
            expr = (f"__dmul_rn({reg[a]}, {reg[a]})" if k == 2 else f"sgb_pow({reg[a]}, {float(k)!r})") \
                if kind == 4 else _SLOW[kind].format(a=reg[a])
        else:
            raise ValueError(f"unknown tape op {op}")
        comp.append(f"const double t{j}{sfx} = {expr};")
        reg[dst] = f"t{j}{sfx}"
    return loads, comp


def group_batch_body(dp, gi, tape, imms, vec: int) -> list[str]:
    """Batched: instance ``i`` for value sets b + 32 v (v < vec), loads of all of them first."""
    n = int(dp.groups[gi]["n"])
    lines, comps = [], []
    shared = None
    for v in range(vec):
        lines.append(f"const i64 b{v} = b + {32 * v}LL;")
        lines.append(f"const bool ok_{v} = b{v} < batch;")
        lines.append(f"const i64 bc{v} = ok_{v} ? b{v} : batch - 1;")
        ld, cp = group_parts(dp, gi, tape, imms, iv="i", sfx=f"_{v}", batched=True, bv=f"bc{v}")
        # the index decode (idx0 / column loads) is the same for every value set: emit it once
        if shared is None:
            shared = [ln for ln in ld if ln.startswith(f"const {_idx_t(False)} idx0")]
            lines = shared[:1] + lines if shared else lines
            opl = [ln for ln in ld if ln.startswith("const u32 op")]  # output positions: per instance
            lines = opl + lines
        ld = [ln.replace(f"idx0_{v}", "idx0_0") for ln in ld
              if not ln.startswith(f"const {_idx_t(False)} idx0") and not ln.startswith("const u32 op")]
        cp = [ln.replace(f"idx0_{v}", "idx0_0") for ln in cp]
        cp = [re.sub(rf"\bop(\d+)_{v}\b", r"op\1_0", ln) for ln in cp]
        lines += ld
        comps += cp
    if shared:
        lines = [shared[0].replace("idx0_0", "idx0_0")] + [ln for ln in lines if ln != shared[0]]
    return lines + comps


def group_vec_body(dp, gi, tape, imms, vec: int, base: str, stride: int, batched=False, window=False,
                   limit: str | None = None, stage: bool = False, keep: set | None = None,
                   lane: str = "threadIdx.x"):
    """VEC instances base + v*stride: every instance's loads first, then the computes.

    ``limit``: instance v is valid only if ``limit`` (with ``{v}`` = v * stride) holds too.
    ``keep``: the tape records of one part of a split root set; ``lane``: the thread's instance
    lane inside the tile (stage position).
    """
    n = int(dp.groups[gi]["n"])
    lines, comps = [], []
    for v in range(vec):
        lines.append(f"const u32 iv{v} = {base} + {v * stride}u;")
        extra = f" && ({limit.format(v=v * stride)})" if limit else ""
        lines.append(f"const bool ok_{v} = iv{v} < {n}u{extra};")
        lines.append(f"const u32 ic{v} = ok_{v} ? iv{v} : {n - 1}u;")
        ld, cp = group_parts(dp, gi, tape, imms, iv=f"ic{v}", sfx=f"_{v}", batched=batched, window=window,
                             stage=f"{lane} + {v * stride}" if stage else None, keep=keep)
        lines += ld
        comps += cp
    return lines + comps


def _check_stores(tape, n_roots: int, gi: int):
    roots = sorted(int(t[7]) for t in tape.tolist() if t[0] == L.T_ST)
    if roots != list(range(n_roots)):
        raise ValueError(f"group {gi}: tape stores roots {roots}, expected 0..{n_roots - 1}")


def _stage_out(rec, vec: int, threads: int = JIT_BLOCK) -> list[str]:
    """Write a staged tile of an instance-major group: its instances' results are one contiguous
    run ``dest_base + tile_start * R ...`` of the value array, stored by consecutive threads."""
    n, R = int(rec["n"]), int(rec["n_roots"])
    rp = L.stage_stride(R)
    st = "__stcs(x + base_ + k_, v_)" if rec["flags"] & L.FLAG_STREAM else "x[base_ + k_] = v_"
    return ["__syncthreads();",
            f"{{ const u32 cnt_ = min({JIT_BLOCK * vec}u, {n}u - (u32)tl.y) * {R}u;",
            f"  const u32 base_ = {int(rec['dest_base'])}u + (u32)tl.y * {R}u;",
            "  #pragma unroll 8",  # shared loads of the write-out in flight together (C3: 78 per thread)
            f"  for (u32 k_ = threadIdx.x; k_ < cnt_; k_ += {threads}u) {{",
            f"    const u32 q_ = k_ / {R}u; const double v_ = stage_[q_ * {rp}u + (k_ - q_ * {R}u)]; {st}; }} }}",
            "__syncthreads();"]


_KEEP_HELPER = r"""
#ifndef SGB_KEEP_HELPER
#define SGB_KEEP_HELPER
__device__ __forceinline__ void st_keep(double *a, double v) {  // store, L2 evict_last
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
#endif
"""


def unit_source(dp, u: int, tapes: dict, imms: dict) -> str:
    """Persistent kernels for tape unit ``u``: a case per group.

    ``sgb_tape_u<u>``: one value set, one instance per thread (tiles of JIT_BLOCK
    instances).  ``sgb_tape_b<u>``: batched, one instance per warp, lanes sweep
    the value sets (tiles of JIT_BLOCK / 32 instances, csrc btiles).
    """
    unit = dp.unit(u)
    out = []
    if any(int(dp.groups[g]["flags"]) & L.FLAG_KEEP for g in range(unit["group_begin"], unit["group_end"])):
        out.append(_KEEP_HELPER)
    split = getattr(dp, "jit_split", {}).get(unit["group_begin"]) if unit["group_end"] - unit["group_begin"] == 1 \
        else None
    nthreads = JIT_BLOCK * (len(split) if split else 1)
    big = max(len(tapes[gi]) for gi in range(unit["group_begin"], unit["group_end"]))
    # batched value sets per lane: 8 for small templates (C5: 2.90 -> 2.47 ms, r45); big templates keep
    # 4 (their register file is full already, and the body is compiled once per value set)
    bvec = BATCH_VEC if big <= BATCH_VEC_SMALL_TAPE else min(BATCH_VEC, 4)
    for batched in (False, True):
        if batched:
            head = [f'extern "C" __global__ void __launch_bounds__({JIT_BLOCK}) sgb_tape_b{u}(',
                    "    Tables T, const int2 *tiles, i64 n_tiles, double *x, i64 ld, i64 batch, double *out,",
                    "    i64 ld_out, int csr) {",
                    "  for (i64 t = blockIdx.x; t < n_tiles; t += gridDim.x) {",
                    "    const int2 tl = tiles[t];",
                    "    const u32 i = (u32)tl.y + (threadIdx.x >> 5);",
                    f"    for (i64 b = threadIdx.x & 31; b < batch; b += {32 * bvec}) {{",
                    "    switch (tl.x) {"]
        else:
            # no register cap: huge templates run best uncapped -- a 2-block cap spilled and measured
            # 2.7x slower on C3 (r24)
            bounds = f"{nthreads}"
            lane = f"(threadIdx.x % {JIT_BLOCK}u)" if split else "threadIdx.x"
            head = [f'extern "C" __global__ void __launch_bounds__({bounds}) sgb_tape_u{u}(',
                    "    Tables T, const int2 *tiles, i64 n_tiles, double *x, double *out, int csr) {",
                    "  extern __shared__ double stage_[];",
                    "  for (i64 t = blockIdx.x; t < n_tiles; t += gridDim.x) {",
                    "    const int2 tl = tiles[t];",
                    f"    const u32 i = (u32)tl.y + {lane};",
                    f"    const u32 part_ = threadIdx.x / {JIT_BLOCK}u;  // root-set part (lower.split_roots)",
                    "    {",
                    "    switch (tl.x) {"]
        out += head
        vec = 1 if batched else max(1, int(unit["variant"]))
        for gi in range(unit["group_begin"], unit["group_end"]):
            rec = dp.groups[gi]
            _check_stores(tapes[gi], int(rec["n_roots"]), gi)
            staged = not batched and bool(rec["flags"] & L.FLAG_IMAJOR)
            out.append(f"    case {gi}: {{")
            if not staged:  # (a staged tile keeps every thread: the block synchronises)
                out.append(f"      if (i >= {int(rec['n'])}u) break;")
            if rec["flags"] & L.FLAG_CSR_ONLY:
                out.append("      if (!csr) break;")
            if batched or not split:
                body = (group_batch_body(dp, gi, tapes[gi], imms[gi], bvec) if batched else
                        group_vec_body(dp, gi, tapes[gi], imms[gi], vec, "i", JIT_BLOCK, stage=staged))
            else:  # part p of the split root set: its roots' cone, the same tile of instances
                body = []
                for p, keep in enumerate(split):
                    body.append(f"if (part_ == {p}u) {{")
                    body += ["  " + ln for ln in group_vec_body(dp, gi, tapes[gi], imms[gi], vec, "i", JIT_BLOCK,
                                                                 stage=staged, keep=keep,
                                                                 lane=f"(threadIdx.x % {JIT_BLOCK}u)")]
                    body.append("}")
            out += ["      " + ln for ln in body]
            if staged:
                out += ["      " + ln for ln in _stage_out(rec, vec, nthreads)]
            out.append("    } break;")
        out += ["    default: break;", "    }", "    }", "  }", "}", ""]
    return "\n".join(out)


# -- NVRTC ------------------------------------------------------------------------------

_nvrtc = None


def _lib():
    global _nvrtc
    if _nvrtc is None:
        last = None
        for name in (os.environ.get("SGB_NVRTC"), "libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12"):
            if not name:
                continue
            try:
                _nvrtc = ctypes.CDLL(name)
                break
            except OSError as e:
                last = e
        if _nvrtc is None:
            raise RuntimeError(f"NVRTC not found: {last}")
    return _nvrtc


def available() -> bool:
    try:
        _lib()
        return True
    except RuntimeError:
        return False


NVRTC_OPTS = (b"--gpu-architecture=sm_100a", b"-fmad=false", b"-std=c++17", b"-default-device", b"-lineinfo",
              b"--extra-device-vectorization")
stats = {"hits": 0, "compiles": 0, "compile_s": 0.0}


def cache_key(src: str) -> str:
    return hashlib.sha1(b"\0".join(NVRTC_OPTS) + b"\0" + src.encode()).hexdigest()


def compile_cubin(src: str, name: str = "sgb_tape.cu") -> bytes:
    """NVRTC -> sm_100a cubin (no GPU needed); cached by source + options hash."""
    import time

    path = CACHE / f"{cache_key(src)}.cubin"
    if path.exists():
        stats["hits"] += 1
        return path.read_bytes()
    t0 = time.perf_counter()
    lib = _lib()
    prog = ctypes.c_void_p()
    rc = lib.nvrtcCreateProgram(ctypes.byref(prog), src.encode(), name.encode(), 0, None, None)
    if rc:
        raise RuntimeError(f"nvrtcCreateProgram failed ({rc})")
    opts = list(NVRTC_OPTS)
    arr = (ctypes.c_char_p * len(opts))(*opts)
    rc = lib.nvrtcCompileProgram(prog, len(opts), arr)
    if rc:
        size = ctypes.c_size_t()
        lib.nvrtcGetProgramLogSize(prog, ctypes.byref(size))
        log = ctypes.create_string_buffer(size.value)
        lib.nvrtcGetProgramLog(prog, log)
        lib.nvrtcDestroyProgram(ctypes.byref(prog))
        raise RuntimeError(f"NVRTC compile failed ({rc}):\n{log.value.decode(errors='replace')[:4000]}")
    size = ctypes.c_size_t()
    lib.nvrtcGetCUBINSize(prog, ctypes.byref(size))
    buf = ctypes.create_string_buffer(size.value)
    lib.nvrtcGetCUBIN(prog, buf)
    lib.nvrtcDestroyProgram(ctypes.byref(prog))
    cubin = buf.raw
    stats["compiles"] += 1
    stats["compile_s"] += time.perf_counter() - t0
    try:
        CACHE.mkdir(parents=True, exist_ok=True)
        tmp = path.with_suffix(f".{os.getpid()}.tmp")
        tmp.write_bytes(cubin)
        os.replace(tmp, path)
    except OSError:
        pass
    return cubin


WINDOW_LOADS = 32  # loads in flight per thread per chunk of a window kernel (C2: 24 0.134 ms, 32 0.128, 40 0.144, r2h)
COPY_UNROLL = 6  # copied outputs per thread in flight
WINDOW_MIN_BLOCKS = 3  # resident windows per SM the window kernel's register budget is sized for
WINDOW_COPY_OVERLAP = False  # first copy batch in flight with the first member chunk
COPY_OVERLAP_LOADS = 9  # registers (in doubles) the first copy batch takes from the first chunk
WBULK_LOADS = 16  # bulk-fed window kernel: shared-memory loads per thread per member chunk


def window_source(dp, u: int, tapes: dict, imms: dict) -> str:
    """CSR-window kernel of unit ``u`` (lower._csr_windows): block w assembles the outputs
    [win_k[w], win_k[w+1]) in shared memory and writes them out with 16-byte streaming stores.

    Work inside a window is block-uniform, so nothing diverges: the outputs copied from the
    value array (inputs, earlier waves' results) first, then the members in chunks -- every
    member of a chunk takes its piece (instance range) with one instance per thread, all the
    chunk's loads (operands and window positions) issued before its computes (WINDOW_LOADS per
    thread) -- each result stored at its FLAG_WPOS16 position in the window.  Members store
    nothing to the value array (the last wave: never re-read), so every output crosses HBM
    once, coalesced.  (Staging the row-aligned members' operand streams and the copies in shared
    memory with cp.async -- one round trip per window -- measured 14-19 % slower on C2, r2e/r2f.)
    """
    unit = dp.unit(u)
    g0, g1 = unit["group_begin"], unit["group_end"]
    J = g1 - g0
    chunks, cur, width = [], [], 0
    for gi in range(g0, g1):
        rec = dp.groups[gi]
        _check_stores(tapes[gi], int(rec["n_roots"]), gi)
        wdt = max(1, int(rec["n_slots"]) + int(rec["n_const"]))
        # the first chunk shares the register budget with the first batch of copies in flight
        cap = WINDOW_LOADS - (COPY_OVERLAP_LOADS if WINDOW_COPY_OVERLAP and not chunks else 0)
        if cur and width + wdt > cap:
            chunks.append(cur)
            cur, width = [], 0
        cur.append(gi)
        width += wdt
    if cur:
        chunks.append(cur)
    B = JIT_BLOCK
    out = [f'extern "C" __global__ void __launch_bounds__({B}, {WINDOW_MIN_BLOCKS}) sgb_window_u{u}(',
           "    Tables T, const int2 *pieces, const i64 *win_k, const i64 *copy_off, const u32 *copy_src,",
           "    const u16 *copy_pos, i64 n_win, const double *x, double *out) {",
           "  extern __shared__ __align__(16) double buf[];",
           f"  __shared__ int2 sp[{J}];",
           "  const int tid = threadIdx.x;",
           "  for (i64 w = blockIdx.x; w < n_win; w += gridDim.x) {",
           f"    for (int j = tid; j < {J}; j += {B}) sp[j] = __ldg(pieces + w * {J} + j);",
           "    const i64 k0 = __ldg(win_k + w);",
           "    const u32 len_ = (u32)(__ldg(win_k + w + 1) - k0);",
           "    const i64 c0_ = __ldg(copy_off + w), c1_ = __ldg(copy_off + w + 1);",
           "    // window position p at bw[p]: out + k0 - head_ is 16-byte aligned, so is buf",
           "    const u32 head_ = (u32)((reinterpret_cast<u64>(out + k0) >> 3) & 1ull);",
           "    double *bw = buf + head_;",
           "    __syncthreads();"]

    def copy_loop(first: str, pre: str) -> list:
        lines = [f"    for (i64 c = {first}; c < c1_; c += {B * COPY_UNROLL}) {{"]
        for q in range(COPY_UNROLL):  # named registers (no local arrays): every copy's loads in flight
            lines.append(f"      const bool {pre}q{q} = c + {q * B} < c1_;")
            lines.append(f"      const u16 {pre}p{q} = {pre}q{q} ? __ldcs(copy_pos + c + {q * B}) : (u16)0;")
            lines.append(f"      const double {pre}v{q} = {pre}q{q} ? __ldg(x + __ldcs(copy_src + c + {q * B})) : 0.0;")
        lines += [f"      if ({pre}q{q}) bw[{pre}p{q}] = {pre}v{q};" for q in range(COPY_UNROLL)]
        return lines + ["    }"]

    if WINDOW_COPY_OVERLAP:  # the first copy batch's loads in flight with the first member chunk's
        out.append("    const i64 cb_ = c0_ + tid;")
        for q in range(COPY_UNROLL):
            out.append(f"    const bool cq{q} = cb_ + {q * B} < c1_;")
            out.append(f"    const u16 cp{q} = cq{q} ? __ldcs(copy_pos + cb_ + {q * B}) : (u16)0;")
            out.append(f"    const double cv{q} = cq{q} ? __ldg(x + __ldcs(copy_src + cb_ + {q * B})) : 0.0;")
    else:
        out += copy_loop("c0_ + tid", "c")
    for k_, chunk in enumerate(chunks):
        if WINDOW_COPY_OVERLAP and k_ == 1:
            out += [f"    if (cq{q}) bw[cp{q}] = cv{q};" for q in range(COPY_UNROLL)]
            out += copy_loop(f"cb_ + {B * COPY_UNROLL}", "d")
        cmax = "0"
        for gi in chunk:
            cmax = f"max({cmax}, sp[{gi - g0}].y)"
        out.append(f"    for (int c0 = 0, cmax_ = {cmax}; c0 < cmax_; c0 += {B}) {{")
        loads, comps = [], []
        for gi in chunk:
            j = gi - g0
            out.append(f"      const bool ok_{j} = c0 + tid < sp[{j}].y;")
            out.append(f"      const u32 i_{j} = ok_{j} ? (u32)(sp[{j}].x + c0 + tid) : 0u;")
            ld, cp = group_parts(dp, gi, tapes[gi], imms[gi], iv=f"i_{j}", sfx=f"_{j}", window=True,
                                 guard=f"ok_{j}")
            loads += ld
            comps += cp
        out += ["      " + ln for ln in loads + comps]
        out.append("    }")
    if WINDOW_COPY_OVERLAP and len(chunks) < 2:
        out += [f"    if (cq{q}) bw[cp{q}] = cv{q};" for q in range(COPY_UNROLL)]
        out += copy_loop(f"cb_ + {B * COPY_UNROLL}", "d")
    out += ["    __syncthreads();",
            "    {  // 16-byte shared loads and streaming stores; the pair straddling k0 writes its second half",
            "      const u32 tot_ = len_ + head_;",
            "      double2 *o2 = reinterpret_cast<double2 *>(out + k0 - head_);",
            "      const double2 *b2 = reinterpret_cast<const double2 *>(buf);",
            f"      for (u32 q = tid; q < (tot_ >> 1); q += {B}) {{",
            "        const double2 v_ = b2[q];",
            "        if (q == 0 && head_) __stcs(out + k0, v_.y); else __stcs(o2 + q, v_);",
            "      }",
            "      if (tid == 0 && (tot_ & 1u)) __stcs(out + k0 + len_ - 1, buf[tot_ - 1]);",
            "    }",
            "    if (w + gridDim.x < n_win) __syncthreads();  // the window buffer is reused (uniform)",
            "  }",
            "}",
            ""]
    return "\n".join(out)


_WBULK_HELPERS = r"""
#ifndef SGB_WBULK_HELPERS
#define SGB_WBULK_HELPERS
__device__ __forceinline__ u32 sgb_smem(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sgb_mbar_init(u64 *b, u32 n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sgb_smem(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void sgb_mbar_expect(u64 *b, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sgb_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void sgb_mbar_expect_only(u64 *b, u32 bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(sgb_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void sgb_mbar_arrive(u64 *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sgb_smem(b)) : "memory");
}
__device__ __forceinline__ void sgb_mbar_wait(u64 *b, u32 parity) {
  asm volatile("{\n .reg .pred P1;\n LAB_WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
               " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n }" ::"r"(sgb_smem(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void sgb_bulk_g2s(void *dst, const void *src, u32 bytes, u64 *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(sgb_smem(dst)), "l"(src), "r"(bytes), "r"(sgb_smem(b)) : "memory");
}
__device__ __forceinline__ void sgb_bar_consumers(u32 n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }
#endif
"""


def _window_chunks(dp, g0: int, members: list, tapes: dict, imms: dict, threads: int,
                   lane: str = "tid", split: bool = False, loads: int | None = None) -> list:
    """Members evaluated from the value array (global loads), chunked so every thread has at
    most WINDOW_LOADS loads in flight: a chunk's loads (operands + window positions) are all
    issued before its computes.  Member j's piece is ``sp[j]``; results go to ``bw[wpos]``;
    instance c0 + ``lane`` per thread.  ``split``: a list of (loads, lines) per chunk."""
    cap = WINDOW_LOADS if loads is None else loads
    chunks, cur, width = [], [], 0
    for gi in members:
        rec = dp.groups[gi]
        _check_stores(tapes[gi], int(rec["n_roots"]), gi)
        wdt = max(1, int(rec["n_slots"]) + int(rec["n_const"]))
        if cur and width + wdt > cap:
            chunks.append(cur)
            cur, width = [], 0
        cur.append(gi)
        width += wdt
    if cur:
        chunks.append(cur)
    out, parts = [], []
    for chunk in chunks:
        lines = []
        cmax = "0"
        for gi in chunk:
            cmax = f"max({cmax}, sp[{gi - g0}].y)"
        if split:  # (the bulk kernel's code size matters more than overlapping passes)
            lines.append("    #pragma unroll 1")
        lines.append(f"    for (int c0 = 0, cmax_ = {cmax}; c0 < cmax_; c0 += {threads}) {{")
        loads, comps = [], []
        for gi in chunk:
            j = gi - g0
            lines.append(f"      const bool ok_{j} = c0 + {lane} < sp[{j}].y;")
            lines.append(f"      const u32 i_{j} = ok_{j} ? (u32)(sp[{j}].x + c0 + {lane}) : 0u;")
            ld, cp = group_parts(dp, gi, tapes[gi], imms[gi], iv=f"i_{j}", sfx=f"_{j}", window=True,
                                 guard=f"ok_{j}")
            loads += ld
            comps += cp
        lines += ["      " + ln for ln in loads + comps]
        lines.append("    }")
        out += lines
        parts.append((sum(max(1, int(dp.groups[gi]["n_slots"]) + int(dp.groups[gi]["n_const"])) for gi in chunk),
                      lines))
    return parts if split else out


def _window_writeout(threads: int) -> list[str]:
    """The assembled window buf[head_ ..] -> out[k0 ..]: 16-byte shared loads and streaming stores
    (out + k0 - head_ is 16-byte aligned; the pair straddling k0 writes its second half)."""
    return ["    {",
            "      const u32 tot_ = len_ + head_;",
            "      double2 *o2 = reinterpret_cast<double2 *>(out + k0 - head_);",
            "      const double2 *b2 = reinterpret_cast<const double2 *>(buf);",
            f"      for (u32 q = tid; q < (tot_ >> 1); q += {threads}) {{",
            "        const double2 v_ = b2[q];",
            "        if (q == 0 && head_) __stcs(out + k0, v_.y); else __stcs(o2 + q, v_);",
            "      }",
            "      if (tid == 0 && (tot_ & 1u)) __stcs(out + k0 + len_ - 1, buf[tot_ - 1]);",
            "    }"]


def wbulk_source(dp, u: int, tapes: dict, imms: dict) -> str:
    """Bulk-fed CSR-window kernel of unit ``u`` (lower.WindowBulk): persistent blocks of
    WBULK_CONSUMERS consumer threads + one producer warp; block b walks windows b, b + grid, ...

    The producer thread copies each window's consumer blob and its merged value-array intervals
    into the next slot of a shared-memory ring with ``cp.async.bulk`` (TMA engine, completion
    counted on the slot's ``full`` mbarrier) as soon as the consumers have released that slot
    (``empty`` mbarrier), so the copies of the next windows run while the consumers evaluate this
    one.  The consumers issue the window's copy gathers first, evaluate the bulk members from the
    ring (operands ``X[run offset + t]``, window positions from the blob), the other members from
    the value array (chunked loads, as window_source), store the copies, release the slot and
    write the window out with 16-byte streaming stores.  Same arithmetic as every other path.
    """
    wb = dp.wbulk
    unit = dp.unit(u)
    g0, g1 = unit["group_begin"], unit["group_end"]
    CT = L.WBULK_CONSUMERS  # threads per member group (one instance each per pass)
    H = L.WBULK_GROUPS  # member groups: chunks of members spread over H x CT consumer threads
    NC = H * CT
    bulk = set(wb.members)
    out = [_WBULK_HELPERS,
           f'extern "C" __global__ void __launch_bounds__({NC + 32}, 1) sgb_wbulk_u{u}(',
           "    Tables T, const unsigned char *meta, const i64 *meta_off, const uint2 *iv, const i64 *iv_off,",
           "    i64 n_win, const double *x, double *out, i64 ring, i64 slot_meta, i64 slot_x, i64 bwb) {",
           "  extern __shared__ __align__(128) unsigned char smem_[];",
           "  __shared__ __align__(8) u64 full_[8], empty_[8];",
           "  const int tid = threadIdx.x;",
           "  double *buf = reinterpret_cast<double *>(smem_);",
           "  unsigned char *ring_ = smem_ + bwb;",
           "  const i64 slot = slot_meta + slot_x;",
           "  const u32 R = (u32)ring;",
           "  if (tid == 0) {",
           "    for (u32 r = 0; r < R; ++r) { sgb_mbar_init(&full_[r], 1); sgb_mbar_init(&empty_[r], 1); }",
           '    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");',
           "  }",
           "  __syncthreads();",
           f"  if (tid >= {NC}) {{  // producer warp: lane l issues the bulk copies of intervals l, l + 32, ...",
           f"    const u32 lane = tid - {NC};",
           "    u32 q = 0;",
           "    for (i64 w = blockIdx.x; w < n_win; w += gridDim.x, ++q) {",
           "      const u32 s = q % R;",
           "      const i64 m0 = __ldg(meta_off + w), m1 = __ldg(meta_off + w + 1);",
           "      const i64 v0 = __ldg(iv_off + w), v1 = __ldg(iv_off + w + 1);",
           "      uint2 e = make_uint2(0u, 0u);",
           "      if (v0 + lane < v1) e = __ldg(iv + v0 + lane);  // the first 32 intervals: loads before the wait",
           "      if (q >= R) sgb_mbar_wait(&empty_[s], ((q / R) - 1u) & 1u);",
           "      unsigned char *sm = ring_ + (i64)s * slot;",
           "      u32 off = 0;",
           "      for (i64 b = v0; b < v1; b += 32) {",
           "        if (b != v0) { e = make_uint2(0u, 0u); if (b + lane < v1) e = __ldg(iv + b + lane); }",
           "        const u32 by = 8u * e.y;",
           "        u32 inc = by;  // inclusive prefix sum of the lanes' bytes",
           "        for (int d = 1; d < 32; d <<= 1) { const u32 t = __shfl_up_sync(0xffffffffu, inc, d); if ((int)lane >= d) inc += t; }",
           "        const u32 tot = __shfl_sync(0xffffffffu, inc, 31);",
           "        if (lane == 0) sgb_mbar_expect_only(&full_[s], tot);  // expected before any of them lands",
           "        __syncwarp();",
           "        if (by) sgb_bulk_g2s(sm + slot_meta + off + inc - by, x + e.x, by, &full_[s]);",
           "        off += tot;",
           "      }",
           "      if (lane == 0) {",
           "        sgb_mbar_expect(&full_[s], (u32)(m1 - m0));  // the blob; the arrival closes the phase",
           "        sgb_bulk_g2s(sm, meta + m0, (u32)(m1 - m0), &full_[s]);",
           "      }",
           "      __syncwarp();",
           "    }",
           "    return;",
           "  }",
           f"  const int grp_ = tid / {CT}, tl_ = tid % {CT};  // member group, instance lane",
           "  u32 q = 0;",
           "  for (i64 w = blockIdx.x; w < n_win; w += gridDim.x, ++q) {",
           "    const u32 s = q % R;",
           "    const unsigned char *sm = ring_ + (i64)s * slot;",
           "    sgb_mbar_wait(&full_[s], (q / R) & 1u);",
           "    const u32 *hd_ = reinterpret_cast<const u32 *>(sm);",
           "    const u32 nc_ = hd_[0], len_ = hd_[3];",
           "    const i64 k0 = *reinterpret_cast<const i64 *>(sm + 16);",
           "    const int2 *sp = reinterpret_cast<const int2 *>(sm + 32);",
           f"    const u16 *roff = reinterpret_cast<const u16 *>(sm + {wb.roff_at});",
           f"    const u16 *woff = reinterpret_cast<const u16 *>(sm + {wb.woff_at});",
           f"    const u16 *wps = reinterpret_cast<const u16 *>(sm + {wb.wpos_at});",
           "    const u32 *csrc = reinterpret_cast<const u32 *>(sm + hd_[1]);",
           "    const u16 *cpos = reinterpret_cast<const u16 *>(sm + hd_[2]);",
           "    const double *X = reinterpret_cast<const double *>(sm + slot_meta);",
           "    const u32 head_ = (u32)((reinterpret_cast<u64>(out + k0) >> 3) & 1ull);",
           "    double *bw = buf + head_;"]
    U = COPY_UNROLL
    for q in range(U):  # first batch of copies: gathers in flight while the members evaluate
        out.append(f"    const bool cq{q} = tid + {q * NC}u < nc_;")
        out.append(f"    const u16 cp{q} = cq{q} ? cpos[tid + {q * NC}u] : (u16)0;")
        out.append(f"    const double cv{q} = cq{q} ? __ldg(x + csrc[tid + {q * NC}u]) : 0.0;")
    # bulk members in chunks of at most WINDOW_LOADS shared-memory loads per thread: a chunk's run /
    # position offsets go to registers once per window, then per pass every operand and position of
    # the chunk is loaded (indices clamped into the piece, no branches) before any result is stored
    info, ro, wo = [], 0, 0
    for j in range(g1 - g0):
        if j not in bulk:
            continue
        rec = dp.groups[g0 + j]
        S, R_ = int(rec["n_slots"]), int(rec["n_roots"])
        _check_stores(tapes[g0 + j], R_, g0 + j)
        info.append((j, S, R_, ro, wo))
        ro += S
        wo += R_
    chunks, cur, width = [], [], 0
    for it in info:
        wdt = it[1] + it[2]
        if cur and width + wdt > WBULK_LOADS:
            chunks.append(cur)
            cur, width = [], 0
        cur.append(it)
        width += wdt
    if cur:
        chunks.append(cur)
    blocks = []  # (load weight, lines) per chunk, spread over the member groups below
    for chunk in chunks:
        out_c = out
        out = []
        out.append("    {")
        cmax = "0"
        for j, S, R_, ro_, wo_ in chunk:
            out.append(f"      const int n_{j} = sp[{j}].y;")
            for s_ in range(S):
                out.append(f"      const u32 ra{s_}_{j} = roff[{ro_ + s_}];")
            for r_ in range(R_):
                out.append(f"      const u32 wa{r_}_{j} = woff[{wo_ + r_}];")
            cmax = f"max({cmax}, n_{j})"
        out.append("      #pragma unroll 1")
        out.append(f"      for (int c0 = 0, cmax_ = {cmax}; c0 < cmax_; c0 += {CT}) {{")
        loads, comps = [], []
        for j, S, R_, ro_, wo_ in chunk:
            gi = g0 + j
            loads.append(f"const bool ok_{j} = c0 + tl_ < n_{j};")
            loads.append(f"const u32 t_{j} = ok_{j} ? (u32)(c0 + tl_) : 0u;")
            for s_ in range(S):
                loads.append(f"const double s{s_}_{j} = X[ra{s_}_{j} + t_{j}];")
            for r_ in range(R_):
                loads.append(f"const u16 wv{r_}_{j} = wps[wa{r_}_{j} + t_{j}];")
                loads.append(f"const u16 wp{r_}_{j} = ok_{j} ? wv{r_}_{j} : (u16)0xFFFF;")
            _, cp = group_parts(dp, gi, tapes[gi], imms[gi], iv=f"t_{j}", sfx=f"_{j}", window=True)
            comps += cp
        out += ["        " + ln for ln in loads + comps]
        out.append("      }")
        out.append("    }")
        blocks.append((sum(c[1] + c[2] for c in chunk), out))
        out = out_c
    blocks += _window_chunks(dp, g0, [g0 + j for j in range(g1 - g0) if j not in bulk], tapes, imms, CT,
                             lane="tl_", split=True, loads=WBULK_LOADS)
    load = [0] * H
    per = [[] for _ in range(H)]
    for wgt, lines in sorted(blocks, key=lambda b: -b[0]):  # heaviest first onto the lightest group
        h = load.index(min(load))
        load[h] += wgt
        per[h].append(lines)
    for h in range(H):
        if per[h]:
            out.append(f"    if (grp_ == {h}) {{")
            for lines in per[h]:
                out += lines
            out.append("    }")
    out += [f"    if (cq{q}) bw[cp{q}] = cv{q};" for q in range(U)]
    out += [f"    for (u32 c = tid + {U * NC}u; c < nc_; c += {U * NC}u) {{"]
    for q in range(U):
        out.append(f"      const bool dq{q} = c + {q * NC}u < nc_;")
        out.append(f"      const u16 dp{q} = dq{q} ? cpos[c + {q * NC}u] : (u16)0;")
        out.append(f"      const double dv{q} = dq{q} ? __ldg(x + csrc[c + {q * NC}u]) : 0.0;")
    out += [f"      if (dq{q}) bw[dp{q}] = dv{q};" for q in range(U)]
    out += ["    }",
            f"    sgb_bar_consumers({NC});",
            "    if (tid == 0) sgb_mbar_arrive(&empty_[s]);  // every read of the slot is done"]
    out += _window_writeout(NC)
    out += [f"    sgb_bar_consumers({NC});  // the window buffer is free again",
            "  }",
            "}",
            ""]
    return "\n".join(out)


def specialise(dp, tapes: dict, imms: dict, units: list[int]) -> tuple[bytes, str]:
    """Compile the given tape units of a lowered plan; returns (cubin, source)."""
    parts = []
    for u in units:
        if dp.unit(u)["flags"] & L.UNIT_BULK:
            parts.append(wbulk_source(dp, u, tapes, imms))
        elif dp.unit(u)["flags"] & L.UNIT_WINDOW:
            parts.append(window_source(dp, u, tapes, imms))
        else:
            parts.append(unit_source(dp, u, tapes, imms))
    src = _PREAMBLE + "\n".join(parts)
    return compile_cubin(src), src


def _pack_u32(vals) -> bytes:
    return struct.pack(f"<{len(vals)}I", *vals)
