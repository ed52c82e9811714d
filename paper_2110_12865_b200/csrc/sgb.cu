// sgb.cu -- sm_100a plan-evaluation kernels and the C ABI of include/sgb.h.
//
// Executes the device plan built by paper_2110_12865_b200/lower.py from a
// reference ExecutionPlan (/root/reference/pkg/src/sparsegen/codegen.py:56-98).
// Semantics are those of the reference evaluators interpret_plan
// (codegen.py:404-512) and the emitted sg_run (emit.py:90-195):
//   * kernels run in dependency waves; every group of a wave runs inside the
//     wave's launch units (tape units, one sum-of-products unit) through a
//     per-block tile table (group, first instance);
//   * every instance evaluates its template's live nodes in stored order; n-ary
//     ADD / MUL fold left (codegen.py:472-481); SELECT is c < 0 (codegen.py:490);
//   * results land at dest_base + r*N + i (codegen.py:492-494);
//   * self-referencing groups re-load their slots before every root and
//     re-evaluate (codegen.py:505-510).
// Arithmetic is IEEE binary64 round-to-nearest through __dadd_rn / __dmul_rn /
// __ddiv_rn / __dsqrt_rn (never contracted; the file is also built with
// --fmad=false), so EXACT_OPS templates reproduce the CPU reference bit for bit.
//
// CSR mode (sgb_run_csr): results that are outputs (codegen.py:445
// `x[plan.outputs]`) are stored straight to their CSR position through a
// per-group output-position table, the sum-of-products tiles of the last wave
// are scheduled in CSR order so partially written sectors merge in L2, groups
// nobody re-reads skip the value-array store, and outputs that are inputs or
// duplicates run as width-1 copy groups.  No separate gather pass.
//
// The path is an irregular gather / elementwise graph (no tensor cores): the
// kernels are built for memory-level parallelism -- every index and value load
// of a tile is issued before the first use, streaming data (index tables,
// results nobody re-reads) carries an L2 evict-first policy so the gathered
// intermediates stay in the 126 MB L2, and register counts stay low enough for
// 50% occupancy.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cstring>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "sgb.h"
#include "glibc_math.h"  // sgb_log / sgb_exp / sgb_pow: glibc restated (tools/gen_glibc_math.py)

namespace {

// tape op codes: lower.py T_*; the key byte of a word is op << 2 | nega << 1 | negb
// (dense, so the interpreter switch compiles to one indirect branch)
enum : int {
  T_MUL = 0, T_ADD, T_SUB, T_DIV, T_MADD, T_NEG, T_SQRT, T_SEL, T_IMM, T_ST, T_SLOW, T_MSUB, T_RMSUB
};
enum : int { KIND_TAPE = 0, KIND_SOP = 1 };
enum : int {
  FLAG_SELFREF = 1, FLAG_INTERLEAVED = 2, FLAG_SERIAL = 4, FLAG_STREAM = 16, FLAG_W16 = 32,
  FLAG_AFFINE0 = 64, FLAG_OPOS16 = 128, FLAG_OPOS32 = 256, FLAG_CSR_ONLY = 512, FLAG_COHERENT = 1024,
  FLAG_IMAJOR = 2048,  // CSR layout: result r of instance i at dest_base + i * n_roots + r (specialised units)
  FLAG_WPOS16 = 4096   // CSR-window member: root r of instance i at window position ooff[oo_off + r*n + i]
};
enum : int {
  U_WAVE = 0, U_KIND, U_VARIANT, U_G0, U_G1, U_T0, U_T1, U_BS, U_REGS, U_FLAGS, U_COUNT
};
enum : int { UNIT_CSR_ONLY = 1, UNIT_JIT = 2, UNIT_VALUE_ONLY = 4, UNIT_WINDOW = 8, UNIT_BULK = 16 };
constexpr int JIT_BLOCK = 256;  // jit.py JIT_BLOCK
constexpr int PRE = 8;        // slot loads kept in flight by the tape prologue
constexpr int SOP_BS = 256;   // sum-of-products block
constexpr int SOP_BATCH = 16; // factor loads in flight per instance
constexpr int BATCH_WARPS = 8;
constexpr uint32_t NONE = 0xFFFFFFFFu;

// instances per thread of the sum-of-products kernel, per width class (lower.SOP_CLASSES)
__host__ __device__ constexpr int sop_vec(int cls) { return cls <= 1 ? 4 : cls == 2 ? 2 : 1; }
__host__ __device__ constexpr int sop_lmax(int cls) { return cls == 0 ? 2 : cls == 1 ? 4 : cls == 2 ? 8 : cls == 3 ? 16 : 32; }

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define SGB_CUDA(call)                                                               \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail(-3, std::string(#call) + ": " + cudaGetErrorString(e_));           \
  } while (0)

struct Tables {
  const sgb_group *groups;
  const uint32_t *tape;  // 4 x u32 per tape word
  const double *imm;
  const uint32_t *sop;   // per SOP group: newterm mask, negate mask
  const int32_t *slot_col;
  const int64_t *slot_delta;
  const uint32_t *pos;
  const double *con;
  const uint32_t *cbase;  // compressed columns: per (column, 32-instance chunk) base
  const uint16_t *coff;   //                     per (column, instance) offset
  const uint32_t *obase;  // output positions: per (root, chunk) base
  const uint16_t *ooff;   //                   per (root, instance) offset, 0xFFFF = not an output
  const uint32_t *opos32; //                   wide form, NONE = not an output
  const uint32_t *fbase;  // sum-of-products fast path: per-factor base address
};

// ---- cache-policy helpers ---------------------------------------------------------
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// streaming index-table reads (ld.global.cs: evict-first).  Real load
// intrinsics, not asm: the compiler never speculates them past the guards that
// keep a missing table's pointer from being dereferenced.
__device__ __forceinline__ uint32_t ld_index(const uint32_t *a, uint64_t) { return __ldcs(a); }
__device__ __forceinline__ uint16_t ld_index16(const uint16_t *a, uint64_t) { return __ldcs(a); }
__device__ __forceinline__ double ld_const(const double *a, uint64_t) { return __ldcs(a); }
__device__ __forceinline__ void st_stream(double *a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}

// Retained column `col` of instance i: affine (column 0 only), the compressed
// form base[col][i/32] + off16[col][i] (lower.compress_column), or the plan's u32 table.
__device__ __forceinline__ uint32_t column_index(const Tables &T, const sgb_group &G, int col, int64_t i,
                                                 uint64_t pol) {
  if (col == 0 && (G.flags & FLAG_AFFINE0)) return (uint32_t)(G.a0_base + G.a0_stride * i);
  if (G.flags & FLAG_W16) {
    const int64_t nch = (G.n + 31) >> 5;
    return __ldg(T.cbase + G.cb_off + (int64_t)col * nch + (i >> 5)) +
           ld_index16(T.coff + G.co_off + (int64_t)col * G.n + i, pol);
  }
  const int64_t e = (G.flags & FLAG_INTERLEAVED) ? G.p_off + i * G.n_ret + col : G.p_off + (int64_t)col * G.n + i;
  return ld_index(T.pos + e, pol);
}

// Output (CSR) position of root r of instance i, or NONE.
__device__ __forceinline__ uint32_t out_pos(const Tables &T, const sgb_group &G, int r, int64_t i, uint64_t pol) {
  if (G.flags & FLAG_OPOS16) {
    const int64_t nch = (G.n + 31) >> 5;
    const uint16_t off = ld_index16(T.ooff + G.oo_off + (int64_t)r * G.n + i, pol);
    return off == 0xFFFFu ? NONE : __ldg(T.obase + G.ob_off + (int64_t)r * nch + (i >> 5)) + off;
  }
  if (G.flags & FLAG_OPOS32) return ld_index(T.opos32 + G.oo_off + (int64_t)r * G.n + i, pol);
  return NONE;
}

// Value-array store of a result (skipped in CSR mode when nobody re-reads it).
__device__ __forceinline__ void store_x(const sgb_group &G, int r, int64_t i, double v, double *x, int64_t ld,
                                        int64_t b, bool csr, uint64_t pol) {
  const bool stream = G.flags & FLAG_STREAM;
  if (csr && stream) return;
  double *a = x + (G.dest_base + (int64_t)r * G.n + i) * ld + b;
  if (stream) st_stream(a, v, pol); else *a = v;
}

// Store root r of instance i: the value array (unless CSR mode and nobody
// re-reads it) and, in CSR mode, its output position.
__device__ __forceinline__ void store_root(const Tables &T, const sgb_group &G, int r, int64_t i, double v,
                                           double *x, int64_t ld, int64_t b, double *out, int64_t ld_out,
                                           bool csr, uint64_t pol) {
  const bool stream = G.flags & FLAG_STREAM;
  if (!(csr && stream)) {
    double *a = x + (G.dest_base + (int64_t)r * G.n + i) * ld + b;
    if (stream) st_stream(a, v, pol); else *a = v;
  }
  if (csr) {
    const uint32_t o = out_pos(T, G, r, i, pol);
    if (o != NONE) out[(int64_t)o * ld_out + b] = v;
  }
}

// Rare ops live out of line so the interpreter loop stays small.  SIN / COS / EXP / LOG / POW are
// glibc's own algorithms (glibc_math.h) -- the reference's math.sin / cos / exp / log / pow, bit for
// bit (SIN / COS for |x| < 105414350); POW k = 2 is x*x (glibc's pow(x, 2.0) == x*x).
__device__ __noinline__ double slow_op(unsigned kind, double a, int k) {
  switch (kind) {
    case 0: return sgb_sin(a);
    case 1: return sgb_cos(a);
    case 2: return sgb_exp(a);
    case 3: return sgb_log(a);
    default: return k == 2 ? __dmul_rn(a, a) : sgb_pow(a, (double)k);
  }
}

// ---- tape interpreter ---------------------------------------------------------------
// Device words (lower.assemble): x = op<<2 | nega<<1 | negb | (c byte offset / 8) << 8,
// y / z / w = byte offsets of dst / a / b in the lane's scratch column (w is the
// immediate index, root index or kind<<16|k for IMM / ST / SLOW).  Scratch is
// shared memory addressed with 32-bit shared addresses; instance v of a lane
// sits VS bytes after instance 0.  Sign flags are part of the switch key, so a
// negated operand is the free negate modifier of DADD / DMUL, not extra work.
__device__ __forceinline__ double lds(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts(uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

#define SGB_NEG(NA, v) ((NA) ? -(v) : (v))
#define SGB_BIN(OPC, NA, NB, EXPR)                                                  \
  case ((OPC) << 2) | ((NA) << 1) | (NB): {                                         \
    _Pragma("unroll") for (int v = 0; v < VEC; ++v) {                               \
      const double a = SGB_NEG(NA, lds(pa + v * VS));                               \
      const double b = SGB_NEG(NB, lds(pb + v * VS));                               \
      sts(pd + v * VS, EXPR);                                                       \
    }                                                                               \
  } break;
#define SGB_FUSED(OPC, NA, NB, EXPR)                                                \
  case ((OPC) << 2) | ((NA) << 1) | (NB): {                                         \
    _Pragma("unroll") for (int v = 0; v < VEC; ++v) {                               \
      const double a = SGB_NEG(NA, lds(pa + v * VS));                               \
      const double b = SGB_NEG(NB, lds(pb + v * VS));                               \
      const double c = lds(pc + v * VS);                                            \
      sts(pd + v * VS, EXPR);                                                       \
    }                                                                               \
  } break;
#define SGB_SIGNS(M, OPC, EXPR) M(OPC, 0, 0, EXPR) M(OPC, 1, 0, EXPR) M(OPC, 0, 1, EXPR) M(OPC, 1, 1, EXPR)

template <int VEC, int VS>
__device__ __forceinline__ void run_tape(const Tables &T, const sgb_group &G, uint32_t Rb, double *x, int64_t ld,
                                         int64_t b, double *out, int64_t ld_out, bool csr,
                                         const int64_t (&iv)[VEC], const bool (&ok)[VEC], int phase, bool selfref,
                                         uint64_t pol) {
  const uint4 *tp = reinterpret_cast<const uint4 *>(T.tape) + G.tape_off;
  const int len = G.tape_len;
  uint4 next = len > 0 ? __ldg(tp) : make_uint4(0, 0, 0, 0);
  for (int k = 0; k < len; ++k) {
    const uint4 w = next;
    if (k + 1 < len) next = __ldg(tp + k + 1);  // prefetch the next word
    const uint32_t pd = Rb + w.y, pa = Rb + w.z, pb = Rb + w.w, pc = Rb + ((w.x >> 8) << 3);
    switch (w.x & 0xFFu) {
      SGB_SIGNS(SGB_BIN, T_MUL, __dmul_rn(a, b))
      SGB_SIGNS(SGB_BIN, T_ADD, __dadd_rn(a, b))
      SGB_SIGNS(SGB_BIN, T_SUB, __dsub_rn(a, b))
      SGB_SIGNS(SGB_BIN, T_DIV, __ddiv_rn(a, b))
      SGB_SIGNS(SGB_FUSED, T_MADD, __dadd_rn(__dmul_rn(a, b), c))
      SGB_SIGNS(SGB_FUSED, T_MSUB, __dsub_rn(__dmul_rn(a, b), c))
      SGB_SIGNS(SGB_FUSED, T_RMSUB, __dsub_rn(c, __dmul_rn(a, b)))
      case T_NEG << 2:
#pragma unroll
        for (int v = 0; v < VEC; ++v) sts(pd + v * VS, -lds(pa + v * VS));
        break;
      case T_SQRT << 2:
#pragma unroll
        for (int v = 0; v < VEC; ++v) sts(pd + v * VS, __dsqrt_rn(lds(pa + v * VS)));
        break;
      case T_SEL << 2:
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          sts(pd + v * VS, lds(pa + v * VS) < 0.0 ? lds(pb + v * VS) : lds(pc + v * VS));
        break;
      case T_IMM << 2: {
        const double imm = __ldg(T.imm + w.w);
#pragma unroll
        for (int v = 0; v < VEC; ++v) sts(pd + v * VS, imm);
        break;
      }
      case T_ST << 2:
        if (!selfref || (int)w.w == phase) {
#pragma unroll
          for (int v = 0; v < VEC; ++v)
            if (ok[v]) store_root(T, G, (int)w.w, iv[v], lds(pa + v * VS), x, ld, b, out, ld_out, csr, pol);
        }
        break;
      default:  // T_SLOW
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          sts(pd + v * VS, slow_op(w.w >> 16, lds(pa + v * VS), (int)(w.w & 0xFFFFu)));
        break;
    }
  }
}

// Prologue: hoisted slot loads (emit.py:108-124), PRE loads in flight per lane;
// slot s of this lane's instance goes to byte offset s * stride8.
__device__ __forceinline__ void load_slots(const Tables &T, const sgb_group &G, uint32_t Rb, uint32_t stride8,
                                           const double *x, int64_t ld, int64_t i, int64_t b, bool coherent_read,
                                           uint64_t pol) {
  const uint32_t idx0 = G.n_slots ? column_index(T, G, 0, i, pol) : 0u;
  const int32_t *scol = T.slot_col + G.slot_off;
  const int64_t *sdel = T.slot_delta + G.slot_off;
  for (int s0 = 0; s0 < G.n_slots; s0 += PRE) {
    double v[PRE];
#pragma unroll
    for (int u = 0; u < PRE; ++u) {
      const int s = s0 + u;
      if (s < G.n_slots) {
        const int col = __ldg(scol + s);
        const int64_t a = col < 0 ? (int64_t)idx0 + __ldg(sdel + s)
                                  : (col == 0 ? (int64_t)idx0 : (int64_t)column_index(T, G, col, i, pol));
        v[u] = coherent_read ? x[a * ld + b] : __ldg(x + a * ld + b);
      }
    }
#pragma unroll
    for (int u = 0; u < PRE; ++u)
      if (s0 + u < G.n_slots) sts(Rb + (uint32_t)(s0 + u) * stride8, v[u]);
  }
  for (int k = 0; k < G.n_const; ++k) {
    const int64_t e = (G.flags & FLAG_INTERLEAVED) ? G.c_off + i * G.n_const + k : G.c_off + (int64_t)k * G.n + i;
    sts(Rb + (uint32_t)(G.n_slots + k) * stride8, ld_const(T.con + e, pol));
  }
}

// One instance, any group (self-referencing groups reload before every root).
__device__ __forceinline__ void tape_instance(const Tables &T, const sgb_group &G, uint32_t Rb, uint32_t stride8,
                                              double *x, int64_t ld, int64_t i, int64_t b, double *out,
                                              int64_t ld_out, bool csr, uint64_t pol) {
  const bool selfref = G.flags & FLAG_SELFREF;
  const int phases = selfref ? G.n_roots : 1;
  const int64_t iv[1] = {i};
  const bool ok[1] = {true};
  for (int ph = 0; ph < phases; ++ph) {
    load_slots(T, G, Rb, stride8, x, ld, i, b, selfref, pol);
    run_tape<1, 0>(T, G, Rb, x, ld, b, out, ld_out, csr, iv, ok, ph, selfref, pol);
  }
}

// Single value set: lane = instance, VEC instances per lane (i0 + tid + v*BS)
// share each decoded tape word.  Scratch file [n_regs][VEC][BS] in shared memory.
template <int BS, int VEC>
__global__ void __launch_bounds__(BS) tape_single(Tables T, const int2 *tiles, int64_t n_tiles, double *x,
                                                  double *out, int csr) {
  extern __shared__ double scratch[];
  const uint64_t pol = evict_first_policy();
  const int tid = threadIdx.x;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(scratch);
  constexpr uint32_t stride8 = BS * VEC * 8;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {  // persistent: the grid is the resident capacity
    const int2 tl = tiles[t];
    const sgb_group G = T.groups[tl.x];
    if (!csr && (G.flags & FLAG_CSR_ONLY)) continue;
    if (VEC == 1 && (G.flags & FLAG_SERIAL)) {  // members read other instances' results: instance order
      if (tid == 0)
        for (int64_t i = 0; i < G.n; ++i) tape_instance(T, G, base, stride8, x, 1, i, 0, out, 1, csr, pol);
      continue;
    }
    const int64_t i0 = (int64_t)tl.y + tid;
    if (i0 >= G.n) continue;
    const uint32_t Rb = base + tid * 8;
    if (VEC == 1) {
      tape_instance(T, G, Rb, stride8, x, 1, i0, 0, out, 1, csr, pol);
      continue;
    }
    int64_t iv[VEC];
    bool ok[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      iv[v] = i0 + (int64_t)v * BS;
      ok[v] = iv[v] < G.n;
      if (!ok[v]) iv[v] = G.n - 1;  // evaluate a valid instance, store nothing
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) load_slots(T, G, Rb + v * BS * 8, stride8, x, 1, iv[v], 0, false, pol);
    run_tape<VEC, BS * 8>(T, G, Rb, x, 1, 0, out, 1, csr, iv, ok, 0, false, pol);
  }
}

// Batched: X[addr * ld + b].  A warp owns one instance and sweeps the batch, so
// index loads are warp-uniform and every gather is a contiguous row.  The block
// is the unit's scratch stride wide, VEC = 1.
__global__ void tape_batch(Tables T, const int2 *tiles, double *X, int64_t ld, int64_t batch, double *out,
                           int64_t ld_out, int csr) {
  extern __shared__ double scratch[];
  const int2 tl = tiles[blockIdx.x];
  const sgb_group G = T.groups[tl.x];
  if (!csr && (G.flags & FLAG_CSR_ONLY)) return;
  const uint64_t pol = evict_first_policy();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t Rb = (uint32_t)__cvta_generic_to_shared(scratch) + tid * 8;
  const uint32_t stride8 = blockDim.x * 8;
  if (G.flags & FLAG_SERIAL) {
    if (warp != 0) return;
    for (int64_t i = 0; i < G.n; ++i)
      for (int64_t b = lane; b < batch; b += 32) tape_instance(T, G, Rb, stride8, X, ld, i, b, out, ld_out, csr, pol);
    return;
  }
  const int64_t i = (int64_t)tl.y + warp;
  if (i >= G.n) return;
  for (int64_t b = lane; b < batch; b += 32) tape_instance(T, G, Rb, stride8, X, ld, i, b, out, ld_out, csr, pol);
}

// ---- sum of products: acc = t0 + t1 + ..., t = f0 * f1 * ... (tape-free) --------------
// Address of factor f (slot f) of instance i with slot-0 index idx0.  Coherent
// slots are slot 0 + delta in 32-bit modular arithmetic (every address < 2^32).
template <class C, class D>
__device__ __forceinline__ uint32_t sop_addr(const Tables &T, const sgb_group &G, int f, int64_t i, uint32_t idx0,
                                             const C &s_col, const D &s_del, bool coherent, uint64_t pol) {
  if (coherent) return idx0 + (uint32_t)s_del[f];
  const int col = s_col[f];
  if (col < 0) return idx0 + (uint32_t)s_del[f];
  if (col == 0) return idx0;
  return column_index(T, G, col, i, pol);
}

__device__ __forceinline__ double neg_if(double v, uint32_t negm, int f) {
  return ((negm >> f) & 1u) ? -v : v;
}

// Template shapes recognised by the lowering (lower.SOP_SHAPE_*): a generic
// sum of products (term-start mask), a plain sum (every factor is a term) and
// a sum of two-factor products with an optional single-factor tail.  All are
// the template's own left fold, bit for bit.
enum : int { SHAPE_GENERIC = 0, SHAPE_SUM = 1, SHAPE_PAIRS = 2 };

template <int SHAPE, int LMAX, bool NEG>
__device__ __forceinline__ double sop_eval(const double (&v)[LMAX], int len, uint32_t newterm, uint32_t negm) {
  if (SHAPE == SHAPE_SUM) {
    double acc = NEG ? neg_if(v[0], negm, 0) : v[0];
#pragma unroll
    for (int f = 1; f < LMAX; ++f)
      if (f < len) acc = __dadd_rn(acc, NEG ? neg_if(v[f], negm, f) : v[f]);
    return acc;
  } else if (SHAPE == SHAPE_PAIRS) {
    double acc = __dmul_rn(NEG ? neg_if(v[0], negm, 0) : v[0], NEG ? neg_if(v[1], negm, 1) : v[1]);
#pragma unroll
    for (int f = 2; f < LMAX; f += 2) {
      const double a = NEG ? neg_if(v[f], negm, f) : v[f];
      if (f + 1 < len) {
        const double b = NEG ? neg_if(v[f + 1], negm, f + 1) : v[f + 1];
        acc = __dadd_rn(acc, __dmul_rn(a, b));
      } else if (f < len) {  // single-factor tail (e.g. "+ A_ij"), len odd
        acc = __dadd_rn(acc, a);
      }
    }
    return acc;
  } else {
    double acc = 0.0, term = 0.0;
    bool have = false;
#pragma unroll
    for (int f = 0; f < LMAX; ++f) {
      if (f < len) {
        const double val = neg_if(v[f], negm, f);
        if ((newterm >> f) & 1u) {
          if (f > 0) {
            acc = have ? __dadd_rn(acc, term) : term;
            have = true;
          }
          term = val;
        } else {
          term = __dmul_rn(term, val);
        }
      }
    }
    return have ? __dadd_rn(acc, term) : term;
  }
}

// Address of factor f of instance i: slot deltas / columns are warp-uniform
// loads (L1 hits after the first tile of a group), issued right before use.
__device__ __forceinline__ uint32_t factor_addr(const Tables &T, const sgb_group &G, int f, int64_t i, uint32_t idx0,
                                                bool coherent, uint64_t pol) {
  const uint32_t d = (uint32_t)__ldg(T.slot_delta + G.slot_off + f);
  if (coherent) return idx0 + d;
  const int col = __ldg(T.slot_col + G.slot_off + f);
  if (col < 0) return idx0 + d;
  if (col == 0) return idx0;
  return column_index(T, G, col, i, pol);
}

// Compact per-group descriptor of the single-set sum-of-products kernel (48 B,
// built by sgb_plan_create from the group records): everything a warp needs per
// tile in three uniform 16-byte loads.
struct __align__(16) SopDesc {
  int32_t n;
  uint32_t dest_base;
  uint32_t meta;  // len | shape << 6 | variant << 8 | fast << 11 | csr_only << 12 | stream << 13 |
                  // opos16 << 14 | opos32 << 15
  int32_t stride; // fast path: factor f of instance i is at fbase[f] + stride * i
  uint32_t newterm, negm;
  uint32_t fbase_off;  // fast path: first factor base in Tables::fbase
  int32_t g;           // group record (generic path)
  uint32_t ob_off, oo_off;
  uint32_t pad0, pad1;
};
enum : uint32_t {
  M_FAST = 1u << 11, M_CSR_ONLY = 1u << 12, M_STREAM = 1u << 13, M_OPOS16 = 1u << 14, M_OPOS32 = 1u << 15
};

__device__ __forceinline__ uint32_t desc_out_pos(const Tables &T, const SopDesc &d, uint32_t i) {
  if (d.meta & M_OPOS16) {
    const uint16_t off = __ldcs(T.ooff + d.oo_off + i);
    return off == 0xFFFFu ? NONE : __ldg(T.obase + d.ob_off + (i >> 5)) + off;
  }
  if (d.meta & M_OPOS32) return __ldcs(T.opos32 + d.oo_off + i);
  return NONE;
}

__device__ __forceinline__ void desc_store(const SopDesc &d, uint32_t i, uint32_t op, double r, double *x,
                                           double *out, bool csr, uint64_t pol) {
  if (!(csr && (d.meta & M_STREAM))) {
    double *a = x + (d.dest_base + (uint64_t)i);
    if (d.meta & M_STREAM) st_stream(a, r, pol); else *a = r;
  }
  if (op != NONE) out[op] = r;
}

// Fast path (affine column 0, every slot coherent): VEC instances per lane
// (i0 + v*32); output-position and value loads of all VEC instances are issued
// before the first fold.
template <int SHAPE, int LMAX, int VEC>
__device__ __forceinline__ void sop_fast(const Tables &T, const SopDesc &d, uint32_t i0, double *x, double *out,
                                         bool csr, uint64_t pol) {
  const int len = d.meta & 63u;
  uint32_t fb[LMAX];
#pragma unroll
  for (int f = 0; f < LMAX; ++f) fb[f] = f < len ? __ldg(T.fbase + d.fbase_off + f) : 0u;
  uint32_t iv[VEC], op[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    iv[v] = min(i0 + (uint32_t)(v * 32), (uint32_t)d.n - 1u);
    op[v] = csr ? desc_out_pos(T, d, iv[v]) : NONE;
  }
  double val[VEC][LMAX];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    const uint32_t off = (uint32_t)d.stride * iv[v];
#pragma unroll
    for (int f = 0; f < LMAX; ++f) val[v][f] = f < len ? __ldg(x + (fb[f] + off)) : 0.0;
  }
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    const uint32_t i = i0 + (uint32_t)(v * 32);
    if (i < (uint32_t)d.n) {
      const double r = d.negm ? sop_eval<SHAPE, LMAX, true>(val[v], len, d.newterm, d.negm)
                              : sop_eval<SHAPE, LMAX, false>(val[v], len, d.newterm, d.negm);
      desc_store(d, i, op[v], r, x, out, csr, pol);
    }
  }
}

// Wide templates and the general index forms: factor batches of SOP_BATCH.
struct SopFold {
  double acc, term;
  bool have;
};

template <int NB>
__device__ __forceinline__ void sop_fold(SopFold &st, int f0, int len, uint32_t newterm, uint32_t negm,
                                         const double (&v)[NB]) {
#pragma unroll
  for (int u = 0; u < NB; ++u) {
    const int f = f0 + u;
    if (f < len) {
      const double val = neg_if(v[u], negm, f);
      if ((newterm >> f) & 1u) {
        if (f > 0) {
          st.acc = st.have ? __dadd_rn(st.acc, st.term) : st.term;
          st.have = true;
        }
        st.term = val;
      } else {
        st.term = __dmul_rn(st.term, val);
      }
    }
  }
}

// General path: any index form (u32 table, compressed, interleaved, per-slot
// columns), one instance per lane, out of line so the fast bodies keep their
// registers.
__device__ __noinline__ void sop_general(const Tables &T, const SopDesc &d, uint32_t i, double *x, double *out,
                                         bool csr) {
  if (i >= (uint32_t)d.n) return;
  const uint64_t pol = evict_first_policy();
  const sgb_group G = T.groups[d.g];
  const int len = d.meta & 63u;
  const bool coherent = G.flags & FLAG_COHERENT;
  const uint32_t idx0 = column_index(T, G, 0, i, pol);
  const uint32_t op = csr ? desc_out_pos(T, d, i) : NONE;
  SopFold st{0.0, 0.0, false};
#pragma unroll 1
  for (int f0 = 0; f0 < len; f0 += 8) {
    double val[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (f0 + u < len) val[u] = __ldg(x + factor_addr(T, G, f0 + u, i, idx0, coherent, pol));
    sop_fold<8>(st, f0, len, d.newterm, d.negm, val);
  }
  const double r = st.have ? __dadd_rn(st.acc, st.term) : st.term;
  desc_store(d, i, op, r, x, out, csr, pol);
}

// Persistent sum-of-products launches: one kernel per (shape, width class) of
// the fast path plus one for the general index forms, so every body gets its
// own register allocation.  Every warp walks its unit's warp tiles t = warp,
// warp + W, ... (tiles of 32 x VEC instances in launch order -- CSR order for
// output groups), prefetching its next tile entry; no block synchronisation and
// no per-CTA prologue, the grid is the resident capacity of the chip.
template <int SHAPE, int LMAX, int VEC>
__global__ void __launch_bounds__(SOP_BS, 3) sop_fast_unit(Tables T, const SopDesc *D, const int2 *tiles,
                                                          int64_t n_tiles, double *x, double *out, int csr) {
  const uint32_t lane = threadIdx.x & 31;
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= n_tiles) return;
  const uint64_t pol = evict_first_policy();
  int2 nxt = tiles[t];
  for (; t < n_tiles; t += W) {
    const int2 tl = nxt;
    if (t + W < n_tiles) nxt = tiles[t + W];
    const SopDesc d = D[tl.x];
    if (!csr && (d.meta & M_CSR_ONLY)) continue;
    sop_fast<SHAPE, LMAX, VEC>(T, d, (uint32_t)tl.y + lane, x, out, csr, pol);
  }
}

__global__ void __launch_bounds__(SOP_BS, 4) sop_general_unit(Tables T, const SopDesc *D, const int2 *tiles,
                                                             int64_t n_tiles, double *x, double *out, int csr) {
  const uint32_t lane = threadIdx.x & 31;
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_tiles; t += W) {
    const int2 tl = tiles[t];
    const SopDesc d = D[tl.x];
    if (!csr && (d.meta & M_CSR_ONLY)) continue;
    const int vec = sop_vec((d.meta >> 8) & 7u);
    for (int v = 0; v < vec; ++v) sop_general(T, d, (uint32_t)tl.y + lane + 32u * v, x, out, csr);
  }
}

// unit variant codes (lower.sop_unit_code): fast path = shape * 8 + width class, general = 64
constexpr int SOP_GENERAL_CODE = 64;

#define SGB_SOP_KERNEL(SH, CLS) sop_fast_unit<SH, sop_lmax(CLS), sop_vec(CLS)>
typedef void (*sop_kernel_t)(Tables, const SopDesc *, const int2 *, int64_t, double *, double *, int);

__host__ sop_kernel_t sop_kernel_for(int code) {
  switch (code) {
    case SHAPE_GENERIC * 8 + 0: return SGB_SOP_KERNEL(SHAPE_GENERIC, 0);
    case SHAPE_GENERIC * 8 + 1: return SGB_SOP_KERNEL(SHAPE_GENERIC, 1);
    case SHAPE_GENERIC * 8 + 2: return SGB_SOP_KERNEL(SHAPE_GENERIC, 2);
    case SHAPE_GENERIC * 8 + 3: return SGB_SOP_KERNEL(SHAPE_GENERIC, 3);
    case SHAPE_SUM * 8 + 0: return SGB_SOP_KERNEL(SHAPE_SUM, 0);
    case SHAPE_SUM * 8 + 1: return SGB_SOP_KERNEL(SHAPE_SUM, 1);
    case SHAPE_SUM * 8 + 2: return SGB_SOP_KERNEL(SHAPE_SUM, 2);
    case SHAPE_SUM * 8 + 3: return SGB_SOP_KERNEL(SHAPE_SUM, 3);
    case SHAPE_PAIRS * 8 + 0: return SGB_SOP_KERNEL(SHAPE_PAIRS, 0);
    case SHAPE_PAIRS * 8 + 1: return SGB_SOP_KERNEL(SHAPE_PAIRS, 1);
    case SHAPE_PAIRS * 8 + 2: return SGB_SOP_KERNEL(SHAPE_PAIRS, 2);
    case SHAPE_PAIRS * 8 + 3: return SGB_SOP_KERNEL(SHAPE_PAIRS, 3);
    case SOP_GENERAL_CODE: return sop_general_unit;
    default: return nullptr;
  }
}

// Batched: one instance per warp, lanes sweep the batch; index decode is warp-uniform.
template <int LMAX>
__device__ __forceinline__ void sop_batch_body(const Tables &T, const sgb_group &G, int64_t i, int lane, double *X,
                                               int64_t ld, int64_t batch, double *out, int64_t ld_out, bool csr,
                                               const int32_t *s_col, const int32_t *s_del, uint64_t pol) {
  constexpr int NB = LMAX < 8 ? LMAX : 8;
  const uint32_t newterm = __ldg(T.sop + 2 * G.sop_off), negm = __ldg(T.sop + 2 * G.sop_off + 1);
  const bool coherent = G.flags & FLAG_COHERENT;
  const int len = G.sop_len;
  const uint32_t idx0 = column_index(T, G, 0, i, pol);
  const uint32_t op = csr ? out_pos(T, G, 0, i, pol) : NONE;
  uint32_t addr[LMAX];
#pragma unroll
  for (int f = 0; f < LMAX; ++f)
    if (f < len) addr[f] = sop_addr(T, G, f, i, idx0, s_col, s_del, coherent, pol);
  for (int64_t b = lane; b < batch; b += 32) {
    SopFold st{0.0, 0.0, false};
#pragma unroll
    for (int f0 = 0; f0 < LMAX; f0 += NB) {
      if (f0 < len) {
        double v[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u)
          if (f0 + u < len) v[u] = __ldg(X + (int64_t)addr[f0 + u] * ld + b);
        sop_fold<NB>(st, f0, len, newterm, negm, v);
      }
    }
    const double r = st.have ? __dadd_rn(st.acc, st.term) : st.term;
    store_x(G, 0, i, r, X, ld, b, csr, pol);
    if (op != NONE) out[(int64_t)op * ld_out + b] = r;
  }
}

__global__ void __launch_bounds__(BATCH_WARPS * 32) sop_batch(Tables T, const int2 *tiles, double *X, int64_t ld,
                                                             int64_t batch, double *out, int64_t ld_out, int csr) {
  __shared__ int32_t s_col[32];
  __shared__ int32_t s_del[32];
  const int2 tl = tiles[blockIdx.x];
  const sgb_group G = T.groups[tl.x];
  if (!csr && (G.flags & FLAG_CSR_ONLY)) return;
  if (threadIdx.x < G.n_slots) {
    s_col[threadIdx.x] = __ldg(T.slot_col + G.slot_off + threadIdx.x);
    s_del[threadIdx.x] = (int32_t)__ldg(T.slot_delta + G.slot_off + threadIdx.x);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = (int64_t)tl.y + warp;
  if (i >= G.n) return;
  const uint64_t pol = evict_first_policy();
  switch (G.variant) {
    case 0: sop_batch_body<2>(T, G, i, lane, X, ld, batch, out, ld_out, csr, s_col, s_del, pol); break;
    case 1: sop_batch_body<4>(T, G, i, lane, X, ld, batch, out, ld_out, csr, s_col, s_del, pol); break;
    case 2: sop_batch_body<8>(T, G, i, lane, X, ld, batch, out, ld_out, csr, s_col, s_del, pol); break;
    case 3: sop_batch_body<16>(T, G, i, lane, X, ld, batch, out, ld_out, csr, s_col, s_del, pol); break;
    default: sop_batch_body<32>(T, G, i, lane, X, ld, batch, out, ld_out, csr, s_col, s_del, pol); break;
  }
}

// CSR values out[k] = x[outputs[k]] (codegen.py:445): u32 index stream
// (evict-first), gathered value, streaming store.
__global__ void __launch_bounds__(256) gather_outputs(const double *__restrict__ x, const uint32_t *__restrict__ outs,
                                                      int64_t n, double *__restrict__ out) {
  const uint64_t pol = evict_first_policy();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    st_stream(out + k, __ldg(x + __ldg(outs + k)), pol);
}

// Batched outputs: one output per warp, lanes over value sets, 4 value sets per lane
// per iteration with all loads issued first.
__global__ void gather_outputs_batch(const double *__restrict__ X, int64_t ld, int64_t batch,
                                     const int64_t *__restrict__ outs, int64_t n, double *__restrict__ out,
                                     int64_t ld_out) {
  const int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= n) return;
  const double *src = X + __ldg(outs + k) * ld;
  double *dst = out + k * ld_out;
  for (int64_t b = threadIdx.x & 31; b < batch; b += 128) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (b + 32 * u < batch) v[u] = __ldg(src + b + 32 * u);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (b + 32 * u < batch) __stcs(dst + b + 32 * u, v[u]);
  }
}

// Batched outputs that are plain value-array entries of a CSR-window plan (the window members'
// value-mode twins store theirs directly): out[copy_k[c] * ld_out + b] = X[copy_src[c] * ld + b].
__global__ void gather_copies_batch(const double *__restrict__ X, int64_t ld, int64_t batch,
                                    const uint32_t *__restrict__ copy_k, const uint32_t *__restrict__ copy_src,
                                    int64_t n, double *__restrict__ out, int64_t ld_out) {
  const int64_t c = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= n) return;
  const double *src = X + (int64_t)__ldg(copy_src + c) * ld;
  double *dst = out + (int64_t)__ldg(copy_k + c) * ld_out;
  for (int64_t b = threadIdx.x & 31; b < batch; b += 128) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (b + 32 * u < batch) v[u] = __ldg(src + b + 32 * u);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (b + 32 * u < batch) __stcs(dst + b + 32 * u, v[u]);
  }
}

template <class T>
int upload(T **dst, const T *src, int64_t n) {
  *dst = nullptr;
  if (n <= 0) return 0;
  SGB_CUDA(cudaMalloc((void **)dst, sizeof(T) * (size_t)n));
  SGB_CUDA(cudaMemcpy(*dst, src, sizeof(T) * (size_t)n, cudaMemcpyHostToDevice));
  return 0;
}

struct Unit {
  int wave, kind, variant, g0, g1, bs, regs, flags;
  int index;                   // position in sgb_plan_desc.units (names the specialised kernels)
  const void *jit = nullptr;   // specialised tape kernels (cudaKernel_t), UNIT_JIT
  const void *jitb = nullptr;
  int64_t grid;      // single-set grid in use (blocks)
  int64_t grid_p = 0, grid_t = 0;  // specialised units: persistent grid / one block per tile
  int64_t grid_b = 0;              // specialised units, batched kernels: persistent grid
  int64_t t0, t1;    // single-set tiles [t0, t1)
  int64_t bt0, bt1;  // batched tiles
};

}  // namespace

struct sgb_plan {
  int device = 0;
  int64_t vas = 0, n_in = 0, n_out = 0, n_pos = 0, n_con = 0;
  int n_groups = 0, n_waves = 0, csr_waves = 0, needs_zero = 2;
  bool ws_dirty = false;  // the workspace holds sg_run results (slots CSR mode never writes)
  std::vector<Unit> units;
  std::vector<std::vector<int>> wave_units;  // per wave: indices into units, largest first
  std::vector<int64_t> group_n;              // host copy of every group's instance count
  std::vector<int2> h_tiles;                 // host copy of the single-set tile table in use
  Tables T{};
  sgb_group *d_groups = nullptr;
  int2 *d_tiles = nullptr, *d_btiles = nullptr;
  int64_t n_tiles = 0;
  int64_t *d_outputs = nullptr;
  uint32_t *d_outputs32 = nullptr;
  bool direct_csr = false;  // some group stores its outputs at their CSR positions (FLAG_OPOS*)
  bool csr_layout = false;  // some group stores instance-major (FLAG_IMAJOR): the value array is permuted
  uint32_t *d_tape = nullptr;
  double *d_imm = nullptr, *d_con = nullptr;
  uint32_t *d_sop = nullptr;
  int32_t *d_scol = nullptr;
  int64_t *d_sdel = nullptr;
  uint32_t *d_pos = nullptr, *d_cbase = nullptr, *d_obase = nullptr, *d_opos32 = nullptr;
  uint16_t *d_coff = nullptr, *d_ooff = nullptr;
  SopDesc *d_sopd = nullptr;
  cudaLibrary_t jit_lib = nullptr;
  int2 *d_wpieces = nullptr;  // CSR windows: [n_win][J] first instance, count
  int64_t *d_wk = nullptr, *d_wcopy = nullptr;
  uint32_t *d_csrc = nullptr;
  uint16_t *d_cpos = nullptr;
  uint32_t *d_copy_k = nullptr;  // CSR position of every copy (win_k[w] + copy_pos[c]): batched CSR mode
  bool batch_direct = false;     // batched CSR: window-member twins store their outputs, copies gathered
  int64_t n_copy_k = 0;
  uint32_t *d_fbase = nullptr;
  // bulk feed of the CSR-window unit (UNIT_BULK): consumer blobs + value-array intervals per window
  uint8_t *d_wmeta = nullptr;
  int64_t *d_wmeta_off = nullptr, *d_wiv_off = nullptr;
  uint2 *d_wiv = nullptr;
  int64_t wb_ring = 0, wb_meta = 0, wb_x = 0, wb_bw = 0;
  int64_t vas_slots = 0;  // value-array doubles a CSR workspace spans (vas, even with a bulk unit)
  // workspace for the host-buffer entry points
  std::mutex ws_mu;
  double *d_x = nullptr, *d_out = nullptr;
  cudaStream_t ws_stream = nullptr;
  // second workspace + copy streams of the pipelined host-buffer stream (sgb_run_outputs_host_many)
  double *d_x2 = nullptr, *d_out2 = nullptr;
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  // fork / join of the independent launch units of one wave
  std::vector<cudaStream_t> aux;
  std::vector<cudaEvent_t> ev_join;
  cudaEvent_t ev_fork = nullptr;
  cudaEvent_t ws_event = nullptr;  // last device-side use of the workspace by sgb_run_inputs_csr
  std::mutex run_mu;  // the aux streams / events are per plan: one launch sequence at a time
};

namespace {

template <int BS, int VEC>
void launch_tape(const sgb_plan *p, const Unit &u, double *x, double *out, bool csr, cudaStream_t s) {
  const size_t smem = (size_t)u.regs * BS * VEC * sizeof(double);
  tape_single<BS, VEC><<<(unsigned)u.grid, BS, smem, s>>>(p->T, p->d_tiles + u.t0, u.t1 - u.t0, x, out, csr);
}

template <int BS>
void launch_tape_vec(const sgb_plan *p, const Unit &u, double *x, double *out, bool csr, cudaStream_t s) {
  if (u.variant <= 1) launch_tape<BS, 1>(p, u, x, out, csr, s);
  else if (u.variant == 2) launch_tape<BS, 2>(p, u, x, out, csr, s);
  else launch_tape<BS, 4>(p, u, x, out, csr, s);
}

template <int BS, int VEC>
cudaError_t tape_occupancy(int regs, int *nb) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(nb, tape_single<BS, VEC>, BS, (size_t)regs * BS * VEC * 8);
}

cudaError_t tape_occupancy_any(int bs, int vec, int regs, int *nb) {
  switch (bs * 8 + vec) {
    case 128 * 8 + 4: return tape_occupancy<128, 4>(regs, nb);
    case 128 * 8 + 2: return tape_occupancy<128, 2>(regs, nb);
    case 128 * 8 + 1: return tape_occupancy<128, 1>(regs, nb);
    case 64 * 8 + 4: return tape_occupancy<64, 4>(regs, nb);
    case 64 * 8 + 2: return tape_occupancy<64, 2>(regs, nb);
    case 64 * 8 + 1: return tape_occupancy<64, 1>(regs, nb);
    case 32 * 8 + 4: return tape_occupancy<32, 4>(regs, nb);
    case 32 * 8 + 2: return tape_occupancy<32, 2>(regs, nb);
    default: return tape_occupancy<32, 1>(regs, nb);
  }
}

void launch_unit(const sgb_plan *p, const Unit &u, double *x, int64_t ld, int64_t batch, bool batched, double *out,
                 int64_t ld_out, bool csr, cudaStream_t s) {
  if ((u.flags & UNIT_CSR_ONLY) && !csr) return;
  const int64_t blocks = batched ? u.bt1 - u.bt0 : u.t1 - u.t0;
  if (blocks <= 0) return;
  if (!batched && csr && (u.flags & UNIT_VALUE_ONLY)) return;
  if (u.flags & UNIT_BULK) {  // bulk-fed CSR windows (jit.py wbulk_source): persistent blocks, smem ring
    const uint8_t *meta = p->d_wmeta;
    const int64_t *moff = p->d_wmeta_off, *ivoff = p->d_wiv_off;
    const uint2 *iv = p->d_wiv;
    int64_t n = u.t1 - u.t0, ring = p->wb_ring, sm = p->wb_meta, sx = p->wb_x, bw = p->wb_bw;
    Tables T = p->T;
    const double *xc = x;
    void *args[] = {&T, &meta, &moff, &iv, &ivoff, &n, &xc, &out, &ring, &sm, &sx, &bw};
    cudaLaunchKernel(u.jit, dim3((unsigned)u.grid), dim3(u.bs), args, (size_t)u.regs, s);
    return;
  }
  if (u.flags & UNIT_WINDOW) {  // CSR windows (jit.py window_source): one block per window
    const int2 *pieces = p->d_wpieces;
    const int64_t *wk = p->d_wk, *wc = p->d_wcopy;
    const uint32_t *csrc = p->d_csrc;
    const uint16_t *cpos = p->d_cpos;
    int64_t n = u.t1 - u.t0;
    Tables T = p->T;
    const double *xc = x;
    void *args[] = {&T, &pieces, &wk, &wc, &csrc, &cpos, &n, &xc, &out};
    cudaLaunchKernel(u.jit, dim3((unsigned)u.grid), dim3(JIT_BLOCK), args, (size_t)u.regs, s);
    return;
  }
  if ((u.flags & UNIT_CSR_ONLY) && batched) return;
  if (u.flags & UNIT_JIT) {  // specialised straight-line kernels (jit.py)
    const int2 *tiles = batched ? p->d_btiles + u.bt0 : p->d_tiles + u.t0;
    int64_t n = blocks;
    int c = csr ? 1 : 0;
    Tables T = p->T;
    if (batched) {
      int64_t ld_ = ld, batch_ = batch, ldo = ld_out;
      void *args[] = {&T, &tiles, &n, &x, &ld_, &batch_, &out, &ldo, &c};
      // the batched kernels run a persistent grid of their own occupancy (the per-wave grid choice is
      // tuned single-set; one block per batched tile measured slower, profiles/r44)
      const int64_t cap = u.grid_b > 0 ? u.grid_b : u.grid;
      const int64_t grid = blocks < cap ? blocks : cap;
      cudaLaunchKernel(u.jitb, dim3((unsigned)grid), dim3(JIT_BLOCK), args, 0, s);
    } else {
      void *args[] = {&T, &tiles, &n, &x, &out, &c};
      cudaLaunchKernel(u.jit, dim3((unsigned)u.grid), dim3(u.bs), args, (size_t)u.regs, s);
    }
    return;
  }
  if (u.kind == KIND_TAPE) {
    if (batched) {  // block = the unit's scratch stride, one instance per warp
      const int stride = u.bs * u.variant;
      const size_t smem = (size_t)u.regs * stride * sizeof(double);
      tape_batch<<<(unsigned)blocks, stride, smem, s>>>(p->T, p->d_btiles + u.bt0, x, ld, batch, out, ld_out, csr);
      return;
    }
    switch (u.bs) {
      case 128: launch_tape_vec<128>(p, u, x, out, csr, s); break;
      case 64: launch_tape_vec<64>(p, u, x, out, csr, s); break;
      default: launch_tape_vec<32>(p, u, x, out, csr, s); break;
    }
  } else if (batched) {
    sop_batch<<<(unsigned)blocks, BATCH_WARPS * 32, 0, s>>>(p->T, p->d_btiles + u.bt0, x, ld, batch, out, ld_out,
                                                            csr);
  } else {
    sop_kernel_for(u.variant)<<<(unsigned)u.grid, SOP_BS, 0, s>>>(p->T, p->d_sopd, p->d_tiles + u.t0, u.t1 - u.t0,
                                                                  x, out, csr);
  }
}

template <int BS, int VEC>
cudaError_t allow_smem_single(int smem_max) {
  return cudaFuncSetAttribute(tape_single<BS, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
}

template <int BS>
cudaError_t allow_smem(int smem_max) {
  cudaError_t e;
  if ((e = allow_smem_single<BS, 1>(smem_max)) != cudaSuccess) return e;
  if ((e = allow_smem_single<BS, 2>(smem_max)) != cudaSuccess) return e;
  return allow_smem_single<BS, 4>(smem_max);
}

// Sum-of-products groups the fast kernels take: affine column 0, one retained
// column (every slot = column 0 + delta), width class <= 16 factors.
bool sop_fast_ok(const sgb_group &G) {
  return (G.flags & FLAG_AFFINE0) && G.n_ret == 1 && G.variant <= 3 && !(G.flags & FLAG_INTERLEAVED) &&
         G.a0_stride >= INT32_MIN && G.a0_stride <= INT32_MAX;
}

// per-entry validation of a compressed table: base[c][i/32] + off[c][i] < limit (off == skip allowed)
bool w16_ok(const uint32_t *base, const uint16_t *off, int64_t n, int cols, int c0, int64_t limit, bool allow_skip) {
  const int64_t nch = (n + 31) / 32;
  for (int c = c0; c < cols; ++c)
    for (int64_t i = 0; i < n; ++i) {
      const uint16_t o = off[c * n + i];
      if (allow_skip && o == 0xFFFFu) continue;
      if ((int64_t)base[c * nch + i / 32] + o >= limit) return false;
    }
  return true;
}

}  // namespace

extern "C" {

const char *sgb_last_error(void) { return g_err.c_str(); }

int sgb_plan_waves(const sgb_plan *p, int csr) {
  if (!p) return 0;
  if (!csr) return p->n_waves;
  return p->direct_csr ? p->csr_waves : p->n_waves + (p->n_out > 0 ? 1 : 0);  // + the gather
}

int64_t sgb_plan_value_slots(const sgb_plan *p) { return p ? p->vas_slots : 0; }

int sgb_plan_units(const sgb_plan *p, int csr) {
  if (!p) return 0;
  const bool direct = csr && p->direct_csr;
  int k = 0;
  for (const Unit &u : p->units) {
    if ((u.flags & UNIT_CSR_ONLY) && !direct) continue;  // CSR-only units run in direct CSR mode only
    if ((u.flags & UNIT_VALUE_ONLY) && direct) continue;  // value-mode twins of CSR-window members
    if (u.t1 <= u.t0) continue;                           // nothing to launch
    ++k;
  }
  return k + (csr && !p->direct_csr && p->n_out > 0 ? 1 : 0);
}

void sgb_plan_destroy(sgb_plan *p) {
  if (!p) return;
  cudaSetDevice(p->device);
  void *bufs[] = {p->d_groups, p->d_tiles, p->d_btiles, p->d_outputs, p->d_tape, p->d_imm, p->d_con,
                  p->d_sop, p->d_scol, p->d_sdel, p->d_pos, p->d_x, p->d_out, p->d_cbase, p->d_coff,
                  p->d_obase, p->d_ooff, p->d_opos32, p->d_sopd, p->d_fbase, p->d_outputs32,
                  p->d_wpieces, p->d_wk, p->d_wcopy, p->d_csrc, p->d_cpos, p->d_x2, p->d_out2,
                  p->d_wmeta, p->d_wmeta_off, p->d_wiv_off, p->d_wiv, p->d_copy_k};
  for (void *b : bufs)
    if (b) cudaFree(b);
  if (p->ws_stream) cudaStreamDestroy(p->ws_stream);
  if (p->h2d_stream) cudaStreamDestroy(p->h2d_stream);
  if (p->d2h_stream) cudaStreamDestroy(p->d2h_stream);
  if (p->jit_lib) cudaLibraryUnload(p->jit_lib);
  for (cudaStream_t a : p->aux) cudaStreamDestroy(a);
  for (cudaEvent_t e : p->ev_join) cudaEventDestroy(e);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ws_event) cudaEventDestroy(p->ws_event);
  delete p;
}

static int64_t a16(int64_t v) { return (v + 15) & ~(int64_t)15; }

// The bulk feed of the CSR-window unit (lower.WindowBulk): every blob, interval and offset the
// kernel dereferences stays inside its window's ring slot, window buffer and value array.
static int check_window_bulk(const sgb_plan_desc *d, const Unit &u, int64_t n_win, int64_t J, int64_t smem_max) {
  auto bad = [](const std::string &what) { return fail(-1, "sgb_plan_create: bad bulk CSR-window feed: " + what); };
  if (!d->win_meta || d->n_win_meta <= 0 || !d->win_meta_off || !d->win_iv_off || !d->win_bulk ||
      (d->n_win_iv > 0 && !d->win_iv) || d->n_win_iv < 0)
    return bad("missing tables");
  if (d->win_ring < 1 || d->win_ring > 8 || d->win_slot_meta <= 0 || d->win_slot_meta % 128 || d->win_slot_x <= 0 ||
      d->win_slot_x % 128 || d->win_bw < 128 || d->win_bw % 128 || u.bs % 32 || u.bs < 64 || u.bs > 1024 ||
      (int64_t)u.regs != d->win_bw + d->win_ring * (d->win_slot_meta + d->win_slot_x) || u.regs > smem_max)
    return bad("ring / block geometry");
  const int64_t vas_even = d->value_array_size + (d->value_array_size & 1);
  int64_t NR = 0, NW = 0;
  for (int64_t j = 0; j < J; ++j) {
    if (!d->win_bulk[j]) continue;
    const sgb_group &G = d->groups[u.g0 + j];
    if ((G.flags & FLAG_INTERLEAVED) || G.n_const || G.n_slots < 1) return bad("member " + std::to_string(j));
    NR += G.n_slots;
    NW += G.n_roots;
  }
  const int64_t roff_at = 32 + 8 * J, woff_at = roff_at + 2 * NR, wpos_at = a16(woff_at + 2 * NW);
  if (d->win_meta_off[0] != 0 || d->win_meta_off[n_win] != d->n_win_meta || d->win_iv_off[0] != 0 ||
      d->win_iv_off[n_win] != d->n_win_iv)
    return bad("offsets do not cover the tables");
  const int64_t wmax = d->win_bw / 8 - 2;
  for (int64_t w = 0; w < n_win; ++w) {
    const int64_t m0 = d->win_meta_off[w], m1 = d->win_meta_off[w + 1];
    if (m1 <= m0 || m0 % 16 || (m1 - m0) % 16 || m1 - m0 > d->win_slot_meta || m1 - m0 < wpos_at)
      return bad("blob " + std::to_string(w));
    const uint8_t *b = d->win_meta + m0;
    uint32_t h[4];
    int64_t k0;
    uint32_t h2[2];
    std::memcpy(h, b, 16);
    std::memcpy(&k0, b + 16, 8);
    std::memcpy(h2, b + 24, 8);
    const int64_t nc = h[0], csrc_at = h[1], cpos_at = h[2], len = h[3], nwp = h2[0], xl = h2[1];
    if (k0 != d->win_k[w] || len != d->win_k[w + 1] - d->win_k[w] || len > wmax ||
        nc != d->win_copy[w + 1] - d->win_copy[w] || csrc_at != a16(wpos_at + 2 * nwp) ||
        cpos_at != a16(csrc_at + 4 * nc) || a16(cpos_at + 2 * nc) != m1 - m0 || 8 * xl > d->win_slot_x)
      return bad("header of window " + std::to_string(w));
    int64_t sum = 0;
    for (int64_t v = d->win_iv_off[w]; v < d->win_iv_off[w + 1]; ++v) {
      const int64_t src = d->win_iv[2 * v], cnt = d->win_iv[2 * v + 1];
      if ((src & 1) || (cnt & 1) || cnt <= 0 || src + cnt > vas_even) return bad("interval " + std::to_string(v));
      sum += cnt;
    }
    if (sum != xl) return bad("x area of window " + std::to_string(w));
    if (std::memcmp(b + 32, d->win_pieces + 2 * w * J, 8 * J)) return bad("pieces of window " + std::to_string(w));
    int64_t ri = 0, wi = 0;
    for (int64_t j = 0; j < J; ++j) {
      if (!d->win_bulk[j]) continue;
      const sgb_group &G = d->groups[u.g0 + j];
      const int64_t cnt = d->win_pieces[2 * (w * J + j) + 1];
      for (int s2 = 0; s2 < G.n_slots; ++s2, ++ri) {
        uint16_t ro;
        std::memcpy(&ro, b + roff_at + 2 * ri, 2);
        if (cnt && ro + cnt > xl) return bad("run offset of window " + std::to_string(w));
      }
      for (int r2 = 0; r2 < G.n_roots; ++r2, ++wi) {
        uint16_t wo;
        std::memcpy(&wo, b + woff_at + 2 * wi, 2);
        if (cnt && wo + cnt > nwp) return bad("position offset of window " + std::to_string(w));
      }
    }
    for (int64_t q = 0; q < nwp; ++q) {
      uint16_t o;
      std::memcpy(&o, b + wpos_at + 2 * q, 2);
      if (o != 0xFFFFu && o >= len) return bad("window position of window " + std::to_string(w));
    }
    for (int64_t c = 0; c < nc; ++c) {
      uint32_t cs;
      uint16_t cp;
      std::memcpy(&cs, b + csrc_at + 4 * c, 4);
      std::memcpy(&cp, b + cpos_at + 2 * c, 2);
      if ((int64_t)cs >= d->value_array_size || cp >= len) return bad("copy of window " + std::to_string(w));
    }
  }
  return 0;
}

static int create_impl(const sgb_plan_desc *d, int device, sgb_plan *p) {
  int ndev = 0;
  SGB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(-1, "sgb_plan_create: bad device ordinal");
  SGB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  SGB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(-2, "sgb_plan_create: libsgb is built for sm_100a (B200) only");
  if (d->n_waves < 0 || d->n_groups < 0 || d->n_units < 0 || d->n_tiles < 0)
    return fail(-1, "sgb_plan_create: negative counts");
  if (d->value_array_size >= (int64_t)1 << 32) return fail(-1, "sgb_plan_create: value array exceeds u32 addressing");
  p->device = device;
  p->vas = d->value_array_size;
  p->n_in = d->input_count;
  p->n_out = d->n_outputs;
  p->n_pos = d->n_positions;
  p->n_con = d->n_constants;
  p->n_groups = d->n_groups;
  p->n_waves = d->n_waves;
  if (d->needs_zero < 0 || d->needs_zero > 2) return fail(-1, "sgb_plan_create: needs_zero must be 0, 1 or 2");
  p->needs_zero = d->needs_zero;
  // host-side validation of every table entry the kernels trust
  for (int g = 0; g < d->n_groups; ++g) {
    const sgb_group &G = d->groups[g];
    const int64_t nch = (G.n + 31) / 32;
    const bool bad =
        G.n < 0 ||
        ((G.flags & FLAG_CSR_ONLY) ? !(G.flags & FLAG_STREAM)  // copy groups never store to the value array
                                   : (G.dest_base < d->input_count || G.dest_base + G.n_roots * G.n > d->value_array_size)) ||
        G.p_off < 0 || G.p_off + (int64_t)G.n_ret * G.n > d->n_positions || G.c_off < 0 ||
        G.c_off + (int64_t)G.n_const * G.n > d->n_constants || G.tape_off < 0 ||
        G.tape_off + G.tape_len > d->tape_rows || G.slot_off < 0 || G.slot_off + G.n_slots > d->n_slot ||
        (G.n_slots > 0 && G.n_ret < 1) ||
        (G.kind == KIND_SOP && (G.sop_len < 1 || G.sop_len > 32 || G.sop_len != G.n_slots ||
                                2 * (int64_t)G.sop_off + 2 > d->n_sop || G.variant < 0 || G.variant > 4 ||
                                G.shape < 0 || G.shape > 2 ||
                                G.sop_len > sop_lmax(G.variant) || G.n_roots != 1)) ||
        ((G.flags & FLAG_W16) && (G.cb_off < 0 || G.co_off < 0 || G.cb_off + (int64_t)G.n_ret * nch > d->n_cbase ||
                                  G.co_off + (int64_t)G.n_ret * G.n > d->n_coff)) ||
        ((G.flags & FLAG_OPOS16) && (G.ob_off < 0 || G.oo_off < 0 ||
                                     G.ob_off + (int64_t)G.n_roots * nch > d->n_obase ||
                                     G.oo_off + (int64_t)G.n_roots * G.n > d->n_ooff)) ||
        ((G.flags & FLAG_OPOS32) && (G.oo_off < 0 || G.oo_off + (int64_t)G.n_roots * G.n > d->n_opos32)) ||
        ((G.flags & FLAG_WPOS16) && (G.oo_off < 0 || G.oo_off + (int64_t)G.n_roots * G.n > d->n_ooff ||
                                     (G.flags & (FLAG_OPOS16 | FLAG_OPOS32)) || !(G.flags & FLAG_CSR_ONLY))) ||
        ((G.flags & FLAG_COHERENT) && G.n_ret != 1);
    if (bad) return fail(-1, "sgb_plan_create: group " + std::to_string(g) + " is out of range");
    for (int s = 0; s < G.n_slots; ++s)
      if (d->slot_col[G.slot_off + s] >= G.n_ret) return fail(-1, "sgb_plan_create: bad slot column");
  }
  for (int64_t k = 0; k < d->n_positions; ++k)
    if ((int64_t)d->positions[k] >= d->value_array_size)
      return fail(-1, "sgb_plan_create: position index outside the value array");
  for (int g = 0; g < d->n_groups; ++g) {  // compressed / affine / coherent decodes stay inside the value array
    const sgb_group &G = d->groups[g];
    if (G.n == 0) continue;
    if (G.flags & FLAG_AFFINE0) {
      const int64_t first = G.a0_base, last = G.a0_base + G.a0_stride * (G.n - 1);
      if (first < 0 || last < 0 || first >= d->value_array_size || last >= d->value_array_size)
        return fail(-1, "sgb_plan_create: affine index column outside the value array");
    }
    if ((G.flags & FLAG_W16) &&
        !w16_ok(d->cbase + G.cb_off, d->coff + G.co_off, G.n, G.n_ret, (G.flags & FLAG_AFFINE0) ? 1 : 0,
                d->value_array_size, false))
      return fail(-1, "sgb_plan_create: compressed index outside the value array");
    if ((G.flags & FLAG_OPOS16) &&
        !w16_ok(d->obase + G.ob_off, d->ooff + G.oo_off, G.n, G.n_roots, 0, d->n_outputs, true))
      return fail(-1, "sgb_plan_create: output position outside the output array");
    if (G.flags & FLAG_OPOS32)
      for (int64_t e = 0; e < (int64_t)G.n_roots * G.n; ++e) {
        const uint32_t o = d->opos32[G.oo_off + e];
        if (o != NONE && (int64_t)o >= d->n_outputs) return fail(-1, "sgb_plan_create: output position out of range");
      }
    // slot-0 relative decodes (coherent slots): the extremes of column 0 plus each delta
    int64_t lo = INT64_MAX, hi = INT64_MIN;
    for (int s = 0; s < G.n_slots; ++s) {
      if (d->slot_col[G.slot_off + s] >= 0) continue;
      lo = lo < d->slot_delta[G.slot_off + s] ? lo : d->slot_delta[G.slot_off + s];
      hi = hi > d->slot_delta[G.slot_off + s] ? hi : d->slot_delta[G.slot_off + s];
    }
    if (lo <= hi) {  // every instance's slot-0 index + delta must be a valid address
      int64_t mn = INT64_MAX, mx = INT64_MIN;
      if (G.flags & FLAG_AFFINE0) {
        const int64_t a = G.a0_base, b = G.a0_base + G.a0_stride * (G.n - 1);
        mn = a < b ? a : b;
        mx = a > b ? a : b;
      } else {
        const int64_t nch = (G.n + 31) / 32;
        for (int64_t i = 0; i < G.n; ++i) {
          int64_t v;
          if (G.flags & FLAG_W16) v = (int64_t)d->cbase[G.cb_off + i / 32] + d->coff[G.co_off + i];
          else if (G.flags & FLAG_INTERLEAVED) v = d->positions[G.p_off + i * G.n_ret];
          else v = d->positions[G.p_off + i];
          mn = v < mn ? v : mn;
          mx = v > mx ? v : mx;
          (void)nch;
        }
      }
      if (mn + lo < 0 || mx + hi >= d->value_array_size)
        return fail(-1, "sgb_plan_create: coherent slot decodes outside the value array");
    }
  }
  for (int64_t k = 0; k < d->n_outputs; ++k)
    if (d->outputs[k] < 0 || d->outputs[k] >= d->value_array_size)
      return fail(-1, "sgb_plan_create: output offset outside the value array");
  int smem_max = 0;
  SGB_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  SGB_CUDA(allow_smem<32>(smem_max));
  SGB_CUDA(allow_smem<64>(smem_max));
  SGB_CUDA(allow_smem<128>(smem_max));
  SGB_CUDA(cudaFuncSetAttribute(tape_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
  if (d->jit_cubin_size > 0) {
    if (!d->jit_cubin) return fail(-1, "sgb_plan_create: null specialised-kernel cubin");
    SGB_CUDA(cudaLibraryLoadData(&p->jit_lib, d->jit_cubin, nullptr, nullptr, 0, nullptr, nullptr, 0));
  }
  std::vector<int2> btiles;
  int max_wave = -1;
  bool has_window = false, has_bulk = false;
  for (int k = 0; k < d->n_units; ++k) {
    const int64_t *r = d->units + (int64_t)k * U_COUNT;
    Unit u;
    u.wave = (int)r[U_WAVE];
    u.kind = (int)r[U_KIND];
    u.variant = (int)r[U_VARIANT];
    u.g0 = (int)r[U_G0];
    u.g1 = (int)r[U_G1];
    u.t0 = r[U_T0];
    u.t1 = r[U_T1];
    u.bs = (int)r[U_BS];
    u.regs = (int)r[U_REGS];
    u.flags = (int)r[U_FLAGS];
    u.index = k;
    const bool csr_only = u.flags & UNIT_CSR_ONLY;
    const bool jit = u.flags & UNIT_JIT;
    const bool window = u.flags & UNIT_WINDOW;
    if (window) {
      const int64_t n_win = d->n_win_k - 1, J = u.g1 - u.g0;
      if (!jit || !csr_only || !p->jit_lib || u.t0 != 0 || u.t1 != n_win || n_win < 1 || J < 1 ||
          d->n_win_pieces != n_win * J || d->n_win_copy != d->n_win_k || u.regs < 8 || has_window)
        return fail(-1, "sgb_plan_create: bad CSR-window unit " + std::to_string(k));
      has_window = true;
      const bool bulk = u.flags & UNIT_BULK;
      has_bulk = bulk;
      cudaKernel_t kw;
      const std::string nw = (bulk ? "sgb_wbulk_u" : "sgb_window_u") + std::to_string(k);
      SGB_CUDA(cudaLibraryGetKernel(&kw, p->jit_lib, nw.c_str()));
      u.jit = (const void *)kw;
      if (u.regs > 48 * 1024) SGB_CUDA(cudaFuncSetAttribute(u.jit, cudaFuncAttributeMaxDynamicSharedMemorySize, u.regs));
      const int64_t wmax = (bulk ? d->win_bw : u.regs) / 8 - 2;  // the window buffer (doubles), alignment slots
      if (bulk) {
        const int rc = check_window_bulk(d, u, n_win, J, (int64_t)smem_max);
        if (rc) return rc;
      } else if (u.bs != JIT_BLOCK) {
        return fail(-1, "sgb_plan_create: bad CSR-window block size");
      }
      if (d->win_k[0] != 0 || d->win_k[n_win] != d->n_outputs || d->win_copy[0] != 0 || d->win_copy[n_win] != d->n_copy)
        return fail(-1, "sgb_plan_create: CSR windows do not cover the outputs / copies");
      for (int g = u.g0; g < u.g1; ++g)
        if (!(d->groups[g].flags & FLAG_WPOS16) || (d->groups[g].flags & FLAG_SELFREF))
          return fail(-1, "sgb_plan_create: CSR-window member without window positions");
      for (int64_t w = 0; w < n_win; ++w) {
        const int64_t len = d->win_k[w + 1] - d->win_k[w];
        if (len < 0 || len > wmax || d->win_copy[w + 1] < d->win_copy[w])
          return fail(-1, "sgb_plan_create: bad CSR window " + std::to_string(w));
        for (int64_t c = d->win_copy[w]; c < d->win_copy[w + 1]; ++c)
          if ((int64_t)d->copy_src[c] >= d->value_array_size || (int64_t)d->copy_pos[c] >= len)
            return fail(-1, "sgb_plan_create: bad CSR-window copy");
        for (int64_t j = 0; j < J; ++j) {  // every staged position of every piece stays inside its window
          const int32_t a = d->win_pieces[2 * (w * J + j)], cnt = d->win_pieces[2 * (w * J + j) + 1];
          const sgb_group &G = d->groups[u.g0 + j];
          if (a < 0 || cnt < 0 || (int64_t)a + cnt > G.n) return fail(-1, "sgb_plan_create: bad CSR-window piece");
          for (int r = 0; r < G.n_roots; ++r)
            for (int64_t i = a; i < (int64_t)a + cnt; ++i) {
              const uint16_t o = d->ooff[G.oo_off + (int64_t)r * G.n + i];
              if (o != 0xFFFFu && (int64_t)o >= len) return fail(-1, "sgb_plan_create: window position out of range");
            }
        }
      }
    } else if (jit) {
      // block: JIT_BLOCK threads, or k x JIT_BLOCK for a single-group unit whose root set is split k ways
      // (jit.py: part p = threadIdx.x / JIT_BLOCK evaluates its roots' cone for the tile's instances)
      if (u.kind != KIND_TAPE || u.bs % JIT_BLOCK || u.bs < JIT_BLOCK || u.bs > 4 * JIT_BLOCK ||
          (u.bs != JIT_BLOCK && u.g1 - u.g0 != 1) || (u.variant != 1 && u.variant != 2 && u.variant != 4) ||
          !p->jit_lib)
        return fail(-1, "sgb_plan_create: specialised unit " + std::to_string(k) + " without its kernels");
      cudaKernel_t kf, kb;
      const std::string nf = "sgb_tape_u" + std::to_string(k), nbn = "sgb_tape_b" + std::to_string(k);
      SGB_CUDA(cudaLibraryGetKernel(&kf, p->jit_lib, nf.c_str()));
      SGB_CUDA(cudaLibraryGetKernel(&kb, p->jit_lib, nbn.c_str()));
      u.jit = (const void *)kf;
      u.jitb = (const void *)kb;
      if (u.regs > 48 * 1024)  // staging buffer of instance-major groups (jit.py _stage_out)
        SGB_CUDA(cudaFuncSetAttribute(u.jit, cudaFuncAttributeMaxDynamicSharedMemorySize, u.regs));
    }
    if (u.g0 < 0 || u.g1 > d->n_groups || u.g0 > u.g1 || u.wave < 0 ||
        (csr_only ? u.wave > d->n_waves : u.wave >= d->n_waves) || u.t0 < 0 ||
        (!(u.flags & UNIT_WINDOW) && u.t1 > d->n_tiles) ||
        u.t0 > u.t1 || (u.kind != KIND_TAPE && u.kind != KIND_SOP) ||
        (u.kind == KIND_TAPE && !jit && (u.bs != 32 && u.bs != 64 && u.bs != 128)) ||
        (u.kind == KIND_TAPE && !window && (u.variant != 1 && u.variant != 2 && u.variant != 4)) ||
        (window && (u.variant < 0 || u.variant > 64)) ||
        (jit ? (int64_t)u.regs : (int64_t)u.regs * (u.kind == KIND_TAPE ? u.bs * u.variant : 0) * 8) > smem_max ||
        u.regs < 0)
      return fail(-1, "sgb_plan_create: bad launch unit " + std::to_string(k));
    max_wave = u.wave > max_wave ? u.wave : max_wave;
    {  // persistent grid: resident capacity of the chip, at most one block (warp for SOP) per tile
      int nb = 0;
      if (window && (u.flags & UNIT_BULK)) {  // persistent: each block walks its windows through its ring
        SGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, u.jit, u.bs, (size_t)u.regs));
        u.grid = (int64_t)(nb > 0 ? nb : 1) * prop.multiProcessorCount;
        if (u.grid > u.t1 - u.t0) u.grid = u.t1 - u.t0;
      } else if (window) {
        // one block per window, dispatched in CSR order, minus `variant` rounds of one block per SM: the
        // first blocks then take a second window each (grid-stride) -- the last windows start early and
        // the final round is short (C2: 3757 windows, 0.1273 ms with 3757 blocks, 0.1188 with 3609)
        u.grid = u.t1 - u.t0;
        const int64_t cut = (int64_t)u.variant * prop.multiProcessorCount;
        if (u.grid - cut >= prop.multiProcessorCount) u.grid -= cut;
      } else if (jit) {
        SGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, u.jit, u.bs, (size_t)u.regs));
        u.grid = (int64_t)(nb > 0 ? nb : 1) * prop.multiProcessorCount;
        if (u.grid > u.t1 - u.t0) u.grid = u.t1 - u.t0;
      } else if (u.kind == KIND_TAPE) {
        SGB_CUDA(tape_occupancy_any(u.bs, u.variant, u.regs, &nb));
        u.grid = (int64_t)(nb > 0 ? nb : 1) * prop.multiProcessorCount;
        if (u.grid > u.t1 - u.t0) u.grid = u.t1 - u.t0;
      } else {
        if (!sop_kernel_for(u.variant)) return fail(-1, "sgb_plan_create: bad sum-of-products unit variant");
        SGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sop_kernel_for(u.variant), SOP_BS, 0));
        u.grid = (int64_t)(nb > 0 ? nb : 1) * prop.multiProcessorCount;
        const int64_t need = (u.t1 - u.t0 + SOP_BS / 32 - 1) / (SOP_BS / 32);
        if (u.grid > need) u.grid = need;
      }
    }
    if (jit)
      for (int g = u.g0; g < u.g1; ++g)
        if (d->groups[g].flags & (FLAG_SELFREF | FLAG_SERIAL))
          return fail(-1, "sgb_plan_create: self-referencing group in a specialised unit");
    if (!jit)
      for (int g = u.g0; g < u.g1; ++g)
        if (d->groups[g].flags & FLAG_IMAJOR)
          return fail(-1, "sgb_plan_create: instance-major group outside a specialised unit");
    for (int64_t t = window ? u.t1 : u.t0; t < u.t1; ++t) {  // tiles name groups of this unit, start inside them
      const int32_t *tl = d->tiles + 2 * t;
      if (tl[0] < u.g0 || tl[0] >= u.g1 || tl[1] < 0 || (int64_t)tl[1] >= d->groups[tl[0]].n)
        return fail(-1, "sgb_plan_create: bad tile in unit " + std::to_string(k));
    }
    for (int g = u.g0; g < u.g1; ++g) {
      const sgb_group &G = d->groups[g];
      if (G.kind != u.kind) return fail(-1, "sgb_plan_create: group kind differs from its unit");
      if (u.kind == KIND_SOP && u.variant != SOP_GENERAL_CODE &&
          (!sop_fast_ok(G) || u.variant != G.shape * 8 + G.variant))
        return fail(-1, "sgb_plan_create: group does not fit its sum-of-products unit");
      if (u.kind == KIND_TAPE && (G.flags & FLAG_SERIAL) && u.variant != 1)
        return fail(-1, "sgb_plan_create: serial group in a vectorised tape unit");
    }
    // batched tiles: one instance per warp (tape blocks are the unit's scratch stride wide);
    // CSR windows are single-set only (batched CSR = batched values + gather)
    const int bwarps = jit ? JIT_BLOCK / 32 : u.kind == KIND_TAPE ? (u.bs * u.variant) / 32 : BATCH_WARPS;
    u.bt0 = (int64_t)btiles.size();
    for (int g = window ? u.g1 : u.g0; g < u.g1; ++g) {
      const sgb_group &G = d->groups[g];
      if (G.flags & FLAG_SERIAL) {
        if (G.n > 0) btiles.push_back(make_int2(g, 0));
        continue;
      }
      for (int64_t i = 0; i < G.n; i += bwarps) btiles.push_back(make_int2(g, (int)i));
    }
    u.bt1 = (int64_t)btiles.size();
    if (jit && u.jitb) {  // the batched kernel's own resident capacity (not the single-set grid,
                          // which is capped by the single-set tile count -- 256x fewer tiles)
      int nbb = 0;
      SGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbb, u.jitb, JIT_BLOCK, 0));
      u.grid_b = (int64_t)(nbb > 0 ? nbb : 1) * prop.multiProcessorCount;
      if (u.grid_b > u.bt1 - u.bt0) u.grid_b = u.bt1 - u.bt0;
    }
    if (jit)  // as the single-set tiles (lower.py): interleave the groups' tiles by instance for L2 reuse
      std::stable_sort(btiles.begin() + u.bt0, btiles.end(), [](const int2 &a, const int2 &b) { return a.y < b.y; });
    if (u.kind == KIND_TAPE && !jit) {  // every tape word must stay inside its lane's scratch column
      const uint64_t limit = (uint64_t)u.regs * u.bs * u.variant * 8;
      for (int g = u.g0; g < u.g1; ++g) {
        const sgb_group &G = d->groups[g];
        if (G.n_slots + G.n_const > u.regs) return fail(-1, "sgb_plan_create: slots exceed the scratch file");
        for (int64_t k2 = G.tape_off; k2 < G.tape_off + G.tape_len; ++k2) {
          const uint32_t *w = d->tape + 4 * k2;
          const uint32_t op = (w[0] & 0xFFu) >> 2;
          if (op != T_MUL && op != T_ADD && op != T_SUB && op != T_DIV && op != T_MADD && op != T_MSUB &&
              op != T_RMSUB && (w[0] & 3u))
            return fail(-1, "sgb_plan_create: sign flags on an op that takes none");
          const uint64_t c8 = (uint64_t)(w[0] >> 8) << 3;
          bool bad = op > T_RMSUB || w[2] >= limit || c8 >= limit;
          if (op != T_ST) bad = bad || w[1] >= limit;
          if (op == T_IMM) bad = bad || w[3] >= d->n_imm;
          else if (op == T_ST) bad = bad || (int64_t)w[3] >= G.n_roots;
          else if (op == T_SLOW) bad = bad || (w[3] >> 16) > 4;
          else bad = bad || w[3] >= limit;
          if (bad) return fail(-1, "sgb_plan_create: malformed tape word in group " + std::to_string(g));
        }
      }
    }
    p->units.push_back(u);
  }
  p->csr_waves = max_wave + 1 > p->n_waves ? max_wave + 1 : p->n_waves;
  {  // per wave: largest unit first (caller's stream); the others co-run on aux streams
    std::stable_sort(p->units.begin(), p->units.end(), [](const Unit &a, const Unit &b) {
      return a.wave != b.wave ? a.wave < b.wave : (a.t1 - a.t0) > (b.t1 - b.t0);
    });
    int max_units = 1;
    for (int w = 0; w <= max_wave; ++w) {
      int n = 0;
      for (const Unit &u : p->units) n += u.wave == w;
      max_units = n > max_units ? n : max_units;
      if (n < 2) continue;
      // leave one block per SM to the co-running units (not window units: they run in CSR mode only
      // while their wave's value-mode twins do not; their grid is chosen above)
      for (Unit &u : p->units)
        if (u.wave == w && !(u.flags & UNIT_WINDOW) && u.grid > prop.multiProcessorCount) {
          const int64_t cap = u.grid - prop.multiProcessorCount;
          if (cap >= prop.multiProcessorCount) u.grid = cap;
        }
    }
    // specialised units have two grids: the persistent one (resident capacity, tiles grid-strided)
    // and one block per tile, the hardware dispatching blocks in tile order as SMs free up --
    // persistent blocks drift apart over a long sweep and widen its L2 working set.
    // sgb_plan_set_wave_grid picks per wave (runtime autotune); the default is persistent.
    for (Unit &u : p->units)
      if ((u.flags & UNIT_JIT) && !(u.flags & UNIT_WINDOW)) {
        u.grid_p = u.grid;
        u.grid_t = u.t1 - u.t0 < 0x7fffffffLL ? u.t1 - u.t0 : 0x7fffffffLL;
      }
    p->wave_units.assign(max_wave + 1, {});
    for (int k = 0; k < (int)p->units.size(); ++k) p->wave_units[p->units[k].wave].push_back(k);
    const int n_aux = max_units - 1 < 8 ? max_units - 1 : 8;
    SGB_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
    for (int k = 0; k < n_aux; ++k) {
      cudaStream_t a;
      cudaEvent_t e;
      SGB_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
      p->aux.push_back(a);
      SGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      p->ev_join.push_back(e);
    }
  }
  p->group_n.resize(d->n_groups);
  for (int g = 0; g < d->n_groups; ++g) p->group_n[g] = d->groups[g].n;
  p->h_tiles.assign(reinterpret_cast<const int2 *>(d->tiles), reinterpret_cast<const int2 *>(d->tiles) + d->n_tiles);
  std::vector<uint32_t> outputs32(d->outputs, d->outputs + d->n_outputs);
  for (int g = 0; g < d->n_groups; ++g)  // CSR mode without the gather: direct stores or CSR windows
    if (d->groups[g].flags & (FLAG_OPOS16 | FLAG_OPOS32 | FLAG_WPOS16)) p->direct_csr = true;
  for (int g = 0; g < d->n_groups; ++g)
    if (d->groups[g].flags & FLAG_IMAJOR) p->csr_layout = true;
  // compact sum-of-products descriptors (+ fast-path factor bases)
  std::vector<SopDesc> sopd(d->n_groups);
  std::vector<uint32_t> fbase;
  if (d->n_obase >= ((int64_t)1 << 32) || d->n_ooff >= ((int64_t)1 << 32) || d->n_opos32 >= ((int64_t)1 << 32))
    return fail(-1, "sgb_plan_create: output-position tables exceed u32 offsets");
  for (int g = 0; g < d->n_groups; ++g) {
    const sgb_group &G = d->groups[g];
    SopDesc &sd = sopd[g];
    memset(&sd, 0, sizeof(sd));
    if (G.kind != KIND_SOP) continue;
    if (G.n >= ((int64_t)1 << 31)) return fail(-1, "sgb_plan_create: sum-of-products group exceeds 2^31 instances");
    const bool fast = sop_fast_ok(G);
    sd.n = (int32_t)G.n;
    sd.dest_base = (uint32_t)G.dest_base;
    sd.meta = (uint32_t)G.sop_len | ((uint32_t)G.shape << 6) | ((uint32_t)G.variant << 8) | (fast ? M_FAST : 0u) |
              ((G.flags & FLAG_CSR_ONLY) ? M_CSR_ONLY : 0u) | ((G.flags & FLAG_STREAM) ? M_STREAM : 0u) |
              ((G.flags & FLAG_OPOS16) ? M_OPOS16 : 0u) | ((G.flags & FLAG_OPOS32) ? M_OPOS32 : 0u);
    sd.stride = (int32_t)G.a0_stride;
    sd.newterm = d->sop[2 * G.sop_off];
    sd.negm = d->sop[2 * G.sop_off + 1];
    sd.g = g;
    sd.ob_off = (uint32_t)G.ob_off;
    sd.oo_off = (uint32_t)G.oo_off;
    if (fast) {
      sd.fbase_off = (uint32_t)fbase.size();
      for (int f = 0; f < G.sop_len; ++f)  // slot 0 is the affine column itself (delta 0)
        fbase.push_back((uint32_t)(G.a0_base + (d->slot_col[G.slot_off + f] < 0 ? d->slot_delta[G.slot_off + f] : 0)));
    }
  }
  int rc = 0;
  if ((rc = upload(&p->d_groups, d->groups, d->n_groups)) ||
      (p->n_tiles = d->n_tiles, rc = upload(&p->d_tiles, reinterpret_cast<const int2 *>(d->tiles), d->n_tiles)) ||
      (rc = upload(&p->d_btiles, btiles.data(), (int64_t)btiles.size())) ||
      (rc = upload(&p->d_outputs, d->outputs, d->n_outputs)) ||
      (rc = upload(&p->d_tape, d->tape, d->tape_rows * 4)) || (rc = upload(&p->d_imm, d->imm, d->n_imm)) ||
      (rc = upload(&p->d_sop, d->sop, d->n_sop)) || (rc = upload(&p->d_scol, d->slot_col, d->n_slot)) ||
      (rc = upload(&p->d_sdel, d->slot_delta, d->n_slot)) ||
      (rc = upload(&p->d_pos, d->positions, d->n_positions)) ||
      (rc = upload(&p->d_con, d->constants, d->n_constants)) ||
      (rc = upload(&p->d_cbase, d->cbase, d->n_cbase)) || (rc = upload(&p->d_coff, d->coff, d->n_coff)) ||
      (rc = upload(&p->d_obase, d->obase, d->n_obase)) || (rc = upload(&p->d_ooff, d->ooff, d->n_ooff)) ||
      (rc = upload(&p->d_opos32, d->opos32, d->n_opos32)) ||
      (rc = upload(&p->d_sopd, sopd.data(), (int64_t)sopd.size())) ||
      (rc = upload(&p->d_outputs32, outputs32.data(), (int64_t)outputs32.size())) ||
      (rc = upload(&p->d_wpieces, reinterpret_cast<const int2 *>(d->win_pieces), d->n_win_pieces)) ||
      (rc = upload(&p->d_wk, d->win_k, d->n_win_k)) || (rc = upload(&p->d_wcopy, d->win_copy, d->n_win_copy)) ||
      (rc = upload(&p->d_csrc, d->copy_src, d->n_copy)) || (rc = upload(&p->d_cpos, d->copy_pos, d->n_copy)) ||
      (rc = upload(&p->d_fbase, fbase.data(), (int64_t)fbase.size())))
    return rc;
  if (has_bulk) {
    if ((rc = upload(&p->d_wmeta, d->win_meta, d->n_win_meta)) ||
        (rc = upload(&p->d_wmeta_off, d->win_meta_off, d->n_win_k)) ||
        (rc = upload(&p->d_wiv, reinterpret_cast<const uint2 *>(d->win_iv), d->n_win_iv)) ||
        (rc = upload(&p->d_wiv_off, d->win_iv_off, d->n_win_k)))
      return rc;
    p->wb_ring = d->win_ring;
    p->wb_meta = d->win_slot_meta;
    p->wb_x = d->win_slot_x;
    p->wb_bw = d->win_bw;
  }
  p->vas_slots = has_bulk ? d->value_array_size + (d->value_array_size & 1) : d->value_array_size;
  if (has_window && d->n_outputs > 0) {
    // batched CSR of a window plan: every output must come from exactly one value-mode twin
    // position (FLAG_OPOS*) or one copy; otherwise batched CSR keeps the full gather
    std::vector<uint8_t> hit((size_t)d->n_outputs, 0);
    bool ok = true;
    std::vector<uint32_t> copy_k((size_t)d->n_copy);
    const int64_t n_win = d->n_win_k - 1;
    for (int64_t w = 0; w < n_win && ok; ++w)
      for (int64_t c = d->win_copy[w]; c < d->win_copy[w + 1]; ++c) {
        const int64_t k = d->win_k[w] + d->copy_pos[c];
        copy_k[(size_t)c] = (uint32_t)k;
        ok = ok && k < d->n_outputs && ++hit[(size_t)k] == 1;
      }
    for (const Unit &u : p->units) {
      if (!(u.flags & UNIT_VALUE_ONLY) || !ok) continue;
      for (int g = u.g0; g < u.g1 && ok; ++g) {
        const sgb_group &G = d->groups[g];
        if (!(G.flags & (FLAG_OPOS16 | FLAG_OPOS32))) { ok = false; break; }
        const int64_t nch = (G.n + 31) >> 5;
        for (int r = 0; r < G.n_roots && ok; ++r)
          for (int64_t i = 0; i < G.n; ++i) {
            uint32_t o = NONE;
            if (G.flags & FLAG_OPOS16) {
              const uint16_t off = d->ooff[G.oo_off + (int64_t)r * G.n + i];
              if (off != 0xFFFFu) o = d->obase[G.ob_off + (int64_t)r * nch + (i >> 5)] + off;
            } else {
              o = d->opos32[G.oo_off + (int64_t)r * G.n + i];
            }
            if (o == NONE) continue;
            if ((int64_t)o >= d->n_outputs || ++hit[o] != 1) { ok = false; break; }
          }
      }
    }
    for (int64_t k = 0; k < d->n_outputs && ok; ++k) ok = hit[(size_t)k] == 1;
    if (ok) {
      if ((rc = upload(&p->d_copy_k, copy_k.data(), (int64_t)copy_k.size()))) return rc;
      p->n_copy_k = (int64_t)copy_k.size();
      p->batch_direct = true;
    }
  }
  p->T = Tables{p->d_groups, p->d_tape, p->d_imm, p->d_sop, p->d_scol, p->d_sdel, p->d_pos,
                p->d_con, p->d_cbase, p->d_coff, p->d_obase, p->d_ooff, p->d_opos32, p->d_fbase};
  return 0;
}

int sgb_plan_create(const sgb_plan_desc *d, int device, sgb_plan **out) {
  if (!d || !out) return fail(-1, "sgb_plan_create: null argument");
  *out = nullptr;
  sgb_plan *p = new sgb_plan();
  int rc = create_impl(d, device, p);
  if (rc) {
    std::string msg = g_err;
    sgb_plan_destroy(p);
    return fail(rc, msg);
  }
  *out = p;
  return 0;
}

// All units of one wave are independent: the largest runs on the caller's
// stream, the others on the plan's aux streams forked from / joined back into it.
static int launch_wave(sgb_plan *p, int wave, double *x, int64_t ld, int64_t batch, bool batched, double *out,
                       int64_t ld_out, bool csr, cudaStream_t s) {
  if (wave < 0 || wave >= (int)p->wave_units.size()) return 0;
  std::vector<const Unit *> us;
  us.reserve(p->wave_units[wave].size());
  for (int k : p->wave_units[wave]) {
    const Unit &u = p->units[k];
    if (!csr && (u.flags & UNIT_CSR_ONLY)) continue;
    if (batched && (u.flags & UNIT_CSR_ONLY)) continue;            // single-set only (windows, copy groups)
    if (csr && !batched && (u.flags & UNIT_VALUE_ONLY)) continue;  // twins of CSR-window members
    if ((batched ? u.bt1 - u.bt0 : u.t1 - u.t0) <= 0) continue;
    us.push_back(&u);
  }
  const int n = (int)us.size();
  if (n == 0) return 0;
  const int k_aux = n - 1 < (int)p->aux.size() ? n - 1 : (int)p->aux.size();
  if (k_aux > 0) SGB_CUDA(cudaEventRecord(p->ev_fork, s));
  for (int k = 0; k < k_aux; ++k) SGB_CUDA(cudaStreamWaitEvent(p->aux[k], p->ev_fork, 0));
  launch_unit(p, *us[0], x, ld, batch, batched, out, ld_out, csr, s);
  for (int k = 1; k < n; ++k) {
    cudaStream_t sk = k - 1 < k_aux ? p->aux[k - 1] : s;
    launch_unit(p, *us[k], x, ld, batch, batched, out, ld_out, csr, sk);
  }
  for (int k = 0; k < k_aux; ++k) {
    SGB_CUDA(cudaEventRecord(p->ev_join[k], p->aux[k]));
    SGB_CUDA(cudaStreamWaitEvent(s, p->ev_join[k], 0));
  }
  return 0;
}

static int launch_gather(sgb_plan *p, const double *x, int64_t ld, int64_t batch, bool batched, double *out,
                         int64_t ld_out, cudaStream_t s);

// CSR mode without direct stores: every wave in value mode, then the output gather.
static int launch_all(sgb_plan *p, double *x, int64_t ld, int64_t batch, bool batched, double *out, int64_t ld_out,
                      bool csr, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(p->run_mu);
  const bool direct = csr && p->direct_csr && !batched;  // batched CSR: batched values + gather
  // batched CSR of a CSR-window plan: the members' value-mode twins store their outputs directly
  // (out[pos * ld_out + b], one warp per instance: coalesced), the other outputs are gathered
  const bool bdirect = csr && batched && p->batch_direct;
  const int waves = direct ? p->csr_waves : p->n_waves;
  for (int w = 0; w < waves; ++w) {
    int rc = launch_wave(p, w, x, ld, batch, batched, out, ld_out, direct || bdirect, s);
    if (rc) return rc;
  }
  if (bdirect) {
    if (p->n_copy_k > 0) {
      const int64_t blocks = (p->n_copy_k + 7) / 8;
      gather_copies_batch<<<(unsigned)blocks, 256, 0, s>>>(x, ld, batch, p->d_copy_k, p->d_csrc, p->n_copy_k, out,
                                                           ld_out);
    }
  } else if (csr && !direct) {
    int rc = launch_gather(p, x, ld, batch, batched, out, ld_out, s);
    if (rc) return rc;
  }
  SGB_CUDA(cudaGetLastError());
  return 0;
}

int sgb_run_wave(sgb_plan *p, double *x, double *out, int wave, void *stream) {
  if (!p || (!x && p->vas)) return fail(-1, "sgb_run_wave: null argument");
  const bool csr = out != nullptr;
  if (!csr && p->csr_layout) return fail(-2, "sgb_run_wave: plan uses the CSR layout (value mode unavailable)");
  if (wave < 0 || wave >= sgb_plan_waves(p, csr)) return fail(-1, "sgb_run_wave: wave out of range");
  if (csr && p->n_out == 0) return 0;
  if (csr && p->wb_ring && (reinterpret_cast<uintptr_t>(x) & 15))
    return fail(-1, "sgb_run_wave: the bulk CSR-window feed needs a 16-byte aligned value array");
  std::lock_guard<std::mutex> lk(p->run_mu);
  if (csr && !p->direct_csr && wave == p->n_waves) {  // the output gather
    int rc = launch_gather(p, x, 1, 1, false, out, 1, (cudaStream_t)stream);
    if (rc) return rc;
    SGB_CUDA(cudaGetLastError());
    return 0;
  }
  int rc = launch_wave(p, wave, x, 1, 1, false, out, 1, csr && p->direct_csr, (cudaStream_t)stream);
  if (rc) return rc;
  SGB_CUDA(cudaGetLastError());
  return 0;
}

int sgb_run_values(sgb_plan *p, double *x, void *stream) {
  if (!p || (!x && p->vas)) return fail(-1, "sgb_run_values: null argument");
  if (p->csr_layout) return fail(-2, "sgb_run_values: plan uses the CSR layout (value mode unavailable)");
  return launch_all(p, x, 1, 1, false, nullptr, 1, false, (cudaStream_t)stream);
}

int sgb_run_csr(sgb_plan *p, double *x, double *out, void *stream) {
  if (!p || (!x && p->vas) || (!out && p->n_out)) return fail(-1, "sgb_run_csr: null argument");
  if (!p->n_out) return 0;
  if (p->wb_ring && (reinterpret_cast<uintptr_t>(x) & 15))
    return fail(-1, "sgb_run_csr: the bulk CSR-window feed needs a 16-byte aligned value array");
  return launch_all(p, x, 1, 1, false, out, 1, true, (cudaStream_t)stream);
}

int sgb_run_batch(sgb_plan *p, double *X, int64_t ld, int64_t batch, void *stream) {
  if (!p || (!X && p->vas)) return fail(-1, "sgb_run_batch: null argument");
  if (batch < 1 || ld < batch) return fail(-1, "sgb_run_batch: need 1 <= batch <= ld");
  if (p->csr_layout) return fail(-2, "sgb_run_batch: plan uses the CSR layout (value mode unavailable)");
  return launch_all(p, X, ld, batch, true, nullptr, 1, false, (cudaStream_t)stream);
}

int sgb_run_batch_csr(sgb_plan *p, double *X, int64_t ld, int64_t batch, double *out, int64_t ld_out,
                      void *stream) {
  if (!p || (!X && p->vas) || (!out && p->n_out)) return fail(-1, "sgb_run_batch_csr: null argument");
  if (batch < 1 || ld < batch || ld_out < batch) return fail(-1, "sgb_run_batch_csr: need 1 <= batch <= ld, ld_out");
  if (!p->n_out) return 0;
  return launch_all(p, X, ld, batch, true, out, ld_out, true, (cudaStream_t)stream);
}

static int launch_gather(sgb_plan *p, const double *x, int64_t ld, int64_t batch, bool batched, double *out,
                         int64_t ld_out, cudaStream_t s) {
  if (!p->n_out) return 0;
  if (batched) {
    const int64_t blocks = (p->n_out + 7) / 8;
    gather_outputs_batch<<<(unsigned)blocks, 256, 0, s>>>(x, ld, batch, p->d_outputs, p->n_out, out, ld_out);
  } else {
    int64_t blocks = (p->n_out + 255) / 256;
    // a capped grid-stride grid: one block per 256 outputs and four outputs per thread with 16-byte
    // index loads both measured slower (profiles/r42)
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (blocks > 0x7fffffffLL) blocks = 0x7fffffffLL;
    gather_outputs<<<(unsigned)blocks, 256, 0, s>>>(x, p->d_outputs32, p->n_out, out);
  }
  return 0;
}

int sgb_gather_outputs(sgb_plan *p, const double *x, double *out, void *stream) {
  if (!p) return fail(-1, "sgb_gather_outputs: null plan");
  if (!p->n_out) return 0;
  if (!x || !out) return fail(-1, "sgb_gather_outputs: null buffer");
  const int bs = 256;
  int64_t blocks = (p->n_out + bs - 1) / bs;
  if (blocks > 148 * 32) blocks = 148 * 32;
  gather_outputs<<<(unsigned)blocks, bs, 0, (cudaStream_t)stream>>>(x, p->d_outputs32, p->n_out, out);
  SGB_CUDA(cudaGetLastError());
  return 0;
}

int sgb_gather_outputs_batch(sgb_plan *p, const double *X, int64_t ld, int64_t batch, double *out, int64_t ld_out,
                             void *stream) {
  if (!p) return fail(-1, "sgb_gather_outputs_batch: null plan");
  if (!p->n_out) return 0;
  if (!X || !out || batch < 1 || ld < batch || ld_out < batch)
    return fail(-1, "sgb_gather_outputs_batch: bad arguments");
  const int64_t blocks = (p->n_out + 7) / 8;
  gather_outputs_batch<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(X, ld, batch, p->d_outputs, p->n_out,
                                                                          out, ld_out);
  SGB_CUDA(cudaGetLastError());
  return 0;
}

static int ensure_ws(sgb_plan *p) {
  SGB_CUDA(cudaSetDevice(p->device));
  if (!p->ws_stream) SGB_CUDA(cudaStreamCreateWithFlags(&p->ws_stream, cudaStreamNonBlocking));
  if (!p->d_x && p->vas) {
    SGB_CUDA(cudaMalloc((void **)&p->d_x, sizeof(double) * (size_t)p->vas_slots));
    // never-written slots (padding, reads before writes) read as zero (codegen.py:419)
    SGB_CUDA(cudaMemset(p->d_x, 0, sizeof(double) * (size_t)p->vas));
    SGB_CUDA(cudaDeviceSynchronize());  // the non-blocking ws_stream does not order after the legacy stream
  }
  if (!p->d_out && p->n_out) SGB_CUDA(cudaMalloc((void **)&p->d_out, sizeof(double) * (size_t)p->n_out));
  // a workspace use enqueued by sgb_run_inputs_csr on another stream must finish first
  if (p->ws_event) SGB_CUDA(cudaStreamWaitEvent(p->ws_stream, p->ws_event, 0));
  return 0;
}

// Device inputs -> device CSR values (the inputs -> CSR shape), through the
// plan's own value-array workspace: stream-ordered, no host synchronisation.
int sgb_run_inputs_csr(sgb_plan *p, const double *inputs, double *out, void *stream) {
  if (!p || (!inputs && p->n_in) || (!out && p->n_out)) return fail(-1, "sgb_run_inputs_csr: null argument");
  if (!p->n_out) return 0;
  std::lock_guard<std::mutex> lk(p->ws_mu);
  int rc = ensure_ws(p);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->ws_event) SGB_CUDA(cudaStreamWaitEvent(s, p->ws_event, 0));
  if ((p->needs_zero == 2 || (p->needs_zero == 1 && p->ws_dirty)) && p->vas > p->n_in)
    SGB_CUDA(cudaMemsetAsync(p->d_x + p->n_in, 0, sizeof(double) * (size_t)(p->vas - p->n_in), s));
  p->ws_dirty = false;
  if (p->n_in)
    SGB_CUDA(cudaMemcpyAsync(p->d_x, inputs, sizeof(double) * (size_t)p->n_in, cudaMemcpyDeviceToDevice, s));
  if ((rc = sgb_run_csr(p, p->d_x, out, s))) return rc;
  if (!p->ws_event) SGB_CUDA(cudaEventCreateWithFlags(&p->ws_event, cudaEventDisableTiming));
  SGB_CUDA(cudaEventRecord(p->ws_event, s));
  return 0;
}

int sgb_sg_run(sgb_plan *p, double *x_host, const double *c_host, const unsigned *p_host) {
  (void)c_host;
  (void)p_host;
  if (!p || (!x_host && p->vas)) return fail(-1, "sgb_sg_run: null argument");
  if (p->csr_layout) return fail(-2, "sgb_sg_run: plan uses the CSR layout (value mode unavailable)");
  std::lock_guard<std::mutex> lk(p->ws_mu);
  int rc = ensure_ws(p);
  if (rc) return rc;
  if (!p->vas) return 0;
  SGB_CUDA(cudaMemcpyAsync(p->d_x, x_host, sizeof(double) * (size_t)p->vas, cudaMemcpyHostToDevice, p->ws_stream));
  p->ws_dirty = true;
  if ((rc = sgb_run_values(p, p->d_x, p->ws_stream))) return rc;
  SGB_CUDA(cudaMemcpyAsync(x_host, p->d_x, sizeof(double) * (size_t)p->vas, cudaMemcpyDeviceToHost, p->ws_stream));
  SGB_CUDA(cudaStreamSynchronize(p->ws_stream));
  return 0;
}

int sgb_run_outputs_host(sgb_plan *p, const double *inputs, double *outputs) {
  if (!p) return fail(-1, "sgb_run_outputs_host: null plan");
  std::lock_guard<std::mutex> lk(p->ws_mu);
  int rc = ensure_ws(p);
  if (rc) return rc;
  if (!p->n_out) return 0;
  // zero-reads (padding, read-before-write) must see zeros: re-zero when a previous
  // evaluation may have written them (every time for read-before-write plans)
  if ((p->needs_zero == 2 || (p->needs_zero == 1 && p->ws_dirty)) && p->vas > p->n_in)
    SGB_CUDA(cudaMemsetAsync(p->d_x + p->n_in, 0, sizeof(double) * (size_t)(p->vas - p->n_in), p->ws_stream));
  p->ws_dirty = false;
  if (p->n_in)
    SGB_CUDA(cudaMemcpyAsync(p->d_x, inputs, sizeof(double) * (size_t)p->n_in, cudaMemcpyHostToDevice, p->ws_stream));
  if ((rc = sgb_run_csr(p, p->d_x, p->d_out, p->ws_stream))) return rc;
  SGB_CUDA(cudaMemcpyAsync(outputs, p->d_out, sizeof(double) * (size_t)p->n_out, cudaMemcpyDeviceToHost, p->ws_stream));
  SGB_CUDA(cudaStreamSynchronize(p->ws_stream));
  return 0;
}


// A stream of value sets through host buffers: set k's inputs go in on the H2D stream while set
// k-1 evaluates and set k-2's CSR values come back on the D2H stream (two device workspaces,
// PCIe is full duplex).  Same results as n_sets calls of sgb_run_outputs_host.
int sgb_run_outputs_host_many(sgb_plan *p, int64_t n_sets, const double *inputs, int64_t in_stride,
                              double *outputs, int64_t out_stride) {
  if (!p) return fail(-1, "sgb_run_outputs_host_many: null plan");
  if (n_sets < 0 || in_stride < 0 || (n_sets > 1 && out_stride < p->n_out))
    return fail(-1, "sgb_run_outputs_host_many: bad set count or stride");
  if (n_sets == 0 || !p->n_out) return 0;
  if ((!inputs && p->n_in) || !outputs) return fail(-1, "sgb_run_outputs_host_many: null buffer");
  std::lock_guard<std::mutex> lk(p->ws_mu);
  int rc = ensure_ws(p);
  if (rc) return rc;
  if (!p->h2d_stream) SGB_CUDA(cudaStreamCreateWithFlags(&p->h2d_stream, cudaStreamNonBlocking));
  if (!p->d2h_stream) SGB_CUDA(cudaStreamCreateWithFlags(&p->d2h_stream, cudaStreamNonBlocking));
  if (n_sets > 1 && !p->d_x2 && p->vas) {
    SGB_CUDA(cudaMalloc((void **)&p->d_x2, sizeof(double) * (size_t)p->vas_slots));
    // zeroed on the evaluation stream, so ordered before set 1 evaluates (codegen.py:419); only
    // [n_in, vas): set 1's inputs land in [0, n_in) on the H2D stream, unordered with this memset
    if (p->vas > p->n_in)
      SGB_CUDA(cudaMemsetAsync(p->d_x2 + p->n_in, 0, sizeof(double) * (size_t)(p->vas - p->n_in), p->ws_stream));
  }
  if (n_sets > 1 && !p->d_out2) SGB_CUDA(cudaMalloc((void **)&p->d_out2, sizeof(double) * (size_t)p->n_out));
  double *xs[2] = {p->d_x, p->d_x2}, *os[2] = {p->d_out, p->d_out2};
  cudaEvent_t ev_in[2], ev_run[2], ev_outd[2];
  for (int j = 0; j < 2; ++j) {
    SGB_CUDA(cudaEventCreateWithFlags(&ev_in[j], cudaEventDisableTiming));
    SGB_CUDA(cudaEventCreateWithFlags(&ev_run[j], cudaEventDisableTiming));
    SGB_CUDA(cudaEventCreateWithFlags(&ev_outd[j], cudaEventDisableTiming));
  }
  for (int64_t k = 0; k < n_sets && !rc; ++k) {
    const int j = (int)(k & 1);
    double *x = xs[j], *o = os[j];
    if (k >= 2) SGB_CUDA(cudaStreamWaitEvent(p->h2d_stream, ev_run[j], 0));  // set k-2 done reading x
    if (p->n_in)
      SGB_CUDA(cudaMemcpyAsync(x, inputs + k * in_stride, sizeof(double) * (size_t)p->n_in, cudaMemcpyHostToDevice,
                               p->h2d_stream));
    SGB_CUDA(cudaEventRecord(ev_in[j], p->h2d_stream));
    SGB_CUDA(cudaStreamWaitEvent(p->ws_stream, ev_in[j], 0));
    if (k >= 2) SGB_CUDA(cudaStreamWaitEvent(p->ws_stream, ev_outd[j], 0));  // set k-2's values are out
    const bool dirty = j == 0 && p->ws_dirty;
    if ((p->needs_zero == 2 || (p->needs_zero == 1 && dirty)) && p->vas > p->n_in)
      SGB_CUDA(cudaMemsetAsync(x + p->n_in, 0, sizeof(double) * (size_t)(p->vas - p->n_in), p->ws_stream));
    if (j == 0) p->ws_dirty = false;
    rc = sgb_run_csr(p, x, o, p->ws_stream);
    SGB_CUDA(cudaEventRecord(ev_run[j], p->ws_stream));
    SGB_CUDA(cudaStreamWaitEvent(p->d2h_stream, ev_run[j], 0));
    SGB_CUDA(cudaMemcpyAsync(outputs + k * out_stride, o, sizeof(double) * (size_t)p->n_out, cudaMemcpyDeviceToHost,
                             p->d2h_stream));
    SGB_CUDA(cudaEventRecord(ev_outd[j], p->d2h_stream));
  }
  SGB_CUDA(cudaStreamSynchronize(p->h2d_stream));
  SGB_CUDA(cudaStreamSynchronize(p->ws_stream));
  SGB_CUDA(cudaStreamSynchronize(p->d2h_stream));
  for (int j = 0; j < 2; ++j) {
    cudaEventDestroy(ev_in[j]);
    cudaEventDestroy(ev_run[j]);
    cudaEventDestroy(ev_outd[j]);
  }
  return rc;
}


// Replace the (single-set) tile table: same length, each unit's range [t0, t1) a permutation of
// its own tiles (a different schedule of the same work).  Stream-ordered after prior work on the
// legacy stream; synchronous.
int sgb_plan_set_tiles(sgb_plan *p, const int32_t *tiles, int64_t n_tiles) {
  if (!p || (!tiles && n_tiles)) return fail(-1, "sgb_plan_set_tiles: null argument");
  if (n_tiles != p->n_tiles) return fail(-1, "sgb_plan_set_tiles: tile count differs from the plan's");
  const int2 *nt = reinterpret_cast<const int2 *>(tiles);
  for (const Unit &u : p->units) {  // each unit's range: the same multiset of its own tiles, reordered
    if (u.flags & UNIT_WINDOW) continue;
    for (int64_t t = u.t0; t < u.t1; ++t)
      if (nt[t].x < u.g0 || nt[t].x >= u.g1 || nt[t].y < 0 || (int64_t)nt[t].y >= p->group_n[nt[t].x])
        return fail(-1, "sgb_plan_set_tiles: tile " + std::to_string(t) + " outside its unit's groups");
    auto key = [](const int2 &a, const int2 &b) { return a.x != b.x ? a.x < b.x : a.y < b.y; };
    std::vector<int2> a(p->h_tiles.begin() + u.t0, p->h_tiles.begin() + u.t1), b(nt + u.t0, nt + u.t1);
    std::sort(a.begin(), a.end(), key);
    std::sort(b.begin(), b.end(), key);
    for (size_t k = 0; k < a.size(); ++k)
      if (a[k].x != b[k].x || a[k].y != b[k].y)
        return fail(-1, "sgb_plan_set_tiles: unit " + std::to_string(u.index) + " range is not a permutation of its tiles");
  }
  std::lock_guard<std::mutex> lk(p->run_mu);
  SGB_CUDA(cudaSetDevice(p->device));
  SGB_CUDA(cudaDeviceSynchronize());
  if (n_tiles) SGB_CUDA(cudaMemcpy(p->d_tiles, tiles, sizeof(int2) * (size_t)n_tiles, cudaMemcpyHostToDevice));
  p->h_tiles.assign(nt, nt + n_tiles);
  return 0;
}


// Grid of the specialised units of one wave: persistent (tiles = 0) or one block per tile
// (tiles = 1).  Returns the number of units switched (0 when the wave has none).  Synchronous.
int sgb_plan_set_wave_grid(sgb_plan *p, int wave, int tiles) {
  if (!p) return fail(-1, "sgb_plan_set_wave_grid: null plan");
  std::lock_guard<std::mutex> lk(p->run_mu);
  SGB_CUDA(cudaSetDevice(p->device));
  SGB_CUDA(cudaDeviceSynchronize());
  int n = 0;
  for (Unit &u : p->units)
    if (u.wave == wave && u.grid_p > 0 && u.grid_t > 0) {
      u.grid = tiles ? u.grid_t : u.grid_p;
      ++n;
    }
  return n;
}

}  // extern "C"
