// sgb.cu -- sm_100a plan-evaluation kernels and the C ABI of include/sgb.h.
//
// Executes the device plan built by paper_2110_12865_b200/lower.py from a
// reference ExecutionPlan (/root/reference/pkg/src/sparsegen/codegen.py:56-98).
// Semantics are those of the reference evaluators interpret_plan
// (codegen.py:404-512) and the emitted sg_run (emit.py:90-195):
//   * kernels run in dependency waves; every group of a wave runs inside the
//     wave's launch units (a tape unit, one sum-of-products unit per width
//     class) through a block -> group table;
//   * every instance evaluates its template's live nodes in stored order; n-ary
//     ADD / MUL fold left (codegen.py:472-481); SELECT is c < 0 (codegen.py:490);
//   * results land at dest_base + r*N + i (codegen.py:492-494);
//   * self-referencing groups re-load their slots before every root and
//     re-evaluate (codegen.py:505-510).
// Arithmetic is IEEE binary64 round-to-nearest through __dadd_rn / __dmul_rn /
// __ddiv_rn / __dsqrt_rn (never contracted; the file is also built with
// --fmad=false), so EXACT_OPS templates reproduce the CPU reference bit for bit.
//
// The path is an irregular gather / elementwise graph (no tensor cores): the
// kernels are built for memory-level parallelism -- every index and value load
// of an instance is issued before the first use, streaming data (index tables,
// results nobody re-reads) carries an L2 evict-first policy so the gathered
// intermediates stay in the 126 MB L2, and the launch units keep register
// counts low enough for high occupancy.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "sgb.h"

namespace {

// tape op codes: lower.py T_*
enum : int {
  T_MUL = 0, T_ADD, T_SUB, T_DIV, T_MADD, T_NEG, T_SQRT, T_SEL, T_IMM, T_ST, T_SLOW, T_MSUB, T_RMSUB
};
enum : int { KIND_TAPE = 0, KIND_SOP = 1 };
enum : int {
  FLAG_SELFREF = 1, FLAG_INTERLEAVED = 2, FLAG_SERIAL = 4, FLAG_STREAM = 16, FLAG_W16 = 32, FLAG_AFFINE0 = 64
};
enum : int { U_WAVE = 0, U_KIND, U_VARIANT, U_G0, U_G1, U_BLOCKS, U_BS, U_REGS, U_COUNT };
constexpr int PRE = 8;  // slot loads kept in flight by the tape prologue
constexpr int MAX_BATCH_WARPS = 8;

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
  const int32_t *sop;
  const int32_t *slot_col;
  const int64_t *slot_delta;
  const uint32_t *pos;
  const double *con;
  const uint32_t *cbase;  // compressed columns: per (column, 32-instance chunk) base
  const uint16_t *coff;   //                     per (column, instance) offset
};

// ---- cache-policy helpers ---------------------------------------------------------
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// streaming index-table read: no L1 allocation, L2 evict-first
__device__ __forceinline__ uint32_t ld_index(const uint32_t *a, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_const(const double *a, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_result(double *a, double v, bool stream, uint64_t pol) {
  if (stream)
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
  else
    *a = v;
}

// Largest g in [g0, g1) with begin[g] <= blk (block -> group table lookup).
__device__ __forceinline__ int find_group(const int64_t *begin, int g0, int g1, int64_t blk) {
  int lo = g0, hi = g1 - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(begin + mid) <= blk) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Retained column `col` of instance i: the plan's u32 table, or the compressed
// form base[col][i/32] + off16[col][i] (lower.compress_columns).
__device__ __forceinline__ uint32_t column_index(const Tables &T, const sgb_group &G, int col, int64_t i,
                                                 bool inter, uint64_t pol) {
  if (col == 0 && (G.flags & FLAG_AFFINE0)) return (uint32_t)(G.a0_base + G.a0_stride * i);
  if (G.flags & FLAG_W16) {
    const int64_t nch = (G.n + 31) >> 5;
    const uint32_t base = __ldg(T.cbase + G.cb_off + (int64_t)col * nch + (i >> 5));
    uint16_t off;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;"
                 : "=h"(off) : "l"(T.coff + G.co_off + (int64_t)col * G.n + i), "l"(pol));
    return base + off;
  }
  const int64_t e = inter ? G.p_off + i * G.n_ret + col : G.p_off + (int64_t)col * G.n + i;
  return ld_index(T.pos + e, pol);
}

// Index decode == slot_addresses (codegen.py:373-388): retained slot -> its
// column of the position table; coherent slot -> slot-0 entry + delta.
__device__ __forceinline__ int64_t slot_addr(const Tables &T, const sgb_group &G, int s, int64_t i,
                                             bool inter, uint32_t idx0, uint64_t pol) {
  const int col = __ldg(T.slot_col + G.slot_off + s);
  if (col < 0) return (int64_t)idx0 + __ldg(T.slot_delta + G.slot_off + s);
  if (col == 0) return idx0;
  return (int64_t)column_index(T, G, col, i, inter, pol);
}

__device__ __forceinline__ uint32_t slot0_index(const Tables &T, const sgb_group &G, int64_t i,
                                                bool inter, uint64_t pol) {
  if (G.n_slots == 0) return 0u;
  return column_index(T, G, 0, i, inter, pol);
}

// ---- double-double integer power (POW k >= 3; k == 2 is an exact x*x) ----------
__device__ __forceinline__ void dd_mul(double ah, double al, double bh, double bl, double &rh,
                                       double &rl) {
  double p = __dmul_rn(ah, bh);
  double e = __fma_rn(ah, bh, -p);
  e = __dadd_rn(e, __dadd_rn(__dmul_rn(ah, bl), __dmul_rn(al, bh)));
  rh = __dadd_rn(p, e);
  rl = __dsub_rn(e, __dsub_rn(rh, p));
}

__device__ __noinline__ double powi(double x, int k) {
  if (k == 2) return __dmul_rn(x, x);  // glibc pow(x, 2.0) == x*x
  double rh = 1.0, rl = 0.0, bh = x, bl = 0.0;
  while (k) {
    if (k & 1) dd_mul(rh, rl, bh, bl, rh, rl);
    k >>= 1;
    if (k) dd_mul(bh, bl, bh, bl, bh, bl);
  }
  double r = __dadd_rn(rh, rl);
  return isfinite(r) ? r : rh;
}

// Rare ops live out of line so the interpreter loop stays small.
__device__ __noinline__ double slow_op(unsigned kind, double a, int k) {
  switch (kind) {
    case 0: return sin(a);
    case 1: return cos(a);
    case 2: return exp(a);
    case 3: return log(a);
    default: return powi(a, k);
  }
}

// ---- tape interpreter ---------------------------------------------------------------
// Device words (lower.assemble): x = op | nega<<6 | negb<<7 | (c byte offset / 8) << 8,
// y / z / w = byte offsets of dst / a / b in the lane's scratch column (w is the
// immediate index, root index or kind<<16|k for IMM / ST / SLOW).  Scratch is
// shared memory addressed with 32-bit shared addresses; instance v of a lane
// sits VS bytes after instance 0.
__device__ __forceinline__ double lds(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts(uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ double flip(double v, uint32_t bit) {  // exact negation when bit = 1
  return __longlong_as_double(__double_as_longlong(v) ^ ((unsigned long long)bit << 63));
}

template <int VEC, int VS>
__device__ __forceinline__ void run_tape(const Tables &T, const sgb_group &G, uint32_t Rb, double *x,
                                         int64_t ld, int64_t b, const int64_t (&iv)[VEC],
                                         const bool (&ok)[VEC], int phase, bool selfref, uint64_t pol) {
  const uint4 *tp = reinterpret_cast<const uint4 *>(T.tape) + G.tape_off;
  const bool stream = G.flags & FLAG_STREAM;
  const int len = G.tape_len;
  uint4 next = len > 0 ? __ldg(tp) : make_uint4(0, 0, 0, 0);
  for (int pc = 0; pc < len; ++pc) {
    const uint4 w = next;
    if (pc + 1 < len) next = __ldg(tp + pc + 1);  // prefetch the next word
    const uint32_t na = (w.x >> 6) & 1u, nb = (w.x >> 7) & 1u;
    const uint32_t cofs = (w.x >> 8) << 3;
    switch (w.x & 63u) {
      case T_MUL:
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          sts(Rb + w.y + v * VS, __dmul_rn(flip(lds(Rb + w.z + v * VS), na), flip(lds(Rb + w.w + v * VS), nb)));
        break;
      case T_ADD:
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          sts(Rb + w.y + v * VS, __dadd_rn(flip(lds(Rb + w.z + v * VS), na), flip(lds(Rb + w.w + v * VS), nb)));
        break;
      case T_SUB:
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          sts(Rb + w.y + v * VS, __dsub_rn(flip(lds(Rb + w.z + v * VS), na), flip(lds(Rb + w.w + v * VS), nb)));
        break;
      case T_MADD:
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const double p = __dmul_rn(flip(lds(Rb + w.z + v * VS), na), flip(lds(Rb + w.w + v * VS), nb));
          sts(Rb + w.y + v * VS, __dadd_rn(p, lds(Rb + cofs + v * VS)));
        }
        break;
      case T_MSUB:
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const double p = __dmul_rn(flip(lds(Rb + w.z + v * VS), na), flip(lds(Rb + w.w + v * VS), nb));
          sts(Rb + w.y + v * VS, __dsub_rn(p, lds(Rb + cofs + v * VS)));
        }
        break;
      case T_RMSUB:
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const double p = __dmul_rn(flip(lds(Rb + w.z + v * VS), na), flip(lds(Rb + w.w + v * VS), nb));
          sts(Rb + w.y + v * VS, __dsub_rn(lds(Rb + cofs + v * VS), p));
        }
        break;
      case T_DIV:
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          sts(Rb + w.y + v * VS, __ddiv_rn(flip(lds(Rb + w.z + v * VS), na), flip(lds(Rb + w.w + v * VS), nb)));
        break;
      case T_NEG:
#pragma unroll
        for (int v = 0; v < VEC; ++v) sts(Rb + w.y + v * VS, -lds(Rb + w.z + v * VS));
        break;
      case T_SQRT:
#pragma unroll
        for (int v = 0; v < VEC; ++v) sts(Rb + w.y + v * VS, __dsqrt_rn(lds(Rb + w.z + v * VS)));
        break;
      case T_SEL:
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          sts(Rb + w.y + v * VS,
              lds(Rb + w.z + v * VS) < 0.0 ? lds(Rb + w.w + v * VS) : lds(Rb + cofs + v * VS));
        break;
      case T_IMM: {
        const double imm = __ldg(T.imm + w.w);
#pragma unroll
        for (int v = 0; v < VEC; ++v) sts(Rb + w.y + v * VS, imm);
        break;
      }
      case T_ST:
        if (!selfref || (int)w.w == phase) {
#pragma unroll
          for (int v = 0; v < VEC; ++v)
            if (ok[v])
              st_result(x + (G.dest_base + (int64_t)w.w * G.n + iv[v]) * ld + b, lds(Rb + w.z + v * VS),
                        stream, pol);
        }
        break;
      default:  // T_SLOW
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          sts(Rb + w.y + v * VS, slow_op(w.w >> 16, lds(Rb + w.z + v * VS), (int)(w.w & 0xFFFFu)));
        break;
    }
  }
}

// Prologue: hoisted slot loads (emit.py:108-124), PRE loads in flight per lane;
// slot s of this lane's instance goes to byte offset s * stride8.
__device__ __forceinline__ void load_slots(const Tables &T, const sgb_group &G, uint32_t Rb, uint32_t stride8,
                                           const double *x, int64_t ld, int64_t i, int64_t b, bool inter,
                                           bool coherent_read, uint64_t pol) {
  const uint32_t idx0 = slot0_index(T, G, i, inter, pol);
  for (int s0 = 0; s0 < G.n_slots; s0 += PRE) {
    double v[PRE];
#pragma unroll
    for (int u = 0; u < PRE; ++u) {
      const int s = s0 + u;
      if (s < G.n_slots) {
        const int64_t a = slot_addr(T, G, s, i, inter, idx0, pol) * ld + b;
        v[u] = coherent_read ? x[a] : __ldg(x + a);
      }
    }
#pragma unroll
    for (int u = 0; u < PRE; ++u)
      if (s0 + u < G.n_slots) sts(Rb + (uint32_t)(s0 + u) * stride8, v[u]);
  }
  for (int k = 0; k < G.n_const; ++k) {
    const int64_t e = inter ? G.c_off + i * G.n_const + k : G.c_off + (int64_t)k * G.n + i;
    sts(Rb + (uint32_t)(G.n_slots + k) * stride8, ld_const(T.con + e, pol));
  }
}

// One instance, any group (self-referencing groups reload before every root).
__device__ __forceinline__ void tape_instance(const Tables &T, const sgb_group &G, uint32_t Rb, uint32_t stride8,
                                              double *x, int64_t ld, int64_t i, int64_t b, uint64_t pol) {
  const bool inter = G.flags & FLAG_INTERLEAVED;
  const bool selfref = G.flags & FLAG_SELFREF;
  const int phases = selfref ? G.n_roots : 1;
  const int64_t iv[1] = {i};
  const bool ok[1] = {true};
  for (int ph = 0; ph < phases; ++ph) {
    load_slots(T, G, Rb, stride8, x, ld, i, b, inter, selfref, pol);
    run_tape<1, 0>(T, G, Rb, x, ld, b, iv, ok, ph, selfref, pol);
  }
}

// Single value set: lane = instance, VEC instances per lane (i0 + v*BS) share each
// decoded tape word.  Scratch file [n_regs][VEC][BS] doubles in shared memory.
template <int BS, int VEC>
__global__ void __launch_bounds__(BS) tape_single(Tables T, const int64_t *blk_begin, int g0, int g1,
                                                  double *x) {
  extern __shared__ double scratch[];
  const int64_t blk = blockIdx.x;
  const int g = find_group(blk_begin, g0, g1, blk);
  const sgb_group G = T.groups[g];
  const uint64_t pol = evict_first_policy();
  const int tid = threadIdx.x;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(scratch);
  constexpr uint32_t stride8 = BS * VEC * 8;
  if (VEC == 1 && (G.flags & FLAG_SERIAL)) {  // members read other instances' results: instance order
    if (tid != 0) return;
    for (int64_t i = 0; i < G.n; ++i) tape_instance(T, G, base, stride8, x, 1, i, 0, pol);
    return;
  }
  const int64_t i0 = (blk - __ldg(blk_begin + g)) * (BS * VEC) + tid;
  if (i0 >= G.n) return;
  const uint32_t Rb = base + tid * 8;
  if (VEC == 1) {
    tape_instance(T, G, Rb, stride8, x, 1, i0, 0, pol);
    return;
  }
  int64_t iv[VEC];
  bool ok[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    iv[v] = i0 + (int64_t)v * BS;
    ok[v] = iv[v] < G.n;
    if (!ok[v]) iv[v] = G.n - 1;  // evaluate a valid instance, store nothing
  }
  const bool inter = G.flags & FLAG_INTERLEAVED;
#pragma unroll
  for (int v = 0; v < VEC; ++v) load_slots(T, G, Rb + v * BS * 8, stride8, x, 1, iv[v], 0, inter, false, pol);
  run_tape<VEC, BS * 8>(T, G, Rb, x, 1, 0, iv, ok, 0, false, pol);
}

// Batched: X[addr * ld + b].  A warp owns one instance and sweeps the batch, so
// index loads are warp-uniform and every gather is a contiguous row.  The block
// is the unit's scratch stride wide (BS = bs * VEC of the unit), VEC = 1.
__global__ void tape_batch(Tables T, const int64_t *blk_begin, int g0, int g1, double *X, int64_t ld,
                           int64_t batch) {
  extern __shared__ double scratch[];
  const int64_t blk = blockIdx.x;
  const int g = find_group(blk_begin, g0, g1, blk);
  const sgb_group G = T.groups[g];
  const uint64_t pol = evict_first_policy();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t Rb = (uint32_t)__cvta_generic_to_shared(scratch) + tid * 8;
  const uint32_t stride8 = blockDim.x * 8;
  if (G.flags & FLAG_SERIAL) {
    if (warp != 0) return;
    for (int64_t i = 0; i < G.n; ++i)
      for (int64_t b = lane; b < batch; b += 32) tape_instance(T, G, Rb, stride8, X, ld, i, b, pol);
    return;
  }
  const int64_t i = (blk - __ldg(blk_begin + g)) * (blockDim.x >> 5) + warp;
  if (i >= G.n) return;
  for (int64_t b = lane; b < batch; b += 32) tape_instance(T, G, Rb, stride8, X, ld, i, b, pol);
}

// ---- sum of products: acc = t0 + t1 + ..., t = f0 * f1 * ... (tape-free) --------------
template <int LMAX>
__device__ __forceinline__ void sop_addrs(const Tables &T, const sgb_group &G, int64_t i,
                                          int64_t (&addr)[LMAX], uint64_t pol) {
  const bool inter = G.flags & FLAG_INTERLEAVED;
  const uint32_t idx0 = slot0_index(T, G, i, inter, pol);
#pragma unroll
  for (int f = 0; f < LMAX; ++f)
    if (f < G.sop_len) addr[f] = slot_addr(T, G, f, i, inter, idx0, pol);
}

template <int LMAX>
__device__ __forceinline__ double sop_fold(const sgb_group &G, uint32_t newterm, uint32_t negm,
                                           const double (&v)[LMAX]) {
  double acc = 0.0, term = 0.0;
  bool have = false;
#pragma unroll
  for (int f = 0; f < LMAX; ++f) {
    if (f < G.sop_len) {
      const double val = ((negm >> f) & 1u) ? -v[f] : v[f];
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

// VEC instances per thread (i0 + v*256): VEC x LMAX independent gathers in flight.
template <int LMAX, int VEC>
__global__ void __launch_bounds__(256) sop_single(Tables T, const int64_t *blk_begin, int g0, int g1,
                                                  double *x) {
  const int64_t blk = blockIdx.x;
  const int g = find_group(blk_begin, g0, g1, blk);
  const sgb_group G = T.groups[g];
  const int64_t i0 = (blk - __ldg(blk_begin + g)) * (256 * VEC) + threadIdx.x;
  if (i0 >= G.n) return;
  const uint64_t pol = evict_first_policy();
  const uint32_t newterm = (uint32_t)__ldg(T.sop + G.sop_off);
  const uint32_t negm = (uint32_t)__ldg(T.sop + G.sop_off + 1);
  int64_t addr[VEC][LMAX];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    const int64_t i = min(i0 + (int64_t)v * 256, G.n - 1);
    sop_addrs<LMAX>(T, G, i, addr[v], pol);
  }
  double val[VEC][LMAX];
#pragma unroll
  for (int v = 0; v < VEC; ++v)
#pragma unroll
    for (int f = 0; f < LMAX; ++f)
      if (f < G.sop_len) val[v][f] = __ldg(x + addr[v][f]);
  const bool stream = G.flags & FLAG_STREAM;
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    const int64_t i = i0 + (int64_t)v * 256;
    if (i < G.n) st_result(x + G.dest_base + i, sop_fold<LMAX>(G, newterm, negm, val[v]), stream, pol);
  }
}

template <int LMAX>
__global__ void __launch_bounds__(256) sop_batch(Tables T, const int64_t *blk_begin, int g0, int g1,
                                                 double *X, int64_t ld, int64_t batch) {
  const int64_t blk = blockIdx.x;
  const int g = find_group(blk_begin, g0, g1, blk);
  const sgb_group G = T.groups[g];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = (blk - __ldg(blk_begin + g)) * (blockDim.x >> 5) + warp;
  if (i >= G.n) return;
  const uint64_t pol = evict_first_policy();
  const uint32_t newterm = (uint32_t)__ldg(T.sop + G.sop_off);
  const uint32_t negm = (uint32_t)__ldg(T.sop + G.sop_off + 1);
  int64_t addr[LMAX];
  sop_addrs<LMAX>(T, G, i, addr, pol);  // warp-uniform: one index fetch per warp
  const bool stream = G.flags & FLAG_STREAM;
  for (int64_t b = lane; b < batch; b += 32) {
    double v[LMAX];
#pragma unroll
    for (int f = 0; f < LMAX; ++f)
      if (f < G.sop_len) v[f] = __ldg(X + addr[f] * ld + b);
    st_result(X + (G.dest_base + i) * ld + b, sop_fold<LMAX>(G, newterm, negm, v), stream, pol);
  }
}

__global__ void gather_outputs(const double *__restrict__ x, const int64_t *__restrict__ outs,
                               int64_t n, double *__restrict__ out) {
  const uint64_t pol = evict_first_policy();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t a;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;"
                 : "=l"(a) : "l"(outs + k), "l"(pol));
    st_result(out + k, __ldg(x + a), true, pol);
  }
}

__global__ void gather_outputs_batch(const double *__restrict__ X, int64_t ld, int64_t batch,
                                     const int64_t *__restrict__ outs, int64_t n,
                                     double *__restrict__ out, int64_t ld_out) {
  const int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= n) return;
  const int64_t src = __ldg(outs + k) * ld;
  for (int64_t b = threadIdx.x & 31; b < batch; b += 32) out[k * ld_out + b] = __ldg(X + src + b);
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
  int wave, kind, variant, g0, g1, bs, regs;
  int64_t blocks;
  int bwarps;       // batched mode: instances (warps) per block
  int64_t bblocks;  // batched mode: blocks
};

}  // namespace

struct sgb_plan {
  int device = 0;
  int64_t vas = 0, n_in = 0, n_out = 0, n_pos = 0, n_con = 0;
  int n_groups = 0, n_waves = 0;
  std::vector<Unit> units;
  Tables T{};
  sgb_group *d_groups = nullptr;
  int64_t *d_blk = nullptr, *d_bblk = nullptr, *d_outputs = nullptr;
  uint32_t *d_tape = nullptr;
  double *d_imm = nullptr, *d_con = nullptr;
  int32_t *d_sop = nullptr, *d_scol = nullptr;
  int64_t *d_sdel = nullptr;
  uint32_t *d_pos = nullptr, *d_cbase = nullptr;
  uint16_t *d_coff = nullptr;
  // workspace for the host-buffer entry points
  std::mutex ws_mu;
  double *d_x = nullptr, *d_out = nullptr;
  cudaStream_t ws_stream = nullptr;
};

namespace {

template <int BS, int VEC>
void launch_tape(const sgb_plan *p, const Unit &u, double *x, cudaStream_t s) {
  const size_t smem = (size_t)u.regs * BS * VEC * sizeof(double);
  tape_single<BS, VEC><<<(unsigned)u.blocks, BS, smem, s>>>(p->T, p->d_blk, u.g0, u.g1, x);
}

template <int BS>
void launch_tape_vec(const sgb_plan *p, const Unit &u, double *x, cudaStream_t s) {
  if (u.variant <= 1) launch_tape<BS, 1>(p, u, x, s);
  else if (u.variant == 2) launch_tape<BS, 2>(p, u, x, s);
  else launch_tape<BS, 4>(p, u, x, s);
}

template <int LMAX>
void launch_sop(const sgb_plan *p, const Unit &u, double *x, int64_t ld, int64_t batch, bool batched,
                cudaStream_t s) {
  if (!batched)
    sop_single<LMAX, (LMAX <= 8 ? 2 : 1)><<<(unsigned)u.blocks, 256, 0, s>>>(p->T, p->d_blk, u.g0, u.g1, x);
  else
    sop_batch<LMAX><<<(unsigned)u.bblocks, 256, 0, s>>>(p->T, p->d_bblk, u.g0, u.g1, x, ld, batch);
}

void launch_unit(const sgb_plan *p, const Unit &u, double *x, int64_t ld, int64_t batch, bool batched,
                 cudaStream_t s) {
  if ((batched ? u.bblocks : u.blocks) == 0) return;
  if (u.kind == KIND_TAPE) {
    if (batched) {  // block = the unit's scratch stride, one instance per warp
      const int stride = u.bs * u.variant;
      const size_t smem = (size_t)u.regs * stride * sizeof(double);
      tape_batch<<<(unsigned)u.bblocks, stride, smem, s>>>(p->T, p->d_bblk, u.g0, u.g1, x, ld, batch);
      return;
    }
    switch (u.bs) {
      case 128: launch_tape_vec<128>(p, u, x, s); break;
      case 64: launch_tape_vec<64>(p, u, x, s); break;
      default: launch_tape_vec<32>(p, u, x, s); break;
    }
  } else {
    switch (u.variant) {
      case 4: launch_sop<4>(p, u, x, ld, batch, batched, s); break;
      case 8: launch_sop<8>(p, u, x, ld, batch, batched, s); break;
      case 16: launch_sop<16>(p, u, x, ld, batch, batched, s); break;
      default: launch_sop<32>(p, u, x, ld, batch, batched, s); break;
    }
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

}  // namespace

extern "C" {

const char *sgb_last_error(void) { return g_err.c_str(); }

int sgb_plan_launches(const sgb_plan *p) { return p ? p->n_waves : 0; }

int sgb_plan_units(const sgb_plan *p) { return p ? (int)p->units.size() : 0; }

void sgb_plan_destroy(sgb_plan *p) {
  if (!p) return;
  cudaSetDevice(p->device);
  void *bufs[] = {p->d_groups, p->d_blk, p->d_bblk, p->d_outputs, p->d_tape, p->d_imm, p->d_con,
                  p->d_sop, p->d_scol, p->d_sdel, p->d_pos, p->d_x, p->d_out, p->d_cbase, p->d_coff};
  for (void *b : bufs)
    if (b) cudaFree(b);
  if (p->ws_stream) cudaStreamDestroy(p->ws_stream);
  delete p;
}

static int create_impl(const sgb_plan_desc *d, int device, sgb_plan *p) {
  int ndev = 0;
  SGB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(-1, "sgb_plan_create: bad device ordinal");
  SGB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  SGB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(-2, "sgb_plan_create: libsgb is built for sm_100a (B200) only");
  if (d->n_waves < 0 || d->n_groups < 0 || d->n_units < 0) return fail(-1, "sgb_plan_create: negative counts");
  p->device = device;
  p->vas = d->value_array_size;
  p->n_in = d->input_count;
  p->n_out = d->n_outputs;
  p->n_pos = d->n_positions;
  p->n_con = d->n_constants;
  p->n_groups = d->n_groups;
  p->n_waves = d->n_waves;
  // host-side validation of every table entry the kernels trust
  for (int g = 0; g < d->n_groups; ++g) {
    const sgb_group &G = d->groups[g];
    const bool bad =
        G.n < 0 || G.dest_base < d->input_count || G.dest_base + G.n_roots * G.n > d->value_array_size ||
        G.p_off < 0 || G.p_off + (int64_t)G.n_ret * G.n > d->n_positions || G.c_off < 0 ||
        G.c_off + (int64_t)G.n_const * G.n > d->n_constants || G.tape_off < 0 ||
        G.tape_off + G.tape_len > d->tape_rows || G.slot_off < 0 || G.slot_off + G.n_slots > d->n_slot ||
        (G.n_slots > 0 && G.n_ret < 1) ||
        (G.kind == KIND_SOP && (G.sop_len > 32 || G.sop_len != G.n_slots || G.sop_off + 2 > d->n_sop)) ||
        ((G.flags & FLAG_W16) && (G.cb_off < 0 || G.co_off < 0 ||
                                  G.cb_off + (int64_t)G.n_ret * ((G.n + 31) / 32) > d->n_cbase ||
                                  G.co_off + (int64_t)G.n_ret * G.n > d->n_coff));
    if (bad) return fail(-1, "sgb_plan_create: group " + std::to_string(g) + " is out of range");
    for (int s = 0; s < G.n_slots; ++s)
      if (d->slot_col[G.slot_off + s] >= G.n_ret) return fail(-1, "sgb_plan_create: bad slot column");
  }
  for (int64_t k = 0; k < d->n_positions; ++k)
    if ((int64_t)d->positions[k] >= d->value_array_size)
      return fail(-1, "sgb_plan_create: position index outside the value array");
  for (int g = 0; g < d->n_groups; ++g) {  // compressed columns decode inside the value array
    const sgb_group &G = d->groups[g];
    if ((G.flags & FLAG_AFFINE0) && G.n > 0) {
      const int64_t first = G.a0_base, last = G.a0_base + G.a0_stride * (G.n - 1);
      if (first < 0 || last < 0 || first >= d->value_array_size || last >= d->value_array_size)
        return fail(-1, "sgb_plan_create: affine index column outside the value array");
    }
    if (!(G.flags & FLAG_W16)) continue;
    const int64_t nch = (G.n + 31) / 32;
    for (int c = (G.flags & FLAG_AFFINE0) ? 1 : 0; c < G.n_ret; ++c)
      for (int64_t i = 0; i < G.n; ++i)
        if ((int64_t)d->cbase[G.cb_off + c * nch + i / 32] + d->coff[G.co_off + c * G.n + i] >= d->value_array_size)
          return fail(-1, "sgb_plan_create: compressed index outside the value array");
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
  std::vector<int64_t> blk(d->n_groups, 0), bblk(d->n_groups, 0);
  for (int k = 0; k < d->n_units; ++k) {
    const int64_t *r = d->units + (int64_t)k * U_COUNT;
    Unit u;
    u.wave = (int)r[U_WAVE];
    u.kind = (int)r[U_KIND];
    u.variant = (int)r[U_VARIANT];
    u.g0 = (int)r[U_G0];
    u.g1 = (int)r[U_G1];
    u.blocks = r[U_BLOCKS];
    u.bs = (int)r[U_BS];
    u.regs = (int)r[U_REGS];
    if (u.g0 < 0 || u.g1 > d->n_groups || u.g0 > u.g1 || u.wave < 0 || u.wave >= d->n_waves ||
        (u.kind == KIND_TAPE && (u.bs != 32 && u.bs != 64 && u.bs != 128)) ||
        (u.kind == KIND_TAPE && (u.variant != 1 && u.variant != 2 && u.variant != 4)) ||
        (int64_t)u.regs * (u.kind == KIND_TAPE ? u.bs * u.variant : 0) * 8 > smem_max)
      return fail(-1, "sgb_plan_create: bad launch unit " + std::to_string(k));
    // batched: one instance per warp; tape blocks are the unit's scratch stride wide
    u.bwarps = u.kind == KIND_TAPE ? (u.bs * u.variant) / 32 : MAX_BATCH_WARPS;
    int64_t acc = 0;
    for (int g = u.g0; g < u.g1; ++g) {
      blk[g] = d->groups[g].blk_begin;
      bblk[g] = acc;
      acc += (d->groups[g].flags & FLAG_SERIAL) ? 1 : (d->groups[g].n + u.bwarps - 1) / u.bwarps;
    }
    u.bblocks = acc;
    if (u.kind == KIND_TAPE) {  // every tape word must stay inside its lane's scratch column
      const uint64_t limit = (uint64_t)u.regs * u.bs * u.variant * 8;
      for (int g = u.g0; g < u.g1; ++g) {
        const sgb_group &G = d->groups[g];
        if (G.n_slots + G.n_const > u.regs) return fail(-1, "sgb_plan_create: slots exceed the scratch file");
        for (int64_t k = G.tape_off; k < G.tape_off + G.tape_len; ++k) {
          const uint32_t *w = d->tape + 4 * k;
          const uint32_t op = w[0] & 63u;
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
  int rc = 0;
  if ((rc = upload(&p->d_groups, d->groups, d->n_groups)) ||
      (rc = upload(&p->d_blk, blk.data(), (int64_t)blk.size())) ||
      (rc = upload(&p->d_bblk, bblk.data(), (int64_t)bblk.size())) ||
      (rc = upload(&p->d_outputs, d->outputs, d->n_outputs)) ||
      (rc = upload(&p->d_tape, d->tape, d->tape_rows * 4)) || (rc = upload(&p->d_imm, d->imm, d->n_imm)) ||
      (rc = upload(&p->d_sop, d->sop, d->n_sop)) || (rc = upload(&p->d_scol, d->slot_col, d->n_slot)) ||
      (rc = upload(&p->d_sdel, d->slot_delta, d->n_slot)) ||
      (rc = upload(&p->d_pos, d->positions, d->n_positions)) ||
      (rc = upload(&p->d_con, d->constants, d->n_constants)) ||
      (rc = upload(&p->d_cbase, d->cbase, d->n_cbase)) || (rc = upload(&p->d_coff, d->coff, d->n_coff)))
    return rc;
  p->T = Tables{p->d_groups, p->d_tape, p->d_imm, p->d_sop, p->d_scol, p->d_sdel,
                p->d_pos, p->d_con, p->d_cbase, p->d_coff};
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

int sgb_run_wave(sgb_plan *p, double *x, int wave, void *stream) {
  if (!p || (!x && p->vas)) return fail(-1, "sgb_run_wave: null argument");
  if (wave < 0 || wave >= p->n_waves) return fail(-1, "sgb_run_wave: wave out of range");
  for (const Unit &u : p->units)
    if (u.wave == wave) launch_unit(p, u, x, 1, 1, false, (cudaStream_t)stream);
  SGB_CUDA(cudaGetLastError());
  return 0;
}

int sgb_run_values(sgb_plan *p, double *x, void *stream) {
  if (!p || (!x && p->vas)) return fail(-1, "sgb_run_values: null argument");
  for (const Unit &u : p->units) launch_unit(p, u, x, 1, 1, false, (cudaStream_t)stream);
  SGB_CUDA(cudaGetLastError());
  return 0;
}

int sgb_run_batch(sgb_plan *p, double *X, int64_t ld, int64_t batch, void *stream) {
  if (!p || (!X && p->vas)) return fail(-1, "sgb_run_batch: null argument");
  if (batch < 1 || ld < batch) return fail(-1, "sgb_run_batch: need 1 <= batch <= ld");
  for (const Unit &u : p->units) launch_unit(p, u, X, ld, batch, true, (cudaStream_t)stream);
  SGB_CUDA(cudaGetLastError());
  return 0;
}

int sgb_gather_outputs(sgb_plan *p, const double *x, double *out, void *stream) {
  if (!p) return fail(-1, "sgb_gather_outputs: null plan");
  if (!p->n_out) return 0;
  if (!x || !out) return fail(-1, "sgb_gather_outputs: null buffer");
  const int bs = 256;
  int64_t blocks = (p->n_out + bs - 1) / bs;
  if (blocks > 148 * 32) blocks = 148 * 32;
  gather_outputs<<<(unsigned)blocks, bs, 0, (cudaStream_t)stream>>>(x, p->d_outputs, p->n_out, out);
  SGB_CUDA(cudaGetLastError());
  return 0;
}

int sgb_gather_outputs_batch(sgb_plan *p, const double *X, int64_t ld, int64_t batch, double *out,
                             int64_t ld_out, void *stream) {
  if (!p) return fail(-1, "sgb_gather_outputs_batch: null plan");
  if (!p->n_out) return 0;
  if (!X || !out || batch < 1 || ld < batch || ld_out < batch)
    return fail(-1, "sgb_gather_outputs_batch: bad arguments");
  const int64_t blocks = (p->n_out + 7) / 8;
  gather_outputs_batch<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(X, ld, batch, p->d_outputs,
                                                                          p->n_out, out, ld_out);
  SGB_CUDA(cudaGetLastError());
  return 0;
}

static int ensure_ws(sgb_plan *p) {
  SGB_CUDA(cudaSetDevice(p->device));
  if (!p->ws_stream) SGB_CUDA(cudaStreamCreateWithFlags(&p->ws_stream, cudaStreamNonBlocking));
  if (!p->d_x && p->vas) SGB_CUDA(cudaMalloc((void **)&p->d_x, sizeof(double) * (size_t)p->vas));
  if (!p->d_out && p->n_out) SGB_CUDA(cudaMalloc((void **)&p->d_out, sizeof(double) * (size_t)p->n_out));
  return 0;
}

int sgb_sg_run(sgb_plan *p, double *x_host, const double *c_host, const unsigned *p_host) {
  (void)c_host;
  (void)p_host;
  if (!p || (!x_host && p->vas)) return fail(-1, "sgb_sg_run: null argument");
  std::lock_guard<std::mutex> lk(p->ws_mu);
  int rc = ensure_ws(p);
  if (rc) return rc;
  if (!p->vas) return 0;
  SGB_CUDA(cudaMemcpyAsync(p->d_x, x_host, sizeof(double) * (size_t)p->vas, cudaMemcpyHostToDevice, p->ws_stream));
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
  if (p->vas) {
    // padding and not-yet-written ranges read as zero (codegen.py:419)
    SGB_CUDA(cudaMemsetAsync(p->d_x + p->n_in, 0, sizeof(double) * (size_t)(p->vas - p->n_in), p->ws_stream));
    if (p->n_in)
      SGB_CUDA(cudaMemcpyAsync(p->d_x, inputs, sizeof(double) * (size_t)p->n_in, cudaMemcpyHostToDevice, p->ws_stream));
    if ((rc = sgb_run_values(p, p->d_x, p->ws_stream))) return rc;
  }
  if (p->n_out) {
    if ((rc = sgb_gather_outputs(p, p->d_x, p->d_out, p->ws_stream))) return rc;
    SGB_CUDA(cudaMemcpyAsync(outputs, p->d_out, sizeof(double) * (size_t)p->n_out, cudaMemcpyDeviceToHost, p->ws_stream));
  }
  SGB_CUDA(cudaStreamSynchronize(p->ws_stream));
  return 0;
}

}  // extern "C"
