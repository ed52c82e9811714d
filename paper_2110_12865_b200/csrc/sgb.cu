// sgb.cu -- sm_100a plan-evaluation kernels and the C ABI of include/sgb.h.
//
// Executes the device plan built by paper_2110_12865_b200/lower.py from a
// reference ExecutionPlan (/root/reference/pkg/src/sparsegen/codegen.py:56-98).
// Semantics are those of the reference evaluators interpret_plan
// (codegen.py:404-512) and the emitted sg_run (emit.py:90-195):
//   * kernels run in dependency waves (one launch per wave, every group of the
//     wave inside that launch, a block -> group table);
//   * every instance evaluates its template's live nodes in stored order; n-ary
//     ADD / MUL fold left (codegen.py:472-481); SELECT is c < 0 (codegen.py:490);
//   * results land at dest_base + r*N + i (codegen.py:492-494);
//   * self-referencing groups re-load their slots before every root and
//     re-evaluate (codegen.py:505-510).
// Arithmetic is IEEE binary64 round-to-nearest through __dadd_rn / __dmul_rn /
// __ddiv_rn / __dsqrt_rn (never contracted; the file is also built with
// --fmad=false), so EXACT_OPS templates reproduce the CPU reference bit for bit.
// No tensor cores: the path is an irregular gather / elementwise graph.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "sgb.h"

namespace {

// op codes: lower.py T_*
enum : int {
  T_ADD = 2, T_SUB = 3, T_MUL = 4, T_DIV = 5, T_NEG = 6, T_SQRT = 7, T_SIN = 8, T_COS = 9,
  T_EXP = 10, T_LOG = 11, T_POW = 12, T_SEL = 13, T_IMM = 20, T_ST = 21
};
enum : int { KIND_TAPE = 0, KIND_SOP = 1 };
enum : int { FLAG_SELFREF = 1, FLAG_INTERLEAVED = 2, FLAG_SERIAL = 4 };
constexpr int SOP_MAX = 32;
constexpr int PRE = 8;           // loads kept in flight by the tape prologue
constexpr int BATCH_WARPS = 8;   // instances per block in batched mode

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
  const int4 *tape;
  const double *imm;
  const int32_t *sop;
  const int32_t *slot_col;
  const int64_t *slot_delta;
  const uint32_t *pos;
  const double *con;
};

// Largest g in [g0, g1) with begin[g] <= blk (block -> group table lookup).
__device__ __forceinline__ int find_group(const int64_t *begin, int g0, int g1, int64_t blk) {
  int lo = g0, hi = g1 - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(begin + mid) <= blk) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Index decode == slot_addresses (codegen.py:373-388): retained slot -> its
// column of the position table; coherent slot -> slot-0 entry + delta.
__device__ __forceinline__ int64_t slot_addr(const Tables &T, const sgb_group &G, int s,
                                             int64_t i, bool inter, uint32_t idx0) {
  const int col = __ldg(T.slot_col + G.slot_off + s);
  if (col < 0) return (int64_t)idx0 + __ldg(T.slot_delta + G.slot_off + s);
  if (col == 0) return idx0;
  const int64_t e = inter ? G.p_off + i * G.n_ret + col : G.p_off + (int64_t)col * G.n + i;
  return (int64_t)__ldg(T.pos + e);
}

__device__ __forceinline__ uint32_t slot0_index(const Tables &T, const sgb_group &G, int64_t i,
                                                bool inter) {
  if (G.n_slots == 0) return 0u;
  const int64_t e = inter ? G.p_off + i * G.n_ret : G.p_off + i;
  return __ldg(T.pos + e);
}

__device__ __forceinline__ double const_slot(const Tables &T, const sgb_group &G, int k,
                                             int64_t i, bool inter) {
  const int64_t e = inter ? G.c_off + i * G.n_const + k : G.c_off + (int64_t)k * G.n + i;
  return __ldg(T.con + e);
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

__device__ double powi(double x, int k) {
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

// Scratch register r of this lane lives at R[r * stride].
__device__ __forceinline__ void run_tape(const Tables &T, const sgb_group &G, double *R, int stride,
                                         double *x, int64_t ld, int64_t i, int64_t b, int phase,
                                         bool selfref) {
  const int4 *tp = T.tape + G.tape_off;
  for (int pc = 0; pc < G.tape_len; ++pc) {
    const int4 ins = __ldg(tp + pc);
    const int op = ins.x & 0xFFFF;
    const unsigned dst = (unsigned)ins.x >> 16;
    const unsigned a = ins.y & 0xFFFF;
    const unsigned bb = (unsigned)ins.y >> 16;
    double v;
    switch (op) {
      case T_ADD: v = __dadd_rn(R[a * stride], R[bb * stride]); break;
      case T_SUB: v = __dsub_rn(R[a * stride], R[bb * stride]); break;
      case T_MUL: v = __dmul_rn(R[a * stride], R[bb * stride]); break;
      case T_DIV: v = __ddiv_rn(R[a * stride], R[bb * stride]); break;
      case T_NEG: v = -R[a * stride]; break;
      case T_SQRT: v = __dsqrt_rn(R[a * stride]); break;
      case T_SIN: v = sin(R[a * stride]); break;
      case T_COS: v = cos(R[a * stride]); break;
      case T_EXP: v = exp(R[a * stride]); break;
      case T_LOG: v = log(R[a * stride]); break;
      case T_POW: v = powi(R[a * stride], ins.w); break;
      case T_SEL: v = (R[a * stride] < 0.0) ? R[bb * stride] : R[(unsigned)ins.z * stride]; break;
      case T_IMM: v = __ldg(T.imm + ins.w); break;
      default:  // T_ST
        if (!selfref || ins.w == phase)
          x[(G.dest_base + (int64_t)ins.w * G.n + i) * ld + b] = R[a * stride];
        continue;
    }
    R[dst * stride] = v;
  }
}

// Prologue: hoisted slot loads (emit.py:108-124), PRE loads in flight per lane.
__device__ __forceinline__ void load_slots(const Tables &T, const sgb_group &G, double *R,
                                           int stride, const double *x, int64_t ld, int64_t i,
                                           int64_t b, bool inter, bool coherent_read) {
  const uint32_t idx0 = slot0_index(T, G, i, inter);
  for (int s0 = 0; s0 < G.n_slots; s0 += PRE) {
    double v[PRE];
#pragma unroll
    for (int u = 0; u < PRE; ++u) {
      const int s = s0 + u;
      if (s < G.n_slots) {
        const int64_t a = slot_addr(T, G, s, i, inter, idx0) * ld + b;
        v[u] = coherent_read ? x[a] : __ldg(x + a);
      }
    }
#pragma unroll
    for (int u = 0; u < PRE; ++u)
      if (s0 + u < G.n_slots) R[(s0 + u) * stride] = v[u];
  }
  for (int k = 0; k < G.n_const; ++k) R[(G.n_slots + k) * stride] = const_slot(T, G, k, i, inter);
}

__device__ __forceinline__ void tape_instance(const Tables &T, const sgb_group &G, double *R,
                                              int stride, double *x, int64_t ld, int64_t i,
                                              int64_t b) {
  const bool inter = G.flags & FLAG_INTERLEAVED;
  const bool selfref = G.flags & FLAG_SELFREF;
  const int phases = selfref ? G.n_roots : 1;
  for (int ph = 0; ph < phases; ++ph) {
    load_slots(T, G, R, stride, x, ld, i, b, inter, selfref);
    run_tape(T, G, R, stride, x, ld, i, b, ph, selfref);
  }
}

// Sum of products of slot loads: acc = t0 + t1 + ..., t = f0 * f1 * ...
__device__ __forceinline__ double sop_eval(const Tables &T, const sgb_group &G, const double *x,
                                           int64_t ld, int64_t i, int64_t b) {
  const bool inter = G.flags & FLAG_INTERLEAVED;
  const uint32_t newterm = (uint32_t)__ldg(T.sop + G.sop_off);
  const uint32_t negm = (uint32_t)__ldg(T.sop + G.sop_off + 1);
  const int L = G.sop_len;
  const uint32_t idx0 = slot0_index(T, G, i, inter);
  double v[SOP_MAX];
#pragma unroll
  for (int f = 0; f < SOP_MAX; ++f)
    if (f < L) v[f] = __ldg(x + slot_addr(T, G, f, i, inter, idx0) * ld + b);
  double acc = 0.0, term = 0.0;
  bool have = false;
#pragma unroll
  for (int f = 0; f < SOP_MAX; ++f) {
    if (f < L) {
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

// One launch per wave, single value set.  blockDim = wave block size.
__global__ void wave_single(Tables T, const int64_t *blk_begin, int g0, int g1, double *x) {
  extern __shared__ double scratch[];
  const int64_t blk = blockIdx.x;
  const int g = find_group(blk_begin, g0, g1, blk);
  const sgb_group G = T.groups[g];
  const int tid = threadIdx.x;
  if (G.flags & FLAG_SERIAL) {  // members read other instances' results: instance order
    if (tid != 0) return;
    for (int64_t i = 0; i < G.n; ++i) tape_instance(T, G, scratch, 1, x, 1, i, 0);
    return;
  }
  const int64_t i = (blk - __ldg(blk_begin + g)) * blockDim.x + tid;
  if (i >= G.n) return;
  if (G.kind == KIND_SOP) {
    x[G.dest_base + i] = sop_eval(T, G, x, 1, i, 0);
  } else {
    tape_instance(T, G, scratch + tid, blockDim.x, x, 1, i, 0);
  }
}

// Batched: X[addr * ld + b].  A warp owns one instance and sweeps the batch,
// so index loads are warp-uniform and every gather is a contiguous row.
__global__ void wave_batch(Tables T, const int64_t *blk_begin, int g0, int g1, double *X,
                           int64_t ld, int64_t batch) {
  extern __shared__ double scratch[];
  const int64_t blk = blockIdx.x;
  const int g = find_group(blk_begin, g0, g1, blk);
  const sgb_group G = T.groups[g];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (G.flags & FLAG_SERIAL) {
    if (warp != 0) return;
    for (int64_t i = 0; i < G.n; ++i)
      for (int64_t b = lane; b < batch; b += 32)
        tape_instance(T, G, scratch + tid, blockDim.x, X, ld, i, b);
    return;
  }
  const int64_t i = (blk - __ldg(blk_begin + g)) * (blockDim.x >> 5) + warp;
  if (i >= G.n) return;
  for (int64_t b = lane; b < batch; b += 32) {
    if (G.kind == KIND_SOP) {
      X[(G.dest_base + i) * ld + b] = sop_eval(T, G, X, ld, i, b);
    } else {
      tape_instance(T, G, scratch + tid, blockDim.x, X, ld, i, b);
    }
  }
}

__global__ void gather_outputs(const double *__restrict__ x, const int64_t *__restrict__ outs,
                               int64_t n, double *__restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = __ldg(x + __ldg(outs + k));
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

}  // namespace

struct sgb_plan {
  int device = 0;
  int64_t vas = 0, n_in = 0, n_out = 0, n_pos = 0, n_con = 0;
  int n_groups = 0, n_waves = 0;
  std::vector<int32_t> wave_group_begin, wave_bs, wave_regs;
  std::vector<int64_t> wave_blocks, wave_bblocks;
  std::vector<int32_t> wave_bwarps;
  Tables T{};
  sgb_group *d_groups = nullptr;
  int64_t *d_blk = nullptr, *d_bblk = nullptr, *d_outputs = nullptr;
  int4 *d_tape = nullptr;
  double *d_imm = nullptr, *d_con = nullptr;
  int32_t *d_sop = nullptr, *d_scol = nullptr;
  int64_t *d_sdel = nullptr;
  uint32_t *d_pos = nullptr;
  // workspace for the host-buffer entry points
  std::mutex ws_mu;
  double *d_x = nullptr, *d_out = nullptr;
  cudaStream_t ws_stream = nullptr;
};

extern "C" {

const char *sgb_last_error(void) { return g_err.c_str(); }

int sgb_plan_launches(const sgb_plan *p) { return p ? p->n_waves : 0; }

void sgb_plan_destroy(sgb_plan *p) {
  if (!p) return;
  cudaSetDevice(p->device);
  void *bufs[] = {p->d_groups, p->d_blk, p->d_bblk, p->d_outputs, p->d_tape, p->d_imm, p->d_con,
                  p->d_sop, p->d_scol, p->d_sdel, p->d_pos, p->d_x, p->d_out};
  for (void *b : bufs)
    if (b) cudaFree(b);
  if (p->ws_stream) cudaStreamDestroy(p->ws_stream);
  delete p;
}

int sgb_plan_create(const sgb_plan_desc *d, int device, sgb_plan **out) {
  if (!d || !out) return fail(-1, "sgb_plan_create: null argument");
  *out = nullptr;
  int ndev = 0;
  SGB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(-1, "sgb_plan_create: bad device ordinal");
  SGB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  SGB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(-2, "sgb_plan_create: libsgb is built for sm_100a (B200) only");
  if (d->n_waves < 0 || d->n_groups < 0) return fail(-1, "sgb_plan_create: negative counts");
  sgb_plan *p = new sgb_plan();
  p->device = device;
  p->vas = d->value_array_size;
  p->n_in = d->input_count;
  p->n_out = d->n_outputs;
  p->n_pos = d->n_positions;
  p->n_con = d->n_constants;
  p->n_groups = d->n_groups;
  p->n_waves = d->n_waves;
  p->wave_group_begin.assign(d->wave_group_begin, d->wave_group_begin + d->n_waves + 1);
  p->wave_blocks.assign(d->wave_blocks, d->wave_blocks + d->n_waves);
  p->wave_bs.assign(d->wave_block_size, d->wave_block_size + d->n_waves);
  p->wave_regs.assign(d->wave_smem_regs, d->wave_smem_regs + d->n_waves);
  // host-side validation of the tables the kernels trust
  for (int g = 0; g < d->n_groups; ++g) {
    const sgb_group &G = d->groups[g];
    if (G.n < 0 || G.dest_base < d->input_count || G.dest_base + G.n_roots * G.n > d->value_array_size ||
        G.p_off + (int64_t)G.n_ret * G.n > d->n_positions ||
        G.c_off + (int64_t)G.n_const * G.n > d->n_constants || G.tape_off + G.tape_len > d->tape_rows ||
        G.slot_off + G.n_slots > d->n_slot || (G.kind == KIND_SOP && (G.sop_len > SOP_MAX || G.sop_off + 2 > d->n_sop))) {
      sgb_plan_destroy(p);
      return fail(-1, "sgb_plan_create: group " + std::to_string(g) + " is out of range");
    }
  }
  for (int64_t k = 0; k < d->n_outputs; ++k)
    if (d->outputs[k] < 0 || d->outputs[k] >= d->value_array_size) {
      sgb_plan_destroy(p);
      return fail(-1, "sgb_plan_create: output offset outside the value array");
    }
  // batched block table: one instance per warp, as many warps per block (<= BATCH_WARPS)
  // as the wave's scratch file allows in shared memory
  int smem_max = 0;
  SGB_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  std::vector<int64_t> bblk(d->n_groups, 0), blk(d->n_groups, 0);
  p->wave_bblocks.assign(d->n_waves, 0);
  p->wave_bwarps.assign(d->n_waves, BATCH_WARPS);
  for (int w = 0; w < d->n_waves; ++w) {
    int warps = BATCH_WARPS;
    while (warps > 1 && (int64_t)p->wave_regs[w] * 32 * warps * 8 > smem_max) warps >>= 1;
    p->wave_bwarps[w] = warps;
    int64_t acc = 0;
    for (int g = d->wave_group_begin[w]; g < d->wave_group_begin[w + 1]; ++g) {
      blk[g] = d->groups[g].blk_begin;
      bblk[g] = acc;
      acc += (d->groups[g].flags & FLAG_SERIAL) ? 1 : (d->groups[g].n + warps - 1) / warps;
    }
    p->wave_bblocks[w] = acc;
  }
  int rc = 0;
  if ((rc = upload(&p->d_groups, d->groups, d->n_groups)) || (rc = upload(&p->d_blk, blk.data(), (int64_t)blk.size())) ||
      (rc = upload(&p->d_bblk, bblk.data(), (int64_t)bblk.size())) ||
      (rc = upload(&p->d_outputs, d->outputs, d->n_outputs)) ||
      (rc = upload(&p->d_tape, (const int4 *)d->tape, d->tape_rows)) ||
      (rc = upload(&p->d_imm, d->imm, d->n_imm)) || (rc = upload(&p->d_sop, d->sop, d->n_sop)) ||
      (rc = upload(&p->d_scol, d->slot_col, d->n_slot)) || (rc = upload(&p->d_sdel, d->slot_delta, d->n_slot)) ||
      (rc = upload(&p->d_pos, d->positions, d->n_positions)) ||
      (rc = upload(&p->d_con, d->constants, d->n_constants))) {
    std::string msg = g_err;
    sgb_plan_destroy(p);
    return fail(rc, msg);
  }
  p->T = Tables{p->d_groups, p->d_tape, p->d_imm, p->d_sop, p->d_scol, p->d_sdel, p->d_pos, p->d_con};
  SGB_CUDA(cudaFuncSetAttribute(wave_single, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
  SGB_CUDA(cudaFuncSetAttribute(wave_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
  for (int w = 0; w < d->n_waves; ++w)
    if ((int64_t)p->wave_regs[w] * p->wave_bs[w] * 8 > smem_max ||
        (int64_t)p->wave_regs[w] * 32 * p->wave_bwarps[w] * 8 > smem_max) {
      sgb_plan_destroy(p);
      return fail(-1, "sgb_plan_create: wave scratch exceeds shared memory");
    }
  *out = p;
  return 0;
}

static void launch_wave(sgb_plan *p, double *x, int w, cudaStream_t s) {
  const int64_t blocks = p->wave_blocks[w];
  if (!blocks) return;
  const int bs = p->wave_bs[w];
  const size_t smem = (size_t)p->wave_regs[w] * bs * sizeof(double);
  wave_single<<<(unsigned)blocks, bs, smem, s>>>(p->T, p->d_blk, p->wave_group_begin[w],
                                                 p->wave_group_begin[w + 1], x);
}

int sgb_run_values(sgb_plan *p, double *x, void *stream) {
  if (!p || (!x && p->vas)) return fail(-1, "sgb_run_values: null argument");
  for (int w = 0; w < p->n_waves; ++w) launch_wave(p, x, w, (cudaStream_t)stream);
  SGB_CUDA(cudaGetLastError());
  return 0;
}

int sgb_run_wave(sgb_plan *p, double *x, int wave, void *stream) {
  if (!p || (!x && p->vas)) return fail(-1, "sgb_run_wave: null argument");
  if (wave < 0 || wave >= p->n_waves) return fail(-1, "sgb_run_wave: wave out of range");
  launch_wave(p, x, wave, (cudaStream_t)stream);
  SGB_CUDA(cudaGetLastError());
  return 0;
}

int sgb_run_batch(sgb_plan *p, double *X, int64_t ld, int64_t batch, void *stream) {
  if (!p || (!X && p->vas)) return fail(-1, "sgb_run_batch: null argument");
  if (batch < 1 || ld < batch) return fail(-1, "sgb_run_batch: need 1 <= batch <= ld");
  cudaStream_t s = (cudaStream_t)stream;
  for (int w = 0; w < p->n_waves; ++w) {
    const int64_t blocks = p->wave_bblocks[w];
    if (!blocks) continue;
    const int bs = 32 * p->wave_bwarps[w];
    const size_t smem = (size_t)p->wave_regs[w] * bs * sizeof(double);
    wave_batch<<<(unsigned)blocks, bs, smem, s>>>(p->T, p->d_bblk, p->wave_group_begin[w],
                                                  p->wave_group_begin[w + 1], X, ld, batch);
  }
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
  const int bs = 256;
  const int64_t blocks = (p->n_out + 7) / 8;
  gather_outputs_batch<<<(unsigned)blocks, bs, 0, (cudaStream_t)stream>>>(X, ld, batch, p->d_outputs,
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
