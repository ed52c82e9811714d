/*
 * sgb.h -- C ABI of the B200 plan-evaluation backend (libsgb.so).
 *
 * Drop-in boundary for the reference's native evaluator.  The reference
 * binds ONE entry point through ctypes, per compiled plan:
 *
 *     void sg_run(double* x, const double* c, const unsigned* p);
 *         /root/reference/pkg/src/sparsegen/emit.py:190 (emitted),
 *         argtypes emit.py:225-231, called by run() emit.py:237-241
 *
 * where x is the full value array (inputs pre-placed at [0, input_count),
 * the rest zero), c the plan's constants and p its u32 positions.  A plan is
 * baked into the reference .so at compile time (compile_plan, emit.py:198-245);
 * here a plan is uploaded once (sgb_plan_create) and the handle replaces the
 * baked-in code:
 *
 *     sgb_sg_run(plan, x, c, p)        == sg_run(x, c, p), host buffers
 *     sgb_run_values(plan, x_dev, s)   == sg_run on a device-resident x
 *     sgb_gather_outputs(plan, ...)    == x[plan.outputs] (codegen.py:445)
 *     sgb_run_csr(plan, x, out, s)     == sg_run + x[plan.outputs] in one pass
 *     sgb_run_outputs_host(plan, ...)  == run(inputs)[plan.outputs], host in/out
 *     sgb_run_batch(plan, X_dev, ...)  == B independent sg_run calls, batch-fastest X
 *
 * Conventions: every call returns 0 on success and a negative code on
 * failure (no exceptions cross the ABI); sgb_last_error() describes the last
 * failure of the calling thread.  A plan's tables and kernels are fixed at
 * create; only its launch configuration changes afterwards (sgb_plan_set_tiles,
 * sgb_plan_set_wave_grid: same tiles, other order / grid, same results).  Calls
 * on one plan serialise their launch sequences (the wave fork/join streams are
 * per plan); distinct x buffers may be in flight at once.  Device calls are
 * stream-ordered with no host synchronisation inside.  `stream` is a cudaStream_t (NULL =
 * legacy default stream).  Only sm_100a (B200) is supported; there is no CPU
 * fallback.
 */
#ifndef SGB_H
#define SGB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sgb_plan sgb_plan;

/* One kernel group of the device plan (== lower.GROUP_DTYPE, 128 bytes).
 * Mirrors one reference KernelPlan (codegen.py:56-85). */
typedef struct sgb_group {
  int64_t n;         /* instances (KernelPlan.instances) */
  int64_t dest_base; /* result r of instance i at dest_base + r*n + i (codegen.py:265); with flags & 2048
                        (CSR layout, specialised units only) at dest_base + i*n_roots + r -- plan addresses
                        are re-mapped to match, and value-mode calls on such a plan return -2 */
  int64_t p_off;     /* KernelPlan.p_base (synthetic copy groups: past the plan's table) */
  int64_t c_off;     /* KernelPlan.c_base */
  int64_t tape_off;  /* first tape row */
  int64_t cb_off;    /* compressed columns (flags & 32): first chunk base in cbase */
  int64_t co_off;    /*                                  first offset in coff */
  int64_t a0_base;   /* affine column 0 (flags & 64): index = a0_base + a0_stride * i */
  int64_t a0_stride;
  int64_t ob_off;    /* output positions (flags & 128): first chunk base in obase */
  int64_t oo_off;    /*   first offset in ooff (flags & 128) or entry in opos32 (flags & 256) */
  int32_t n_roots, n_slots, n_ret, n_const;
  int32_t tape_len, n_regs, kind, flags; /* flags: lower.FLAG_* (8192: the specialised kernel stores with an
                                             L2 evict_last hint -- code generation only) */
  int32_t slot_off, sop_off, sop_len, unit;
  int32_t variant; /* sum-of-products width class (factors <= 2, 4, 8, 16, 32) */
  int32_t shape;   /* sum-of-products shape: 0 generic, 1 plain sum, 2 two-factor products (+ single tail) */
} sgb_group;

/* Host-side device plan handed to sgb_plan_create (all pointers host memory,
 * copied during the call). */
typedef struct sgb_plan_desc {
  int64_t value_array_size; /* ExecutionPlan.value_array_size */
  int64_t input_count;      /* ExecutionPlan.input_count */
  int32_t n_groups;
  int32_t n_waves;          /* value-mode waves; a CSR-only unit may use wave n_waves */
  int32_t n_units;
  int32_t needs_zero;       /* 0: no load reads an unwritten slot; 1: some read slots nothing writes
                               (zero the buffer once); 2: some read slots a later wave writes
                               (re-zero before every evaluation, codegen.py:419, 434-443) */
  const sgb_group *groups;  /* ordered by (wave, launch unit) */
  const int64_t *units;     /* [n_units][10]: wave, kind (0 tape, 1 sum-of-products), variant (tape VEC),
                               group_begin, group_end, tile_begin, tile_end, block_size,
                               scratch registers per lane, flags (1 = CSR mode only,
                               2 = specialised unit in jit_cubin, 4 = value mode only,
                               8 = CSR windows: tile range = window range) */
  const int32_t *tiles;     /* [n_tiles][2]: group, first instance -- one block each, in launch order */
  int64_t n_tiles;
  const uint32_t *tape;     /* [tape_rows][4] device tape words, see lower.assemble() */
  int64_t tape_rows;
  const double *imm;
  int64_t n_imm;
  const uint32_t *sop;      /* per sum-of-products group: newterm mask, negate mask */
  int64_t n_sop;
  const int32_t *slot_col;   /* per slot: retained column or -1 (coherent) */
  const int64_t *slot_delta; /* per slot: coherence delta from slot 0 */
  int64_t n_slot;
  const uint32_t *positions; /* ExecutionPlan.positions (u32, unchanged) + copy-group columns */
  int64_t n_positions;
  const double *constants; /* ExecutionPlan.constants (f64, unchanged) */
  int64_t n_constants;
  const uint32_t *cbase; /* compressed index columns: base per (column, 32 instances) */
  int64_t n_cbase;
  const uint16_t *coff; /* compressed index columns: offset per (column, instance) */
  int64_t n_coff;
  const uint32_t *obase; /* output positions: base per (root, 32 instances) */
  int64_t n_obase;
  const uint16_t *ooff; /* output positions: offset per (root, instance), 0xFFFF = not an output */
  int64_t n_ooff;
  const uint32_t *opos32; /* output positions, wide form, 0xFFFFFFFF = not an output */
  int64_t n_opos32;
  const int64_t *outputs; /* ExecutionPlan.outputs */
  int64_t n_outputs;
  const void *jit_cubin;  /* sm_100a cubin with the specialised units (units flag 2): kernels
                             sgb_tape_u<unit> / sgb_tape_b<unit> / sgb_window_u<unit> (jit.py) */
  int64_t jit_cubin_size;
  /* CSR windows (units flag 8, at most one such unit, lower._csr_windows): window w assembles the
     outputs [win_k[w], win_k[w+1]) in shared memory; member j (= group group_begin + j of the unit,
     flags 4096: root r of instance i goes to window position ooff[oo_off + r*n + i], 0xFFFF none)
     contributes instances [first, first + count) = win_pieces[w*J + j]; the outputs no member
     produces are copied from the value array: copy_src[c] -> window position copy_pos[c] for
     c in [win_copy[w], win_copy[w+1]). */
  const int32_t *win_pieces; /* [n_windows * J][2]: first instance, instance count */
  int64_t n_win_pieces;      /* n_windows * J pairs */
  const int64_t *win_k;      /* [n_windows + 1]: window start positions, win_k[n_windows] = n_outputs */
  int64_t n_win_k;
  const int64_t *win_copy;   /* [n_windows + 1]: first copy of each window */
  int64_t n_win_copy;
  const uint32_t *copy_src;  /* [n_copy] value-array address of each copied output */
  const uint16_t *copy_pos;  /* [n_copy] its position in its window */
  int64_t n_copy;
  /* Bulk feed of the CSR-window unit (units flag 16 on the window unit, lower.WindowBulk): a
     persistent block of block_size threads (consumers + one producer warp) walks windows
     blockIdx.x, blockIdx.x + gridDim.x, ...; per window its producer thread copies the consumer
     blob win_meta[win_meta_off[w] .. win_meta_off[w+1]) and the value-array intervals
     win_iv[win_iv_off[w] .. win_iv_off[w+1]) (first element, element count; both even) with
     cp.async.bulk into a ring slot of win_slot_meta + win_slot_x bytes (win_ring slots after a
     win_bw-byte window buffer); win_bulk[j] = 1 marks the members fed from the ring.  A plan with
     such a unit reads value-array slot value_array_size (padding) when that size is odd: see
     sgb_plan_value_slots. */
  const uint8_t *win_meta;
  int64_t n_win_meta;
  const int64_t *win_meta_off; /* [n_windows + 1] when n_win_meta > 0 */
  const uint32_t *win_iv;      /* [n_win_iv][2] */
  int64_t n_win_iv;
  const int64_t *win_iv_off;   /* [n_windows + 1] */
  const int32_t *win_bulk;     /* [J] */
  int64_t win_ring, win_slot_meta, win_slot_x, win_bw;
} sgb_plan_desc;

/* Upload a device plan to `device`.  Replaces compile_plan (emit.py:198-245). */
int sgb_plan_create(const sgb_plan_desc *desc, int device, sgb_plan **out);
void sgb_plan_destroy(sgb_plan *plan);

/* sg_run semantics on device memory: x_dev[value_array_size], inputs placed,
 * everything else zero.  All dependency waves are launched on `stream`. */
int sgb_run_values(sgb_plan *plan, double *x_dev, void *stream);

/* inputs -> CSR values: out_dev[k] == x[outputs[k]] after sg_run (codegen.py:445).
 * x_dev holds the inputs and serves as scratch for intermediates; it must be
 * 16-byte aligned and readable for sgb_plan_value_slots(plan) doubles.  With CSR
 * windows (the default lowering when the last wave qualifies) the last wave
 * assembles the CSR array window by window in shared memory and writes it
 * coalesced -- no separate gather; otherwise the value waves run and one
 * u32-indexed gather copies the outputs. */
int sgb_run_csr(sgb_plan *plan, double *x_dev, double *out_dev, void *stream);

/* inputs -> CSR values on device buffers: inputs_dev[input_count] -> out_dev[n_outputs] (SURVEY.md
 * §8(b)), through the plan's own value-array workspace; stream-ordered, no host synchronisation.
 * Calls sharing a plan serialise on that workspace (one evaluation in flight per plan). */
int sgb_run_inputs_csr(sgb_plan *plan, const double *inputs_dev, double *out_dev, void *stream);

/* One dependency wave (waves in order 0..sgb_plan_waves(plan, csr)-1); out_dev
 * NULL = value mode (sgb_run_values), else CSR mode (sgb_run_csr).  For
 * per-launch timing and profiling. */
int sgb_run_wave(sgb_plan *plan, double *x_dev, double *out_dev, int wave, void *stream);

/* Swap in another schedule of the same tiles (int32 pairs group, first
 * instance; n_tiles equal to the plan's, every unit's range a permutation of
 * its own tiles).  Results are unchanged; used by the runtime's per-wave
 * schedule autotuning.  Synchronous. */
int sgb_plan_set_tiles(sgb_plan *plan, const int32_t *tiles, int64_t n_tiles);

/* Launch grid of the specialised units of one wave: tiles = 0 a persistent
 * grid sized to the resident capacity (blocks stride over the tiles), 1 one
 * block per tile (dispatched in tile order).  Returns how many units were
 * switched (>= 0) or a negative error code.  Synchronous. */
int sgb_plan_set_wave_grid(sgb_plan *plan, int wave, int tiles);

/* out_dev[k] = x_dev[outputs[k]]  (codegen.py:445). */
int sgb_gather_outputs(sgb_plan *plan, const double *x_dev, double *out_dev, void *stream);

/* The reference ABI with host buffers: copies x in, runs, copies x back.
 * c / p must be the plan's own tables (they were uploaded at create time and
 * may be NULL). */
int sgb_sg_run(sgb_plan *plan, double *x_host, const double *c_host, const unsigned *p_host);

/* Host inputs[input_count] -> host outputs[n_outputs] through sgb_run_csr;
 * only those bytes cross PCIe.  Synchronous. */
int sgb_run_outputs_host(sgb_plan *plan, const double *inputs_host, double *outputs_host);

/* n_sets independent value sets through host buffers, pipelined: set k's
 * inputs (inputs_host + k * in_stride, in_stride >= 0, 0 = the same inputs
 * every set) copy in while set k-1 evaluates and set k-2's CSR values
 * (outputs_host + k * out_stride) copy out.  Equals n_sets calls of
 * sgb_run_outputs_host (emit.py:237-241 per set); use pinned host memory for
 * the copies to overlap.  Synchronous. */
int sgb_run_outputs_host_many(sgb_plan *plan, int64_t n_sets, const double *inputs_host, int64_t in_stride,
                              double *outputs_host, int64_t out_stride);

/* Batched evaluation: X_dev[addr * ld + b] for b < batch (ld >= batch),
 * inputs placed, results written in place.  Independent value sets share one
 * pass over the index tables. */
int sgb_run_batch(sgb_plan *plan, double *X_dev, int64_t ld, int64_t batch, void *stream);

/* Batched CSR mode: out_dev[k * ld_out + b] == X[outputs[k] * ld + b] after sgb_run_batch. */
int sgb_run_batch_csr(sgb_plan *plan, double *X_dev, int64_t ld, int64_t batch, double *out_dev, int64_t ld_out,
                      void *stream);

/* Outputs of a batched evaluation: out_dev[k * ld_out + b] = X_dev[outputs[k] * ld + b]. */
int sgb_gather_outputs_batch(sgb_plan *plan, const double *X_dev, int64_t ld, int64_t batch,
                             double *out_dev, int64_t ld_out, void *stream);

/* Dependency waves of the plan in value mode (csr = 0) or CSR mode (csr = 1). */
int sgb_plan_waves(const sgb_plan *plan, int csr);

/* Kernel launches one evaluation issues in value / CSR mode. */
int sgb_plan_units(const sgb_plan *plan, int csr);

/* Doubles a CSR-mode value-array workspace must span: value_array_size, rounded up to even
 * when the plan has a bulk-fed CSR-window unit (its 16-byte bulk copies may read the padding
 * slot; its value is never used). */
int64_t sgb_plan_value_slots(const sgb_plan *plan);

const char *sgb_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* SGB_H */
