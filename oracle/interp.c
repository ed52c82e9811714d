/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library,
 * and only as the checker or the timed CPU baseline, never as the product.
 *
 * Plain-C restatement of the reference CPU evaluator `interpret_plan`
 * (/root/reference/pkg/src/sparsegen/codegen.py:404-446) and its kernel body
 * `_run_kernel` / `_eval_scalar` (codegen.py:449-557):
 *
 *   x = zeros(value_array_size); x[:input_count] = inputs       (:419-420)
 *   for kp in plan.kernels (schedule order):                    (:428)
 *     addresses = slot_addresses(plan, kp)                       (:373-388)
 *     for every instance, every live template node ascending:    (:459-495)
 *       VAR -> x[addr] or constant column; CONST -> payload;
 *       ADD / MUL fold LEFT over the stored child order;         (:472-481)
 *       SUB, DIV, NEG, SQRT, SIN, COS, EXP, LOG, POW(k), SELECT(c<0) (:482-557)
 *     roots stored at dest_base + r*N + i                        (:492-494)
 *     self-referencing kernels re-load every slot before each root and
 *     re-evaluate from scratch                                   (:497-512)
 *
 * Compiled with -ffp-contract=off and without fast-math: every operation is
 * one IEEE-754 binary64 operation in round-to-nearest, so the result is bit
 * identical to the numpy lane path and to CPython floats.  SIN/COS/EXP/LOG/POW
 * call glibc libm exactly like CPython's math module (codegen.py:545-555).
 *
 * Flat plan encoding (built by oracle/oracle.py from any ExecutionPlan):
 *   kern[k*KF + ...]  int64 per-kernel fields (see KF_* below)
 *   slot_col[], slot_delta[]   per active position slot: retained column or -1,
 *                              coherence delta
 *   node_op[], node_a0[], node_na[], node_pay[]  live template nodes
 *     (node_a0/node_na index arg_list[]; node_pay = CONST value, or for VAR
 *      the slot: s >= 0 position slot, -(k+1) constant slot k)
 *   arg_list[]  child indices, kernel-local live-node numbering
 *   roots[]     kernel-local live-node index per root
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { VAR = 0, CONST, ADD, SUB, MUL, DIV, NEG, SQRT, SIN, COS, EXP, LOG, POW, SELECT };

enum {
  KF_N = 0, KF_NROOTS, KF_DEST, KF_SELFREF, KF_INTERLEAVED, KF_PBASE, KF_CBASE,
  KF_NRET, KF_NCONST, KF_SLOT0, KF_NSLOTS, KF_NODE0, KF_NNODES, KF_ROOT0, KF_COUNT
};

static double eval_nodes(int64_t nn, const int32_t *op, const int64_t *a0, const int32_t *na,
                         const double *pay, const int32_t *args, double *v,
                         const double *bind_x, const double *bind_c) {
  for (int64_t j = 0; j < nn; ++j) {
    const int32_t *a = args + a0[j];
    double r;
    switch (op[j]) {
      case VAR: {
        int64_t s = (int64_t)pay[j];
        r = s >= 0 ? bind_x[s] : bind_c[-s - 1];
        break;
      }
      case CONST: r = pay[j]; break;
      case ADD: r = v[a[0]]; for (int k = 1; k < na[j]; ++k) r = r + v[a[k]]; break;
      case MUL: r = v[a[0]]; for (int k = 1; k < na[j]; ++k) r = r * v[a[k]]; break;
      case SUB: r = v[a[0]] - v[a[1]]; break;
      case DIV: r = v[a[0]] / v[a[1]]; break;
      case NEG: r = -v[a[0]]; break;
      case SQRT: r = sqrt(v[a[0]]); break;
      case SIN: r = sin(v[a[0]]); break;
      case COS: r = cos(v[a[0]]); break;
      case EXP: r = exp(v[a[0]]); break;
      case LOG: r = log(v[a[0]]); break;
      case POW: r = pow(v[a[0]], v[a[1]]); break;
      default: r = (v[a[0]] < 0.0) ? v[a[1]] : v[a[2]]; break;
    }
    v[j] = r;
  }
  return 0.0;
}

/* Runs the whole plan in place on x (inputs pre-placed, rest zero). 0 = ok. */
int oracle_run(double *x, int64_t value_array_size, int64_t n_kernels, const int64_t *kern,
               const int32_t *slot_col, const int64_t *slot_delta, const int32_t *node_op,
               const int64_t *node_a0, const int32_t *node_na, const double *node_pay,
               const int32_t *arg_list, const int32_t *roots, const uint32_t *p,
               const double *c) {
  for (int64_t k = 0; k < n_kernels; ++k) {
    const int64_t *f = kern + k * KF_COUNT;
    const int64_t n = f[KF_N], nroots = f[KF_NROOTS], dest = f[KF_DEST];
    const int selfref = (int)f[KF_SELFREF], inter = (int)f[KF_INTERLEAVED];
    const int64_t pb = f[KF_PBASE], cb = f[KF_CBASE], nret = f[KF_NRET], ncon = f[KF_NCONST];
    const int32_t *scol = slot_col + f[KF_SLOT0];
    const int64_t *sdel = slot_delta + f[KF_SLOT0];
    const int64_t nslots = f[KF_NSLOTS], nn = f[KF_NNODES];
    const int32_t *op = node_op + f[KF_NODE0];
    const int64_t *a0 = node_a0 + f[KF_NODE0];
    const int32_t *na = node_na + f[KF_NODE0];
    const double *pay = node_pay + f[KF_NODE0];
    const int32_t *rt = roots + f[KF_ROOT0];
    double *v = (double *)malloc(sizeof(double) * (size_t)(nn > 0 ? nn : 1));
    double *bx = (double *)malloc(sizeof(double) * (size_t)(nslots > 0 ? nslots : 1));
    double *bc = (double *)malloc(sizeof(double) * (size_t)(ncon > 0 ? ncon : 1));
    int64_t *addr = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nslots > 0 ? nslots : 1));
    if (!v || !bx || !bc || !addr) return -1;
    for (int64_t i = 0; i < n; ++i) {
      /* slot_addresses (codegen.py:373-388) */
      for (int64_t s = 0; s < nslots; ++s) {
        int64_t col = scol[s] >= 0 ? scol[s] : 0;
        int64_t e = inter ? pb + i * nret + col : pb + col * n + i;
        int64_t a = (int64_t)p[e] + (scol[s] >= 0 ? 0 : sdel[s]);
        if (a < 0 || a >= value_array_size) return -2;
        addr[s] = a;
      }
      for (int64_t s = 0; s < ncon; ++s)
        bc[s] = inter ? c[cb + i * ncon + s] : c[cb + s * n + i];
      if (!selfref) {
        for (int64_t s = 0; s < nslots; ++s) bx[s] = x[addr[s]];
        eval_nodes(nn, op, a0, na, pay, arg_list, v, bx, bc);
        for (int64_t r = 0; r < nroots; ++r) x[dest + r * n + i] = v[rt[r]];
      } else {
        /* results stored so far are visible to later members (:505-510) */
        for (int64_t r = 0; r < nroots; ++r) {
          for (int64_t s = 0; s < nslots; ++s) bx[s] = x[addr[s]];
          eval_nodes(nn, op, a0, na, pay, arg_list, v, bx, bc);
          x[dest + r * n + i] = v[rt[r]];
        }
      }
    }
    free(v); free(bx); free(bc); free(addr);
  }
  return 0;
}
