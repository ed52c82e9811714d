"""ORACLE / CPU BASELINE -- TEST INFRASTRUCTURE ONLY (see oracle/README.md).

numpy restatement of the reference's interpreter ``interpret_plan`` /
``_run_kernel`` / ``_eval_scalar`` (/root/reference/pkg/src/sparsegen/
codegen.py:404-557), the reference's own single-core CPU evaluator.  bench.py
times it as the "interpreter" leg of ``cpu_baseline`` (SURVEY.md §8(d) CPU
reference item 2); the product never imports it.

Kernels run in plan order on a zero-initialised value array.  A template
whose live nodes are all exact ops (codegen.py:43-53) and that does not read
its own results runs lane-parallel: one numpy vector op per live node over the
kernel's N instances, n-ary ADD / MUL folded left in stored child order.  Any
other template (SIN / COS / EXP / LOG / POW, or self-referencing) runs the
scalar path: per instance, per node, Python floats and ``math`` (glibc); a
self-referencing kernel re-reads its slots before every root.  ``max_scalar``
bounds the scalar path for timing: only the first ``max_scalar`` instances of
such a kernel are evaluated and the run reports how many were skipped.
"""

from __future__ import annotations

import math

import numpy as np

# OpKind values of the reference (expr.py:55-70)
VAR, CONST, ADD, SUB, MUL, DIV, NEG, SQRT, SIN, COS, EXP, LOG, POW, SELECT = range(14)
EXACT = {VAR, CONST, ADD, SUB, MUL, DIV, NEG, SQRT, SELECT}


def _live(tmpl, roots):
    seen = set()
    stack = list(roots)
    while stack:
        i = stack.pop()
        if i in seen:
            continue
        seen.add(i)
        stack.extend(tmpl.args[i])
    return sorted(seen)


def _addr_columns(plan, kp):
    n, r = kp.instances, len(kp.retained)
    seg = np.asarray(plan.positions[kp.p_base: kp.p_base + r * n], dtype=np.int64)
    tab = seg.reshape(r, n) if kp.layout == "coalesced" else seg.reshape(n, r).T
    col_of = {s: k for k, s in enumerate(kp.retained)}
    return [tab[col_of[s]] if s in col_of else tab[0] + delta for s, delta in enumerate(kp.coherence)]


def _const_columns(plan, kp):
    n, c = kp.instances, len(kp.const_vars)
    seg = np.asarray(plan.constants[kp.c_base: kp.c_base + c * n], dtype=np.float64)
    return list(seg.reshape(c, n) if kp.layout == "coalesced" else seg.reshape(n, c).T)


def _lanes(kp, live, x, cols, consts):
    tmpl = kp.template_arena
    slot = {v: s for s, v in enumerate(kp.pos_vars)}
    cslot = {v: s for s, v in enumerate(kp.const_vars)}
    val: dict[int, np.ndarray] = {}
    for i in live:
        op, a = int(tmpl.ops[i]), tmpl.args[i]
        if op == VAR:
            p = tmpl.payload[i]
            val[i] = x[cols[slot[p]]] if p in slot else consts[cslot[p]]
        elif op == CONST:
            val[i] = np.full(kp.instances, tmpl.payload[i])
        elif op in (ADD, MUL):
            acc = val[a[0]].copy()
            for c in a[1:]:
                acc = acc + val[c] if op == ADD else acc * val[c]
            val[i] = acc
        elif op == SUB:
            val[i] = val[a[0]] - val[a[1]]
        elif op == DIV:
            val[i] = val[a[0]] / val[a[1]]
        elif op == NEG:
            val[i] = -val[a[0]]
        elif op == SQRT:
            val[i] = np.sqrt(val[a[0]])
        else:
            val[i] = np.where(val[a[0]] < 0.0, val[a[1]], val[a[2]])
    for r, root in enumerate(kp.template_roots):
        x[kp.dest_base + r * kp.instances: kp.dest_base + (r + 1) * kp.instances] = val[root]


_SCALAR = {SQRT: math.sqrt, SIN: math.sin, COS: math.cos, EXP: math.exp, LOG: math.log, NEG: lambda v: -v}


def _scalar(kp, live, x, cols, consts, count):
    tmpl = kp.template_arena
    slot = {v: s for s, v in enumerate(kp.pos_vars)}
    cslot = {v: s for s, v in enumerate(kp.const_vars)}
    n = kp.instances
    for inst in range(count):
        bind = {p: float(consts[s][inst]) for p, s in cslot.items()}
        val: dict[int, float] = {}
        for r, root in enumerate(kp.template_roots):
            if r == 0 or kp.self_referencing:  # stored roots are visible to later ones
                bind.update({p: float(x[cols[s][inst]]) for p, s in slot.items()})
                if kp.self_referencing:
                    val = {}
            for i in live:
                if i in val:
                    continue
                op, a = int(tmpl.ops[i]), tmpl.args[i]
                if op == VAR:
                    val[i] = bind[tmpl.payload[i]]
                elif op == CONST:
                    val[i] = float(tmpl.payload[i])
                elif op in (ADD, MUL):
                    acc = val[a[0]]
                    for c in a[1:]:
                        acc = acc + val[c] if op == ADD else acc * val[c]
                    val[i] = acc
                elif op == SUB:
                    val[i] = val[a[0]] - val[a[1]]
                elif op == DIV:
                    val[i] = val[a[0]] / val[a[1]]
                elif op == POW:
                    val[i] = math.pow(val[a[0]], val[a[1]])
                elif op == SELECT:
                    val[i] = val[a[1]] if val[a[0]] < 0.0 else val[a[2]]
                else:
                    val[i] = _SCALAR[op](val[a[0]])
            x[kp.dest_base + r * n + inst] = val[root]


def interpret(plan, inputs, max_scalar: int | None = None):
    """Value array after ``interpret_plan``; returns (x, scalar instances skipped)."""
    x = np.zeros(int(plan.value_array_size), np.float64)
    x[: plan.input_count] = np.asarray(inputs, dtype=np.float64)
    skipped = 0
    for kp in plan.kernels:
        live = _live(kp.template_arena, kp.template_roots)
        cols, consts = _addr_columns(plan, kp), _const_columns(plan, kp)
        exact = all(int(kp.template_arena.ops[i]) in EXACT for i in live)
        if exact and not kp.self_referencing:
            _lanes(kp, live, x, cols, consts)
        else:
            count = kp.instances if max_scalar is None else min(kp.instances, max_scalar)
            skipped += kp.instances - count
            _scalar(kp, live, x, cols, consts, count)
    return x, skipped
