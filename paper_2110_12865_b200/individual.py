"""``evaluate_outputs_individually`` on the B200 -- the naive per-output baseline (codegen.py:560-616).

The reference evaluates every traced output on its own: a post-order walk of the output's DAG
with a memo private to that output (shared subexpressions inside one output are computed once,
nothing is shared between outputs), n-ary ADD / MUL folded left, transcendentals through
``math``.  It is the baseline the paper's plans are measured against (acceptance #10,
test_acceptance.py:364-386; ``sparsegen bench``, cli.py:146-175).

Here each output's reachable sub-DAG becomes a one-root template whose position slots are the
input variables it reads; outputs with the same template structure become instances of one
group -- still no value shared between outputs, every instance recomputes its whole DAG -- and
the resulting ``ExecutionPlan`` runs on the device kernels like any plan.  The arithmetic is the
output's own node by node, so values equal the reference's bit for bit (SIN / COS / EXP / LOG /
POW through the device restatements of glibc, csrc/glibc_math.h).
"""

from __future__ import annotations

import numpy as np

from .plan import ExecutionPlan, KernelPlan, OpKind, Template


def _output_template(arena, root: int):
    """(structure key, template, root, input variable ids in slot order) of one output's DAG."""
    ops, args, payload = arena.ops, arena.args, arena.payload
    order, seen, stack = [], set(), [(int(root), False)]
    while stack:  # iterative post-order (children before parents, child order kept)
        n, done = stack.pop()
        if done:
            order.append(n)
            continue
        if n in seen:
            continue
        seen.add(n)
        stack.append((n, True))
        for c in reversed(args[n]):
            if int(c) not in seen:
                stack.append((int(c), False))
    local, slots, key = {}, [], []
    T = Template()
    for n in order:
        op = int(ops[n])
        if op == OpKind.VAR:
            if n not in local:
                slots.append(int(payload[n]))
                local[n] = T.var(len(slots) - 1)
            key.append(("v", local[n]))
            continue
        if op == OpKind.CONST:
            local[n] = T.const(float(payload[n]))
            key.append(("c", np.float64(payload[n]).view(np.uint64).item()))
            continue
        cs = tuple(local[int(c)] for c in args[n])
        local[n] = T.apply(op, cs)
        key.append((op, cs))
    return tuple(key), T, local[int(root)], slots


def individual_plan(arena, outputs, input_count: int) -> ExecutionPlan:
    """An ExecutionPlan evaluating every output on its own (codegen.py:560-616 semantics)."""
    groups: dict = {}
    for k, root in enumerate(outputs):
        key, T, r, slots = _output_template(arena, int(root))
        g = groups.setdefault(key, {"T": T, "root": r, "cols": [], "outs": []})
        g["cols"].append(slots)
        g["outs"].append(k)
    kernels, pos = [], []
    cursor, p_next = int(input_count), 0
    outs = np.zeros(len(outputs), np.int64)
    for gi, g in enumerate(groups.values()):
        cols = np.asarray(g["cols"], np.int64).reshape(len(g["outs"]), -1)  # (N, S)
        n, S = cols.shape
        dest = (cursor + 3) // 4 * 4
        cursor = dest + n
        kernels.append(KernelPlan(
            name=f"individual{gi}", level=0, dest_kind="output", instances=n, n_roots=1, dest_base=dest,
            template_arena=g["T"], template_roots=[g["root"]], template_locals=[], pos_vars=list(range(S)),
            const_vars=[], coherence=[0] + [None] * (S - 1) if S else [], retained=list(range(S)),
            p_base=p_next, c_base=0, layout="coalesced"))
        pos.append(cols.T.reshape(-1))
        p_next += cols.size
        outs[np.asarray(g["outs"])] = dest + np.arange(n)
    return ExecutionPlan(value_array_size=cursor, input_count=int(input_count), vector_width=4, outputs=outs,
                         kernels=kernels,
                         positions=np.concatenate(pos).astype(np.uint32) if pos else np.zeros(0, np.uint32),
                         constants=np.zeros(0, np.float64), metadata={"program": "evaluate_outputs_individually"})


def evaluate_outputs_individually(arena, outputs, input_values, device: int = 0) -> np.ndarray:
    """GPU counterpart of ``evaluate_outputs_individually(arena, outputs, input_values)``
    (codegen.py:560-616): one value per output, every output evaluated without sharing."""
    from .lower import lower_plan
    from .runtime import DevicePlan

    vals = np.ascontiguousarray(input_values, dtype=np.float64)
    plan = individual_plan(arena, list(outputs), vals.size)
    if not plan.kernels:
        return np.zeros(0)
    dp = DevicePlan(plan, device=device, lowered=lower_plan(plan, jit=False))
    return dp.run_outputs_host(vals)
