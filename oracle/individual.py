"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/README.md).

Restatement of the reference's naive baseline ``evaluate_outputs_individually(arena, outputs,
input_values)`` (/root/reference/pkg/src/sparsegen/codegen.py:560-616): every output evaluated on
its own by an iterative post-order walk with a memo private to that output, n-ary ADD / MUL
folded left in stored child order, SELECT on ``c < 0``, transcendentals through ``math`` (glibc).
The checker for ``paper_2110_12865_b200.evaluate_outputs_individually``.
"""

from __future__ import annotations

import math

import numpy as np

_UNARY = {6: lambda v: -v, 7: math.sqrt, 8: math.sin, 9: math.cos, 10: math.exp, 11: math.log}


def evaluate_outputs_individually(arena, outputs, input_values) -> np.ndarray:
    ops, args, payload = arena.ops, arena.args, arena.payload
    out = np.zeros(len(outputs))
    for k, root in enumerate(outputs):
        val: dict[int, float] = {}
        stack = [int(root)]
        while stack:
            i = stack[-1]
            if i in val:
                stack.pop()
                continue
            todo = [int(c) for c in args[i] if int(c) not in val]
            if todo:
                stack.extend(todo)
                continue
            stack.pop()
            op, a = int(ops[i]), args[i]
            if op == 0:
                val[i] = float(input_values[payload[i]])
            elif op == 1:
                val[i] = float(payload[i])
            elif op in (2, 4):
                acc = val[a[0]]
                for c in a[1:]:
                    acc = acc + val[c] if op == 2 else acc * val[c]
                val[i] = acc
            elif op == 3:
                val[i] = val[a[0]] - val[a[1]]
            elif op == 5:
                val[i] = val[a[0]] / val[a[1]] if val[a[1]] != 0 else math.copysign(math.inf, val[a[0]]) * (
                    math.copysign(1.0, val[a[1]])) if val[a[0]] != 0 else math.nan
            elif op == 12:
                try:
                    val[i] = math.pow(val[a[0]], val[a[1]])
                except OverflowError:
                    val[i] = math.inf if val[a[0]] > 0 or float(val[a[1]]) % 2 == 0 else -math.inf
            elif op == 13:
                val[i] = val[a[1]] if val[a[0]] < 0.0 else val[a[2]]
            else:
                val[i] = _UNARY[op](val[a[0]])
        out[k] = val[int(root)]
    return out
