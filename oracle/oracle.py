"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/README.md).

ctypes glue for ``interp.c``, the C restatement of the reference CPU evaluator
``interpret_plan`` (/root/reference/pkg/src/sparsegen/codegen.py:404-446).
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  The product path (``paper_2110_12865_b200``) never does.

The encoding reads a plan only through the reference's own field names
(codegen.py:56-98), so it accepts reference ``ExecutionPlan`` objects and the
package's wire-format mirror alike, and it is independent of the device-plan
lowering it is used to check.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"
LIB = BUILD / "liboracle.so"

# kernel field layout shared with interp.c (KF_*)
KF = ["N", "NROOTS", "DEST", "SELFREF", "INTERLEAVED", "PBASE", "CBASE", "NRET", "NCONST",
      "SLOT0", "NSLOTS", "NODE0", "NNODES", "ROOT0"]


def build(force: bool = False) -> Path:
    """gcc -O2 -ffp-contract=off (no fast-math): IEEE binary64, glibc libm."""
    src = HERE / "interp.c"
    if LIB.exists() and not force and LIB.stat().st_mtime >= src.stat().st_mtime:
        return LIB
    BUILD.mkdir(parents=True, exist_ok=True)
    tmp = LIB.with_suffix(f".{os.getpid()}.tmp")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                    "-o", str(tmp), str(src), "-lm"], check=True)
    os.replace(tmp, LIB)
    return LIB


_dll = None


def _lib():
    global _dll
    if _dll is None:
        _dll = ctypes.CDLL(str(build()))
        _dll.oracle_run.restype = ctypes.c_int
    return _dll


def _reachable(tmpl, roots):
    n = len(tmpl.ops)
    need = bytearray(n)
    for r in roots:
        need[r] = 1
    for i in range(n - 1, -1, -1):
        if need[i]:
            for c in tmpl.args[i]:
                need[c] = 1
    return [i for i in range(n) if need[i]]


def encode_plan(plan) -> dict:
    """Flatten a plan into the arrays interp.c walks."""
    kern, slot_col, slot_delta = [], [], []
    node_op, node_a0, node_na, node_pay, arg_list, roots = [], [], [], [], [], []
    for kp in plan.kernels:
        tmpl = kp.template_arena
        live = _reachable(tmpl, kp.template_roots)
        local = {ref: j for j, ref in enumerate(live)}
        slot_of = {v: s for s, v in enumerate(kp.pos_vars)}
        cslot_of = {v: s for s, v in enumerate(kp.const_vars)}
        ridx = {s: k for k, s in enumerate(kp.retained)}
        fields = dict(
            N=kp.instances, NROOTS=kp.n_roots, DEST=kp.dest_base,
            SELFREF=int(bool(kp.self_referencing)), INTERLEAVED=int(kp.layout == "interleaved"),
            PBASE=kp.p_base, CBASE=kp.c_base, NRET=len(kp.retained), NCONST=len(kp.const_vars),
            SLOT0=len(slot_col), NSLOTS=len(kp.pos_vars), NODE0=len(node_op), NNODES=len(live),
            ROOT0=len(roots),
        )
        kern.extend(int(fields[k]) for k in KF)
        for s, coh in enumerate(kp.coherence):
            slot_col.append(ridx.get(s, -1))
            slot_delta.append(0 if s in ridx else int(coh))
        for ref in live:
            op = int(tmpl.ops[ref])
            node_op.append(op)
            node_a0.append(len(arg_list))
            node_na.append(len(tmpl.args[ref]))
            arg_list.extend(local[c] for c in tmpl.args[ref])
            if op == 0:
                v = tmpl.payload[ref]
                node_pay.append(float(slot_of[v]) if v in slot_of else float(-(cslot_of[v] + 1)))
            elif op == 1:
                node_pay.append(float(tmpl.payload[ref]))
            else:
                node_pay.append(0.0)
        roots.extend(local[r] for r in kp.template_roots)
    return dict(
        n_kernels=len(plan.kernels),
        kern=np.asarray(kern, np.int64),
        slot_col=np.asarray(slot_col, np.int32),
        slot_delta=np.asarray(slot_delta, np.int64),
        node_op=np.asarray(node_op, np.int32),
        node_a0=np.asarray(node_a0, np.int64),
        node_na=np.asarray(node_na, np.int32),
        node_pay=np.asarray(node_pay, np.float64),
        arg_list=np.asarray(arg_list, np.int32),
        roots=np.asarray(roots, np.int32),
        p=np.ascontiguousarray(plan.positions, dtype=np.uint32),
        c=np.ascontiguousarray(plan.constants, dtype=np.float64),
    )


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a.size else ctypes.c_void_p(0)


def run_values(plan, inputs, enc=None) -> np.ndarray:
    """Full value array, exactly like ``interpret_plan(plan, inputs).values``."""
    inputs = np.asarray(inputs, dtype=np.float64)
    if inputs.shape != (plan.input_count,):
        raise ValueError(f"plan expects {plan.input_count} input values, got {inputs.size}")
    enc = enc or encode_plan(plan)
    x = np.zeros(plan.value_array_size, dtype=np.float64)
    x[: plan.input_count] = inputs
    rc = _lib().oracle_run(
        _ptr(x), ctypes.c_int64(plan.value_array_size), ctypes.c_int64(enc["n_kernels"]),
        _ptr(enc["kern"]), _ptr(enc["slot_col"]), _ptr(enc["slot_delta"]), _ptr(enc["node_op"]),
        _ptr(enc["node_a0"]), _ptr(enc["node_na"]), _ptr(enc["node_pay"]), _ptr(enc["arg_list"]),
        _ptr(enc["roots"]), _ptr(enc["p"]), _ptr(enc["c"]),
    )
    if rc != 0:
        raise ValueError(f"oracle: plan decode failed (code {rc})")
    return x


def run_outputs(plan, inputs, enc=None) -> np.ndarray:
    x = run_values(plan, inputs, enc)
    return x[np.asarray(plan.outputs, dtype=np.int64)] if len(plan.outputs) else np.zeros(0)
