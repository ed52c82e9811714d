"""evaluate_outputs_individually: the naive per-output baseline (codegen.py:560-616), on the B200.

The oracle restatement (oracle/individual.py) is pinned to the reference's own function where the
reference is importable; the device plan (individual.individual_plan) is proven on CPU through the
device-plan emulator and on the GPU through the kernels, bit for bit against the oracle.
"""

import math
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import bits

REF = Path("/root/reference/pkg/src")


def synthetic_arena(n=300, seed=0):
    """sin / cos / exp / log / x**3 / select / sqrt over pairs of inputs (the transc37 program, larger)."""
    from paper_2110_12865_b200.plan import OpKind, Template

    T = Template()
    outs = []
    for k in range(n):
        x, y = T.var(2 * k), T.var(2 * k + 1)
        s = T.apply(OpKind.MUL, (T.apply(OpKind.SIN, (x,)), T.apply(OpKind.COS, (y,))))
        e = T.apply(OpKind.EXP, (T.apply(OpKind.DIV, (x, T.apply(OpKind.ADD, (y, T.const(3.0)))),),))
        lg = T.apply(OpKind.LOG, (T.apply(OpKind.ADD, (y, T.const(1.5))),))
        p3 = T.apply(OpKind.POW, (x, T.const(3.0)))
        sel = T.apply(OpKind.SELECT, (T.apply(OpKind.SUB, (x, y)), T.apply(OpKind.MUL, (x, T.const(2.0))),
                                      T.apply(OpKind.SQRT, (y,))))
        outs.append(T.apply(OpKind.ADD, (T.apply(OpKind.SUB, (T.apply(OpKind.ADD, (s, e)), lg)), p3, sel)))
    inputs = np.random.default_rng(seed).uniform(0.5, 2.0, 2 * n)
    return T, outs, inputs


def test_device_plan_equals_oracle_on_cpu():
    import device_plan_emu as emu
    from oracle.individual import evaluate_outputs_individually
    from paper_2110_12865_b200.individual import individual_plan
    from paper_2110_12865_b200.lower import lower_plan

    T, outs, inputs = synthetic_arena()
    plan = individual_plan(T, outs, inputs.size)
    assert len(plan.kernels) == 1 and plan.kernels[0].instances == len(outs)  # one structure, 300 instances
    got = emu.run_csr(lower_plan(plan, jit=False), inputs)
    assert np.array_equal(bits(got), bits(evaluate_outputs_individually(T, outs, inputs)))


@pytest.mark.skipif(not REF.exists(), reason="the reference package is not installed here")
@pytest.mark.parametrize("program,pattern", [("expr3", "random:40,4,2"), ("lpow3", "grid:5x5"),
                                             ("energy-hessian", "grid:3x3")])
def test_oracle_equals_reference_evaluate_outputs_individually(program, pattern):
    sys.path.insert(0, str(REF))
    from sparsegen.codegen import evaluate_outputs_individually as ref_eoi
    from sparsegen.programs import ProgramSpec, trace_program

    import device_plan_emu as emu
    from oracle.individual import evaluate_outputs_individually
    from paper_2110_12865_b200.individual import individual_plan
    from paper_2110_12865_b200.lower import lower_plan

    tr = trace_program(ProgramSpec(program, pattern, seed=3))
    vals = np.random.default_rng(3).uniform(0.5, 2.0, tr.arena.var_count)
    want = np.asarray(ref_eoi(tr.arena, tr.outputs, list(vals)), dtype=np.float64)
    assert np.array_equal(bits(evaluate_outputs_individually(tr.arena, tr.outputs, vals)), bits(want))
    plan = individual_plan(tr.arena, tr.outputs, tr.arena.var_count)
    assert np.array_equal(bits(emu.run_csr(lower_plan(plan, jit=False), vals)), bits(want))


@pytest.mark.gpu
def test_evaluate_outputs_individually_on_the_gpu():
    from oracle.individual import evaluate_outputs_individually as oracle_eoi
    from paper_2110_12865_b200 import evaluate_outputs_individually

    T, outs, inputs = synthetic_arena(n=2000, seed=4)
    got = evaluate_outputs_individually(T, outs, inputs)
    assert np.array_equal(bits(got), bits(oracle_eoi(T, outs, inputs)))
