"""The reference's own cross-backend tests, run with this package's ``compile_plan``.

The reference proves its native evaluator with five tests in pkg/tests/test_emit.py:81-142 and
acceptance criterion 9 (test_acceptance.py:346-361): ``compile_plan(plan, work_dir)`` must
return a runner whose full value array / CSR outputs equal ``interpret_plan``'s with
``np.array_equal``.  The same assertions run here with ``paper_2110_12865_b200.compile_plan`` --
the GPU backend behind the C ABI -- on the same plans and the same inputs
(``_inputs(arena, seed)`` = default_rng(seed).uniform(0.5, 2.0)), the reference's plans and
``interpret_plan`` results recorded as golden fixtures by tests/golden/make_golden.py (the
reference package is not installed on the GPU box):

    test_compiled_matches_interpreter_bitwise                        product_n24_s3_seed21
    test_compiled_matches_interpreter_with_simplify_and_transcendentals  transc37
    test_compiled_handles_blocks_and_self_references                 selfref
    test_interleaved_layout_compiles_and_agrees                      toy256_interleaved
    test_criterion_09_cross_backend_equivalence                      acc9_{expr3,lpow3}_{nosimp,simp}
"""

import numpy as np
import pytest

from conftest import golden_case

pytestmark = pytest.mark.gpu


def _ref(name):
    g = golden_case(name)
    return g.plan, g.inputs, g.values, g.values[np.asarray(g.plan.outputs, np.int64)]


def test_compiled_matches_interpreter_bitwise(tmp_path):
    """test_emit.py:81-91"""
    from paper_2110_12865_b200 import compile_plan

    plan, vals, ref_values, ref_outputs = _ref("product_n24_s3_seed21")
    run = compile_plan(plan, tmp_path)
    assert run is not None
    x = run(vals)
    assert np.array_equal(x[np.array(plan.outputs)], ref_outputs)
    assert np.array_equal(x, ref_values)


def test_compiled_matches_interpreter_with_simplify_and_transcendentals(tmp_path):
    """test_emit.py:94-113: sin, cos, exp, log, x**3 and select over 37 instances, simplify on."""
    from paper_2110_12865_b200 import compile_plan

    plan, vals, _, ref_outputs = _ref("transc37")
    run = compile_plan(plan, tmp_path)
    assert run is not None
    x = run(vals)
    assert np.array_equal(x[np.array(plan.outputs)], ref_outputs)


def test_compiled_handles_blocks_and_self_references(tmp_path):
    """test_emit.py:116-130"""
    from paper_2110_12865_b200 import compile_plan

    plan, vals, _, ref_outputs = _ref("selfref")
    assert np.array_equal(vals, np.array([1.25, -2.5]))
    run = compile_plan(plan, tmp_path)
    assert run is not None
    x = run(vals)
    assert np.array_equal(x[np.array(plan.outputs)], ref_outputs)


def test_interleaved_layout_compiles_and_agrees(tmp_path):
    """test_emit.py:133-142"""
    from paper_2110_12865_b200 import compile_plan

    plan, vals, _, ref_outputs = _ref("toy256_interleaved")
    assert all(kp.layout == "interleaved" for kp in plan.kernels)
    run = compile_plan(plan, tmp_path, parallel="pragma")
    assert run is not None
    x = run(vals)
    assert np.array_equal(x[np.array(plan.outputs)], ref_outputs)


def test_criterion_09_cross_backend_equivalence(tmp_path):
    """test_acceptance.py:346-361: expr3 on random:120,5,2 and lpow3 on grid:10x10, simplify off and on."""
    from paper_2110_12865_b200 import compile_plan

    for name in ("expr3", "lpow3"):
        for simplify_on in (False, True):
            plan, vals, _, ref_outputs = _ref(f"acc9_{name}_{'simp' if simplify_on else 'nosimp'}")
            run = compile_plan(plan, tmp_path)
            assert run is not None, "compilation failed"
            x = run(vals)
            assert np.array_equal(x[np.array(plan.outputs)], ref_outputs), (
                f"{name} simplify={simplify_on}: compiled output differs")
