"""Scalable plan builders pinned against the reference trace (tests/golden/lmlt_*).

The builder never traces; these tests prove its plan computes exactly the
expressions the reference builds -- outputs bit-identical to eval_numeric of
the reference trace and the same CSR pattern.
"""

import numpy as np
import pytest

import device_plan_emu as emu
from conftest import Golden, bits
from oracle import oracle
from paper_2110_12865_b200.lower import lower_plan
from paper_2110_12865_b200.programs import structhash as S
from paper_2110_12865_b200.programs.mesh import build_lmlt_plan, lmlt_inputs, random_pattern_rows

SIZES = (3, 4, 7, 12)


@pytest.mark.parametrize("w", SIZES)
def test_lmlt_builder_matches_reference_trace(w):
    g = Golden(f"lmlt_w{w}")
    plan, row_ptr, col_idx = build_lmlt_plan(w)
    assert np.array_equal(row_ptr, g.vec["row_ptr"])
    assert np.array_equal(col_idx, g.vec["col_idx"])
    out = oracle.run_outputs(plan, g.inputs)
    assert np.array_equal(bits(out), bits(g.oracle))


@pytest.mark.parametrize("w", SIZES)
def test_lmlt_builder_lowering_bitwise(w):
    g = Golden(f"lmlt_w{w}")
    plan, _, _ = build_lmlt_plan(w)
    x = emu.run_values(lower_plan(plan, jit=False), g.inputs)
    assert np.array_equal(bits(x[np.asarray(plan.outputs)]), bits(g.oracle))


def test_inputs_match_fixture_convention():
    g = Golden("lmlt_w7")
    assert np.array_equal(lmlt_inputs(7), g.inputs)


def test_random_pattern_restatement():
    # sparse.py:199-208: per row, sorted rng.choice(n, k, replace=False)
    cols = random_pattern_rows(50, 6, 7)
    rng = np.random.default_rng(7)
    for i in range(50):
        assert cols[i].tolist() == sorted(rng.choice(50, size=6, replace=False).tolist())


def test_structured_layout_is_coherent_at_scale():
    plan, _, _ = build_lmlt_plan(60)
    big = [k for k in plan.kernels if k.instances == 3600]
    assert len(big) >= 20
    assert all(len(k.retained) == 1 for k in big)  # one index column (slot 0) per group


def test_struct_hash_restatement_matches_reference():
    ref = pytest.importorskip("sparsegen.expr", reason="reference package not importable here")
    arena = ref.ExprArena()
    a, b, c = arena.var(0), arena.var(1), arena.var(2)
    e = (a - b) * (c - a) + (b - c) * (a - b)
    sh_e = S.sh_apply(S.SUB, [S.SH_VAR, S.SH_VAR])
    t = S.sh_apply(S.MUL, [sh_e, sh_e])
    assert arena.struct_hash[e.ref] == S.sh_apply(S.ADD, [t, t])
    assert arena.struct_hash[ref.sym_sqrt(e).ref] == S.sh_apply(S.SQRT, [S.sh_apply(S.ADD, [t, t])])


@pytest.mark.parametrize("m", [1, 2])
def test_fem_builder_matches_reference_trace(m):
    """C3: the template-instancing Neo-Hookean builder == the reference trace (tests/golden/fem_nh_m*):
    same CSR pattern, every output bit-identical to eval_numeric."""
    from paper_2110_12865_b200.programs.fem import build_fem_plan, fem_inputs

    g = Golden(f"fem_nh_m{m}")
    plan, row_ptr, col_idx = build_fem_plan(m)
    assert np.array_equal(row_ptr, g.vec["row_ptr"])
    assert np.array_equal(col_idx, g.vec["col_idx"])
    assert np.array_equal(fem_inputs(m), g.inputs)
    out = oracle.run_outputs(plan, g.inputs)
    assert np.array_equal(bits(out), bits(g.oracle))
    x = emu.run_values(lower_plan(plan, jit=False), g.inputs)
    assert np.array_equal(bits(x[np.asarray(plan.outputs)]), bits(g.oracle))


def test_fem_element_template_counts():
    from paper_2110_12865_b200.plan import reachable
    from paper_2110_12865_b200.programs.fem import element_template

    T, roots, sh, rank = element_template()
    assert len(roots) == 78
    assert len(reachable(T, roots)) < 3000  # hand-structured: ~1.5k ops, not the 68k of naive autodiff


@pytest.mark.parametrize("w", [3, 5])
def test_arap_builder_matches_reference_trace(w):
    """C4: the ARAP builder (L via the C2 cotan restatement, per-valence rotation / rhs templates)
    == the reference trace (tests/golden/arap_w*): same L pattern, every output bit-identical."""
    from paper_2110_12865_b200.programs.arap import arap_inputs, build_arap_plan

    g = Golden(f"arap_w{w}")
    plan, row_ptr, col_idx = build_arap_plan(w)
    assert np.array_equal(row_ptr, g.vec["row_ptr"])
    assert np.array_equal(col_idx, g.vec["col_idx"])
    assert np.array_equal(arap_inputs(w), g.inputs)
    out = oracle.run_outputs(plan, g.inputs)
    assert np.array_equal(bits(out), bits(g.oracle))
    x = emu.run_values(lower_plan(plan, jit=False), g.inputs)
    assert np.array_equal(bits(x[np.asarray(plan.outputs)]), bits(g.oracle))


@pytest.mark.parametrize("w,m,w4", [(60, 6, 40), (33, 5, 21)])
def test_builder_patterns_equal_scipy_boolean_products(w, m, w4):
    """C2 / C3 / C4 CSR patterns from the builders == scipy boolean products of the mesh alone
    (tools/check_patterns.py; the full BASELINE sizes are checked by `--full`, profiles/r2/patterns_full.json)."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
    import check_patterns

    res = check_patterns.check(w, m, w4)
    assert all(r["match"] for r in res.values()), res
