"""C3's program is the Neo-Hookean Hessian it claims to be.

``programs.fem.element_hessian`` writes the 12x12 element Hessian in closed form
(dP/dF through the chain rule).  The builder tests prove the device plan equals the
reference's trace of THAT formula; these tests pin the formula itself:

* against central finite differences of the energy
  Psi = vol (mu/2 (I_C - 3) - mu log J + lam/2 (log J)^2), F = Ds Dm^-1, in plain floats;
* against the reference's own reverse-mode ``sparsegen.autodiff.hessian`` of the same Psi
  traced with the reference's ``Sym`` (autodiff.py:111-129), evaluated by ``eval_numeric``
  (expr.py:423-484) -- where the reference is importable (the build container).
"""

import math
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2110_12865_b200.programs.fem import LAM, MU, element_hessian

REF = Path("/root/reference/pkg/src")


def energy(x, dm, vol, log=math.log):
    X = [[x[3 * a + i] for i in range(3)] for a in range(4)]
    Ds = [[X[k + 1][i] - X[0][i] for k in range(3)] for i in range(3)]
    D = [[dm[3 * k + j] for j in range(3)] for k in range(3)]
    F = [[Ds[i][0] * D[0][j] + Ds[i][1] * D[1][j] + Ds[i][2] * D[2][j] for j in range(3)] for i in range(3)]
    J = (F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) - F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0])
         + F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]))
    ic = sum(F[i][j] * F[i][j] for i in range(3) for j in range(3))
    lj = log(J)
    return vol * (MU / 2 * (ic - 3) - MU * lj + LAM / 2 * lj * lj)


def _tet(seed):
    rng = np.random.default_rng(seed)
    rest = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float) + rng.uniform(-0.1, 0.1, (4, 3))
    Dm = np.stack([rest[k + 1] - rest[0] for k in range(3)], axis=1)
    dm = np.linalg.inv(Dm).reshape(-1)
    vol = abs(np.linalg.det(Dm)) / 6
    x = (rest + rng.uniform(-0.1, 0.1, (4, 3))).reshape(-1)
    return x, dm, vol


def _upper(H):
    return np.array([H[d1][d2] for d1 in range(12) for d2 in range(d1, 12)])


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_element_hessian_matches_finite_differences(seed):
    x, dm, vol = _tet(seed)
    h = 1e-5
    H = np.zeros((12, 12))
    for a in range(12):
        for b in range(12):
            def e(da, db):
                y = x.copy()
                y[a] += da
                y[b] += db
                return energy(y, dm, vol)
            H[a, b] = (e(h, h) - e(h, -h) - e(-h, h) + e(-h, -h)) / (4 * h * h)
    got = np.array(element_hessian(list(x), list(dm), vol, math.log))
    want = _upper(H)
    assert np.allclose(got, want, rtol=1e-5, atol=1e-5 * np.abs(want).max())


@pytest.mark.skipif(not REF.exists(), reason="the reference package is not installed here")
@pytest.mark.parametrize("seed", [0, 5])
def test_element_hessian_matches_reference_autodiff(seed):
    sys.path.insert(0, str(REF))
    from sparsegen.autodiff import hessian
    from sparsegen.expr import ExprArena, eval_numeric, sym_log

    x, dm, vol = _tet(seed)
    arena = ExprArena()
    xs = [arena.var(v) for v in range(12)]
    psi = energy(xs, list(dm), vol, log=sym_log)
    H = hessian(arena, psi.ref, range(12))
    refs = [H[(d1, d2)] for d1 in range(12) for d2 in range(d1, 12)]
    want = np.array(eval_numeric(arena, refs, {v: float(x[v]) for v in range(12)}))
    got = np.array(element_hessian(list(x), list(dm), vol, math.log))
    assert np.allclose(got, want, rtol=1e-10, atol=1e-12 * np.abs(want).max())
