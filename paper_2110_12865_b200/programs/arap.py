"""ARAP system matrix + right-hand side on a grid mesh (config C4).

The program, one local/global iteration of
as-rigid-as-possible deformation:

* system matrix: the cotan Laplacian L of the rest pose (``build_operator``,
  sparse.py:343-395) -- it is also where the edge weights come from,
  w_ij = -L_ij;
* local step, per vertex i: covariance S_i = sum_j w_ij E_ij e_ij^T with rest
  edges E_ij = P_j - P_i and deformed edges e_ij = p_j - p_i (neighbours j in
  the CSR order of L's row), rotation R_i by Gram-Schmidt orthonormalisation
  of S_i's columns (see arap_rotation);
* right-hand side b_i = sum_j (w_ij / 2) (R_i + R_j) (P_i - P_j).

Outputs: L's values in CSR order, then b (3 per vertex).  Inputs: rest
coordinates (3v..3v+2) then deformed coordinates (3n + 3v ..).

Every arithmetic node the per-vertex functions create is binary, so the
value of the program does not depend on the child order commutative nodes
get in an arena: the builder can trace one vertex per valence class with
``symtrace`` and instance it, and still match the reference trace bit for
bit (tests/test_builders.py against tests/golden/arap_w*).
"""

from __future__ import annotations

import numpy as np

from .mesh import build_cotan
from .planbuild import PlanBuilder
from .symtrace import Arena, sym_sqrt


def arap_rotation(Pi, pi, nbrs, sqrt):
    """R_i (row-major, 9 values).  nbrs: list of (w_ij, P_j, p_j) in neighbour order.

    Covariance S_i = sum_j w_ij E_ij e_ij^T; rotation by Gram-Schmidt on S_i's
    columns (c1 = s1/|s1|, c2 = normalised s2 - (c1.s2) c1, c3 = c1 x c2): a
    shallow, division-safe orthonormalisation that equals the polar factor for
    pure rotations and stays close to it for the small deformations of a local
    step.  (Iterated polar schemes -- Newton-Schulz, McAdams -- make the
    reference planner's tree walks exponential in the iteration count: 4 s for
    one Newton-Schulz step, 82 s for two on a 3x3 mesh.)
    """
    S = None
    for w, Pj, pj in nbrs:
        E = [Pj[c] - Pi[c] for c in range(3)]
        e = [pj[c] - pi[c] for c in range(3)]
        t = [[(w * E[a]) * e[b] for b in range(3)] for a in range(3)]
        S = t if S is None else [[S[a][b] + t[a][b] for b in range(3)] for a in range(3)]
    s1 = [S[a][0] for a in range(3)]
    s2 = [S[a][1] for a in range(3)]
    n1 = sqrt(s1[0] * s1[0] + s1[1] * s1[1] + s1[2] * s1[2])
    c1 = [s1[a] / n1 for a in range(3)]
    d = c1[0] * s2[0] + c1[1] * s2[1] + c1[2] * s2[2]
    u2 = [s2[a] - d * c1[a] for a in range(3)]
    n2 = sqrt(u2[0] * u2[0] + u2[1] * u2[1] + u2[2] * u2[2])
    c2 = [u2[a] / n2 for a in range(3)]
    c3 = [c1[1] * c2[2] - c1[2] * c2[1], c1[2] * c2[0] - c1[0] * c2[2], c1[0] * c2[1] - c1[1] * c2[0]]
    cols = (c1, c2, c3)
    return [cols[b][a] for a in range(3) for b in range(3)]


def arap_rhs(Ri, Pi, nbrs):
    """b_i (3 values).  nbrs: list of (w_ij, R_j (9), P_j) in neighbour order."""
    b = None
    for w, Rj, Pj in nbrs:
        D = [Pi[c] - Pj[c] for c in range(3)]
        hw = 0.5 * w
        t = []
        for a in range(3):
            q = (Ri[3 * a] + Rj[3 * a]) * D[0]
            for c in (1, 2):
                q = q + (Ri[3 * a + c] + Rj[3 * a + c]) * D[c]
            t.append(hw * q)
        b = t if b is None else [b[a] + t[a] for a in range(3)]
    return b


# -- inputs -------------------------------------------------------------------------


def arap_inputs(w: int, seed: int = 0) -> np.ndarray:
    """Rest = jittered grid (as C2), deformed = rest + smooth displacement + small noise (seed)."""
    n = w * w
    rng = np.random.default_rng(seed)
    xy = np.stack(np.meshgrid(np.arange(w, dtype=np.float64), np.arange(w, dtype=np.float64),
                              indexing="xy"), -1).reshape(n, 2)
    rest = np.zeros((n, 3))
    rest[:, :2] = xy
    rest += rng.uniform(-0.25, 0.25, (n, 3))
    x, y = rest[:, 0], rest[:, 1]
    disp = np.stack([0.3 * np.sin(0.05 * y), 0.3 * np.cos(0.05 * x), 0.2 * np.sin(0.03 * (x + y))], axis=1)
    cur = rest + disp + rng.uniform(-0.02, 0.02, (n, 3))
    return np.concatenate([rest.reshape(-1), cur.reshape(-1)])


# -- template-instancing builder -------------------------------------------------------


def _rotation_template(v: int):
    """Slots: P_i (0-2), p_i (3-5), per neighbour k: L_ij (6+7k), P_j (7+7k..), p_j (10+7k..)."""
    A = Arena()
    Pi = [A.var(c) for c in range(3)]
    pi = [A.var(3 + c) for c in range(3)]
    nb = []
    for k in range(v):
        s = 6 + 7 * k
        nb.append((-A.var(s), [A.var(s + 1 + c) for c in range(3)], [A.var(s + 4 + c) for c in range(3)]))
    roots = [r.ref for r in arap_rotation(Pi, pi, nb, sym_sqrt)]
    return A.to_template(roots)


def _rhs_template(v: int):
    """Slots: R_i (0-8), P_i (9-11), per neighbour k: L_ij (12+13k), R_j (13+13k..), P_j (22+13k..)."""
    A = Arena()
    Ri = [A.var(c) for c in range(9)]
    Pi = [A.var(9 + c) for c in range(3)]
    nb = []
    for k in range(v):
        s = 12 + 13 * k
        nb.append((-A.var(s), [A.var(s + 1 + c) for c in range(9)], [A.var(s + 10 + c) for c in range(3)]))
    roots = [r.ref for r in arap_rhs(Ri, Pi, nb)]
    return A.to_template(roots)


def build_arap_plan(w: int, vector_width: int = 4):
    """ExecutionPlan of L's CSR values then b (3 per vertex).  Returns (plan, row_ptr, col_idx) of L."""
    n = w * w
    B = PlanBuilder(6 * n, vector_width)
    cot = build_cotan(B, w, with_mass=False)
    L_row, L_col, L_addr, L_ptr = cot["L_row"], cot["L_col"], cot["L_addr"], cot["L_ptr"]
    offd = L_row != L_col
    val = np.diff(L_ptr) - 1  # neighbours per vertex (row length minus the diagonal)
    nb_col = L_col[offd]  # neighbours in CSR order, row by row
    nb_addr = L_addr[offd]
    nb_start = np.concatenate([[0], np.cumsum(val)[:-1]])
    R_addr = np.empty((9, n), np.int64)
    for v in np.unique(val).tolist():
        verts = np.flatnonzero(val == v)
        cols = [3 * verts + c for c in range(3)] + [3 * n + 3 * verts + c for c in range(3)]
        for k in range(v):
            j = nb_col[nb_start[verts] + k]
            cols += [nb_addr[nb_start[verts] + k]] + [3 * j + c for c in range(3)] + \
                    [3 * n + 3 * j + c for c in range(3)]
        T, roots = _rotation_template(v)
        scales = [3] * 6 + [1, 3, 3, 3, 3, 3, 3] * v  # positions 3/vertex, L entries 1/anchor
        R_addr[:, verts] = B.add_affine_classes(f"rot{v}", 1, T, roots, cols, verts, scales, dest_kind="block")
    b_addr = np.empty((3, n), np.int64)
    for v in np.unique(val).tolist():
        verts = np.flatnonzero(val == v)
        cols = [R_addr[c, verts] for c in range(9)] + [3 * verts + c for c in range(3)]
        for k in range(v):
            j = nb_col[nb_start[verts] + k]
            cols += [nb_addr[nb_start[verts] + k]] + [R_addr[c, j] for c in range(9)] + [3 * j + c for c in range(3)]
        T, roots = _rhs_template(v)
        scales = [1] * 9 + [3] * 3 + ([1] * 10 + [3] * 3) * v
        b_addr[:, verts] = B.add_affine_classes(f"rhs{v}", 0, T, roots, cols, verts, scales, dest_kind="output")
    outputs = np.concatenate([L_addr, b_addr.T.reshape(-1)])
    plan = B.finish(outputs, {"program": "arap", "w": w, "rotation": "gram-schmidt"})
    return plan, L_ptr, L_col
