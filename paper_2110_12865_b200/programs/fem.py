"""Neo-Hookean tetrahedral FEM Hessian assembled directly to CSR (config C3).

The program: a Kuhn 6-tet subdivision of an m^3 cube
grid; per tet the energy density Psi = mu/2 (I_C - 3) - mu log J + lam/2
(log J)^2 with F = Ds Dm^-1, and the element Hessian written out through the
chain rule -- H_(a i),(b k) = vol * sum_jl G_aj dP_ij/dF_kl G_bl with the
closed-form Neo-Hookean second derivative

    dP_ij/dF_kl = mu d_ik d_jl + (mu - lam log J) Finv_jk Finv_li + lam Finv_ji Finv_lk

(the "hand-structured energy" of SURVEY.md §7.4 H2: ~1.5k FP64 operations per
tet instead of the 68k of naive autodiff).  Per-tet rest data (Dm^-1, vol)
are input variables, so every tet is an instance of one template; the 78
upper-triangle entries of each 12x12 block are assembled to the symmetric
CSR Hessian with ``from_triplets`` (sparse.py:73-99): each cell is the n-ary
sum of its contributions in the reference's canonical order, ascending
(struct hash, arena index) (expr.py:245-251).

``element_hessian`` is written once against the ``Sym`` protocol: the golden
fixtures trace it with the reference (tests/golden/make_fem_golden.py); the
template-instancing builder ``build_fem_plan`` traces ONE tet with
``symtrace`` and instances it with numpy, bit-identical to the reference trace
(tests/test_builders.py).
"""

from __future__ import annotations

import itertools

import numpy as np

from ..plan import OpKind, Template
from .planbuild import PlanBuilder
from .symtrace import Arena, sym_log

MU, LAM = 1.0, 10.0
N_ELEM_VARS = 10  # Dm^-1 (row-major) + rest volume


def element_hessian(x, dm, vol, log, mu=MU, lam=LAM):
    """Upper triangle (d1 <= d2, row-major) of the 12x12 Neo-Hookean Hessian of one tet.

    x: 12 position values (vertex a, axis i at 3a + i); dm: Dm^-1 row-major (9);
    vol: rest volume.  Any Sym type (reference or symtrace) or floats.
    """
    X = [[x[3 * a + i] for i in range(3)] for a in range(4)]
    Ds = [[X[k + 1][i] - X[0][i] for k in range(3)] for i in range(3)]  # Ds[i][k]
    D = [[dm[3 * k + j] for j in range(3)] for k in range(3)]  # Dm^-1[k][j]
    F = [[Ds[i][0] * D[0][j] + Ds[i][1] * D[1][j] + Ds[i][2] * D[2][j] for j in range(3)] for i in range(3)]
    C = [[F[1][1] * F[2][2] - F[1][2] * F[2][1], F[1][2] * F[2][0] - F[1][0] * F[2][2],
          F[1][0] * F[2][1] - F[1][1] * F[2][0]],
         [F[0][2] * F[2][1] - F[0][1] * F[2][2], F[0][0] * F[2][2] - F[0][2] * F[2][0],
          F[0][1] * F[2][0] - F[0][0] * F[2][1]],
         [F[0][1] * F[1][2] - F[0][2] * F[1][1], F[0][2] * F[1][0] - F[0][0] * F[1][2],
          F[0][0] * F[1][1] - F[0][1] * F[1][0]]]  # cofactors of F
    J = F[0][0] * C[0][0] + F[0][1] * C[0][1] + F[0][2] * C[0][2]
    Finv = [[C[i][j] / J for i in range(3)] for j in range(3)]  # Finv[j][i] = cof(F)_ij / J
    logJ = log(J)
    alpha = mu - lam * logJ
    P = {}
    for i, j, k, l_ in itertools.product(range(3), repeat=4):
        t = alpha * Finv[j][k] * Finv[l_][i] + lam * Finv[j][i] * Finv[l_][k]
        P[i, j, k, l_] = mu + t if (i == k and j == l_) else t
    G = [[-(D[0][j] + D[1][j] + D[2][j]) for j in range(3)]] + [D[k] for k in range(3)]  # dN_a/dX (4x3)
    T = {}
    for i, k in itertools.product(range(3), repeat=2):
        for j in range(3):
            for b in range(4):
                acc = P[i, j, k, 0] * G[b][0]
                for l_ in (1, 2):
                    acc = acc + P[i, j, k, l_] * G[b][l_]
                T[i, k, j, b] = acc
    out = []
    for d1 in range(12):
        a, i = divmod(d1, 3)
        for d2 in range(d1, 12):
            b, k = divmod(d2, 3)
            s = G[a][0] * T[i, k, 0, b]
            for j in (1, 2):
                s = s + G[a][j] * T[i, k, j, b]
            out.append(vol * s)
    return out


UPPER = [(d1, d2) for d1 in range(12) for d2 in range(d1, 12)]  # element root order


# -- mesh ---------------------------------------------------------------------------


def kuhn_tets(m: int) -> np.ndarray:
    """(6 m^3, 4) vertex ids: cube (x fastest, then y, z), permutation order of itertools, positive volume."""
    n1 = m + 1
    vid = lambda x, y, z: x + n1 * (y + n1 * z)  # noqa: E731
    unit = np.eye(3, dtype=np.int64)
    tets = []
    for z, y, x in itertools.product(range(m), range(m), range(m)):
        c = np.array([x, y, z])
        for perm in itertools.permutations(range(3)):
            p1 = c + unit[perm[0]]
            p2 = p1 + unit[perm[1]]
            p3 = c + 1
            t = [vid(*c), vid(*p1), vid(*p2), vid(*p3)]
            # Kuhn tet orientation = permutation parity: swap to keep det(Dm) > 0
            inv = sum(1 for a in range(3) for b in range(a + 1, 3) if perm[a] > perm[b])
            if inv % 2 == 1:
                t[1], t[2] = t[2], t[1]
            tets.append(t)
    return np.asarray(tets, dtype=np.int64).reshape(-1, 4)


def rest_positions(m: int) -> np.ndarray:
    n1 = m + 1
    z, y, x = np.meshgrid(np.arange(n1), np.arange(n1), np.arange(n1), indexing="ij")
    return np.stack([x.reshape(-1), y.reshape(-1), z.reshape(-1)], axis=1).astype(np.float64)


def rest_data(m: int, tets: np.ndarray):
    """Per tet: Dm^-1 (row-major, 9) and rest volume -- element input values."""
    Xr = rest_positions(m)
    Dm = np.stack([Xr[tets[:, k + 1]] - Xr[tets[:, 0]] for k in range(3)], axis=2)  # [e, i, k]
    vol = np.abs(np.linalg.det(Dm)) / 6.0
    return np.linalg.inv(Dm).reshape(-1, 9), vol


def fem_inputs(m: int, seed: int = 0) -> np.ndarray:
    """Deformed positions (rest + U(-0.1, 0.1)^3, seed) then per tet Dm^-1 and vol."""
    tets = kuhn_tets(m)
    Xr = rest_positions(m)
    x = Xr + np.random.default_rng(seed).uniform(-0.1, 0.1, Xr.shape)
    dminv, vol = rest_data(m, tets)
    elem = np.concatenate([dminv, vol[:, None]], axis=1)
    return np.concatenate([x.reshape(-1), elem.reshape(-1)])


# -- template-instancing builder -------------------------------------------------------


def element_template():
    """ONE traced tet (symtrace): template, roots, per-root struct hash and creation rank."""
    A = Arena()
    x = [A.var(s) for s in range(12)]
    dm = [A.var(12 + k) for k in range(9)]
    vol = A.var(21)
    roots = [r.ref for r in element_hessian(x, dm, vol, sym_log)]
    sh = np.array([A.sh[r] for r in roots], dtype=object)
    rank = np.array(roots, dtype=np.int64)  # arena index: creation order inside the tet
    T, troots = A.to_template(roots)
    return T, troots, sh, rank


def shared_nodes(T, roots) -> list[int]:
    """Non-leaf nodes with two or more consumers, ascending: the template's stack locals
    (what local_decompose would keep, decompose.py:346-388); arithmetic is unchanged."""
    from ..plan import reachable

    live = reachable(T, roots)
    uses: dict[int, int] = {}
    for ref in live:
        for c in T.args[ref]:
            uses[c] = uses.get(c, 0) + 1
    return [ref for ref in live if T.ops[ref] not in (OpKind.VAR, OpKind.CONST) and uses.get(ref, 0) >= 2]


def _sum_template(k: int):
    T = Template()
    vs = [T.var(s) for s in range(k)]
    return T, [T.apply(OpKind.ADD, vs)]


def build_fem_plan(m: int, vector_width: int = 4):
    """ExecutionPlan of the assembled Neo-Hookean Hessian (CSR outputs) on the m^3 Kuhn mesh.

    Returns ``(plan, row_ptr, col_idx)``.  Inputs: 3 nv positions then 10 per tet
    (fem_inputs).
    """
    tets = kuhn_tets(m)
    ne = len(tets)
    nv = (m + 1) ** 3
    ndof = 3 * nv
    B = PlanBuilder(ndof + N_ELEM_VARS * ne, vector_width)
    T, troots, sh, rank = element_template()
    # element group: slots 0..11 positions, 12..21 element data
    cols = [3 * tets[:, a] + i for a in range(4) for i in range(3)]
    cols += [ndof + N_ELEM_VARS * np.arange(ne, dtype=np.int64) + k for k in range(N_ELEM_VARS)]
    res = B.add_group("nh_elem", 0, T, troots, cols, dest_kind="block",
                      locals_=shared_nodes(T, troots))  # (78, ne)
    # triplets (cell, contribution): both halves of every off-diagonal entry
    nq = len(UPPER)
    d1 = np.array([u for u, _ in UPPER])
    d2 = np.array([v for _, v in UPPER])
    g1 = 3 * tets[:, d1 // 3] + d1 % 3  # (ne, nq)
    g2 = 3 * tets[:, d2 // 3] + d2 % 3
    q = np.broadcast_to(np.arange(nq), (ne, nq))
    e = np.broadcast_to(np.arange(ne)[:, None], (ne, nq))
    off = d1 != d2
    rows = np.concatenate([g1.reshape(-1), g2[:, off].reshape(-1)])
    colsc = np.concatenate([g2.reshape(-1), g1[:, off].reshape(-1)])
    qq = np.concatenate([q.reshape(-1), q[:, off].reshape(-1)])
    ee = np.concatenate([e.reshape(-1), e[:, off].reshape(-1)])
    # canonical summand order inside a cell: (struct hash, arena index) = (sh[q], tet, rank[q])
    sh_rank = {h: r for r, h in enumerate(sorted(set(sh.tolist())))}
    shq = np.array([sh_rank[h] for h in sh.tolist()], dtype=np.int64)
    cell = rows * ndof + colsc
    # cells (r, c) and (c, r) sum the same contributions: the reference's hash-consing
    # makes them ONE node (expr.py:252-255) -- sums are built for r <= c only
    upper = rows <= colsc
    ucell_all = np.unique(cell)
    cell_u, q_u, e_u = cell[upper], qq[upper], ee[upper]
    order = np.lexsort((rank[q_u], e_u, shq[q_u], cell_u))
    cell_s, q_s, e_s = cell_u[order], q_u[order], e_u[order]
    addr = res[q_s, e_s]
    starts = np.flatnonzero(np.concatenate([[True], cell_s[1:] != cell_s[:-1]]))
    counts = np.diff(np.concatenate([starts, [cell_s.size]]))
    ucell = cell_s[starts]
    up_addr = np.empty(ucell.size, dtype=np.int64)
    single = counts == 1
    up_addr[single] = addr[starts[single]]
    for k in np.unique(counts[~single]).tolist():
        sel = np.flatnonzero(counts == k)
        slot_cols = [addr[starts[sel] + j] for j in range(k)]
        tk, rk = _sum_template(k)
        up_addr[sel] = B.add_group(f"nh_sum{k}", 1, tk, rk, slot_cols, dest_kind="output")[0]
    r = ucell_all // ndof
    c = ucell_all % ndof
    canon = np.minimum(r, c) * ndof + np.maximum(r, c)
    out_addr = up_addr[np.searchsorted(ucell, canon)]
    ucell = ucell_all
    row_ptr = np.zeros(ndof + 1, dtype=np.int64)
    np.add.at(row_ptr, r + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    plan = B.finish(out_addr, {"program": "neo-hookean-hessian", "m": m, "tets": ne, "mu": MU, "lam": LAM})
    return plan, row_ptr, c
