"""Template-instancing builder for L.M.L^T + A on a cotan grid mesh (configs C2, C5).

The reference builds this plan by tracing::

    L, M = build_operator(arena, MeshLaplacianSpec("grid", w, w, weighting="cotan"),
                          vertex_vars=vertex_coordinate_vars(arena, n), with_mass=True)
    A, _ = symbolic_matrix(arena, n, n, random_pattern(n, 6, seed=7), first_var=3n)
    out  = sp_add(sp_mul(sp_mul(L, M), sp_transpose(L)), A)

which costs ~17 s of tracing + ~28 s of planning and 1.5 GB per 10^4 vertices
 and cannot reach 10^6 vertices.  This builder produces an
ExecutionPlan for the SAME expressions -- every output bit-identical to
``eval_numeric`` of the reference trace -- with numpy index arithmetic:

* per face (sparse.py:319-340, face order sparse.py:266-276): three cotan
  weights and the area share, one 4-root kernel per face orientation (all nine
  coordinate loads are offset-coherent: one index column per group);
* L diagonal = left-fold sum of the vertex's weights in creation order
  (face, corner) -- ``from_triplets`` sorts equal-structure summands by arena
  index, i.e. creation order (sparse.py:73-99, expr.py:245-251); L off-diagonal
  = -w (boundary) or -w1 + -w2; M diagonal = area shares in face order;
* LM_ik = L_ik * M_kk (sp_mul with a diagonal right factor: one term);
* P_ij = sum over k of LM_ik * L_jk, summands in the reference's canonical
  order -- ascending (structural hash of the term, k) (sparse.py:102-139);
  the structural hash of each term class is recomputed by ``structhash``;
* out = P (+ A_ij) in CSR order (sp_add, sparse.py:142-168); entries only in
  A are the input values themselves.

Pinned against the reference's own plans and eval_numeric outputs at small
sizes (tests/golden/lmlt_w*, tests/test_builders.py).
"""

from __future__ import annotations

import numpy as np

from ..plan import OpKind, Template
from . import structhash as S
from .planbuild import PlanBuilder


# -- the random A pattern (sparse.py:199-208) ---------------------------------------


def random_pattern_rows(n: int, nnz_per_row: int, seed: int) -> np.ndarray:
    """Column indices, (n, nnz) sorted per row, exactly as ``random_pattern``."""
    if nnz_per_row > n:
        raise ValueError("nnz_per_row cannot exceed the matrix dimension")
    rng = np.random.default_rng(seed)
    out = np.empty((n, nnz_per_row), dtype=np.int64)
    for i in range(n):
        out[i] = np.sort(rng.choice(n, size=nnz_per_row, replace=False))
    return out


# -- the per-face template (face_operator_terms, sparse.py:319-340) --------------------


def face_template():
    """Slots 0..8 = (x,y,z) of corners i, j, k.  Roots: w_jk, w_ki, w_ij, area."""
    T = Template()
    p = [[T.var(3 * v + c) for c in range(3)] for v in range(3)]
    sub = lambda a, b: T.apply(OpKind.SUB, (a, b))  # noqa: E731
    neg = lambda a: T.apply(OpKind.NEG, (a,))  # noqa: E731
    mul = lambda a, b: T.apply(OpKind.MUL, (a, b))  # noqa: E731
    add = lambda a, b: T.apply(OpKind.ADD, (a, b))  # noqa: E731

    def edge(P, Q):  # _edge: [b - a for a, b in zip(p, q)]
        return [sub(b, a) for a, b in zip(P, Q)]

    def dot(u, v):  # _dot: ((u0 v0) + u1 v1) + u2 v2
        acc = mul(u[0], v[0])
        for a, b in zip(u[1:], v[1:]):
            acc = add(acc, mul(a, b))
        return acc

    pi, pj, pk = p
    eij, ejk, eki = edge(pi, pj), edge(pj, pk), edge(pk, pi)
    u, v = eij, [neg(c) for c in eki]
    uv = dot(u, v)
    dbl_area = T.apply(OpKind.SQRT, (sub(mul(dot(u, u), dot(v, v)), mul(uv, uv)),))
    half = T.const(0.5)

    def weight(a, b):
        return T.apply(OpKind.DIV, (mul(dot(a, b), half), dbl_area))

    roots = [
        weight([neg(c) for c in eij], eki),  # edge (j, k), opposite corner i
        weight([neg(c) for c in ejk], eij),  # edge (k, i)
        weight([neg(c) for c in eki], ejk),  # edge (i, j)
        mul(dbl_area, T.const(1.0 / 6.0)),
    ]
    return T, roots


def _face_struct_hashes():
    """Struct hashes of a cotan weight and of an area share (one face traced symbolically)."""
    V = S.SH_VAR
    e = S.sh_apply(S.SUB, [V, V])
    ne = S.sh_apply(S.NEG, [e])

    def dot(hu, hv):
        acc = S.sh_apply(S.MUL, [hu, hv])
        for _ in range(2):
            acc = S.sh_apply(S.ADD, [acc, S.sh_apply(S.MUL, [hu, hv])])
        return acc

    uv = dot(e, ne)
    area2 = S.sh_apply(S.SQRT, [S.sh_apply(S.SUB, [S.sh_apply(S.MUL, [dot(e, e), dot(ne, ne)]),
                                                   S.sh_apply(S.MUL, [uv, uv])])])
    w = S.sh_apply(S.DIV, [S.sh_apply(S.MUL, [dot(ne, e), S.SH_CONST]), area2])
    area = S.sh_apply(S.MUL, [area2, S.SH_CONST])
    return w, area


# -- small templates -----------------------------------------------------------------


def _sum_template(n: int, neg: bool = False):
    """v0 + v1 + ... (n-ary, left fold); with ``neg`` every summand is -v."""
    T = Template()
    vs = [T.var(s) for s in range(n)]
    if neg:
        vs = [T.apply(OpKind.NEG, (v,)) for v in vs]
    if n == 1:
        return T, [vs[0]]
    return T, [T.apply(OpKind.ADD, vs)]


def _product_template():
    T = Template()
    return T, [T.apply(OpKind.MUL, (T.var(0), T.var(1)))]


def _sop_template(m: int, with_a: bool):
    """(LM_1*L_1 + ... + LM_m*L_m) [+ a]; slots 2t, 2t+1 per term, a last."""
    T = Template()
    terms = [T.apply(OpKind.MUL, (T.var(2 * t), T.var(2 * t + 1))) for t in range(m)]
    p = terms[0] if m == 1 else T.apply(OpKind.ADD, terms)
    if with_a:
        p = T.apply(OpKind.ADD, (p, T.var(2 * m)))
    return T, [p]


# -- grid mesh topology (GridMesh.faces, sparse.py:266-276) ------------------------------


def grid_faces(w: int, h: int) -> np.ndarray:
    """(2*(w-1)*(h-1), 3) faces in the reference order: per quad (v00,v10,v11), (v00,v11,v01)."""
    y, x = np.meshgrid(np.arange(h - 1), np.arange(w - 1), indexing="ij")
    v00 = (y * w + x).reshape(-1)
    f = np.empty((2 * v00.size, 3), dtype=np.int64)
    f[0::2] = np.stack([v00, v00 + 1, v00 + w + 1], 1)
    f[1::2] = np.stack([v00, v00 + w + 1, v00 + w], 1)
    return f


def _ragged_groups(keys: np.ndarray):
    """Sorted keys -> (unique keys, start offsets, counts)."""
    if keys.size == 0:
        return keys, np.zeros(0, np.int64), np.zeros(0, np.int64)
    change = np.flatnonzero(np.diff(keys)) + 1
    starts = np.concatenate([[0], change])
    counts = np.diff(np.concatenate([starts, [keys.size]]))
    return keys[starts], starts, counts


def build_cotan(B, w: int, with_mass: bool = True):
    """Cotan Laplacian L (and lumped mass M) of the w x w grid mesh as plan groups.

    Restates ``build_operator(..., weighting="cotan", with_mass)`` (sparse.py:343-395)
    over vertex coordinates at inputs 3v..3v+2.  Returns a dict of numpy arrays:
    L in CSR order (L_row, L_col, L_addr, L_sh, L_ptr), per undirected edge
    (ekeys = a*n+b with a<b, eaddr), the diagonal (ldiag_addr) and, with mass,
    m_addr / m_sh (M diagonal).
    """
    n = w * w
    F = grid_faces(w, w)
    nf = len(F)
    sh_w, sh_area = _face_struct_hashes()
    gap = 2 * w + 8  # structured consumers reach at most w+1 anchors past either end

    # ---- per-face weights and area shares: anchor = the quad's lower-left vertex ----
    gap = 2 * w + 8  # structured consumers reach at most w+1 anchors past either end
    tmpl, roots = face_template()
    v00 = np.repeat(np.arange(nf // 2) // (w - 1) * w + np.arange(nf // 2) % (w - 1), 2)
    cols = [3 * F[:, v] + c for v in range(3) for c in range(3)]
    res = B.add_structured("face", 3, tmpl, roots, cols, v00, n, scales=[3] * 9, gap=gap)
    w_addr = res[:3].T.copy()  # weight of corner c of face f
    area_addr = res[3].copy()

    # ---- L diagonal: weights of both edge ends, creation order (face, corner) ----
    # corner c's weight belongs to the edge opposite corner c: (j,k), (k,i), (i,j)
    ends = np.array([[1, 2], [2, 0], [0, 1]])
    vert = F[:, ends].reshape(nf, 6)  # (f, c, end)
    fid = np.repeat(np.arange(nf), 6)
    cid = np.tile(np.repeat(np.arange(3), 2), nf)
    vv = vert.reshape(-1)
    order = np.lexsort((cid, fid, vv))
    vv, fid, cid = vv[order], fid[order], cid[order]
    verts, starts, counts = _ragged_groups(vv)
    assert len(verts) == n
    ldiag_addr = np.empty(n, np.int64)
    ldiag_sh = np.empty(n, dtype=object)
    for cnt in np.unique(counts):
        sel = np.flatnonzero(counts == cnt)
        cols = [w_addr[fid[starts[sel] + s], cid[starts[sel] + s]] for s in range(cnt)]
        T, r = _sum_template(int(cnt))
        ldiag_addr[verts[sel]] = B.add_structured(f"ldiag{cnt}", 2, T, r, cols, verts[sel], n, gap=gap)[0]
        ldiag_sh[verts[sel]] = S.sh_apply(S.ADD, [sh_w] * int(cnt))

    # ---- L off-diagonal per undirected edge: -w or -w1 + -w2 ----
    a_e = np.minimum(vert[:, 0::2], vert[:, 1::2]).reshape(-1)  # (f, c)
    b_e = np.maximum(vert[:, 0::2], vert[:, 1::2]).reshape(-1)
    wa = w_addr.reshape(-1)
    ekey = a_e * n + b_e
    order = np.argsort(ekey, kind="stable")  # stable: creation order inside an edge
    ekey_s, wa_s = ekey[order], wa[order]
    ekeys, estarts, ecounts = _ragged_groups(ekey_s)
    eaddr = np.empty(len(ekeys), np.int64)
    esh = np.empty(len(ekeys), dtype=object)
    sh_negw = S.sh_apply(S.NEG, [sh_w])
    for cnt in np.unique(ecounts):
        sel = np.flatnonzero(ecounts == cnt)
        cols = [wa_s[estarts[sel] + s] for s in range(cnt)]
        T, r = _sum_template(int(cnt), neg=True)
        eaddr[sel] = B.add_structured(f"loff{cnt}", 2, T, r, cols, ekeys[sel] // n, n, gap=gap)[0]
        esh[sel] = sh_negw if cnt == 1 else S.sh_apply(S.ADD, [sh_negw] * int(cnt))

    m_addr = m_sh = None
    if with_mass:
        # ---- M diagonal: area shares in face order ----
        mv = F.reshape(-1)
        mf = np.repeat(np.arange(nf), 3)
        order = np.lexsort((mf, mv))
        mv, mf = mv[order], mf[order]
        mverts, mstarts, mcounts = _ragged_groups(mv)
        m_addr = np.empty(n, np.int64)
        m_sh = np.empty(n, dtype=object)
        for cnt in np.unique(mcounts):
            sel = np.flatnonzero(mcounts == cnt)
            if cnt == 1:
                m_addr[mverts[sel]] = area_addr[mf[mstarts[sel]]]
                m_sh[mverts[sel]] = sh_area
                continue
            cols = [area_addr[mf[mstarts[sel] + s]] for s in range(cnt)]
            T, r = _sum_template(int(cnt))
            m_addr[mverts[sel]] = B.add_structured(f"mdiag{cnt}", 2, T, r, cols, mverts[sel], n, gap=gap)[0]
            m_sh[mverts[sel]] = S.sh_apply(S.ADD, [sh_area] * int(cnt))

    # ---- L in CSR: diagonal + both directions of every edge ----
    ea, eb = ekeys // n, ekeys % n
    rows = np.concatenate([np.arange(n), ea, eb])
    cols_ = np.concatenate([np.arange(n), eb, ea])
    laddr = np.concatenate([ldiag_addr, eaddr, eaddr])
    lsh = np.concatenate([ldiag_sh, esh, esh])
    order = np.lexsort((cols_, rows))
    L_row, L_col, L_addr, L_sh = rows[order], cols_[order], laddr[order], lsh[order]
    L_ptr = np.zeros(n + 1, np.int64)
    np.add.at(L_ptr, L_row + 1, 1)
    L_ptr = np.cumsum(L_ptr)

    return dict(L_row=L_row, L_col=L_col, L_addr=L_addr, L_sh=L_sh, L_ptr=L_ptr, ekeys=ekeys, eaddr=eaddr,
                ldiag_addr=ldiag_addr, m_addr=m_addr, m_sh=m_sh, gap=gap)


def build_lmlt_plan(w: int, a_nnz: int = 6, a_seed: int = 7, a_cols: np.ndarray | None = None,
                    vector_width: int = 4):
    """ExecutionPlan for out = L.M.L^T + A on a w x w cotan grid mesh.

    Returns ``(plan, row_ptr, col_idx)``; ``plan.outputs`` follow the CSR order
    of ``out``.  Inputs: 3n coordinates (vertex v at 3v..3v+2), then the
    n*a_nnz values of A in pattern order (first_var = 3n).
    """
    n = w * w
    if a_cols is None:
        a_cols = random_pattern_rows(n, min(a_nnz, n), a_seed)
    a_nnz = a_cols.shape[1]
    input_count = 3 * n + n * a_nnz
    B = PlanBuilder(input_count, vector_width)
    F = grid_faces(w, w)
    nf = len(F)
    sh_w, sh_area = _face_struct_hashes()

    cot = build_cotan(B, w, with_mass=True)
    L_row, L_col, L_addr, L_sh, L_ptr = cot["L_row"], cot["L_col"], cot["L_addr"], cot["L_sh"], cot["L_ptr"]
    m_addr, m_sh, gap = cot["m_addr"], cot["m_sh"], cot["gap"]

    # ---- LM = L * M (one term per entry) ----
    T, r = _product_template()
    lm_addr = B.add_structured("lm", 1, T, r, [L_addr, m_addr[L_col]], L_row, n, gap=gap)[0]
    # struct-hash classes: intern the (few) distinct hashes as small ints
    classes: dict[int, int] = {}
    cls_val: list[int] = []

    def intern(h):
        if h not in classes:
            classes[h] = len(cls_val)
            cls_val.append(h)
        return classes[h]

    L_cls = np.array([intern(h) for h in L_sh], np.int64)
    lm_h = {}
    lm_cls = np.empty(len(L_row), np.int64)
    m_cls_col = np.array([intern(h) for h in m_sh[L_col]], np.int64)
    for a_c, m_c in set(zip(L_cls.tolist(), m_cls_col.tolist())):
        lm_h[(a_c, m_c)] = intern(S.sh_apply(S.MUL, [cls_val[a_c], cls_val[m_c]]))
    for (a_c, m_c), h in lm_h.items():
        lm_cls[(L_cls == a_c) & (m_cls_col == m_c)] = h

    # ---- P = (LM) L^T: triples (i, k, j) from row i of L and row k of L ----
    rl = np.diff(L_ptr)
    rep = rl[L_col]  # entries of row k for each (i, k)
    tri_a = np.repeat(np.arange(len(L_row)), rep)  # LM entry (i, k)
    off = np.arange(tri_a.size) - np.repeat(np.cumsum(rep) - rep, rep)
    tri_b = L_ptr[L_col[tri_a]] + off  # L entry (k, j) == L_jk (symmetric)
    ti, tk, tj = L_row[tri_a], L_col[tri_a], L_col[tri_b]
    # term struct class -> canonical order key (sh, k)
    pair = lm_cls[tri_a] * len(cls_val) + L_cls[tri_b]
    upairs, inv = np.unique(pair, return_inverse=True)
    term_sh = np.array([S.sh_apply(S.MUL, [cls_val[p // len(cls_val)], cls_val[p % len(cls_val)]])
                        for p in upairs.tolist()], dtype=object)
    rank = np.argsort(np.argsort(term_sh.astype(np.uint64), kind="stable"), kind="stable")
    term_rank = rank[inv]
    order = np.lexsort((tk, term_rank, tj, ti))
    ti, tj, tri_a, tri_b = ti[order], tj[order], tri_a[order], tri_b[order]
    pkey = ti * n + tj
    pkeys, pstarts, pcounts = _ragged_groups(pkey)

    # ---- out = P + A in CSR order ----
    a_rows = np.repeat(np.arange(n), a_nnz)
    a_key = a_rows * n + a_cols.reshape(-1)
    a_var = 3 * n + np.arange(n * a_nnz)
    out_keys = np.union1d(pkeys, a_key)
    in_p = np.searchsorted(pkeys, out_keys)
    in_p_ok = (in_p < len(pkeys)) & (pkeys[np.minimum(in_p, len(pkeys) - 1)] == out_keys)
    a_pos = np.searchsorted(a_key, out_keys)  # a_key is sorted (rows, sorted cols)
    in_a_ok = (a_pos < len(a_key)) & (a_key[np.minimum(a_pos, len(a_key) - 1)] == out_keys)
    outputs = np.empty(len(out_keys), np.int64)
    only_a = ~in_p_ok
    outputs[only_a] = a_var[a_pos[only_a]]
    pi_idx = in_p[in_p_ok]  # which P entry
    has_a = in_a_ok[in_p_ok]
    out_slot = np.flatnonzero(in_p_ok)
    m_of = pcounts[pi_idx]
    for m in np.unique(m_of):
        for wa_flag in (False, True):
            sel = np.flatnonzero((m_of == m) & (has_a == wa_flag))
            if sel.size == 0:
                continue
            st = pstarts[pi_idx[sel]]
            cols = []
            for t in range(int(m)):
                cols.append(lm_addr[tri_a[st + t]])
                cols.append(L_addr[tri_b[st + t]])
            if wa_flag:
                cols.append(a_var[a_pos[out_slot[sel]]])
            T, r = _sop_template(int(m), wa_flag)
            res = B.add_structured(f"out{m}{'a' if wa_flag else ''}", 0, T, r, cols,
                                   out_keys[out_slot[sel]] // n, n, dest_kind="output")
            outputs[out_slot[sel]] = res[0]
    out_rows = out_keys // n
    row_ptr = np.zeros(n + 1, np.int64)
    np.add.at(row_ptr, out_rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    col_idx = out_keys % n
    plan = B.finish(outputs, {"program": "lmlt", "w": w, "a_nnz": a_nnz, "a_seed": a_seed,
                              "builder": "paper_2110_12865_b200.programs.mesh"})
    return plan, row_ptr, col_idx


def lmlt_inputs(w: int, a_nnz: int = 6, seed: int = 0) -> np.ndarray:
    """Jittered grid coordinates (no degenerate triangle) + A values in U(0.5, 2)."""
    n = w * w
    rng = np.random.default_rng(seed)
    xy = np.stack(np.meshgrid(np.arange(w, dtype=np.float64), np.arange(w, dtype=np.float64),
                              indexing="xy"), -1).reshape(n, 2)
    pos = np.zeros((n, 3))
    pos[:, :2] = xy
    pos += rng.uniform(-0.25, 0.25, (n, 3))
    a = np.random.default_rng(seed + 1).uniform(0.5, 2.0, n * min(a_nnz, n))
    return np.concatenate([pos.reshape(-1), a])
