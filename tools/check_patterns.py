"""The builders' CSR sparsity patterns == independent scipy boolean products.

The template-instancing builders (programs/mesh.py, fem.py, arap.py) produce the CSR pattern
(row_ptr, col_idx) of the output along with the plan.  Here every pattern is rebuilt from the
mesh alone with scipy.sparse -- the grid stencil for C2 / C4 (the reference's GridMesh faces,
sparse.py:266-276: quads split along the (x, y) -> (x+1, y+1) diagonal), tet incidence for C3 --
and compared entry for entry:

* C2 out = L.M.L^T + A:  pattern(L) = I + grid adjacency; pattern(out) = pattern(L)^2 | pattern(A)
  (M diagonal; A = random_pattern(n, 6, seed 7), sparse.py:199-208);
* C3 Hessian: vertex adjacency V = B^T B (B the tet-vertex incidence), pattern = V kron ones(3, 3);
* C4 system matrix: pattern(L) as in C2.

    python tools/check_patterns.py [--full]     (full = the BASELINE sizes: w=1000, m=55, w4=708)
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def grid_laplacian_pattern(w: int) -> sp.csr_matrix:
    """I + adjacency of the w x w grid mesh triangulated along the (+1, +1) diagonal of every quad."""
    n = w * w
    y, x = np.divmod(np.arange(n), w)
    rows, cols = [np.arange(n)], [np.arange(n)]
    for dx, dy in ((1, 0), (0, 1), (1, 1)):
        ok = (x + dx < w) & (y + dy < w)
        a = np.flatnonzero(ok)
        b = a + dx + dy * w
        rows += [a, b]
        cols += [b, a]
    r, c = np.concatenate(rows), np.concatenate(cols)
    return sp.csr_matrix((np.ones(r.size, np.int8), (r, c)), shape=(n, n))


def lmlt_pattern(w: int) -> sp.csr_matrix:
    from paper_2110_12865_b200.programs.mesh import random_pattern_rows

    n = w * w
    L = grid_laplacian_pattern(w).astype(np.int64)
    P = (L @ L).astype(bool).astype(np.int8)
    a = random_pattern_rows(n, min(6, n), 7)
    A = sp.csr_matrix((np.ones(a.size, np.int8), (np.repeat(np.arange(n), a.shape[1]), a.reshape(-1))), shape=(n, n))
    return (P + A).astype(bool).tocsr()


def hessian_pattern(m: int) -> sp.csr_matrix:
    from paper_2110_12865_b200.programs.fem import kuhn_tets

    t = kuhn_tets(m)
    nv = (m + 1) ** 3
    B = sp.csr_matrix((np.ones(t.size, np.int64), (np.repeat(np.arange(len(t)), 4), t.reshape(-1))),
                      shape=(len(t), nv))
    V = (B.T @ B).astype(bool).astype(np.int8)
    return sp.kron(V, np.ones((3, 3), np.int8), format="csr").astype(bool)


def same(row_ptr, col_idx, M: sp.csr_matrix) -> bool:
    M = M.tocsr()
    M.sort_indices()
    return (np.array_equal(np.asarray(row_ptr, np.int64), M.indptr.astype(np.int64))
            and np.array_equal(np.asarray(col_idx, np.int64), M.indices.astype(np.int64)))


def check(w: int, m: int, w4: int) -> dict:
    from paper_2110_12865_b200.programs.arap import build_arap_plan
    from paper_2110_12865_b200.programs.fem import build_fem_plan
    from paper_2110_12865_b200.programs.mesh import build_lmlt_plan

    out = {}
    for name, build, ref in (("c2", lambda: build_lmlt_plan(w), lambda: lmlt_pattern(w)),
                             ("c3", lambda: build_fem_plan(m), lambda: hessian_pattern(m)),
                             ("c4", lambda: build_arap_plan(w4), lambda: grid_laplacian_pattern(w4))):
        t0 = time.perf_counter()
        plan, rp, ci = build()
        M = ref()
        out[name] = {"nnz": int(len(ci)), "rows": int(len(rp) - 1), "match": bool(same(rp, ci, M)),
                     "scipy_nnz": int(M.nnz), "seconds": round(time.perf_counter() - t0, 1)}
        if name in ("c2", "c3"):
            out[name]["outputs_are_the_pattern"] = len(plan.outputs) == len(ci)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    args = ap.parse_args()
    sizes = dict(w=1000, m=55, w4=708) if args.full else dict(w=60, m=6, w4=40)
    res = {"sizes": sizes, "patterns": check(**sizes)}
    print(json.dumps(res))
    if args.full:
        (ROOT / "profiles" / "r2" / "patterns_full.json").write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
