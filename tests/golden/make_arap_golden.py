"""Golden fixtures for ARAP system matrix + rhs (config C4), traced by the reference (run HERE only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_arap_golden.py

``paper_2110_12865_b200.programs.arap`` run with the reference's ``Sym``: L from
``build_operator(weighting="cotan")`` over the rest coordinates, per-vertex
rotations (tagged blocks) and right-hand sides; outputs = L's CSR values then b.
"""

import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent.parent))
sys.setrecursionlimit(100000)

from make_golden import emit  # noqa: E402
from sparsegen.codegen import PlanConfig  # noqa: E402
from sparsegen.decompose import TraceSession  # noqa: E402
from sparsegen.expr import ExprArena, Sym, sym_sqrt  # noqa: E402
from sparsegen.sparse import MeshLaplacianSpec, build_operator, vertex_coordinate_vars  # noqa: E402

from paper_2110_12865_b200.programs import arap  # noqa: E402


def arap_session(w):
    arena = ExprArena()
    n = w * w
    rest = vertex_coordinate_vars(arena, n)
    L = build_operator(arena, MeshLaplacianSpec(builder="grid", w=w, h=w, weighting="cotan"), vertex_vars=rest)
    cur = [[Sym(arena, arena.make_var(3 * n + 3 * v + c)) for c in range(3)] for v in range(n)]
    session = TraceSession(arena)

    def nbrs(i):
        lo, hi = L.row_ptr[i], L.row_ptr[i + 1]
        return [(L.col_idx[k], -Sym(arena, L.values[k])) for k in range(lo, hi) if L.col_idx[k] != i]

    R = []
    for i in range(n):
        Ri = arap.arap_rotation(rest[i], cur[i], [(wv, rest[j], cur[j]) for j, wv in nbrs(i)], sym_sqrt)
        fresh = [r for r in dict.fromkeys(x.ref for x in Ri) if r not in session._tagged]
        if fresh:
            session.tag_block(fresh, block_id=i)
        R.append(Ri)
    b = []
    for i in range(n):
        b += arap.arap_rhs(R[i], rest[i], [(wv, R[j], rest[j]) for j, wv in nbrs(i)])
    session.add_outputs(list(L.values) + [x.ref for x in b])
    return session, L


DEFECT = ("the reference's build_plan groups rhs terms whose commutative children are ordered differently per "
          "instance (ADD(R_i, R_j) sorted by arena index) and harvests their leaves in the template's order: its "
          "interpret_plan outputs differ from eval_numeric (up to 37% relative); builders match eval_numeric")


def main():
    off = PlanConfig(simplify_enabled=False)
    for w in (3, 5):
        sess, L = arap_session(w)
        emit(f"arap_w{w}", sess, off, 0, {"source": "SURVEY.md §8(d) C4 (ARAP system matrix + rhs)", "w": w,
                                          "reference_plan_defect": DEFECT}, csr=L, inputs=arap.arap_inputs(w))


if __name__ == "__main__":
    main()
