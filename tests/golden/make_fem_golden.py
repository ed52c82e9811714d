"""Golden fixtures for the Neo-Hookean FEM Hessian (config C3), traced by the reference (run HERE only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fem_golden.py

The program is ``paper_2110_12865_b200.programs.fem.element_hessian`` run with
the reference's ``Sym`` over the reference's arena: per tet the 78 upper-
triangle Hessian entries, tagged as one block (programs.py:275-294 style),
assembled with ``from_triplets`` (sparse.py:73-99) into the symmetric CSR
Hessian whose values are the session outputs; plan by ``build_plan`` with
simplify off; values by ``interpret_plan``; oracle by ``eval_numeric``
(written through make_golden.emit).
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
from sparsegen.expr import ExprArena, Sym, sym_log  # noqa: E402
from sparsegen.sparse import from_triplets  # noqa: E402

from paper_2110_12865_b200.programs import fem  # noqa: E402


def fem_session(m):
    arena = ExprArena()
    tets = fem.kuhn_tets(m)
    nv = (m + 1) ** 3
    ndof = 3 * nv
    pos = [Sym(arena, arena.make_var(v)) for v in range(ndof)]
    session = TraceSession(arena)
    trips = []
    for e, t in enumerate(tets.tolist()):
        x = [pos[3 * t[a] + i] for a in range(4) for i in range(3)]
        base = ndof + fem.N_ELEM_VARS * e
        dm = [Sym(arena, arena.make_var(base + k)) for k in range(9)]
        vol = Sym(arena, arena.make_var(base + 9))
        entries = [s.ref for s in fem.element_hessian(x, dm, vol, sym_log)]
        fresh = [r for r in dict.fromkeys(entries) if r not in session._tagged]
        if fresh:
            session.tag_block(fresh, block_id=e)
        for (d1, d2), ref in zip(fem.UPPER, entries):
            g1 = 3 * t[d1 // 3] + d1 % 3
            g2 = 3 * t[d2 // 3] + d2 % 3
            trips.append((g1, g2, ref))
            if d1 != d2:
                trips.append((g2, g1, ref))
    H = from_triplets(arena, ndof, ndof, trips)
    session.add_outputs(H.values)
    return session, H


def main():
    off = PlanConfig(simplify_enabled=False)
    for m in (1, 2):
        sess, H = fem_session(m)
        emit(f"fem_nh_m{m}", sess, off, 0, {"source": "SURVEY.md §8(d) C3 (Neo-Hookean, hand-structured Hessian)",
                                          "m": m}, csr=H, inputs=fem.fem_inputs(m))


if __name__ == "__main__":
    main()
