"""Generate the golden plan fixtures from the reference package (run HERE only).

Usage (in the build container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture directory holds exactly what the reference itself produced:

* ``manifest.json`` + ``data.blob`` -- ``sparsegen.codegen.save_plan`` output
  (codegen.py:708-717), i.e. the reference plan wire format;
* ``vectors.npz`` -- ``inputs`` (the reference's input convention
  ``default_rng(seed).uniform(0.5, 2.0, var_count)``, test_codegen.py:24-26),
  ``values`` (``interpret_plan(plan, inputs).values``, codegen.py:404-446;
  the interpreter's ``outputs`` are ``values[plan.outputs]``), ``oracle``
  (``eval_numeric`` of the traced outputs, expr.py:423-484 -- stored only when
  it is not bit-identical to the interpreter's outputs, which meta.json
  records as ``oracle_bitwise``), and for sparse programs the CSR
  ``row_ptr`` / ``col_idx`` of the result matrix (sparse.py:27-58);
* ``meta.json`` -- how it was made (program, pattern, seed, config flags).

The fixtures pin the oracle restatement (oracle/) and the GPU backend; the
GPU box never needs /root/reference.
"""

from __future__ import annotations

import json
import shutil
import sys
from pathlib import Path

import numpy as np

sys.setrecursionlimit(100000)

from sparsegen.codegen import PlanConfig, build_plan, interpret_plan, save_plan  # noqa: E402
from sparsegen.decompose import TraceSession  # noqa: E402
from sparsegen.expr import (  # noqa: E402
    ExprArena,
    OpKind,
    eval_numeric,
    sym_cos,
    sym_exp,
    sym_log,
    sym_select,
    sym_sin,
    sym_sqrt,
)
from sparsegen.programs import ProgramSpec, trace_program  # noqa: E402
from sparsegen.sparse import (  # noqa: E402
    GridMesh,
    MeshLaplacianSpec,
    build_operator,
    random_pattern,
    sp_add,
    sp_mul,
    sp_transpose,
    symbolic_matrix,
    vertex_coordinate_vars,
)

OUT = Path(__file__).resolve().parent


def _inputs(arena, seed):
    return np.random.default_rng(seed).uniform(0.5, 2.0, arena.var_count)


def emit(name, session, cfg, seed, meta, csr=None, inputs=None):
    plan = build_plan(session, cfg)
    vals = _inputs(session.arena, seed) if inputs is None else inputs
    res = interpret_plan(plan, vals, check_schedule=True)
    oracle = np.array(eval_numeric(session.arena, session.outputs, list(vals)), dtype=np.float64)
    d = OUT / name
    if d.exists():
        shutil.rmtree(d)
    save_plan(plan, d)
    stats = d / "stats.json"
    if stats.exists():
        stats.unlink()  # wall-clock stage times are not deterministic
    bitwise = bool(np.array_equal(res.outputs.view(np.uint64), oracle.view(np.uint64)))
    # outputs == values[plan.outputs]; the oracle is stored only where it differs
    # (simplify on reassociates, F5), otherwise it equals outputs bit for bit
    arrays = dict(inputs=np.asarray(vals, dtype=np.float64), values=res.values)
    if not bitwise:
        arrays["oracle"] = oracle
    if csr is not None:
        arrays["row_ptr"] = np.asarray(csr.row_ptr, dtype=np.int64)
        arrays["col_idx"] = np.asarray(csr.col_idx, dtype=np.int64)
    np.savez_compressed(d / "vectors.npz", **arrays)
    m = dict(meta)
    m.update(
        name=name,
        seed=seed,
        config=cfg.describe(),
        t_ref=cfg.t_ref,
        t_compl=cfg.t_compl,
        kernels=len(plan.kernels),
        outputs=len(plan.outputs),
        violations=res.violations,
        oracle_bitwise=bitwise,
    )
    (d / "meta.json").write_text(json.dumps(m, indent=1, sort_keys=True) + "\n")
    print(f"{name:40s} kernels={len(plan.kernels):4d} outputs={len(plan.outputs):7d} "
          f"|P|={plan.positions.size:8d} |C|={plan.constants.size:6d} "
          f"oracle_bitwise={m['oracle_bitwise']}")


# -- the reference's own test programs (pkg/tests) --------------------------------------


def toy_256_group():
    """test_codegen.py:39-58"""
    arena = ExprArena()
    outs = []
    rng = np.random.default_rng(11)
    for k in range(256):
        base = 4 * k
        x0, x1, x2 = arena.var(base), arena.var(base + 1), arena.var(base + 2)
        c0 = arena.const(float(rng.integers(2, 40)))
        c1 = arena.const(float(rng.integers(2, 40)) + 0.5)
        t = x0 * x1
        outs.append((c0 * t + 2.0 * c1 * x2 * sym_sqrt(t)).ref)
    arena.make_var(1023)
    return TraceSession(arena, outputs=outs)


def trace_product_program(n=24, seed=3):
    """test_codegen.py:29-36"""
    arena = ExprArena()
    A, nxt = symbolic_matrix(arena, n, n, random_pattern(n, 3, seed=seed))
    B, nxt = symbolic_matrix(arena, n, n, random_pattern(n, 3, seed=seed + 1), first_var=nxt)
    C, nxt = symbolic_matrix(arena, n, n, random_pattern(n, 3, seed=seed + 2), first_var=nxt)
    out = sp_mul(sp_add(A, B), sp_add(sp_mul(A, B), C))
    return TraceSession(arena, outputs=list(out.values)), out


def coordinate_toy(instances=96):
    """test_acceptance.py:307-320"""
    arena = ExprArena()
    outs = []
    rng = np.random.default_rng(31)
    for k in range(instances):
        x0, x1, x2 = arena.var(3 * k), arena.var(3 * k + 1), arena.var(3 * k + 2)
        c0 = arena.const(float(rng.integers(2, 30)) + 0.25)
        t = x0 * x1
        outs.append((c0 * t + 2.0 * x2 * sym_sqrt(t)).ref)
    return TraceSession(arena, outputs=outs)


def transcendental_37():
    """test_emit.py:94-113 (sin/cos/exp/log/pow^3/select, 37 instances)."""
    arena = ExprArena()
    outs = []
    for k in range(37):
        x = arena.var(2 * k)
        y = arena.var(2 * k + 1)
        e = sym_sin(x) * sym_cos(y) + sym_exp(x / (y + 3.0)) - sym_log(y + 1.5) + x**3
        e = e + sym_select(x - y, x * 2.0, y * 0.5)
        outs.append(e.ref)
    return TraceSession(arena, outputs=outs)


def self_ref_block():
    """test_codegen.py:240-250 / test_emit.py:116-130"""
    arena = ExprArena()
    a, b = arena.var(0), arena.var(1)
    m0 = (a * b + a).ref
    m1 = arena.apply(OpKind.MUL, (m0, b.ref))
    session = TraceSession(arena, outputs=[m0, m1])
    session.tag_block([m0, m1], block_id=0)
    return session


def self_ref_many(n=300):
    """Self-referencing blocks with many instances (lane-parallel edge case)."""
    arena = ExprArena()
    session = TraceSession(arena)
    for k in range(n):
        a, b = arena.var(2 * k), arena.var(2 * k + 1)
        m0 = (a * b + a).ref
        m1 = arena.apply(OpKind.MUL, (m0, b.ref))
        m2 = arena.apply(OpKind.ADD, (m1, m0, a.ref))
        session.add_outputs([m0, m1, m2])
        session.tag_block([m0, m1, m2], block_id=k)
    return session


def tagged_pair():
    """test_codegen.py:222-237"""
    arena = ExprArena()
    a, b = arena.var(0), arena.var(1)
    q = sym_sqrt(a * a + b * b)
    out0 = (b * q + a).ref
    out1 = (a * q + b).ref
    session = TraceSession(arena, outputs=[out0, out1])
    session.tag_block([out0, out1], block_id=0)
    return session


def select_nan_edge():
    """SELECT on exact zero and negative zero conditions, division by zero -> inf."""
    arena = ExprArena()
    outs = []
    for k in range(64):
        x = arena.var(2 * k)
        y = arena.var(2 * k + 1)
        e = sym_select(x - y, x / (y - y), -x)
        outs.append((e * 1.0 + x).ref)
    return TraceSession(arena, outputs=outs)


def lmlt_session(w):
    """SURVEY §8(d) C2 construction: L.M.L^T + A on a w x w cotan grid mesh."""
    arena = ExprArena()
    mesh = GridMesh(w, w)
    n = mesh.nverts
    coords = vertex_coordinate_vars(arena, n)
    spec = MeshLaplacianSpec(builder="grid", w=w, h=w, weighting="cotan")
    L, M = build_operator(arena, spec, vertex_vars=coords, with_mass=True)
    A, _ = symbolic_matrix(arena, n, n, random_pattern(n, min(6, n), seed=7), first_var=3 * n)
    out = sp_add(sp_mul(sp_mul(L, M), sp_transpose(L)), A)
    return TraceSession(arena, outputs=list(out.values)), out


def lmlt_inputs(w, seed=0):
    """Jittered grid coordinates (no degenerate triangle) + A values in U(0.5, 2)."""
    n = w * w
    rng = np.random.default_rng(seed)
    xy = np.stack(np.meshgrid(np.arange(w, dtype=np.float64), np.arange(w, dtype=np.float64),
                              indexing="xy"), -1).reshape(n, 2)
    pos = np.zeros((n, 3))
    pos[:, :2] = xy
    pos += rng.uniform(-0.25, 0.25, (n, 3))
    a = np.random.default_rng(seed + 1).uniform(0.5, 2.0, 6 * n if n >= 6 else n * n)
    return np.concatenate([pos.reshape(-1), a])


def spgemm_session(n, nnz, seeds=(1, 2)):
    """C = A.B with random_pattern(n, nnz, seed) inputs."""
    arena = ExprArena()
    A, nxt = symbolic_matrix(arena, n, n, random_pattern(n, nnz, seeds[0]))
    B, _ = symbolic_matrix(arena, n, n, random_pattern(n, nnz, seeds[1]), first_var=nxt)
    C = sp_mul(A, B)
    return TraceSession(arena, outputs=list(C.values)), C


def main(which=None):
    off = PlanConfig(simplify_enabled=False)
    on = PlanConfig(simplify_enabled=True)
    jobs = []

    def job(name, fn):
        if which is None or name.startswith(tuple(which)):
            jobs.append((name, fn))

    job("toy256", lambda: emit("toy256", toy_256_group(), off, 12, {"source": "test_codegen.py:39-58"}))
    job("toy256_interleaved", lambda: emit(
        "toy256_interleaved", toy_256_group(),
        PlanConfig(simplify_enabled=False, coalesce=False, coherence=False), 23,
        {"source": "test_emit.py:133-142"}))
    for s in (3, 4, 5):
        def _p(s=s):
            sess, out = trace_product_program(24, s)
            emit(f"product_n24_s{s}", sess, off, 7, {"source": "test_codegen.py:29-36"}, csr=out)
        job(f"product_n24_s{s}", _p)

    def _p21():  # test_emit.py:81-91 (test_compiled_matches_interpreter_bitwise): inputs seed 21
        sess, out = trace_product_program(24, 3)
        emit("product_n24_s3_seed21", sess, off, 21, {"source": "test_emit.py:81-91"}, csr=out)
    job("product_n24_s3_seed21", _p21)

    def _p0():
        sess, out = trace_product_program(24, 3)
        emit("product_n24_s3_tcompl0", sess, PlanConfig(simplify_enabled=False, t_compl=0), 9,
             {"source": "test_codegen.py:73-79"}, csr=out)
    job("product_n24_s3_tcompl0", _p0)

    def _ps():
        sess, out = trace_product_program(24, 3)
        emit("product_n24_s3_simplify", sess, on, 8, {"source": "test_codegen.py:99-105"}, csr=out)
    job("product_n24_s3_simplify", _ps)

    for name in ("expr1", "expr2", "expr3"):
        for seed in ((1, 2) if name == "expr3" else (1,)):
            def _a(name=name, seed=seed):
                tr = trace_program(ProgramSpec(name, f"random:200,6,{seed}", seed=seed))
                emit(f"acc1_{name}_s{seed}", tr.session, off, seed,
                     {"source": "test_acceptance.py:41-53", "program": name,
                      "pattern": f"random:200,6,{seed}"}, csr=tr.detail["result"])
            job(f"acc1_{name}_s{seed}", _a)
    for name, pattern in (("expr3", "random:120,5,2"), ("lpow3", "grid:10x10")):
        for simp in (False, True):
            def _b(name=name, pattern=pattern, simp=simp):
                tr = trace_program(ProgramSpec(name, pattern, seed=13))
                emit(f"acc9_{name}_{'simp' if simp else 'nosimp'}", tr.session,
                     on if simp else off, 13,
                     {"source": "test_acceptance.py:346-361", "program": name, "pattern": pattern},
                     csr=tr.detail["result"])
            job(f"acc9_{name}_{'simp' if simp else 'nosimp'}", _b)
    job("coord96", lambda: emit("coord96", coordinate_toy(), off, 17, {"source": "test_acceptance.py:307-343"}))
    job("coord96_baseline", lambda: emit(
        "coord96_baseline", coordinate_toy(),
        PlanConfig(simplify_enabled=False, coalesce=False, coherence=False), 17,
        {"source": "test_acceptance.py:307-343"}))
    job("transc37", lambda: emit("transc37", transcendental_37(), on, 22, {"source": "test_emit.py:94-113"}))
    job("transc37_nosimp", lambda: emit("transc37_nosimp", transcendental_37(), off, 22, {"source": "test_emit.py:94-113"}))
    job("selfref", lambda: emit("selfref", self_ref_block(), off, 0, {"source": "test_codegen.py:240-250"},
                                inputs=np.array([1.25, -2.5])))
    job("selfref300", lambda: emit("selfref300", self_ref_many(), off, 3, {"source": "self-referencing blocks, 300 instances"}))
    job("tagged_pair", lambda: emit("tagged_pair", tagged_pair(), off, 0, {"source": "test_codegen.py:222-237"},
                                    inputs=np.array([3.0, 4.0])))
    job("select_edge", lambda: emit("select_edge", select_nan_edge(), off, 5, {"source": "SELECT/inf edge cases"}))

    small = {
        "expr1": "random:20,3,4", "expr2": "random:20,3,4", "expr3": "random:20,3,4",
        "lpow2": "grid:4x4", "lpow3": "grid:4x4", "lpow4": "grid:3x3",
        "cotan": "grid:3x3", "energy-hessian": "grid:3x3",
    }
    for name, pattern in small.items():
        for simp in (False, True):
            def _c(name=name, pattern=pattern, simp=simp):
                tr = trace_program(ProgramSpec(name, pattern, seed=0))
                emit(f"cli_{name}_{'simp' if simp else 'nosimp'}", tr.session, on if simp else off, 0,
                     {"source": "test_cli.py:120-135", "program": name, "pattern": pattern})
            job(f"cli_{name}_{'simp' if simp else 'nosimp'}", _c)
    for name, pattern, tag in (("cotan", "grid:4x4", True), ("cotan", "grid:6x5", False),
                               ("energy-hessian", "grid:4x4", True), ("lpow3", "grid:6x6", True)):
        def _d(name=name, pattern=pattern, tag=tag):
            tr = trace_program(ProgramSpec(name, pattern, seed=0, tag=tag))
            emit(f"prog_{name}_{pattern.split(':')[1]}_{'tag' if tag else 'notag'}", tr.session,
                 off, 4, {"source": "test_programs.py:81-164", "program": name, "pattern": pattern})
        job(f"prog_{name}_{pattern.split(':')[1]}_{'tag' if tag else 'notag'}", _d)

    # C2 (L.M.L^T + A, cotan grid mesh) at small sizes: pins the scalable builder
    for w in (3, 4, 7, 12):
        def _l(w=w):
            sess, out = lmlt_session(w)
            emit(f"lmlt_w{w}", sess, off, 0, {"source": "SURVEY.md §8(d) C2", "w": w},
                 csr=out, inputs=lmlt_inputs(w))
        job(f"lmlt_w{w}", _l)
    # C1 spgemm (2k x 2k, 10 nnz/row) at full size and a small case
    for n, nnz in ((60, 4), (2000, 10)):
        def _s(n=n, nnz=nnz):
            sess, out = spgemm_session(n, nnz)
            emit(f"spgemm_n{n}_k{nnz}", sess, off, 0, {"source": "SURVEY.md §8(d) C1", "n": n, "nnz": nnz},
                 csr=out)
        job(f"spgemm_n{n}_k{nnz}", _s)

    for name, fn in jobs:
        fn()


if __name__ == "__main__":
    main(sys.argv[1:] or None)
