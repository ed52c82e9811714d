"""C1's CPU reference is "plan build + evaluate": the reference's
own trace of C = A.B (random_pattern 2000 x 2000, 10 nnz/row, seeds 1, 2; sparse.py:102-139,
199-246) plus ``build_plan`` (codegen.py:127-314), timed here -- the reference package exists only
in the build container, not on the GPU box -- and written to profiles/r2/c1_plan_build.json, which
bench.py reports beside the evaluation timings it measures on the box.

    python tools/ref_plan_build.py [--reps 3]
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    from sparsegen.codegen import PlanConfig, build_plan
    from sparsegen.expr import ExprArena
    from sparsegen.programs import TraceSession
    from sparsegen.sparse import random_pattern, sp_mul, symbolic_matrix

    trace_s, plan_s = [], []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        arena = ExprArena()
        A, nxt = symbolic_matrix(arena, 2000, 2000, random_pattern(2000, 10, 1))
        B, _ = symbolic_matrix(arena, 2000, 2000, random_pattern(2000, 10, 2), first_var=nxt)
        C = sp_mul(A, B)
        session = TraceSession(arena, outputs=list(C.values))
        t1 = time.perf_counter()
        plan = build_plan(session, PlanConfig(simplify_enabled=False))
        t2 = time.perf_counter()
        trace_s.append(t1 - t0)
        plan_s.append(t2 - t1)
    cpu = "unknown"
    for line in Path("/proc/cpuinfo").read_text().splitlines():
        if line.startswith("model name"):
            cpu = line.split(":", 1)[1].strip()
            break
    rec = {"config": "C1 spgemm 2000x2000, 10 nnz/row (seeds 1, 2)", "out_nnz": len(plan.outputs),
           "trace_s": min(trace_s), "build_plan_s": min(plan_s), "reps": args.reps,
           "how": "reference sparsegen (symbolic_matrix + sp_mul trace, build_plan simplify off), min of reps, "
                  "one core", "cpu": cpu, "host": platform.node(), "threads": 1,
           "measured_in": "build container (the reference is not installed on the GPU box)"}
    out = ROOT / "profiles" / "r2" / "c1_plan_build.json"
    out.write_text(json.dumps(rec, indent=1) + "\n")
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
