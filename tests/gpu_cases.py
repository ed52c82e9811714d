"""Which lowerings the GPU parity suite runs, and the NVRTC pre-compilation of their cubins.

The specialised kernels (paper_2110_12865_b200/jit.py) are compiled by NVRTC
when a plan is lowered.  NVRTC needs no GPU, so ``warm()`` -- called by
``__graft_entry__.build()`` on the CPU host -- compiles every cubin the GPU
suite needs into the in-tree cache (jit.CACHE), which travels with the
repository to the GPU box: ``pytest -m gpu`` on a cold box then spends its
time on the GPU, not in NVRTC.

Default lowering (``jit_min_n`` = 4096) runs for every fixture; every group
specialised (``jit_min_n=0``) and the CSR layout (``relayout="all"``) run for
the subsets below, which cover every template shape in the fixtures (sums of
products, multi-root element templates, transcendental / select / POW tapes,
interleaved and coherent index forms).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

# every group specialised (jit_min_n = 0): specialised == hand-written, tile schedules, shards
JIT_CASES = ["lmlt_w7", "lmlt_w12", "prog_energy-hessian_4x4_tag", "transc37", "transc37_nosimp",
             "toy256_interleaved", "tagged_pair", "acc9_lpow3_simp", "spgemm_n60_k4", "selfref", "coord96",
             "select_edge", "prog_cotan_4x4_tag", "cli_lpow4_simp", "fem_nh_m1", "arap_w3"]
# CSR layout (multi-root groups stored instance-major): every fixture with a relayout candidate
# at jit_min_n = 0 plus representatives without one
LAYOUT_CASES = ["fem_nh_m1", "fem_nh_m2", "prog_energy-hessian_4x4_tag", "arap_w3", "arap_w5", "prog_cotan_4x4_tag",
                "lmlt_w7", "transc37", "selfref", "toy256_interleaved"]

# CSR windows forced on (csr_window=True): the fixtures whose last wave qualifies with at most 25
# members (the default lowering applies windows only to big plans, lower.lower_plan)
WINDOW_CASES = ["acc1_expr2_s1", "acc9_lpow3_nosimp", "acc9_lpow3_simp", "arap_w3", "arap_w5", "cli_expr2_nosimp",
                "cli_expr2_simp", "cli_lpow2_simp", "cli_lpow3_simp", "cli_lpow4_nosimp", "cli_lpow4_simp", "coord96",
                "coord96_baseline", "lmlt_w12", "lmlt_w3", "lmlt_w4", "lmlt_w7", "product_n24_s3_tcompl0",
                "prog_lpow3_6x6_tag", "select_edge", "spgemm_n2000_k10", "spgemm_n60_k4", "tagged_pair", "toy256",
                "toy256_interleaved", "transc37", "transc37_nosimp"]


def lowering_specs(names: list[str]) -> list[tuple[str, tuple]]:
    specs = [(n, ()) for n in names]
    specs += [(n, (("jit_min_n", 0),)) for n in JIT_CASES]
    specs += [(n, (("jit_min_n", 0), ("relayout", r))) for n in LAYOUT_CASES for r in ("all", "auto")]
    specs += [(n, (("csr_window", False),)) for n in names]
    specs += [(n, (("csr_window", True),)) for n in WINDOW_CASES]
    specs += [(n, (("direct_csr", True),)) for n in names]
    specs += [(n, (("relayout", r), ("wbulk", b))) for n in BUILDER_CASES for r in (False, "auto")
              for b in (True, False)]
    return specs


# builder plans the GPU suite runs beyond the fixtures: C2 (CSR windows), C3 (CSR layout), C4 (gather)
# at small sizes
BUILDER_CASES = {"lmlt_w70": ("mesh", 70), "lmlt_w65": ("mesh", 65), "fem_m9": ("fem", 9), "arap_w70": ("arap", 70)}


def builder_plan(name: str):
    sys.path.insert(0, str(ROOT))
    from paper_2110_12865_b200.programs.arap import arap_inputs, build_arap_plan
    from paper_2110_12865_b200.programs.fem import build_fem_plan, fem_inputs
    from paper_2110_12865_b200.programs.mesh import build_lmlt_plan, lmlt_inputs

    kind, size = BUILDER_CASES[name]
    build, inputs = {"mesh": (build_lmlt_plan, lmlt_inputs), "fem": (build_fem_plan, fem_inputs),
                     "arap": (build_arap_plan, arap_inputs)}[kind]
    return build(size)[0], inputs(size, seed=1)


def _lower_one(spec):
    name, kw = spec
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    from conftest import Golden
    from paper_2110_12865_b200 import jit
    from paper_2110_12865_b200.lower import lower_plan

    plan = builder_plan(name)[0] if name in BUILDER_CASES else Golden(name).plan
    lower_plan(plan, **dict(kw))
    return jit.stats["compiles"]


def warm(processes: int | None = None) -> int:
    """Compile every cubin the GPU suite lowers (cache hits are free); returns NVRTC compiles."""
    import multiprocessing as mp

    sys.path.insert(0, str(ROOT / "tests"))
    from conftest import golden_names
    from paper_2110_12865_b200 import jit

    if not jit.available():
        return 0
    specs = lowering_specs(golden_names())
    # biggest first so the long compiles overlap
    specs.sort(key=lambda s: -(10 ** 9 if s[0] in BUILDER_CASES else
                               sum(p.stat().st_size for p in (ROOT / "tests" / "golden" / s[0]).iterdir())))
    procs = processes or min(len(specs), os.cpu_count() or 1)
    with mp.get_context("spawn").Pool(procs) as pool:
        return sum(pool.map(_lower_one, specs, chunksize=1))


if __name__ == "__main__":
    import time

    t0 = time.perf_counter()
    n = warm()
    print(f"warm: {n} NVRTC compiles in {time.perf_counter() - t0:.1f}s")
