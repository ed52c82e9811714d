"""ORACLE / CPU BASELINE RECIPE -- TEST INFRASTRUCTURE ONLY.

Generates the reference's OWN native evaluator for the bench plans: the C99
translation unit that ``sparsegen.emit.emit_kernel_source``
(/root/reference/pkg/src/sparsegen/emit.py:153-195) emits for a plan, written
to ``oracle/ref_emitted/<key>.c`` together with a fingerprint of the plan it was
emitted for.  bench.py compiles it on the GPU box with the reference's flags
(``cc -O3 -ffp-contract=off -fPIC -shared ... -lm``, emit.py:220, plus
``-fopenmp`` for the all-core figure) and times ``sg_run`` as the
``cpu_baseline`` (kind "reference").

Runs only where /root/reference exists (this build container);
The emitted sources are committed (``oracle/ref_emitted/``, a few hundred KB): they are the
reference's output for the bench plans, like the golden fixtures, so the reference arm never has
to fall back to the restated emitter on a box without /root/reference.
The emitter is used unmodified: it reads only the plan fields
(codegen.py:56-98), so the template-instancing builder's plans go through it
as they are.

    python oracle/make_ref.py [--w 1000]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
REF_DIR = HERE / "ref_emitted"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def plan_fingerprint(plan) -> str:
    """Identity of everything the emitted source bakes in (layout + templates)."""
    h = hashlib.sha1()
    h.update(np.ascontiguousarray(plan.positions, dtype=np.uint32).tobytes())
    h.update(np.asarray(plan.outputs, dtype=np.int64).tobytes())
    for kp in plan.kernels:
        h.update(repr((kp.name, kp.instances, kp.n_roots, kp.dest_base, kp.p_base, kp.c_base, kp.layout,
                       list(kp.pos_vars), list(kp.const_vars), list(kp.coherence), list(kp.retained),
                       len(kp.template_arena.ops), list(kp.template_roots))).encode())
    h.update(repr((plan.value_array_size, plan.input_count, plan.vector_width)).encode())
    return h.hexdigest()


def builder_hash() -> str:
    sys.path.insert(0, str(ROOT))
    from paper_2110_12865_b200.programs import builder_hash as bh

    return bh()


def up_to_date(key: str) -> bool:
    """Cheap staleness check for build(): same builder sources as when the source was emitted."""
    meta = REF_DIR / f"{key}.json"
    return (REF_DIR / f"{key}.c").exists() and meta.exists() and \
        json.loads(meta.read_text()).get("builder_hash") == builder_hash()


def reference_emitter():
    if not REFERENCE_SRC.exists():
        raise RuntimeError("/root/reference is not present: the reference emitter cannot run here")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    sys.setrecursionlimit(max(sys.getrecursionlimit(), 100000))  # emit.py:53-87 recurses
    from sparsegen.emit import emit_kernel_source

    return emit_kernel_source


def emit_for_plan(plan, key: str, parallel: str = "pragma") -> Path:
    emit = reference_emitter()
    REF_DIR.mkdir(parents=True, exist_ok=True)
    src = REF_DIR / f"{key}.c"
    src.write_text(emit(plan, parallel=parallel))
    (REF_DIR / f"{key}.json").write_text(json.dumps({
        "key": key, "fingerprint": plan_fingerprint(plan), "parallel": parallel, "builder_hash": builder_hash(),
        "emitter": "sparsegen.emit.emit_kernel_source (/root/reference/pkg/src/sparsegen/emit.py:153-195)",
    }, indent=1))
    return src


def lookup(plan, key: str):
    """(source path, fingerprint ok) for a plan, or (None, False)."""
    src, meta = REF_DIR / f"{key}.c", REF_DIR / f"{key}.json"
    if not src.exists() or not meta.exists():
        return None, False
    return src, json.loads(meta.read_text()).get("fingerprint") == plan_fingerprint(plan)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--w", type=int, default=1000)
    ap.add_argument("--if-stale", action="store_true")
    ap.add_argument("--golden", nargs="*", default=["spgemm_n2000_k10"],
                    help="also emit for these reference-built golden plans (bench C1)")
    args = ap.parse_args()
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2110_12865_b200.plan import load_plan

    for name in args.golden:
        if args.if_stale and (REF_DIR / f"{name}.c").exists():
            continue
        src = emit_for_plan(load_plan(ROOT / "tests" / "golden" / name), name)
        print(f"wrote {src}")
    ns = bench.parse_args(["--w", str(args.w)])
    for cfg in ("c2", "c5", "c3", "c4"):
        key = bench.workload_key(cfg, ns)
        if args.if_stale and up_to_date(key):
            print(f"oracle/ref_emitted/{key}.c is up to date")
            continue
        key, plan = bench.build_workload(cfg, ns)
        src = emit_for_plan(plan, key)
        print(f"wrote {src} ({src.stat().st_size / 1e6:.1f} MB) for {key}")



if __name__ == "__main__":
    main()
