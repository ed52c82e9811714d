"""ORACLE / CPU BASELINE -- TEST INFRASTRUCTURE ONLY (see oracle/README.md).

Restatement of the reference's native CPU evaluator: ``emit_kernel_source`` +
``compile_plan`` (/root/reference/pkg/src/sparsegen/emit.py:153-245).  Used by
bench.py's ``cpu_baseline`` / ``--impl reference`` legs as the timed CPU
reference and by tests as a second checker; the product never imports it.

Same program shape as the reference emitter:

* one ``static void kN(double* x, const double* c, const unsigned* p)`` per
  kernel, an outer chunk loop over ``instances / vector_width`` (annotated
  ``#pragma omp parallel for`` when ``parallel="pragma"``) around an inner
  ``#pragma omp simd`` loop of ``vector_width``, plus a scalar tail
  (emit.py:166-188);
* hoisted slot loads ``x{s}`` through the coalesced / interleaved index
  tables, coherent slots as ``p[slot0] + delta`` (emit.py:108-124), constant
  slots ``c{s}`` (emit.py:121-124);
* the template's live nodes evaluated in stored order with the left-fold of
  n-ary ADD / MUL (emit.py:63-71), ``pow(b, k.0)`` (emit.py:81-83) and
  ``(c < 0.0 ? t : f)`` (emit.py:84-86); self-referencing kernels load
  through ``x`` again for every root (emit.py:96, 114-124, interpreter
  semantics codegen.py:505-510);
* ``sg_run`` calls the kernels in schedule order (emit.py:190-193);
* compiled with the reference flags ``cc -O3 -ffp-contract=off -fPIC -shared
  ... -lm`` (emit.py:220), plus ``-fopenmp`` for the all-core baseline.

Differences (documented, arithmetic-neutral): every live node becomes a
``const double`` local instead of only the ``local_decompose`` set (the
expression is identical, the compiler allocates registers), and rendering is
iterative (the reference printer recurses and overflows on deep templates,
SURVEY H6).
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
CACHE = HERE / "_build" / "emitted"

_OPS = {2: "+", 3: "-", 4: "*", 5: "/"}
_FUNC = {7: "sqrt", 8: "sin", 9: "cos", 10: "exp", 11: "log"}


def _c_double(v: float) -> str:
    """Round-trip literal (emit.py:37-41)."""
    v = float(v)
    if v == int(v) and abs(v) < 1e16:
        return f"{int(v)}.0"
    return repr(v)


def _reachable(tmpl, roots):
    n = len(tmpl.ops)
    need = bytearray(n)
    for r in roots:
        need[r] = 1
    for i in range(n - 1, -1, -1):
        if need[i]:
            for c in tmpl.args[i]:
                need[c] = 1
    return [i for i in range(n) if need[i]]


def _kernel_body(kp, idx: str) -> list[str]:
    n = kp.instances
    ridx = {s: k for k, s in enumerate(kp.retained)}
    nret = len(kp.retained)
    ncon = len(kp.const_vars)

    def p_entry(r):
        if kp.layout == "coalesced":
            return f"p[{kp.p_base + r * n}L + {idx}]"
        return f"p[{kp.p_base}L + {idx}*{nret}L + {r}]"

    def c_entry(s):
        if kp.layout == "coalesced":
            return f"c[{kp.c_base + s * n}L + {idx}]"
        return f"c[{kp.c_base}L + {idx}*{ncon}L + {s}]"

    loads = {}
    for s, coh in enumerate(kp.coherence):
        if s in ridx:
            loads[s] = f"x[{p_entry(ridx[s])}]"
        else:
            loads[s] = f"x[(long){p_entry(0)} + ({int(coh)}L)]"
    tmpl = kp.template_arena
    slot_of = {v: s for s, v in enumerate(kp.pos_vars)}
    cslot_of = {v: s for s, v in enumerate(kp.const_vars)}
    live = _reachable(tmpl, kp.template_roots)
    lines = []
    if not kp.self_referencing:
        for s in range(len(kp.pos_vars)):
            lines.append(f"const double x{s} = {loads[s]};")
    for s in range(ncon):
        lines.append(f"const double c{s} = {c_entry(s)};")

    def render_nodes(root_filter=None):
        out = []
        name = {}
        for ref in live:
            op = int(tmpl.ops[ref])
            a = tmpl.args[ref]
            if op == 0:
                v = tmpl.payload[ref]
                if v in slot_of:
                    s = slot_of[v]
                    name[ref] = f"x{s}" if not kp.self_referencing else f"({loads[s]})"
                else:
                    name[ref] = f"c{cslot_of[v]}"
                continue
            if op == 1:
                name[ref] = _c_double(tmpl.payload[ref])
                continue
            if op in (2, 4):
                acc = name[a[0]]
                for ch in a[1:]:
                    acc = f"({acc} {_OPS[op]} {name[ch]})"
                expr = acc
            elif op in (3, 5):
                expr = f"({name[a[0]]} {_OPS[op]} {name[a[1]]})"
            elif op == 6:
                expr = f"(-{name[a[0]]})"
            elif op in _FUNC:
                expr = f"{_FUNC[op]}({name[a[0]]})"
            elif op == 12:
                expr = f"pow({name[a[0]]}, {_c_double(tmpl.payload[a[1]])})"
            elif op == 13:
                expr = f"({name[a[0]]} < 0.0 ? {name[a[1]]} : {name[a[2]]})"
            else:
                raise ValueError(f"unknown op {op}")
            out.append(f"const double t{ref} = {expr};")
            name[ref] = f"t{ref}"
        return out, name

    if not kp.self_referencing:
        body, name = render_nodes()
        lines += body
        for r, root in enumerate(kp.template_roots):
            lines.append(f"x[{kp.dest_base + r * n}L + {idx}] = {name[root]};")
    else:
        for r, root in enumerate(kp.template_roots):
            body, name = render_nodes()
            lines.append("{")
            lines += body
            lines.append(f"x[{kp.dest_base + r * n}L + {idx}] = {name[root]};")
            lines.append("}")
    return lines


def emit_kernel_source(plan, parallel: str = "none") -> str:
    if parallel not in ("none", "pragma"):
        raise ValueError(f"parallel must be 'none' or 'pragma', got {parallel!r}")
    w = int(plan.vector_width)
    out = ["/* generated kernel source; compile with: cc -O3 -ffp-contract=off */",
           "#include <math.h>", ""]
    for k, kp in enumerate(plan.kernels):
        n = kp.instances
        full = n // w
        out.append(f"static void k{k}(double* x, const double* c, const unsigned* p) {{")
        body = _kernel_body(kp, "i")
        if full:
            if parallel == "pragma":
                out.append("    #pragma omp parallel for")
            out.append(f"    for (long ii = 0; ii < {full}L; ++ii) {{")
            out.append("        #pragma omp simd")
            out.append(f"        for (long j = 0; j < {w}; ++j) {{")
            out.append(f"            const long i = ii*{w} + j;")
            out += ["            " + ln for ln in body]
            out.append("        }")
            out.append("    }")
        if full * w < n:
            out.append(f"    for (long i = {full * w}L; i < {n}L; ++i) {{")
            out += ["        " + ln for ln in body]
            out.append("    }")
        out.append("}")
        out.append("")
    out.append("void sg_run(double* x, const double* c, const unsigned* p) {")
    for k in range(len(plan.kernels)):
        out.append(f"    k{k}(x, c, p);")
    out.append("}")
    return "\n".join(out) + "\n"


def compile_plan(plan, parallel: str = "none", openmp: bool = False, work_dir=None):
    """Emit + ``cc -O3 -ffp-contract=off -fPIC -shared`` (emit.py:220) -> run(x)."""
    src_text = emit_kernel_source(plan, parallel=parallel)
    tag = hashlib.sha1((src_text + str(openmp)).encode()).hexdigest()[:16]
    work = Path(work_dir) if work_dir else CACHE
    work.mkdir(parents=True, exist_ok=True)
    src = work / f"k_{tag}.c"
    lib = work / f"k_{tag}{'_omp' if openmp else ''}.so"
    if not lib.exists():
        src.write_text(src_text)
        cmd = ["cc", "-O3", "-ffp-contract=off", "-fPIC", "-shared"]
        if openmp:
            cmd.append("-fopenmp")
        tmp = lib.with_suffix(f".{os.getpid()}.tmp")
        cmd += ["-o", str(tmp), str(src), "-lm"]
        subprocess.run(cmd, check=True, capture_output=True)
        os.replace(tmp, lib)
    dll = ctypes.CDLL(str(lib))
    dll.sg_run.restype = None
    dll.sg_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    constants = np.ascontiguousarray(plan.constants, dtype=np.float64)
    positions = np.ascontiguousarray(plan.positions, dtype=np.uint32)

    def sg_run(x: np.ndarray) -> np.ndarray:
        dll.sg_run(x.ctypes.data, constants.ctypes.data if constants.size else None,
                   positions.ctypes.data if positions.size else None)
        return x

    def run(inputs) -> np.ndarray:
        x = np.zeros(plan.value_array_size, dtype=np.float64)
        x[: plan.input_count] = np.asarray(inputs, dtype=np.float64)
        return sg_run(x)

    run.sg_run = sg_run
    run.library_path = lib
    run.source_path = src
    return run
