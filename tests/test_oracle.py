"""The oracle (oracle/interp.c) pinned against the reference's own outputs."""

import numpy as np
import pytest

from conftest import bits
from oracle import oracle


def test_oracle_matches_reference_interpreter_bitwise(golden):
    # interpret_plan(...).values of the reference, full value array, as uint64
    x = oracle.run_values(golden.plan, golden.inputs)
    assert np.array_equal(bits(x), bits(golden.values))


def test_oracle_outputs_match_eval_numeric(golden):
    out = oracle.run_outputs(golden.plan, golden.inputs)
    if golden.meta.get("reference_plan_defect"):
        # the reference's own plan is wrong here (meta.json says why); pin that it still is
        o = golden.oracle
        assert not np.allclose(out, o, rtol=1e-6, atol=0)
        return
    if golden.meta["oracle_bitwise"]:
        assert np.array_equal(bits(out), bits(golden.oracle))
    else:
        # simplify on: the reference's own contract (cli.py:118-122)
        o = golden.oracle
        assert np.all(np.abs(out - o) <= 1e-12 * np.maximum(1.0, np.maximum(np.abs(out), np.abs(o))))


def test_oracle_rejects_wrong_input_length(golden):
    import pytest

    with pytest.raises(ValueError):
        oracle.run_values(golden.plan, np.zeros(golden.plan.input_count + 1))


REF_EMIT_CASES = ["toy256", "lmlt_w7", "transc37_nosimp", "selfref", "toy256_interleaved", "spgemm_n60_k4",
                  "prog_energy-hessian_4x4_tag"]


@pytest.mark.parametrize("name", REF_EMIT_CASES)
def test_reference_emitted_c_matches_fixture_and_port(name, tmp_path):
    """The reference's own emit_kernel_source (emit.py:153-195), compiled with its flags (emit.py:220),
    reproduces the fixture values -- and so does the restated emitter used as the fallback CPU baseline."""
    import ctypes
    import subprocess

    from conftest import Golden, REFERENCE_SRC, bits
    from oracle import emit_c, make_ref

    if not REFERENCE_SRC.exists():
        pytest.skip("reference not present (GPU box)")
    g = Golden(name)
    src = tmp_path / "k.c"
    src.write_text(make_ref.reference_emitter()(g.plan, parallel="pragma"))
    lib = tmp_path / "k.so"
    subprocess.run(["cc", "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-o", str(lib), str(src), "-lm"],
                   check=True, capture_output=True)
    dll = ctypes.CDLL(str(lib))
    dll.sg_run.argtypes = [ctypes.c_void_p] * 3
    con = np.ascontiguousarray(g.plan.constants, dtype=np.float64)
    pos = np.ascontiguousarray(g.plan.positions, dtype=np.uint32)
    x = np.zeros(g.plan.value_array_size)
    x[: g.plan.input_count] = g.inputs
    dll.sg_run(x.ctypes.data, con.ctypes.data if con.size else None, pos.ctypes.data if pos.size else None)
    if g.exact:
        assert np.array_equal(bits(x), bits(g.values))
    else:  # libm transcendentals: glibc on both sides, still expect equality
        assert np.allclose(x, g.values, rtol=1e-12, atol=0, equal_nan=True)
    port = emit_c.compile_plan(g.plan, parallel="pragma", work_dir=tmp_path)(g.inputs)
    assert np.array_equal(bits(port), bits(x))


def test_numpy_interpreter_restatement_matches_reference(golden):
    """oracle/interp_np.py (the timed single-core interpreter leg of bench.py) == interpret_plan, bitwise."""
    from oracle import interp_np

    x, skipped = interp_np.interpret(golden.plan, golden.inputs)
    assert skipped == 0
    assert np.array_equal(bits(x), bits(golden.values))


def test_glibc_math_header_matches_this_libm():
    """csrc/glibc_math.h holds this image's glibc tables (__log_data, __exp_data, __pow_log_data), and
    the restatements it implements equal math.log / math.exp / math.pow -- the reference's LOG / EXP /
    POW -- bit for bit on a random sample (tools/gen_glibc_math.py)."""
    import re
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root / "tools"))
    import gen_glibc_math as g

    t = g.read_tables(g.libm_path())
    text = (root / "paper_2110_12865_b200" / "csrc" / "glibc_math.h").read_text()
    hexf = r"(-?0x[0-9a-f.]+p[-+]\d+)"
    tab = [float.fromhex(v) for v in re.findall(hexf, text.split("sgb_log_tab")[1])[: 2 * g.N_TAB]]
    assert tab == list(t["log_tab"])
    ptab = [float.fromhex(v) for v in re.findall(hexf, text.split("sgb_pow_tab")[1])[: 3 * g.N_TAB]]
    assert ptab == [t["pow_tab"][4 * j + q] for j in range(g.N_TAB) for q in (0, 2, 3)]
    etab = [int(v, 16) for v in re.findall(r"0x([0-9a-f]{16})ull", text.split("sgb_exp_tab")[1])[: 2 * g.N_TAB]]
    assert etab == list(t["exp_tab"])
    sct = [float.fromhex(v) for v in re.findall(hexf, text.split("sgb_sincostab")[1])[:440]]
    assert sct == list(t["sincostab"])
    assert g.verify(t, 3000) == []
