"""Device-plan lowering, proven on CPU through an emulator of the kernels."""

import numpy as np
import pytest

import device_plan_emu as emu
from conftest import bits
from paper_2110_12865_b200.lower import (
    KIND_SOP, KIND_TAPE, compute_waves, lower_plan, recognise_sop,
)
from paper_2110_12865_b200 import lower as L
from paper_2110_12865_b200.plan import load_plan


def test_emulated_device_plan_matches_reference_bitwise(golden):
    dp = lower_plan(golden.plan, jit=False)
    x = emu.run_values(dp, golden.inputs)
    assert np.array_equal(bits(x), bits(golden.values))


def test_emulated_csr_mode_matches_reference_outputs(golden):
    """CSR mode: producers store outputs at their CSR positions, copy groups cover the rest."""
    dp = lower_plan(golden.plan, direct_csr=True, jit=False)
    emu.check_tiles(dp)
    out = emu.run_csr(dp, golden.inputs)
    assert np.array_equal(bits(out), bits(golden.outputs))


@pytest.mark.parametrize("wbulk", [False, True])
@pytest.mark.parametrize("jit_min_n", [None, 0])
def test_emulated_csr_windows_match_reference_outputs(golden, jit_min_n, wbulk):
    """CSR windows (lower._csr_windows, jit.window_source / wbulk_source): every output lands exactly
    once, from its member's piece or the window's copy list, bit for bit; with the bulk feed the
    emulator rebuilds every ring slot from the blobs and intervals (lower.WindowBulk); plans that do
    not qualify keep the gather."""
    dp = lower_plan(golden.plan, csr_window=True, jit_min_n=jit_min_n, jit_compile=False, wbulk=wbulk)
    assert (dp.wbulk is not None) <= wbulk
    out = emu.run_csr(dp, golden.inputs)
    want = golden.outputs
    if golden.exact:
        assert np.array_equal(bits(out), bits(want))
    else:
        assert np.allclose(out, want, rtol=1e-12, atol=1e-12)
    if dp.windows is not None:
        wn = dp.windows
        assert wn.k[0] == 0 and wn.k[-1] == len(golden.plan.outputs) and np.all(np.diff(wn.k) > 0)
        assert np.diff(wn.k).max() <= L.WIN_MAX
        # every position written once: copies + member results partition each window
        hits = np.zeros(len(golden.plan.outputs), np.int64)
        u = dp.unit(dp.window_units[0][0])
        for w in range(wn.k.size - 1):
            k0 = int(wn.k[w])
            c0, c1 = wn.copy_off[w], wn.copy_off[w + 1]
            np.add.at(hits, k0 + wn.copy_pos[c0:c1].astype(np.int64), 1)
            for gi in range(u["group_begin"], u["group_end"]):
                a, cnt = (int(v) for v in wn.pieces[w, gi - u["group_begin"]])
                g = dp.groups[gi]
                n = int(g["n"])
                for r in range(int(g["n_roots"])):
                    o = dp.ooff[int(g["oo_off"]) + r * n + a: int(g["oo_off"]) + r * n + a + cnt].astype(np.int64)
                    np.add.at(hits, k0 + o[o != 0xFFFF], 1)
        assert np.all(hits == 1)


def test_csr_windows_on_the_c2_builder_plan():
    """On the mesh builder's L.M.L^T+A plan the windows qualify, hold ~WIN_ROWS rows, and the anchor
    pieces are one block pass."""
    from paper_2110_12865_b200.programs.mesh import build_lmlt_plan, lmlt_inputs

    from oracle import oracle

    plan, _, _ = build_lmlt_plan(40)
    ins = lmlt_inputs(40, seed=3)
    want = bits(oracle.run_outputs(plan, ins))
    for wbulk in (False, True):
        dp = lower_plan(plan, csr_window=True, jit_compile=False, wbulk=wbulk)
        assert dp.windows is not None and len(dp.window_units) == 1
        cnt = dp.windows.pieces[:, :, 1]
        assert np.median(cnt.max(axis=1)) <= 256
        assert np.array_equal(bits(emu.run_csr(dp, ins)), want)
        if wbulk:  # every bulk member's runs are merged into aligned intervals of the value array
            wb = dp.wbulk
            assert wb is not None and len(wb.members) >= 10
            assert np.all(wb.iv % 2 == 0) and np.all(wb.iv[:, 1] > 0)
            assert np.all(wb.meta_off % 16 == 0) and wb.smem <= L.WBULK_SMEM


def test_waves_respect_producers(golden):
    plan = golden.plan
    waves = compute_waves(plan)
    from paper_2110_12865_b200.plan import slot_addresses

    ranges = [(kp.dest_base, kp.dest_base + kp.n_roots * kp.instances) for kp in plan.kernels]
    for k, kp in enumerate(plan.kernels):
        reads = np.concatenate(slot_addresses(plan, kp)) if kp.pos_vars else np.zeros(0, np.int64)
        for j, (lo, hi) in enumerate(ranges):
            if j != k and np.any((reads >= lo) & (reads < hi)):
                if j < k:
                    assert waves[j] < waves[k]
                else:  # read before write in schedule order: must still see zeros
                    assert waves[k] < waves[j]


def test_lmlt_is_mostly_sum_of_products():
    plan = load_plan("tests/golden/lmlt_w12")
    dp = lower_plan(plan, direct_csr=True, jit=False)
    n_sop = int(np.sum(dp.groups["kind"] == KIND_SOP))
    assert n_sop >= len(plan.kernels) // 2
    assert dp.n_waves == 5  # L.M.L^T + A needs 5 waves
    # the output groups write their CSR positions directly
    assert np.sum((dp.groups["flags"] & (L.FLAG_OPOS16 | L.FLAG_OPOS32)) != 0) >= 5


def test_builder_plan_csr_mode_copy_group():
    """Builder plan: A-only outputs are input slots -> one CSR-only copy group in the last wave."""
    from oracle import oracle
    from paper_2110_12865_b200.programs.mesh import build_lmlt_plan, lmlt_inputs

    plan, _, _ = build_lmlt_plan(20)
    dp = lower_plan(plan, direct_csr=True, jit=False)
    copy = (dp.groups["flags"] & L.FLAG_CSR_ONLY) != 0
    assert copy.sum() == 1 and dp.needs_zero == L.ZERO_ONCE  # structural gaps read as zero
    assert int(dp.units[-1][0]) == dp.n_waves - 1  # no extra CSR-only wave: sources are inputs
    inputs = lmlt_inputs(20)
    assert np.array_equal(bits(emu.run_csr(dp, inputs)), bits(oracle.run_outputs(plan, inputs)))


def test_sop_rejects_right_nested_products():
    plan = load_plan("tests/golden/acc1_expr2_s1")
    kp = plan.kernels[0]  # v0 * (v1 * v2): not a left fold of three factors
    assert recognise_sop(kp) is None


def test_broken_schedule_still_matches_interpreter(tmp_path):
    # a producer moved behind its consumers (test_codegen.py:209-216): the
    # reference reads zeros; the wave builder must reproduce that
    from oracle import oracle

    plan = load_plan("tests/golden/product_n24_s3_tcompl0")
    plan.kernels.append(plan.kernels.pop(0))
    inputs = np.random.default_rng(0).uniform(0.5, 2.0, plan.input_count)
    want = oracle.run_values(plan, inputs)
    dp = lower_plan(plan, jit=False)
    assert dp.needs_zero == L.ZERO_EVERY
    got = emu.run_values(dp, inputs)
    assert np.array_equal(bits(got), bits(want))


def test_tape_register_reuse_bounded():
    plan = load_plan("tests/golden/prog_energy-hessian_4x4_tag")
    dp = lower_plan(plan, jit=False)
    for kl, kp in zip(dp.kernels, plan.kernels):
        if kl.kind == KIND_TAPE:
            live = len(kp.template_arena.ops)
            assert kl.n_regs <= live + len(kp.pos_vars) + len(kp.const_vars)


def test_sop_shapes():
    N, NEG = L.SOP_NEWTERM, L.SOP_NEG
    assert L.sop_shape([N, N | NEG, N]) == L.SOP_SHAPE_SUM
    assert L.sop_shape([N, 0, N, 0]) == L.SOP_SHAPE_PAIRS
    assert L.sop_shape([N, 0, N | NEG, 0, N]) == L.SOP_SHAPE_PAIRS  # two products + single tail
    assert L.sop_shape([N, 0, 0]) == L.SOP_SHAPE_GENERIC  # one three-factor product
    assert L.sop_shape([N, 0, N]) == L.SOP_SHAPE_PAIRS
    assert L.sop_shape([N, N, 0]) == L.SOP_SHAPE_GENERIC


JIT_CASES = ["lmlt_w7", "prog_energy-hessian_4x4_tag", "transc37", "toy256_interleaved", "tagged_pair",
             "acc9_lpow3_simp", "spgemm_n60_k4", "selfref", "coord96"]


@pytest.mark.parametrize("name", JIT_CASES)
def test_specialised_tape_units_compile(name):
    """jit.py: the tape units compile to sm_100a cubins with NVRTC (no GPU needed)."""
    from conftest import Golden
    from paper_2110_12865_b200 import jit

    if not jit.available():
        pytest.skip("NVRTC not available")
    dp = lower_plan(Golden(name).plan, jit=True, jit_min_n=0)
    n_jit = sum(1 for u in range(len(dp.units)) if dp.unit(u)["flags"] & L.UNIT_JIT)
    n_plain = sum(1 for kl in dp.kernels if not kl.flags & (L.FLAG_SELFREF | L.FLAG_SERIAL))
    assert (n_jit > 0) == (n_plain > 0)
    if n_jit:
        assert dp.jit_cubin[:4] == b"\x7fELF" and "sgb_tape_u" in dp.jit_source


def test_emulated_csr_layout_matches_reference_outputs(golden):
    """CSR layout (every eligible multi-root group instance-major): same CSR values bit for bit,
    and the relaid value array is a permutation of the reference one inside each moved range."""
    dp = lower_plan(golden.plan, jit=False, jit_min_n=0, relayout="all")
    emu.check_tiles(dp)
    out = emu.run_csr(dp, golden.inputs)
    assert np.array_equal(bits(out), bits(golden.outputs))
    for k in dp.csr_layout:
        kp = golden.plan.kernels[k]
        assert kp.n_roots > 1
        gi = [j for j in range(len(dp.groups)) if dp.groups[j]["flags"] & L.FLAG_IMAJOR
              and dp.groups[j]["dest_base"] == kp.dest_base]
        assert len(gi) == 1


def test_relaid_plan_remap_is_a_bijection():
    plan = load_plan(__import__("conftest").GOLDEN / "lmlt_w7")
    multi = [k for k, kp in enumerate(plan.kernels) if kp.n_roots > 1]
    if not multi:
        pytest.skip("no multi-root group")
    rp = L._RelaidPlan(plan, multi)
    a = np.arange(plan.value_array_size, dtype=np.int64)
    b = rp.remap(a)
    assert np.array_equal(np.sort(b), a)
    for k in multi:
        kp = plan.kernels[k]
        r, i = 1, kp.instances - 1
        assert b[kp.dest_base + r * kp.instances + i] == kp.dest_base + i * kp.n_roots + r


def test_window_rounds_are_balanced(monkeypatch):
    """Between one and WIN_BALANCE_ROUNDS rounds of resident windows the lowering re-chooses the rows
    per window for whole rounds; the windows still cover every output once, bit for bit."""
    from paper_2110_12865_b200.programs.mesh import build_lmlt_plan, lmlt_inputs

    from oracle import oracle

    plan, _, _ = build_lmlt_plan(40)
    monkeypatch.setattr(L, "WIN_ROWS", 64)
    monkeypatch.setattr(L, "WIN_BALANCE_ROUNDS", 1000)
    base = lower_plan(plan, csr_window=True, jit_compile=False)
    n0 = base.windows.k.size - 1
    slots = max(2, n0 // 3 + 1)  # a partial last round
    monkeypatch.setattr(L, "WIN_SLOTS", slots)
    dp = lower_plan(plan, csr_window=True, jit_compile=False)
    n = dp.windows.k.size - 1
    assert n % slots == 0 or n >= (n // slots) * slots + slots - slots // 8, (n0, n, slots)
    assert np.all(np.diff(dp.windows.k) > 0) and np.diff(dp.windows.k).max() <= L.WIN_MAX
    ins = lmlt_inputs(40, seed=5)
    assert np.array_equal(bits(emu.run_csr(dp, ins)), bits(oracle.run_outputs(plan, ins)))
