"""B200 parity: the CUDA path (through the C ABI) against the reference's outputs.

Bar: bit-exact (uint64 compare of the FULL value array) for
plans whose templates use only EXACT_OPS (codegen.py:43-53) and POW k=2;
SIN/COS/EXP/LOG/POW k>=3 within |g - o| <= 1e-12 * max(1, |g|, |o|)
(cli.py:118-122) because CUDA's libm is not glibc.

Cost control (a cold B200 box runs this file in a few minutes): lowerings and
device plans are shared per (fixture, lowering) through conftest.lowered /
conftest.device_plan, every NVRTC cubin is pre-compiled by
__graft_entry__.build() (tests/gpu_cases.py), autotuning is off except in its
own test, and the every-group-specialised / CSR-layout lowerings run on the
subsets of tests/gpu_cases.py.  The most informative tests run first.
"""

import numpy as np
import pytest

from conftest import bits, device_plan, golden_case, lowered
from gpu_cases import BUILDER_CASES, JIT_CASES, LAYOUT_CASES, WINDOW_CASES, builder_plan

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _close(got, want):
    got, want = np.asarray(got), np.asarray(want)
    same = bits(got) == bits(want)
    both_nan = np.isnan(got) & np.isnan(want)
    rel = np.abs(got - want) <= TOL * np.maximum(1.0, np.maximum(np.abs(got), np.abs(want)))
    return bool(np.all(same | both_nan | rel))


def check(got, golden):
    if golden.exact:
        assert np.array_equal(bits(got), bits(golden.values)), "bitwise mismatch"
    else:
        assert _close(got, golden.values)


def cmp_outputs(golden):
    want = golden.outputs
    return (lambda g: np.array_equal(bits(g), bits(want))) if golden.exact else (lambda g: _close(g, want))


def test_compile_plan_values(golden):
    from paper_2110_12865_b200 import compile_plan

    run = compile_plan(golden.plan)
    x = run(golden.inputs)
    check(x, golden)
    # the native library that ran is the in-tree one
    assert run.library_path.name == "libsgb.so"
    assert np.array_equal(bits(run.outputs(golden.inputs)), bits(x[np.asarray(golden.plan.outputs, np.int64)]))


@pytest.mark.parametrize("name", sorted(BUILDER_CASES))
@pytest.mark.parametrize("relayout", [False, "auto"])
@pytest.mark.parametrize("wbulk", [True, False])
def test_builder_plans_default_lowering(name, relayout, wbulk):
    """The config builders' plans at small sizes through the default lowering (CSR windows on the mesh
    plans -- bulk-fed through the shared-memory ring or not --, the CSR layout on the FEM plan):
    run_csr, every wave one at a time, the captured graph and the host path == the oracle, bit for bit."""
    import torch

    from oracle import oracle
    from paper_2110_12865_b200 import DevicePlan, lower_plan

    plan, inputs = builder_plan(name)
    dp = DevicePlan(plan, lowered=lower_plan(plan, relayout=relayout, wbulk=wbulk))
    if name.startswith("lmlt"):
        assert (dp.lowered.wbulk is not None) == wbulk
        assert dp.value_slots == dp.value_array_size + (dp.value_array_size % 2 if wbulk else 0)
    want = oracle.run_outputs(plan, inputs)
    x = dp.new_values(inputs)
    out = dp.run_csr(x)
    torch.cuda.synchronize()
    assert np.array_equal(bits(out.cpu().numpy()), bits(want))
    assert np.array_equal(bits(dp.run_outputs_host(inputs)), bits(want))
    out.fill_(float("nan"))
    x = dp.new_values(inputs)
    for w in range(dp.csr_launches):
        dp.run_wave(x, w, out)
    torch.cuda.synchronize()
    assert np.array_equal(bits(out.cpu().numpy()), bits(want))
    graph = dp.capture_csr(dp.new_values(inputs), out)
    out.fill_(float("nan"))
    graph.replay()
    torch.cuda.synchronize()
    assert np.array_equal(bits(out.cpu().numpy()), bits(want))
    # batched CSR (window plans: the members' value-mode twins store their outputs, copies gathered)
    rng = np.random.default_rng(5)
    sets = [inputs] + [inputs * rng.uniform(0.9, 1.1, inputs.size) for _ in range(2)]
    X = torch.zeros((dp.value_array_size, 3), dtype=torch.float64, device="cuda")
    X[: dp.input_count] = torch.from_numpy(np.stack(sets, axis=1)).cuda()
    outb = dp.run_batch_csr(X)
    torch.cuda.synchronize()
    for j, ins in enumerate(sets):
        assert np.array_equal(bits(outb[:, j].cpu().numpy()), bits(oracle.run_outputs(plan, ins)))
    if name.startswith("lmlt"):
        assert dp.lowered.windows is not None  # the CSR windows ran


@pytest.mark.parametrize("name", LAYOUT_CASES)
@pytest.mark.parametrize("relayout", ["all", "auto"])
def test_csr_layout(name, relayout):
    """CSR layout (multi-root groups stored instance-major, lower.choose_relayout): CSR values equal the
    reference's, on the device path, the captured graph, the host-buffer path and batched; value-mode
    calls are refused (the value array is permuted)."""
    import torch

    from paper_2110_12865_b200 import SgbError

    golden = golden_case(name)
    plan = golden.plan
    dp = device_plan(name, jit_min_n=0, relayout=relayout)
    cmp = cmp_outputs(golden)
    x = dp.new_values(golden.inputs)
    out = torch.full((len(plan.outputs),), float("nan"), dtype=torch.float64, device=x.device)
    dp.run_csr(x, out)
    torch.cuda.synchronize()
    assert cmp(out.cpu().numpy())
    assert cmp(dp.run_outputs_host(golden.inputs))
    many = dp.run_outputs_host_many(np.stack([golden.inputs] * 3))
    for k in range(3):
        assert cmp(many[k])
    if dp.lowered.needs_zero != 2:
        graph = dp.capture_csr(dp.new_values(golden.inputs), out)
        out.fill_(float("nan"))
        graph.replay()
        torch.cuda.synchronize()
        assert cmp(out.cpu().numpy())
    X = torch.zeros((plan.value_array_size, 5), dtype=torch.float64, device="cuda")
    X[: plan.input_count] = torch.from_numpy(np.repeat(golden.inputs[:, None], 5, axis=1)).cuda()
    o = dp.run_batch_csr(X).cpu().numpy()
    for b in range(5):
        assert cmp(o[:, b])
    if dp.csr_layout:
        with pytest.raises(SgbError):
            dp.run_values(dp.new_values(golden.inputs))
        with pytest.raises(SgbError):
            dp.sg_run(np.zeros(plan.value_array_size))


def test_outputs_host_many(golden):
    """The pipelined host-buffer stream (sgb_run_outputs_host_many): every set equals the reference's
    values, distinct value sets stay distinct (set k's inputs scaled), one repeated input set works."""
    import torch

    plan = golden.plan
    dp = device_plan(golden.name)
    cmp = cmp_outputs(golden)
    n = 5
    ins = np.stack([golden.inputs] * n)
    ins[1] *= 1.5
    ins[3] *= 0.75
    got = dp.run_outputs_host_many(ins)
    for k in (0, 2, 4):
        assert cmp(got[k])
    for k in (1, 3):
        ref = dp.run_outputs_host(ins[k])
        assert np.array_equal(bits(got[k]), bits(ref))
    rep = dp.run_outputs_host_many(golden.inputs, np.empty((4, len(plan.outputs))))
    for k in range(4):
        assert cmp(rep[k])
    assert cmp(dp.run_outputs_host(golden.inputs))  # the single-set path after the stream
    # chunked batched stream: 3 chunks of 2 value sets
    sets = np.stack([golden.inputs * f for f in (1.0, 1.5, 0.75, 1.25, 1.0, 2.0)])  # (6, n_in)
    hin = torch.from_numpy(np.ascontiguousarray(sets.reshape(3, 2, -1).transpose(0, 2, 1)))
    hout = torch.empty((3, len(plan.outputs), 2), dtype=torch.float64)
    dp.run_batch_outputs_host(hin, hout)
    for k in range(6):
        assert np.array_equal(bits(hout[k // 2, :, k % 2].numpy()), bits(dp.run_outputs_host(sets[k])))
    # device inputs -> device CSR values through the plan's own workspace (sgb_run_inputs_csr), on a
    # side stream, interleaved with the host-buffer path that shares the workspace
    s = torch.cuda.Stream()
    for k in (1, 3, 0):
        with torch.cuda.stream(s):
            o = dp.run_inputs_csr(torch.from_numpy(ins[k]).cuda(), stream=s)
        s.synchronize()
        assert np.array_equal(bits(o.cpu().numpy()), bits(dp.run_outputs_host(ins[k])))


def test_interpret_plan_outputs(golden):
    from paper_2110_12865_b200 import interpret_plan

    res = interpret_plan(golden.plan, golden.inputs, check_schedule=True, device_plan=device_plan(golden.name))
    check(res.values, golden)
    if golden.exact and golden.meta["oracle_bitwise"]:
        assert np.array_equal(bits(res.outputs), bits(golden.oracle))
    assert res.violations == golden.meta["violations"]


def test_device_resident_run_on_torch(golden):
    import torch

    dp = device_plan(golden.name)
    x = dp.new_values(golden.inputs)
    dp.run_values(x)
    out = dp.gather_outputs(x)
    torch.cuda.synchronize()
    check(x.cpu().numpy(), golden)
    assert np.array_equal(bits(out.cpu().numpy()), bits(x.cpu().numpy()[np.asarray(golden.plan.outputs, np.int64)]))


@pytest.mark.parametrize("mode", ["gather", "window", "direct", "interpreter"])
def test_csr_mode(golden, mode):
    """sgb_run_csr: value waves + gather; CSR windows (the last wave assembles the CSR array in shared
    memory, lower._csr_windows); direct scattered stores; the hand-written kernels only."""
    import torch

    if mode == "window" and golden.name not in WINDOW_CASES:
        pytest.skip("CSR windows forced on: the fixtures of gpu_cases.WINDOW_CASES")
    kw = {"gather": dict(csr_window=False), "window": dict(csr_window=True), "direct": dict(direct_csr=True),
          "interpreter": dict(jit=False)}[mode]
    dp = device_plan(golden.name, **kw)
    x = dp.new_values(golden.inputs)
    out = torch.full((len(golden.plan.outputs),), float("nan"), dtype=torch.float64, device=x.device)
    dp.run_csr(x, out)
    first = out.cpu().numpy().copy()
    if dp.lowered.needs_zero != 2:  # re-running on the same buffer is valid unless reads precede writes
        dp.run_csr(x, out)
    torch.cuda.synchronize()
    cmp = cmp_outputs(golden)
    for got in (first, out.cpu().numpy()):
        assert cmp(got)
    if mode == "window" and dp.lowered.windows is not None:
        assert dp.csr_launches == dp.launches  # no gather launch
        assert cmp(dp.run_outputs_host(golden.inputs))
        if dp.lowered.needs_zero != 2:
            graph = dp.capture_csr(dp.new_values(golden.inputs), out)
            out.fill_(float("nan"))
            graph.replay()
            torch.cuda.synchronize()
            assert cmp(out.cpu().numpy())
        x = dp.new_values(golden.inputs)  # value mode runs the members' value-only twins
        dp.run_values(x)
        check(x.cpu().numpy(), golden)


@pytest.mark.parametrize("name", JIT_CASES)
@pytest.mark.parametrize("batch", [0, 5, 64, 300])
def test_specialised_kernels_match_hand_written(name, batch):
    """Every group specialised (jit.py, jit_min_n=0) == the hand-written kernels only, bit for bit,
    single value set and batched (300 value sets: the batched kernels' lane loop runs twice)."""
    import torch

    golden = golden_case(name)
    plan = golden.plan
    rng = np.random.default_rng(batch)
    ins = rng.uniform(0.5, 2.0, (max(batch, 1), plan.input_count))
    ins[0] = golden.inputs
    outs = []
    for kw in (dict(jit=False), dict(jit_min_n=0)):
        dp = device_plan(name, **kw)
        if batch:
            X = torch.zeros((plan.value_array_size, batch), dtype=torch.float64, device="cuda")
            X[: plan.input_count] = torch.from_numpy(ins.T.copy()).cuda()
            dp.run_batch(X)
            o = dp.run_batch_csr(torch.where(torch.arange(plan.value_array_size, device="cuda")[:, None]
                                             < plan.input_count, X, torch.zeros_like(X)))
            outs.append((X.cpu().numpy(), o.cpu().numpy()))
        else:
            x = dp.new_values(golden.inputs)
            dp.run_values(x)
            outs.append((x.cpu().numpy(), dp.run_csr(dp.new_values(golden.inputs)).cpu().numpy()))
        torch.cuda.synchronize()
    if not batch:
        check(outs[1][0], golden)
    assert np.array_equal(bits(outs[0][0]), bits(outs[1][0]))
    assert np.array_equal(bits(outs[0][1]), bits(outs[1][1]))


def test_run_wave_by_wave_equals_run(golden):
    import torch

    dp = device_plan(golden.name)
    x = dp.new_values(golden.inputs)
    for w in range(dp.launches):
        dp.run_wave(x, w)
    x2 = dp.new_values(golden.inputs)
    out = torch.empty(len(golden.plan.outputs), dtype=torch.float64, device=x.device)
    for w in range(dp.csr_launches):
        dp.run_wave(x2, w, out=out)
    torch.cuda.synchronize()
    check(x.cpu().numpy(), golden)
    assert np.array_equal(bits(out.cpu().numpy()), bits(x.cpu().numpy()[np.asarray(golden.plan.outputs, np.int64)]))


@pytest.mark.parametrize("batch", [1, 5, 64])
def test_batched_matches_single(golden, batch):
    """B independent value sets in one pass == B single evaluations."""
    import torch

    from oracle import oracle

    plan = golden.plan
    dp = device_plan(golden.name)
    rng = np.random.default_rng(batch)
    ins = rng.uniform(0.5, 2.0, (batch, plan.input_count))
    ins[0] = golden.inputs
    X = torch.zeros((plan.value_array_size, batch), dtype=torch.float64, device="cuda")
    X[: plan.input_count] = torch.from_numpy(ins.T.copy()).cuda()
    dp.run_batch(X)
    got = X.cpu().numpy()
    check(got[:, 0], golden)
    for b in range(1, min(batch, 4)):
        want = oracle.run_values(plan, ins[b])
        if golden.exact:
            assert np.array_equal(bits(got[:, b]), bits(want))
        else:
            assert _close(got[:, b], want)
    outs = dp.gather_outputs_batch(X).cpu().numpy()
    assert np.array_equal(bits(outs[:, 0]), bits(got[np.asarray(plan.outputs, np.int64), 0]))
    # batched CSR mode on a fresh buffer == the gathered outputs of the value-mode run
    X2 = torch.zeros_like(X)
    X2[: plan.input_count] = torch.from_numpy(ins.T.copy()).cuda()
    csr = dp.run_batch_csr(X2).cpu().numpy()
    assert np.array_equal(bits(csr), bits(outs))


def test_wrong_input_length_raises():
    from paper_2110_12865_b200 import compile_plan, interpret_plan

    g = golden_case("toy256")
    with pytest.raises(ValueError):
        interpret_plan(g.plan, [1.0, 2.0])
    run = compile_plan(g.plan)
    with pytest.raises(ValueError):
        run(np.zeros(3))


@pytest.mark.parametrize("name", ["lmlt_w12", "spgemm_n60_k4", "prog_energy-hessian_4x4_tag", "fem_nh_m2", "arap_w5"])
def test_cuda_graph_replay_equals_run(name):
    """capture_csr: a replayed CUDA graph of one evaluation (all units, aux streams, gather) == sgb_run_csr."""
    import torch

    g = golden_case(name)
    dp = device_plan(name)
    x = dp.new_values(g.inputs)
    out = torch.empty(len(g.plan.outputs), dtype=torch.float64, device=x.device)
    want = dp.run_csr(dp.new_values(g.inputs)).cpu().numpy()
    graph = dp.capture_csr(x, out)
    out.fill_(float("nan"))
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    assert np.array_equal(bits(out.cpu().numpy()), bits(want))


@pytest.mark.parametrize("name", JIT_CASES)
def test_tile_schedules_bitwise(name):
    """Both tile schedules lower_plan offers (instance / fraction interleave of multi-group specialised
    units) and both grids give the same bits; sgb_plan_set_tiles refuses a table of another length
    and a table that is not a per-unit permutation of the plan's tiles."""
    import torch

    from paper_2110_12865_b200 import DevicePlan, SgbError

    golden = golden_case(name)
    lw = lowered(name, jit_min_n=0)
    dp = DevicePlan(golden.plan, lowered=lw)  # its own: the schedule and grids change
    x = dp.new_values(golden.inputs)
    want = dp.run_csr(x).cpu().numpy()
    assert cmp_outputs(golden)(want)
    if lw.tiles_alt is not None:
        for t in (lw.tiles_alt, lw.tiles):
            dp.set_tiles(t)
            got = dp.run_csr(dp.new_values(golden.inputs)).cpu().numpy()
            torch.cuda.synchronize()
            assert np.array_equal(bits(got), bits(want))
    for w in range(dp.csr_launches):  # both grids of the specialised units, every wave
        for tiles in (True, False):
            dp.set_wave_grid(w, tiles)
            got = dp.run_csr(dp.new_values(golden.inputs)).cpu().numpy()
            assert np.array_equal(bits(got), bits(want))
    with pytest.raises(SgbError):
        dp.set_tiles(np.zeros((len(lw.tiles) + 1, 2), np.int32))
    if len(lw.tiles):
        bad = np.array(lw.tiles, np.int32).reshape(-1, 2).copy()
        bad[0, 1] = 2 ** 30  # past the end of its group
        with pytest.raises(SgbError):
            dp.set_tiles(bad)


def test_autotune_keeps_bits():
    """DevicePlan.autotune (per-wave schedule x grid) changes launch configurations, never results."""
    import torch

    from paper_2110_12865_b200 import DevicePlan

    for name in ("lmlt_w12", "fem_nh_m2"):
        g = golden_case(name)
        dp = DevicePlan(g.plan, lowered=lowered(name, jit_min_n=0))
        before = dp.run_csr(dp.new_values(g.inputs)).cpu().numpy()
        dp.autotune(reps=2)
        after = dp.run_csr(dp.new_values(g.inputs)).cpu().numpy()
        torch.cuda.synchronize()
        assert np.array_equal(bits(before), bits(after))
        assert cmp_outputs(g)(after)


@pytest.mark.parametrize("world", [2, 3])
def test_output_shards_on_device(golden, world):
    """One evaluation with its CSR outputs split (shard.shard_device_plan): each shard's device plan,
    running only the tiles of its producer cone, gives the full evaluation's slice bit for bit."""
    from paper_2110_12865_b200 import DevicePlan
    from paper_2110_12865_b200.shard import shard_bounds, shard_device_plan

    plan = golden.plan
    kw = dict(jit_min_n=0) if golden.name in JIT_CASES else {}
    lw = lowered(golden.name, **kw)
    if lw.needs_zero == 2:
        pytest.skip("reads before writes: output sharding refuses the plan")
    full = device_plan(golden.name, **kw).run_outputs_host(golden.inputs)
    n_out = len(plan.outputs)
    for r in range(world):
        lo, hi = shard_bounds(lw, n_out, world, r)
        if hi == lo:
            continue
        view, slw = shard_device_plan(plan, lw, lo, hi)
        dp = DevicePlan(view, lowered=slw)
        got = dp.run_csr(dp.new_values(golden.inputs)).cpu().numpy()
        assert np.array_equal(bits(got), bits(full[lo:hi]))
        assert np.array_equal(bits(dp.run_outputs_host(golden.inputs)), bits(full[lo:hi]))


def _unary_plan(n, op, k=None):
    """One group of n instances, template op(v0) (POW: v0 ** k) over the inputs."""
    from paper_2110_12865_b200.plan import Template
    from paper_2110_12865_b200.programs.planbuild import PlanBuilder

    T = Template()
    args = (T.var(0),) if k is None else (T.var(0), T.const(float(k)))
    root = T.apply(op, args)
    B = PlanBuilder(n)
    res = B.add_group("probe", 0, T, [root], [np.arange(n, dtype=np.int64)])
    return B.finish(res[0], {"program": "transcendental probe"})


def _ref_math(fn, *a):
    import math

    try:
        return fn(*a)
    except OverflowError:
        return math.inf
    except ValueError:
        return math.nan


@pytest.mark.parametrize("jit", [True, False])
@pytest.mark.parametrize("op", ["log", "exp", "pow3", "pow4", "pow7", "sin", "cos"])
def test_device_transcendentals_match_glibc_bitwise(op, jit):
    """LOG / EXP / POW on the device (csrc/glibc_math.h, glibc's algorithms restated) == the
    reference's math.log / math.exp / math.pow (glibc), bit for bit, on ~3M values covering every
    branch (both log paths, the whole exponent range, subnormals, exp's under/overflow scaling,
    negative bases of odd and even powers), through the specialised and the interpreter kernels."""
    import math
    import sys
    from pathlib import Path

    from paper_2110_12865_b200 import DevicePlan, lower_plan
    from paper_2110_12865_b200.plan import OpKind

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
    import gen_glibc_math as g

    n = 3 << 20
    if op == "log":
        xs, kind, k, fn = np.concatenate([g.samples(n, seed=11), [1.0, math.inf, math.nan]]), OpKind.LOG, None, math.log
    elif op == "exp":
        xs, kind, k, fn = np.concatenate([g.exp_samples(n, seed=12), [0.0, -math.inf, math.inf, 709.8, -746.0]]), \
            OpKind.EXP, None, math.exp
    elif op in ("sin", "cos"):  # the whole finite range (glibc's __branred beyond 105414350)
        xs = np.concatenate([g.sincos_samples(n, seed=13), [0.0, -0.0, 1e-300, 2.426265, 105414349.0,
                                                             105414350.0, -1e22, 1.7976931348623157e308]])
        kind, k, fn = (OpKind.SIN, None, math.sin) if op == "sin" else (OpKind.COS, None, math.cos)
    else:
        k = int(op[3:])
        rng = np.random.default_rng(k)
        xs = np.concatenate([rng.uniform(-3.0, 3.0, n // 2), np.exp(rng.uniform(-200, 200, n // 2)) *
                             rng.choice([-1.0, 1.0], n // 2), [0.0, -0.0, 1e300, -1e300, 5e-324]])
        kind = OpKind.POW

        def fn(v, k=k):  # math.pow raises on overflow; glibc returns the signed infinity
            try:
                return math.pow(v, float(k))
            except OverflowError:
                return -math.inf if v < 0 and k % 2 else math.inf
    plan = _unary_plan(xs.size, kind, k)
    dp = DevicePlan(plan, lowered=lower_plan(plan, jit=jit))
    got = dp.run_outputs_host(xs)
    want = np.array([_ref_math(fn, v) for v in xs.tolist()])
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    bad = np.flatnonzero(bits(got[~nan]) != bits(want[~nan]))
    assert bad.size == 0, f"{bad.size} of {xs.size} differ, e.g. {xs[~nan][bad[:3]]}"


@pytest.mark.parametrize("world", [4])
def test_plan_shards_on_device(world):
    """bench.py's --split outputs path: each rank's own plan (shard.shard_plan) lowered with its
    whole-kept kernels' tiles filtered (shard.shard_device), on the device == the full evaluation's
    CSR slice, bit for bit."""
    import torch

    from oracle import oracle
    from paper_2110_12865_b200 import DevicePlan
    from paper_2110_12865_b200.shard import shard_device, shard_outputs, shard_plan

    plan, inputs = builder_plan("lmlt_w70")
    full = oracle.run_outputs(plan, inputs)
    for r in (0, world - 1):
        lo, hi = shard_outputs(len(plan.outputs), world, r)
        view, lw = shard_device(shard_plan(plan, lo, hi), relayout=False)
        dp = DevicePlan(view, lowered=lw)
        out = dp.run_csr(dp.new_values(inputs))
        torch.cuda.synchronize()
        assert np.array_equal(bits(out.cpu().numpy()), bits(full[lo:hi]))
