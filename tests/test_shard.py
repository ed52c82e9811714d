"""Multi-process sharding of value sets on CPU: gloo, world size 2.

The N>1 bench path shards independent value sets across ranks with no
collective in the step and gathers CSR blocks only on request; here every rank
evaluates its shard with the oracle (the GPU is not needed to check the
partitioning logic) and the gathered result must equal the single-process
evaluation of all value sets.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_12865_b200.shard import gather_csr, max_over_ranks, shard_value_sets


@pytest.mark.parametrize("total,world", [(256, 1), (256, 2), (256, 8), (7, 3), (3, 8), (0, 2)])
def test_shards_cover_every_value_set_once(total, world):
    seen = []
    for r in range(world):
        first, count = shard_value_sets(total, world, r)
        seen.extend(range(first, first + count))
    assert seen == list(range(total))
    sizes = [shard_value_sets(total, world, r)[1] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path

        root = Path(__file__).resolve().parent.parent
        sys.path.insert(0, str(root))
        sys.path.insert(0, str(root / "tests"))
        from conftest import Golden
        from oracle import oracle

        g = Golden("lmlt_w7")
        plan = g.plan
        first, count = shard_value_sets(total, world, rank)
        enc = oracle.encode_plan(plan)
        block = np.stack([oracle.run_outputs(plan, np.random.default_rng(s).uniform(0.5, 2.0, plan.input_count),
                                             enc) for s in range(first, first + count)], axis=1) \
            if count else np.zeros((len(plan.outputs), 0))
        full = gather_csr(torch.from_numpy(np.ascontiguousarray(block)), total)
        slowest = max_over_ranks(float(rank + 1))
        if rank == 0:
            np.save(result_path, full.numpy())
            assert slowest == float(world)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [5, 6])
def test_gloo_world2_gather_equals_single_process(tmp_path, total):
    world = 2
    path = tmp_path / "full.npy"
    mp.spawn(_worker, args=(world, _free_port(), total, str(path)), nprocs=world, join=True)
    got = np.load(path)
    from conftest import Golden, bits
    from oracle import oracle

    g = Golden("lmlt_w7")
    want = np.stack([oracle.run_outputs(g.plan, np.random.default_rng(s).uniform(0.5, 2.0, g.plan.input_count))
                     for s in range(total)], axis=1)
    assert got.shape == want.shape
    assert np.array_equal(bits(got), bits(want))


# -- one evaluation, output nonzeros partitioned (shard.shard_device_plan) --------------------


@pytest.mark.parametrize("name", ["lmlt_w12", "spgemm_n2000_k10", "acc1_expr2_s1"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_output_shards_with_csr_windows(name, world):
    """CSR-window plans shard at window boundaries (shard.shard_bounds): each rank keeps its windows,
    re-based, and its output cone's tiles; the shards tile the outputs and equal the full evaluation."""
    from conftest import Golden, bits

    import device_plan_emu as emu
    from paper_2110_12865_b200 import lower_plan
    from paper_2110_12865_b200.shard import shard_bounds, shard_device_plan

    g = Golden(name)
    lw = lower_plan(g.plan, csr_window=True, jit_compile=False)
    assert lw.windows is not None
    full = emu.run_csr(lw, g.inputs)
    n_out = len(g.plan.outputs)
    covered = []
    for r in range(world):
        lo, hi = shard_bounds(lw, n_out, world, r)
        covered.extend(range(lo, hi))
        if hi == lo:
            continue
        view, slw = shard_device_plan(g.plan, lw, lo, hi)
        assert slw.windows.k[0] == 0 and slw.windows.k[-1] == hi - lo
        got = emu.run_csr(slw, g.inputs, by_tiles=True)
        assert np.array_equal(bits(got), bits(full[lo:hi]))
    assert covered == list(range(n_out))


@pytest.mark.parametrize("name", ["lmlt_w7", "spgemm_n60_k4", "prog_energy-hessian_4x4_tag"])
@pytest.mark.parametrize("world", [2, 3])
def test_output_shards_match_full_evaluation(name, world):
    """Every rank's output cone, evaluated alone by the device-plan emulator over its filtered tile
    table, gives the full evaluation's CSR values [lo, hi) bit for bit; the shards tile the outputs."""
    from conftest import Golden, bits

    import device_plan_emu as emu
    from paper_2110_12865_b200 import lower_plan
    from paper_2110_12865_b200.shard import shard_device_plan, shard_outputs

    g = Golden(name)
    lw = lower_plan(g.plan, jit=False)
    full = emu.run_csr(lw, g.inputs)
    n_out = len(g.plan.outputs)
    covered = []
    for r in range(world):
        lo, hi = shard_outputs(n_out, world, r)
        covered.extend(range(lo, hi))
        view, slw = shard_device_plan(g.plan, lw, lo, hi)
        assert len(view.outputs) == hi - lo and len(slw.outputs) == hi - lo
        assert len(slw.tiles) <= len(lw.tiles)
        got = emu.run_csr(slw, g.inputs, by_tiles=True)
        assert np.array_equal(bits(got), bits(full[lo:hi]))
    assert covered == list(range(n_out))


def test_output_cone_shrinks_with_the_slice():
    """On a mesh plan the cone of half the outputs is well under the whole plan."""
    from conftest import Golden

    from paper_2110_12865_b200.shard import output_cone

    g = Golden("lmlt_w7")
    n_out = len(g.plan.outputs)
    whole = sum(int(m.sum()) for m in output_cone(g.plan, 0, n_out).values())
    half = sum(int(m.sum()) for m in output_cone(g.plan, 0, n_out // 2).values())
    assert 0 < half < whole


def _split_worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path

        root = Path(__file__).resolve().parent.parent
        sys.path.insert(0, str(root))
        sys.path.insert(0, str(root / "tests"))
        import device_plan_emu as emu
        from conftest import Golden

        from paper_2110_12865_b200 import lower_plan
        from paper_2110_12865_b200.shard import shard_device_plan, shard_outputs

        g = Golden("lmlt_w7")
        n_out = len(g.plan.outputs)
        lo, hi = shard_outputs(n_out, world, rank)
        _, slw = shard_device_plan(g.plan, lower_plan(g.plan, jit=False), lo, hi)
        mine = torch.from_numpy(emu.run_csr(slw, g.inputs, by_tiles=True))
        width = max(shard_outputs(n_out, world, r)[1] - shard_outputs(n_out, world, r)[0] for r in range(world))
        send = torch.zeros(width, dtype=torch.float64)
        send[: hi - lo] = mine
        parts = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(parts, send)
        if rank == 0:
            full = torch.cat([parts[r][: shard_outputs(n_out, world, r)[1] - shard_outputs(n_out, world, r)[0]]
                              for r in range(world)])
            np.save(result_path, full.numpy())
    finally:
        dist.destroy_process_group()


def test_gloo_world2_output_split_equals_oracle(tmp_path):
    """Two processes each evaluate half of one evaluation's CSR outputs from their producer cone;
    the gathered halves equal the oracle's full evaluation bit for bit."""
    world = 2
    path = tmp_path / "split.npy"
    mp.spawn(_split_worker, args=(world, _free_port(), str(path)), nprocs=world, join=True)
    from conftest import Golden, bits
    from oracle import oracle

    g = Golden("lmlt_w7")
    assert np.array_equal(bits(np.load(path)), bits(oracle.run_outputs(g.plan, g.inputs)))


def test_bench_emulated_eight_ranks_via_the_bench_entry_point():
    """`python bench.py --gpus 8 --emulate`: the bench's own spawn (torchrun, 8 ranks, gloo), CSR-window
    aligned output shards, max-over-ranks timing and the all-gather of the slices; the gathered
    evaluation equals the oracle bit for bit and the line reports n_gpus = 8."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, SGB_PLAN_CACHE=str(Path(os.environ.get("TMPDIR", "/tmp")) / "sgb_plan_cache_emu"))
    env.pop("WORLD_SIZE", None)
    proc = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "8", "--emulate", "--w", "14",
                           "--steps", "1"], capture_output=True, text=True, timeout=600, env=env)
    assert proc.returncode == 0, proc.stderr[-3000:]
    line = json.loads([ln for ln in proc.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 8 and line["config"]["parity"] == "bitwise"
    assert len(line["config"]["shards"]) == 8


@pytest.mark.parametrize("name", ["lmlt_w12", "spgemm_n2000_k10", "prog_energy-hessian_4x4_tag", "fem_nh_m2",
                                  "acc1_expr2_s1", "toy256_interleaved", "coord96"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_plan_shards_are_plans_of_their_own(name, world):
    """shard.shard_plan: each rank's ExecutionPlan (its producer cone, kernels cut to the instance
    ranges it needs) lowers and evaluates -- in every output mode -- to the full evaluation's CSR slice
    bit for bit."""
    from conftest import Golden, bits

    import device_plan_emu as emu
    from paper_2110_12865_b200 import lower_plan
    from paper_2110_12865_b200.shard import shard_outputs, shard_plan

    g = Golden(name)
    full = g.outputs
    n_out = len(g.plan.outputs)
    for r in range(world):
        lo, hi = shard_outputs(n_out, world, r)
        if hi == lo:
            continue
        sp = shard_plan(g.plan, lo, hi)
        for kw in (dict(jit=False), dict(csr_window=True, jit_compile=False)):
            got = emu.run_csr(lower_plan(sp, **kw), g.inputs)
            if g.exact:
                assert np.array_equal(bits(got), bits(full[lo:hi])), (r, kw)
            else:
                assert np.allclose(got, full[lo:hi], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("world", [2, 8])
def test_shard_device_filters_the_kernels_kept_whole(world):
    """shard.shard_device: a rank's shard lowered and its whole-kept (multi-root) kernels' tiles cut to
    the instances its outputs need -- fewer tiles than the shard's own lowering, the same CSR slice
    bit for bit (emulated over the filtered tiles)."""
    from conftest import bits

    import device_plan_emu as emu
    from oracle import oracle
    from paper_2110_12865_b200 import lower_plan
    from paper_2110_12865_b200.programs.mesh import build_lmlt_plan, lmlt_inputs
    from paper_2110_12865_b200.shard import shard_device, shard_outputs, shard_plan

    plan = build_lmlt_plan(48)[0]
    ins = lmlt_inputs(48, seed=2)
    full = oracle.run_outputs(plan, ins)
    for r in (0, world - 1):
        lo, hi = shard_outputs(len(plan.outputs), world, r)
        sp = shard_plan(plan, lo, hi)
        view, lw = shard_device(sp, relayout=False, jit_compile=False)
        assert np.asarray(lw.tiles).shape[0] < np.asarray(lower_plan(sp, relayout=False, jit_compile=False).tiles).shape[0]
        got = emu.run_csr(lw, ins, by_tiles=True)
        assert np.array_equal(bits(got), bits(full[lo:hi]))


def test_plan_shards_hold_their_share_of_the_tables():
    """On a mesh plan 8 shards together hold about one copy of the index tables (the cone overlap
    is a few grid rows per boundary, multi-root kernels whole), not 8."""
    from paper_2110_12865_b200.programs.mesh import build_lmlt_plan
    from paper_2110_12865_b200.shard import shard_outputs, shard_plan

    plan, _, _ = build_lmlt_plan(120)
    full = np.asarray(plan.positions).size
    parts = [shard_plan(plan, *shard_outputs(len(plan.outputs), 8, r)).positions.size for r in range(8)]
    assert sum(parts) <= 1.5 * full  # multi-root kernels (the 4-root face groups) are kept whole
    assert max(parts) <= 0.2 * full
