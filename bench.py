#!/usr/bin/env python
"""Benchmark: fp64 plan evaluation on B200 (arXiv 2110.12865 hot path), all five BASELINE configs.

Headline (default) = BASELINE.json configs[1] (C2): out = L.M.L^T + A on the
cotan Laplacian of a 1000 x 1000 grid mesh (10^6 vertices, ~25M output
nonzeros), plan built by the template-instancing builder
(paper_2110_12865_b200.programs.mesh; bit-identical to the reference trace,
tests/test_builders.py).  One step = one CSR-mode evaluation (sgb_run_csr) on
inputs already resident in HBM, replayed as a CUDA graph; the value array
(~385 MB), the CSR output (~200 MB) and the tables exceed the 126 MB L2.

At N = 1 the same line carries ``other_configs`` -- C1 spgemm 2k (the
reference's own plan), C3 Neo-Hookean 1M tets, C4 ARAP 500k vertices, C5
batched 1M-nnz x 256 value sets -- each with its own timing, parity, roofline,
CPU baseline and end-to-end figure.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2] [--only]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU; `--gpus N` alone spawns them)

N > 1: by default one C2 evaluation with its CSR outputs
split across the ranks -- each rank evaluates the producer cone of its slice
(shard.shard_device_plan), no collective in the step (strong scaling); the
NCCL all-gather of the slices is timed separately.  ``--split replicas`` runs
one full evaluation per rank (weak scaling); ``--config c5`` shards the 256
value sets.  Timing is the max over ranks of CUDA-event time.

``--impl reference`` times the reference's CPU evaluator on the same plan:
the reference's own emitted C (``sparsegen.emit.emit_kernel_source``,
oracle/make_ref.py -> oracle/ref_emitted/) built with its flags
(``cc -O3 -ffp-contract=off``, emit.py:220) plus -fopenmp on every host thread.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import pickle
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "output nonzeros/s & achieved HBM GB/s (fp64 eval, fixed pattern) vs CPU ref"
UNIT = "output nnz/s"
CONFIGS = ("c2", "c1", "c3", "c4", "c5")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# -- workloads (BASELINE.json configs) ------------------------------------------


def workload_key(cfg: str, args) -> str:
    if cfg == "c1":
        return "spgemm_n2000_k10"
    if cfg == "c3":
        return f"fem_nh_m{args.m}"
    if cfg == "c4":
        return f"arap_w{args.w4}"
    w = args.w5 if cfg == "c5" else args.w
    return f"lmlt_w{w}_a6_s7_split0"


def _build(cfg: str, args):
    if cfg == "c3":
        from paper_2110_12865_b200.programs.fem import build_fem_plan

        return build_fem_plan(args.m)[0]
    if cfg == "c4":
        from paper_2110_12865_b200.programs.arap import build_arap_plan

        return build_arap_plan(args.w4)[0]
    from paper_2110_12865_b200.programs.mesh import build_lmlt_plan

    return build_lmlt_plan(args.w5 if cfg == "c5" else args.w)[0]


def build_workload(cfg: str, args, rank: int = 0, barrier=None):
    """(key, plan): C1 is the reference's own saved plan; the others come from the builders, cached on
    disk for the other ranks and later runs (keyed by the builder sources)."""
    key = workload_key(cfg, args)
    if cfg == "c1":
        from paper_2110_12865_b200 import load_plan

        return key, load_plan(ROOT / "tests" / "golden" / key)
    cache_dir = Path(os.environ.get("SGB_PLAN_CACHE", Path(tempfile.gettempdir()) / "sgb_plan_cache"))
    from paper_2110_12865_b200.programs import builder_hash

    path = cache_dir / f"{key}.{builder_hash()[:12]}.v2.pkl"
    if rank == 0 and not path.exists():
        t0 = time.perf_counter()
        plan = _build(cfg, args)
        log(f"[bench] built plan {key} in {time.perf_counter() - t0:.1f}s")
        cache_dir.mkdir(parents=True, exist_ok=True)
        tmp = path.with_suffix(f".{os.getpid()}.tmp")
        with open(tmp, "wb") as fh:
            pickle.dump(plan, fh, protocol=pickle.HIGHEST_PROTOCOL)
        os.replace(tmp, path)
    if barrier is not None:
        barrier()
    with open(path, "rb") as fh:
        plan = pickle.load(fh)
    return key, plan


def workload_inputs(cfg: str, args, seed: int = 0, plan=None) -> np.ndarray:
    if cfg == "c1":
        if seed == 0:
            with np.load(ROOT / "tests" / "golden" / "spgemm_n2000_k10" / "vectors.npz") as z:
                return z["inputs"]
        return np.random.default_rng(seed).uniform(0.5, 2.0, int(plan.input_count))
    if cfg == "c3":
        from paper_2110_12865_b200.programs.fem import fem_inputs

        return fem_inputs(args.m, seed=seed)
    if cfg == "c4":
        from paper_2110_12865_b200.programs.arap import arap_inputs

        return arap_inputs(args.w4, seed=seed)
    from paper_2110_12865_b200.programs.mesh import lmlt_inputs

    return lmlt_inputs(args.w5 if cfg == "c5" else args.w, seed=seed)


def workload_name(cfg: str, args, n_out: int) -> str:
    if cfg == "c1":
        return f"C1 spgemm C=A.B, random CSR 2000x2000 10 nnz/row, {n_out} out nnz (the reference's own plan)"
    if cfg == "c3":
        return (f"C3 Neo-Hookean tet FEM Hessian assembled to CSR, Kuhn mesh of {args.m}^3 cubes "
                f"({6 * args.m ** 3} tets), mu=1 lam=10, {n_out} output nnz")
    if cfg == "c4":
        return f"C4 ARAP system matrix + rhs on a {args.w4}x{args.w4} grid mesh, {n_out} outputs"
    if cfg == "c5":
        return (f"C5 batched: L.M.L^T+A plan on a {args.w5}x{args.w5} grid ({n_out} out nnz) x {args.batch} "
                f"value sets")
    return (f"C2 L.M.L^T+A, cotan Laplacian of a {args.w}x{args.w} grid mesh "
            f"({args.w * args.w} vertices), A random 6 nnz/row (seed 7), {n_out} output nnz")


def config_dict(cfg: str, args, plan) -> dict:
    """The workload description both arms print (identical keys and values)."""
    n_out = len(plan.outputs)
    d = {"workload": workload_name(cfg, args, n_out), "config": cfg, "plan": workload_key(cfg, args),
         "out_nnz": n_out, "value_array": int(plan.value_array_size), "inputs": int(plan.input_count),
         "kernels": len(plan.kernels), "index_entries": int(np.asarray(plan.positions).size)}
    if cfg == "c5":
        d["value_sets"] = args.batch
    return d


# -- clocks ---------------------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.file = None

    def __enter__(self):
        try:
            self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.gpu)], stdout=self.file, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None:
            return None
        self.file.flush()
        rows = []
        for line in Path(self.file.name).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), float(parts[3]), parts[4:]))
            except ValueError:
                continue
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for _, _, _, r in rows for k, v in enumerate(r[1:5]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "power_w_max": max(r[2] for r in rows), "samples": len(rows), "reasons": reasons}


# -- CPU reference (the reference's own evaluators, on the box's host cores) ---------------------


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def reference_library(plan, key: str, openmp: bool, extra_sources=()):
    """Compile the reference's emitted C for ``plan`` (oracle/ref_emitted/<key>.c, the output of
    sparsegen.emit.emit_kernel_source) with the reference flags (emit.py:220), or the restated emitter
    (oracle/emit_c.py, kind "port") when no emitted source matches the plan.  (ctypes lib, kind, what)."""
    from oracle import make_ref

    src, ok = make_ref.lookup(plan, key)
    kind, what = "reference", f"sparsegen.emit.emit_kernel_source output (oracle/ref_emitted/{key}.c)"
    if src is None or not ok:
        from oracle import emit_c

        src = Path(tempfile.gettempdir()) / f"sgb_port_{key}_{os.getpid()}.c"
        src.write_text(emit_c.emit_kernel_source(plan, parallel="pragma"))
        kind, what = "port", "emitted C restated by oracle/emit_c.py (emit.py:153-245)"
        log(f"[bench] no reference-emitted source matches {key}: timing the restated emitter")
    tag = "omp" if openmp else "1t"
    lib = Path(tempfile.gettempdir()) / f"sgb_ref_{key}_{tag}_{len(extra_sources)}_{os.getpid()}.so"
    cmd = ["cc", "-O3", "-ffp-contract=off", "-fPIC", "-shared"] + (["-fopenmp"] if openmp else []) + \
        ["-o", str(lib), str(src)] + [str(s) for s in extra_sources] + ["-lm"]
    subprocess.run(cmd, check=True, capture_output=True)
    dll = ctypes.CDLL(str(lib))
    dll.sg_run.restype = None
    dll.sg_run.argtypes = [ctypes.c_void_p] * 3
    return dll, kind, what


def _sg_run_fn(dll, plan):
    con = np.ascontiguousarray(plan.constants, dtype=np.float64)
    pos = np.ascontiguousarray(plan.positions, dtype=np.uint32)

    def sg_run(x):
        dll.sg_run(x.ctypes.data, con.ctypes.data if con.size else None, pos.ctypes.data if pos.size else None)
        return x

    sg_run.keep = (dll, con, pos)
    return sg_run


def time_sg_run(sg_run, plan, inputs, budget_s: float, max_evals: int) -> tuple[float, int, np.ndarray]:
    """Mean seconds per sg_run over up to max_evals calls (budget-bounded), after one warm-up."""
    x = np.zeros(int(plan.value_array_size), np.float64)
    x[: plan.input_count] = inputs
    sg_run(x)
    times = []
    t_start = time.perf_counter()
    while len(times) < max_evals and (not times or time.perf_counter() - t_start < budget_s):
        t0 = time.perf_counter()
        sg_run(x)
        times.append(time.perf_counter() - t0)
    return statistics.mean(times), len(times), x


def cpu_baseline(cfg: str, args, plan, key: str, inputs, gpu_out=None, budget_s: float = 8.0) -> dict:
    """SURVEY.md §8(d) CPU reference, timed on this box's host cores: the reference's emitted-C
    ``sg_run`` with OpenMP on every host thread (the line's ``value``) and on one thread, the
    reference interpreter (numpy restatement, oracle/interp_np.py) on one core, plus C1's reference
    plan build and C5's OpenMP-over-value-sets variant."""
    n_out = len(plan.outputs)
    cores = host_cores()
    os.environ["OMP_NUM_THREADS"] = str(cores)
    legs = {}
    dll, kind, what = reference_library(plan, key, openmp=True)
    t_all, n_all, x = time_sg_run(_sg_run_fn(dll, plan), plan, inputs, budget_s, args.cpu_steps)
    legs["sg_run_all_cores"] = {"value": n_out / t_all, "ms": t_all * 1e3, "evals": n_all, "threads": cores}
    parity = None
    if gpu_out is not None:
        got = x[np.asarray(plan.outputs, np.int64)]
        parity = bool(np.array_equal(got.view(np.uint64), np.asarray(gpu_out).view(np.uint64)))
    dll1, _, _ = reference_library(plan, key, openmp=False)
    t_1, n_1, _ = time_sg_run(_sg_run_fn(dll1, plan), plan, inputs, budget_s / 2, max(3, args.cpu_steps // 4))
    legs["sg_run_one_thread"] = {"value": n_out / t_1, "ms": t_1 * 1e3, "evals": n_1, "threads": 1}
    # the reference interpreter (interpret_plan, codegen.py:404-557) on one core; its scalar path
    # (LOG / POW / self-referencing kernels) is capped at a bounded number of instances per kernel
    from oracle import interp_np

    cap = 20000
    t0 = time.perf_counter()
    _, skipped = interp_np.interpret(plan, inputs, max_scalar=cap)
    t_i = time.perf_counter() - t0
    legs["interpret_plan_one_core"] = {
        "value": n_out / t_i if not skipped else None, "s": t_i, "threads": 1,
        "sample": ("one full evaluation (oracle/interp_np.py, the numpy restatement of interpret_plan)"
                   if not skipped else
                   f"scalar-path kernels capped at {cap} instances ({skipped} instances skipped): {t_i:.1f} s is a "
                   "lower bound on one evaluation, so no rate is reported")}
    if cfg == "c1":
        pb = ROOT / "profiles" / "r2" / "c1_plan_build.json"
        if pb.exists():
            rec = json.loads(pb.read_text())
            build_s = rec["trace_s"] + rec["build_plan_s"]
            legs["plan_build_plus_evaluate"] = {
                "value": n_out / (build_s + t_all), "plan_build_s": build_s, "evaluate_ms": t_all * 1e3,
                "source": f"{pb.relative_to(ROOT)} (reference trace + build_plan, one core, {rec['cpu']}, "
                          f"{rec['measured_in']}) + the all-core sg_run measured here"}
    if cfg == "c5":
        legs["omp_over_value_sets"] = omp_over_sets(plan, key, args, budget_s)
    return {"value": n_out / t_all, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": (f"{n_all} full sg_run evaluations of the {key} plan ({n_out} nnz): {what}, cc -O3 "
                       f"-ffp-contract=off -fopenmp on {cores} threads of {cpu_model()}"),
            "matches_gpu_bitwise": parity, "legs": legs}


def omp_over_sets(plan, key: str, args, budget_s: float) -> dict:
    """C5's strongest CPU figure: one OpenMP thread per value set, each sg_run serial (oracle/omp_sets.c)."""
    cores = host_cores()
    os.environ["OMP_MAX_ACTIVE_LEVELS"] = "1"
    dll, kind, _ = reference_library(plan, key, openmp=True, extra_sources=[ROOT / "oracle" / "omp_sets.c"])
    dll.sg_run_sets.restype = None
    dll.sg_run_sets.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    n_sets = min(args.batch, 2 * cores)
    xs = [np.zeros(int(plan.value_array_size), np.float64) for _ in range(n_sets)]
    for s, x in enumerate(xs):
        x[: plan.input_count] = workload_inputs("c5", args, seed=s)
    ptrs = (ctypes.c_void_p * n_sets)(*[x.ctypes.data for x in xs])
    con = np.ascontiguousarray(plan.constants, dtype=np.float64)
    pos = np.ascontiguousarray(plan.positions, dtype=np.uint32)

    def run():
        dll.sg_run_sets(n_sets, ptrs, con.ctypes.data if con.size else None, pos.ctypes.data if pos.size else None)

    run()
    reps, t0 = 0, time.perf_counter()
    while reps < 3 or (time.perf_counter() - t0 < budget_s / 2 and reps < 20):
        run()
        reps += 1
    t = (time.perf_counter() - t0) / reps
    return {"value": n_sets * len(plan.outputs) / t, "threads": cores, "value_sets_per_call": n_sets,
            "ms_per_call": t * 1e3, "kind": kind,
            "sample": "one OpenMP thread per value set, each sg_run serial (the emitted kernels' own OpenMP regions "
                      "nest inside and run on one thread)"}


# -- GPU measurement --------------------------------------------------------------------------------


def peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def parity_vs_oracle(plan, inputs, got, exact: bool, lo: int = 0, hi: int | None = None) -> str:
    from oracle import oracle

    want = oracle.run_outputs(plan, inputs)[lo:hi]
    got = np.asarray(got)
    if np.array_equal(got.view(np.uint64), want.view(np.uint64)):
        return "bitwise"
    rel = np.abs(got - want) / np.maximum(1.0, np.maximum(np.abs(got), np.abs(want)))
    if not exact and float(np.nanmax(rel)) <= 1e-12:
        return f"within 1e-12 (max rel {float(np.nanmax(rel)):.2e}; transcendental ops, CUDA libm vs glibc)"
    return f"MISMATCH (max rel {float(np.nanmax(rel)):.2e})"


def output_mode(dp) -> str:
    if getattr(dp.lowered, "windows", None) is not None:
        return ("CSR windows: the last wave assembles the CSR array window by window in shared memory "
                "(lower._csr_windows, jit.window_source), no gather")
    if np.any(dp.lowered.groups["flags"] & 384):
        return "CSR, direct stores"
    return "value-array waves + u32-indexed output gather"


def measure_eval(cfg: str, args, rank: int, world: int, barrier, split=None) -> dict:
    """One CSR-mode evaluation per step (C1-C4), device-resident inputs, CUDA-graph replay; per-launch
    times from a wave-by-wave pass; e2e through the host-buffer C ABI; CPU baseline on rank 0."""
    import torch
    import torch.distributed as dist

    from paper_2110_12865_b200 import DevicePlan
    from paper_2110_12865_b200.metrics import csr_wave_traffic, plan_balg, wave_traffic

    local = torch.cuda.current_device()
    key, plan = build_workload(cfg, args, rank, barrier)
    full_plan = plan
    n_total = len(plan.outputs)
    cfgd = config_dict(cfg, args, plan)
    split_info = None
    lo, hi = 0, n_total
    if split is not None:  # one evaluation, CSR outputs split: this rank's own plan shard (its producer cone)
        from paper_2110_12865_b200.shard import shard_outputs, shard_plan

        s_world, s_rank = split
        lo, hi = shard_outputs(n_total, s_world, s_rank)
        plan = shard_plan(full_plan, lo, hi)
        split_info = {"world": s_world, "rank": s_rank, "outputs": [lo, hi],
                      "index_entries_kept": int(plan.positions.size),
                      "index_entries_full": int(np.asarray(full_plan.positions).size),
                      "kernels_kept": len(plan.kernels)}
        from paper_2110_12865_b200.shard import shard_device

        view, lw = shard_device(plan, relayout=os.environ.get("SGB_RELAYOUT", "auto"))
        dp = DevicePlan(view, device=local, lowered=lw)
        inputs = workload_inputs(cfg, args, seed=0, plan=full_plan)
    else:
        inputs = workload_inputs(cfg, args, seed=rank, plan=plan)
        dp = DevicePlan(plan, device=local, csr_layout=True)
    n_out = len(plan.outputs)
    if dp.lowered.needs_zero == 2:
        raise SystemExit("bench: the plan reads slots later waves write; re-zeroing per step is not benchmarked")
    x = dp.new_values(inputs)
    out = torch.empty(n_out, dtype=torch.float64, device=x.device)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        dp.run_csr(x, out)
    torch.cuda.synchronize()
    parity = None
    if rank == 0:
        parity = parity_vs_oracle(full_plan, inputs, out.cpu().numpy(), dp.lowered.exact, lo, hi)
        log(f"[bench {cfg}] parity vs oracle: {parity}")
    small = cfg == "c1"  # 3.5 MB per evaluation: L2-resident unless flushed
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=x.device) if small else None
    n_w = dp.csr_launches
    sampler = ClockSampler(local)
    with sampler:
        t_end = time.perf_counter() + 1.0  # settle clocks on real work (untimed)
        while time.perf_counter() < t_end:
            for _ in range(20):
                dp.run_csr(x, out)
            torch.cuda.synchronize()
        graph = dp.capture_csr(x, out)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if barrier:
            barrier()
        torch.cuda.synchronize()
        for e0, e1 in evs:
            if flush is not None:
                flush.fill_(1.0)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        if barrier:
            barrier()
        wev = [[torch.cuda.Event(enable_timing=True) for _ in range(n_w + 1)] for _ in range(args.steps)]
        for e in wev:  # per-launch breakdown: one wave at a time, events between the launches
            if flush is not None:
                flush.fill_(1.0)
            for w in range(n_w):
                e[w].record(stream)
                dp.run_wave(x, w, out=out)
            e[n_w].record(stream)
        torch.cuda.synchronize()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    ms = statistics.mean(step_ms)
    per_launch = np.array([[e[j].elapsed_time(e[j + 1]) for j in range(n_w)] for e in wev]).mean(axis=0)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=x.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    job_out = n_total if split_info and split_info["world"] == world else world * n_out
    value = job_out / (ms * 1e-3)

    # end to end through the public host-buffer API, pinned host memory, copies inside the timed region
    want_bits = out.cpu().numpy().view(np.uint64)
    if small:  # launch-bound per value set: value sets stream in batched chunks (sgb_run_batch_csr)
        n_chunks, cb = 8, max(1, args.e2e_steps * 20 // 8)
        k_sets = n_chunks * cb
        hin = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(inputs[None, :, None],
                                                                    (n_chunks, inputs.size, cb)))).pin_memory()
        hout = torch.empty((n_chunks, n_out, cb), dtype=torch.float64).pin_memory()
        dp.run_batch_outputs_host(hin, hout)  # warm
        t0 = time.perf_counter()
        dp.run_batch_outputs_host(hin, hout)
        e2e_s = (time.perf_counter() - t0) / k_sets
        e2e_ok = bool(np.all(hout.numpy().view(np.uint64) == want_bits[None, :, None]))
        api = (f"DevicePlan.run_batch_outputs_host: {k_sets} value sets from pinned host memory in {n_chunks} "
               f"chunks of {cb} (sgb_run_batch_csr per chunk), copies and evaluation pipelined on three streams")
    else:
        k_sets = max(args.e2e_steps, 2)
        ins_h = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(inputs, (k_sets, inputs.size)))).pin_memory()
        outs_h = torch.empty((k_sets, n_out), dtype=torch.float64).pin_memory()
        dp.run_outputs_host_many(ins_h.numpy()[:2], outs_h.numpy()[:2])  # warm (second workspace)
        if barrier:
            barrier()
        t0 = time.perf_counter()
        dp.run_outputs_host_many(ins_h.numpy(), outs_h.numpy())
        e2e_s = (time.perf_counter() - t0) / k_sets
        e2e_ok = bool(all(np.array_equal(outs_h[k].numpy().view(np.uint64), want_bits) for k in range(k_sets)))
        api = (f"DevicePlan.run_outputs_host_many -> sgb_run_outputs_host_many: {k_sets} value sets from pinned "
               "host memory, per-set copy in / evaluate / copy out pipelined on three streams")
        del ins_h, outs_h
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=x.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    gather_ms = None
    if split_info and world > 1:  # NCCL all-gather of the slices (not in the step)
        gather_ms = time_slice_gather(out, world, barrier)
    if rank != 0:
        return {}

    direct = bool(np.any(dp.lowered.groups["flags"] & (384 | 4096)))
    traffic = csr_wave_traffic(plan, dp.lowered) if direct else wave_traffic(plan, dp.lowered)
    traffic = traffic[:n_w]
    dom = int(np.argmax(per_launch))
    peak, peak_src = peak_gbs()
    achieved = traffic[dom].bytes / (per_launch[dom] * 1e-3) / 1e9
    balg = plan_balg(plan)
    whole = balg / (ms * 1e-3) / 1e9
    cpu = None
    if world == 1 and not split_info and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args, full_plan, key, inputs, gpu_out=out.cpu().numpy())
    if split_info:
        par = (f"one evaluation, CSR outputs split {split_info['world']} ways (shard.shard_plan): each rank holds its "
               f"own plan shard -- rank 0 outputs {split_info['outputs']}, {split_info['index_entries_kept']} of "
               f"{split_info['index_entries_full']} index entries; no collective in the step")
    else:
        par = "single GPU" if world == 1 else f"replicas x{world}: one full evaluation per GPU per step"
    cfgd.update({
        "parallelism": par, "split": split_info, "nccl_allgather_ms": gather_ms,
        "l2": ("flushed (512 MB write) before every timed evaluation" if small else
               "no flush: value array + tables exceed the 126 MB L2"),
        "clock_settle": "1 s of untimed evaluations before the timed region",
        "parity": parity, "mode": output_mode(dp),
        "launch": "CUDA graph of one sgb_run_csr evaluation replayed per step; per-launch times from a separate "
                  "wave-by-wave pass",
        "layout": (f"CSR layout: plan groups {dp.lowered.csr_layout} store instance-major" if dp.csr_layout
                   else "reference value-array layout"),
        "tile_schedule": ({str(w): o for w, o in dp.tile_order.items()} if dp.tile_order else None),
    })
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "ms_per_step_min": min(step_ms), "higher_is_better": True,
        "scaling": "strong" if split_info else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfgd,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": traffic[dom].name, "algorithmic_bytes": traffic[dom].bytes,
                     "avg_launch_ms": float(per_launch[dom]), "peak_source": peak_src,
                     "traffic_note": ("not measurable in a timed run: ncu --set full DRAM bytes per launch of "
                                      "this kernel are in profiles/r2/ncu_full_*.txt"),
                     "whole_evaluation": {"balg_bytes": int(balg), "achieved": whole, "frac": whole / peak,
                                          "definition": "SURVEY 8(d) single-pass B_alg of the plan / ms_per_step"}},
        "launches": [{"name": t.name, "ms": float(m), "alg_bytes": t.bytes,
                      "gbs": t.bytes / (m * 1e-3) / 1e9 if m > 0 else None} for t, m in zip(traffic, per_launch)],
        "e2e": {"value": job_out / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * int(plan.input_count),
                "d2h_bytes_per_step": 8 * n_out, "api": api, "matches_device_run": e2e_ok},
        "gpu_launches": args.steps * dp.csr_units, "clocks": sampler.summary(), "cpu_baseline": cpu,
    }


def time_slice_gather(out, world: int, barrier) -> float:
    """NCCL all-gather of every rank's CSR slice (padded to the largest), max over ranks."""
    import torch
    import torch.distributed as dist

    width = torch.tensor([out.numel()], device=out.device)
    dist.all_reduce(width, op=dist.ReduceOp.MAX)
    send = torch.zeros(int(width.item()), dtype=torch.float64, device=out.device)
    send[: out.numel()] = out
    parts = [torch.empty_like(send) for _ in range(world)]
    for _ in range(2):
        dist.all_gather(parts, send)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dist.all_gather(parts, send)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=out.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measure_batched(args, rank: int, world: int, barrier) -> dict:
    """C5: the L.M.L^T+A plan on a 200 x 200 grid (991,912 out nnz) x 256 value sets, the value sets
    sharded across the ranks (the 256 sets are the whole job); no collective in the step."""
    import torch

    from paper_2110_12865_b200 import DevicePlan
    from paper_2110_12865_b200.metrics import plan_balg, wave_traffic
    from paper_2110_12865_b200.shard import gather_csr, max_over_ranks, shard_value_sets

    local = torch.cuda.current_device()
    key, plan = build_workload("c5", args, rank, barrier)
    n_out, n_in = len(plan.outputs), int(plan.input_count)
    total = args.batch
    per = [shard_value_sets(total, world, r)[1] for r in range(world)]
    first, b = shard_value_sets(total, world, rank)
    host_in = np.stack([workload_inputs("c5", args, seed=s_) for s_ in range(first, first + b)], axis=1)
    dp = DevicePlan(plan, device=local, csr_layout=True)
    X = torch.zeros((plan.value_array_size, b), dtype=torch.float64, device=f"cuda:{local}")
    X[:n_in] = torch.from_numpy(host_in).to(X.device)
    out = torch.empty((n_out, b), dtype=torch.float64, device=X.device)
    for _ in range(args.warmup):
        dp.run_batch_csr(X, out)
    torch.cuda.synchronize()
    parity = None
    if rank == 0:
        from oracle import oracle

        enc = oracle.encode_plan(plan)
        ok = all(np.array_equal(oracle.run_outputs(plan, host_in[:, j], enc).view(np.uint64),
                                out[:, j].cpu().numpy().view(np.uint64)) for j in range(min(b, 3)))
        parity = "bitwise (value sets 0-2 vs oracle)" if ok else "MISMATCH"
        log(f"[bench c5] parity: {parity}")
    stream = torch.cuda.current_stream()
    sampler = ClockSampler(local)
    steps = max(3, args.steps // 4)
    with sampler:
        t_end = time.perf_counter() + 1.0
        while time.perf_counter() < t_end:
            dp.run_batch_csr(X, out)
            torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        if barrier:
            barrier()
        torch.cuda.synchronize()
        for e0, e1 in evs:
            e0.record(stream)
            dp.run_batch_csr(X, out)
            e1.record(stream)
        torch.cuda.synchronize()
        if barrier:
            barrier()
    ms = max_over_ranks(statistics.mean(e0.elapsed_time(e1) for e0, e1 in evs), X.device)
    gather_ms = None
    if world > 1:  # NCCL gather of every rank's CSR block to rank 0 (not in the step)
        for _ in range(2):
            gather_csr(out, total)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        gather_csr(out, total)
        e1.record(stream)
        torch.cuda.synchronize()
        gather_ms = max_over_ranks(e0.elapsed_time(e1), X.device)
    # e2e: the rank's value sets from pinned host memory in chunks (run_batch_outputs_host)
    n_chunks = next(c for c in (8, 4, 2, 1) if b % c == 0 and b // c >= 1)
    cb = b // n_chunks
    hin = torch.from_numpy(np.ascontiguousarray(host_in.reshape(n_in, n_chunks, cb).transpose(1, 0, 2))).pin_memory()
    hout = torch.empty((n_chunks, n_out, cb), dtype=torch.float64).pin_memory()
    want = out.cpu().numpy()
    del X
    torch.cuda.empty_cache()
    dp.run_batch_outputs_host(hin, hout)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dp.run_batch_outputs_host(hin, hout)
    e2e_s = max_over_ranks(time.perf_counter() - t0, out.device)
    e2e_ok = bool(np.array_equal(hout.numpy().transpose(1, 0, 2).reshape(n_out, b).view(np.uint64),
                                 want.view(np.uint64)))
    if rank != 0:
        return {}
    traffic = wave_traffic(plan, dp.lowered, batch=b)
    step_bytes = sum(t.bytes for t in traffic)
    peak, peak_src = peak_gbs()
    achieved = step_bytes / (ms * 1e-3) / 1e9
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline("c5", args, plan, key, host_in[:, 0], gpu_out=want[:, 0])
        cpu["sample"] += " (one value set per sg_run call: the reference has no batch API)"
    cfgd = config_dict("c5", args, plan)
    cfgd.update({"parallelism": f"value sets sharded over {world} GPU(s) ({per} per rank), plan replicated, no "
                                "collective in the step",
                 "l2": "no flush: X (%.1f GB per rank) exceeds L2" % (plan.value_array_size * b * 8 / 1e9),
                 "parity": parity, "nccl_gather_ms": gather_ms, "mode": "batched CSR (sgb_run_batch_csr)"})
    bal = plan_balg(plan)
    return {
        "metric": METRIC, "value": total * n_out / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfgd,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": "whole batched step (waves + gather)", "algorithmic_bytes": step_bytes,
                     "peak_source": peak_src,
                     "whole_evaluation": {"balg_bytes": int(bal) * total,
                                          "achieved": bal * total / (ms * 1e-3) / 1e9,
                                          "frac": bal * total / (ms * 1e-3) / 1e9 / peak,
                                          "definition": "256 x the single-pass B_alg (tables re-read per set)"}},
        "e2e": {"value": total * n_out / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * n_in * b,
                "d2h_bytes_per_step": 8 * n_out * b,
                "api": (f"DevicePlan.run_batch_outputs_host: {n_chunks} chunks of {cb} value sets per rank from "
                        "pinned host memory, copy in / sgb_run_batch_csr / copy out pipelined on three streams"),
                "matches_device_run": e2e_ok},
        "gpu_launches": steps * dp.csr_units, "clocks": sampler.summary(), "cpu_baseline": cpu,
    }


def measure_emulated(args, rank: int, world: int, barrier) -> dict:
    """``--emulate``: the N-rank orchestration of ``measure_eval`` on CPU -- gloo, the device-plan
    emulator (tests/device_plan_emu.py) in place of the GPU -- so the multi-rank path (spawn, CSR
    window-aligned output shards, max-over-ranks timing, the all-gather of the slices) is testable
    without GPUs (tests/test_shard.py).  Test infrastructure: never a bench number."""
    import torch
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT / "tests"))
    import device_plan_emu as emu

    from paper_2110_12865_b200.shard import max_over_ranks, shard_device, shard_outputs, shard_plan

    cfg = args.config
    key, plan = build_workload(cfg, args, rank, barrier)
    n_total = len(plan.outputs)
    lo, hi = shard_outputs(n_total, world, rank)
    _, slw = shard_device(shard_plan(plan, lo, hi), relayout=False, jit_compile=False, csr_window=True)
    inputs = workload_inputs(cfg, args, seed=0, plan=plan)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        mine = emu.run_csr(slw, inputs, by_tiles=True)  # the same tile-filtered shard the GPU path runs
    sec = max_over_ranks((time.perf_counter() - t0) / args.steps)
    width = torch.tensor([hi - lo])
    dist.all_reduce(width, op=dist.ReduceOp.MAX)
    send = torch.zeros(int(width.item()), dtype=torch.float64)
    send[: hi - lo] = torch.from_numpy(mine)
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send)
    bounds = [shard_outputs(n_total, world, r) for r in range(world)]
    full = torch.cat([parts[r][: b - a] for r, (a, b) in enumerate(bounds)]).numpy()
    if rank != 0:
        return {}
    from oracle import oracle

    ok = bool(np.array_equal(full.view(np.uint64), oracle.run_outputs(plan, inputs).view(np.uint64)))
    return {"metric": METRIC, "value": n_total / sec, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "emulated": True,
            "config": dict(config_dict(cfg, args, plan), parity="bitwise" if ok else "MISMATCH",
                           shards=[list(b) for b in bounds],
                           parallelism=f"CPU emulation, gloo x{world}: one evaluation, each rank its own plan shard "
                                       "(shard.shard_plan), slices all-gathered and compared with the oracle")}


def compact(line: dict) -> dict:
    """The other_configs entry of a config's full line."""
    roof = line.get("roofline", {})
    whole = roof.get("whole_evaluation", {})
    return {
        "workload": line["config"]["workload"], "value": line["value"], "unit": line["unit"],
        "ms_per_step": line["ms_per_step"], "steps": line["steps"], "parity": line["config"].get("parity"),
        "mode": line["config"].get("mode"),
        "roofline": {"kernel": roof.get("kernel"), "achieved": roof.get("achieved"), "frac": roof.get("frac"),
                     "whole_evaluation_gbs": whole.get("achieved"), "whole_evaluation_frac": whole.get("frac")},
        "launches": line.get("launches"), "e2e": line.get("e2e"), "clocks": line.get("clocks"),
        "cpu_baseline": line.get("cpu_baseline"), "gpu_launches": line.get("gpu_launches"),
    }


# -- the reference arm ------------------------------------------------------------------------------


def run_reference(args) -> int:
    """``--impl reference``: the reference's CPU evaluator (its emitted C, all host threads) on the
    headline config; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg = args.config
    key, plan = build_workload(cfg, args)
    n_out = len(plan.outputs)
    inputs = workload_inputs(cfg, args, seed=0, plan=plan)
    cores = host_cores()
    os.environ["OMP_NUM_THREADS"] = str(cores)
    dll, kind, what = reference_library(plan, key, openmp=True)
    t, n, _ = time_sg_run(_sg_run_fn(dll, plan), plan, inputs, budget_s=120.0, max_evals=args.steps)
    v = n_out / t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": n,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(cfg, args, plan),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"full plan, {n} sg_run evaluations after 1 warm-up; {what}, cc -O3 "
                                   f"-ffp-contract=off -fopenmp, {cpu_model()}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# -- main -------------------------------------------------------------------------------------------


def spawn(args, argv) -> int:
    """``--gpus N`` without a torchrun environment: re-run this command under torchrun, N ranks."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + list(argv)
    return subprocess.call(cmd)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=CONFIGS, default="c2",
                    help="headline config: c2 (default, BASELINE configs[1]), c1 spgemm, c3 FEM, c4 ARAP, c5 batched")
    ap.add_argument("--only", action="store_true", help="N=1: the headline config only (no other_configs)")
    ap.add_argument("--w", type=int, default=1000, help="C2 grid width (1000 -> 10^6 vertices)")
    ap.add_argument("--m", type=int, default=55, help="C3 cubes per axis (55 -> 998,250 tets)")
    ap.add_argument("--w4", type=int, default=708, help="C4 grid width (708 -> 501,264 vertices)")
    ap.add_argument("--w5", type=int, default=200, help="C5 grid width")
    ap.add_argument("--batch", type=int, default=256, help="C5 value sets (whole job)")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=20)
    ap.add_argument("--split", choices=("outputs", "replicas"), default="outputs",
                    help="N>1, C1-C4: one evaluation with its CSR outputs split across ranks (strong scaling), "
                         "or one full evaluation per rank (weak)")
    ap.add_argument("--split-world", type=int, default=0,
                    help="N=1: time one rank's share of an outputs split this many ways")
    ap.add_argument("--split-rank", type=int, default=0)
    ap.add_argument("--emulate", action="store_true",
                    help="test infrastructure: the multi-rank path on CPU (gloo + the device-plan emulator)")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    return args


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    args = parse_args(argv)
    rank, world, local = dist_env()
    if (args.gpus > 1 or args.emulate) and "WORLD_SIZE" not in os.environ:
        return spawn(args, argv)
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        log(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
        return 2
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    if args.emulate:
        dist.init_process_group("gloo")
        line = measure_emulated(args, rank, world, dist.barrier)
        if rank == 0:
            print(json.dumps(line), flush=True)
        dist.destroy_process_group()
        return 0

    torch.cuda.set_device(local)
    barrier = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        barrier = dist.barrier
    t0 = time.perf_counter()
    if args.config == "c5":
        line = measure_batched(args, rank, world, barrier)
    else:
        split = None
        if world > 1 and args.split == "outputs":
            split = (world, rank)
        elif args.split_world > 1:
            split = (args.split_world, args.split_rank)
        line = measure_eval(args.config, args, rank, world, barrier, split)
    if rank == 0 and world == 1 and not args.only and args.split_world <= 1:
        others = {}
        for cfg in CONFIGS:
            if cfg == args.config:
                continue
            t1 = time.perf_counter()
            try:
                sub = measure_batched(args, 0, 1, None) if cfg == "c5" else measure_eval(cfg, args, 0, 1, None)
                others[cfg] = compact(sub)
            except Exception as e:  # noqa: BLE001 -- one config failing must not lose the headline line
                others[cfg] = {"error": f"{type(e).__name__}: {e}"}
            log(f"[bench] {cfg} done in {time.perf_counter() - t1:.0f}s")
        line["other_configs"] = others
    if rank == 0:
        line["bench_wall_s"] = time.perf_counter() - t0
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
