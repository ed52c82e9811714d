#!/usr/bin/env python
"""Benchmark: fp64 plan evaluation on B200 (arXiv 2110.12865 hot path).

Default workload = BASELINE.json configs[1] (C2): out = L.M.L^T + A on the
cotan Laplacian of a 1000 x 1000 grid mesh (10^6 vertices, ~25M output
nonzeros), plan built by the template-instancing builder
(paper_2110_12865_b200.programs.mesh; bit-identical to the reference trace,
tests/test_builders.py).  One step = one CSR-mode evaluation (sgb_run_csr:
every dependency wave, outputs stored at their CSR positions by the producing
kernels) on inputs already resident in HBM; the value array (~385 MB), the
25M-entry CSR output (~200 MB) and the tables exceed the 126 MB L2, so no
explicit flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

N > 1: every rank evaluates the plan on its own input value set (independent
value sets sharded across GPUs: weak scaling, no data-path collective); the
timed region is bracketed by barriers and the max over ranks is reported.

`--impl reference` times the reference's CPU evaluator (the emitted-C
`sg_run`, restated in oracle/emit_c.py, built with the reference flags
`-O3 -ffp-contract=off` plus -fopenmp, all host threads) on the same plan.
"""

from __future__ import annotations

import argparse
import dataclasses
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


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# -- workload -----------------------------------------------------------------------


def _config(args) -> str:
    return getattr(args, "config", "c2") or "c2"


def workload_key(args) -> str:
    if _config(args) == "c3":
        return f"fem_nh_m{args.m}"
    if _config(args) == "c4":
        return f"arap_w{args.w4}"
    return f"lmlt_w{args.w}_a6_s7_split{os.environ.get('SGB_SPLIT', '0')}"


def _build(args):
    cfg = _config(args)
    if cfg == "c3":
        from paper_2110_12865_b200.programs.fem import build_fem_plan

        return build_fem_plan(args.m)
    if cfg == "c4":
        from paper_2110_12865_b200.programs.arap import build_arap_plan

        return build_arap_plan(args.w4)
    from paper_2110_12865_b200.programs.mesh import build_lmlt_plan

    return build_lmlt_plan(args.w)


def build_workload(args, rank: int, world: int, barrier=None):
    """Plan + CSR pattern for the configured workload, cached across ranks."""
    key = workload_key(args)
    cache_dir = Path(os.environ.get("SGB_PLAN_CACHE", Path(tempfile.gettempdir()) / "sgb_plan_cache"))
    from paper_2110_12865_b200.programs import builder_hash  # a cache is valid only for its builder sources

    path = cache_dir / f"{key}.{builder_hash()[:12]}.pkl"
    if rank == 0 and not path.exists():
        t0 = time.perf_counter()
        plan, row_ptr, col_idx = _build(args)
        log(f"[bench] built plan {key} in {time.perf_counter() - t0:.1f}s")
        cache_dir.mkdir(parents=True, exist_ok=True)
        tmp = path.with_suffix(f".{os.getpid()}.tmp")
        with open(tmp, "wb") as fh:
            pickle.dump((plan, row_ptr, col_idx), fh, protocol=pickle.HIGHEST_PROTOCOL)
        os.replace(tmp, path)
    if barrier is not None:
        barrier()
    with open(path, "rb") as fh:
        plan, row_ptr, col_idx = pickle.load(fh)
    return key, plan, row_ptr, col_idx


def workload_inputs(args, seed: int):
    cfg = _config(args)
    if cfg == "c3":
        from paper_2110_12865_b200.programs.fem import fem_inputs

        return fem_inputs(args.m, seed=seed)
    if cfg == "c4":
        from paper_2110_12865_b200.programs.arap import arap_inputs

        return arap_inputs(args.w4, seed=seed)
    from paper_2110_12865_b200.programs.mesh import lmlt_inputs

    return lmlt_inputs(args.w, seed=seed)


def workload_name(args, n_out):
    cfg = _config(args)
    if cfg == "c3":
        return (f"C3 Neo-Hookean tet FEM Hessian assembled to CSR, Kuhn mesh of {args.m}^3 cubes "
                f"({6 * args.m ** 3} tets), mu=1 lam=10, {n_out} output nnz")
    if cfg == "c4":
        return f"C4 ARAP system matrix + rhs on a {args.w4}x{args.w4} grid mesh, {n_out} outputs"
    return (f"C2 L.M.L^T+A, cotan Laplacian of a {args.w}x{args.w} grid mesh "
            f"({args.w * args.w} vertices), A random 6 nnz/row (seed 7), {n_out} output nnz")


# -- clocks ------------------------------------------------------------------------


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


# -- CPU reference -------------------------------------------------------------------


def _reference_sg_run(plan, key):
    """The reference's own emitted C for this plan (oracle/_ref, made by oracle/make_ref.py), or None."""
    import ctypes

    from oracle import make_ref

    src, ok = make_ref.lookup(plan, key)
    if src is None or not ok:
        return None
    lib = Path(tempfile.gettempdir()) / f"sgb_ref_{key}_{os.getpid()}.so"
    # emit.py:220 flags + -fopenmp (the emitted source carries `#pragma omp parallel for`)
    subprocess.run(["cc", "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-fopenmp", "-o", str(lib), str(src), "-lm"],
                   check=True, capture_output=True)
    dll = ctypes.CDLL(str(lib))
    dll.sg_run.restype = None
    dll.sg_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    con = np.ascontiguousarray(plan.constants, dtype=np.float64)
    pos = np.ascontiguousarray(plan.positions, dtype=np.uint32)

    def sg_run(x):
        dll.sg_run(x.ctypes.data, con.ctypes.data if con.size else None, pos.ctypes.data if pos.size else None)
        return x

    sg_run.keep = (dll, con, pos)
    return sg_run


def cpu_reference(plan, inputs, steps: int, warmup: int, budget_s: float = 20.0, key: str | None = None):
    """The reference's native evaluator (emitted-C sg_run) with OpenMP on every host thread.

    Prefers the reference's own emitted source (oracle/_ref/<key>.c, kind "reference"); falls back
    to the restated emitter (oracle/emit_c.py, kind "port") when it is absent or stale.
    """
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    sg_run = _reference_sg_run(plan, key) if key else None
    kind, what = "reference", f"sparsegen.emit.emit_kernel_source output (oracle/_ref/{key}.c)"
    if sg_run is None:
        from oracle import emit_c

        sg_run = emit_c.compile_plan(plan, parallel="pragma", openmp=True).sg_run
        kind, what = "port", "emitted C restated by oracle/emit_c.py (emit.py:153-245)"
    x = np.zeros(plan.value_array_size, np.float64)
    for _ in range(max(warmup, 1)):
        x[:] = 0.0
        x[: plan.input_count] = inputs
        sg_run(x)
    times = []
    t_start = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        sg_run(x)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    t = statistics.mean(times)
    return {"seconds_per_eval": t, "evals": len(times), "cores": cores, "x": x, "kind": kind, "what": what}


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# -- main ----------------------------------------------------------------------------


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    key, plan, _, _ = build_workload(args, 0, 1)
    n_out = len(plan.outputs)
    inputs = workload_inputs(args, seed=0)
    res = cpu_reference(plan, inputs, args.steps, args.warmup, budget_s=120.0, key=key)
    v = n_out / res["seconds_per_eval"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": res["evals"], "warmup": args.warmup, "ms_per_step": res["seconds_per_eval"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": workload_name(args, n_out), "w": args.w},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": res["cores"], "kind": res["kind"],
                         "sample": f"full plan, {res['evals']} sg_run evaluations after {args.warmup} warm-up; "
                                   f"{res['what']}, cc -O3 -ffp-contract=off -fopenmp, {cpu_model()}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _peak_gbs():
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    if peaks_path.exists():
        return float(json.loads(peaks_path.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def run_batched(args):
    """C5: one L.M.L^T+A plan (GridMesh(200,200), 991,912 out nnz) x 256 value sets, the value sets
    sharded across the ranks (strong scaling: the 256 sets are the whole job); no collective in the
    step.  ``--gather`` adds the NCCL gather of every rank's CSR block to rank 0 (timed separately)."""
    import torch
    import torch.distributed as dist

    from paper_2110_12865_b200 import DevicePlan
    from paper_2110_12865_b200.metrics import plan_balg, wave_traffic
    from paper_2110_12865_b200.programs.mesh import lmlt_inputs

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    barrier = dist.barrier if world > 1 else None
    args.w = args.w5
    key, plan, _, _ = build_workload(args, rank, world, barrier)
    n_out, n_in = len(plan.outputs), int(plan.input_count)
    from paper_2110_12865_b200.shard import gather_csr, max_over_ranks, shard_value_sets

    total = args.batch
    per = [shard_value_sets(total, world, r)[1] for r in range(world)]
    first, b = shard_value_sets(total, world, rank)
    sets = list(range(first, first + b))  # value set s = lmlt_inputs(seed=s)
    host_in = np.stack([lmlt_inputs(args.w, seed=s_) for s_ in sets], axis=1)  # [n_in, b]
    dp = DevicePlan(plan, device=local, csr_layout=args.layout == "csr")
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
    with sampler:
        t_end = time.perf_counter() + 1.0
        while time.perf_counter() < t_end:
            dp.run_batch_csr(X, out)
            torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
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
    ms = max_over_ranks(sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps, X.device)
    gather_ms = None
    if args.gather and world > 1:  # NCCL gather of every rank's CSR block to rank 0 (not in the step)
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
    # e2e through the public API: host inputs (pinned) -> device -> batched CSR -> host, the rank's
    # value sets in chunks whose copies in / evaluation / copies out overlap (run_batch_outputs_host)
    n_chunks = next(c for c in (8, 4, 2, 1) if b % c == 0 and b // c >= 1)
    cb = b // n_chunks
    hin = torch.from_numpy(np.ascontiguousarray(host_in.reshape(n_in, n_chunks, cb).transpose(1, 0, 2))).pin_memory()
    hout = torch.empty((n_chunks, n_out, cb), dtype=torch.float64).pin_memory()
    del X  # the chunk workspaces replace the whole-batch array
    torch.cuda.empty_cache()
    dp.run_batch_outputs_host(hin, hout)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        dp.run_batch_outputs_host(hin, hout)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.e2e_steps, out.device)
    e2e_ok = bool(np.array_equal(hout.numpy().transpose(1, 0, 2).reshape(n_out, b).view(np.uint64),
                                 out.cpu().numpy().view(np.uint64)))
    if rank != 0:
        dist.destroy_process_group()
        return 0
    traffic = wave_traffic(plan, dp.lowered, batch=b)
    step_bytes = sum(t.bytes for t in traffic)
    peak, peak_src = _peak_gbs()
    achieved = step_bytes / (ms * 1e-3) / 1e9  # whole step (per-launch events are not recorded here)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        k_cpu = 8  # bounded sample: 8 value sets through the reference's emitted sg_run (OpenMP)
        res = cpu_reference(plan, host_in[:, 0], k_cpu, 1, key=key)
        cpu = {"value": n_out / res["seconds_per_eval"], "unit": UNIT, "cores": res["cores"], "kind": res["kind"],
               "sample": f"{res['evals']} sequential sg_run evaluations of one value set (the reference has no batch "
                         f"API; SURVEY 8(d) C5); {res['what']}, cc -O3 -ffp-contract=off -fopenmp"}
    line = {
        "metric": METRIC, "value": total * n_out / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C5 batched: L.M.L^T+A plan on a {args.w}x{args.w} grid ({n_out} out nnz) x "
                               f"{total} value sets, {per} per rank", "out_nnz": n_out, "value_sets": total,
                   "parallelism": f"value sets sharded over {world} GPU(s), plan replicated, no collective in the step",
                   "l2": "no flush: X (%.1f GB per rank) exceeds L2" % (plan.value_array_size * b * 8 / 1e9),
                   "parity": parity, "nccl_gather_ms": gather_ms},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": "whole batched step (waves + gather)", "algorithmic_bytes": step_bytes,
                     "peak_source": peak_src, "balg_single_pass_per_set": plan_balg(plan)},
        "e2e": {"value": total * n_out / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * n_in * b,
                "d2h_bytes_per_step": 8 * n_out * b,
                "api": (f"DevicePlan.run_batch_outputs_host: {n_chunks} chunks of {cb} value sets per rank from pinned "
                        "host memory, copy in / sgb_run_batch_csr / copy out pipelined on three streams"),
                "matches_device_run": e2e_ok},
        "gpu_launches": dp.csr_units, "clocks": sampler.summary(), "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_spgemm(args):
    """C1: C = A.B, random CSR 2000x2000, 10 nnz/row -- the reference's own plan (tests/golden/spgemm_n2000_k10,
    written by sparsegen.codegen.save_plan).  3.5 MB per evaluation sits in L2, so every step flushes L2
    (untimed) before the timed evaluation."""
    import torch

    from paper_2110_12865_b200 import DevicePlan, load_plan

    gdir = ROOT / "tests" / "golden" / "spgemm_n2000_k10"
    plan = load_plan(gdir)
    with np.load(gdir / "vectors.npz") as z:
        inputs, ref_values = z["inputs"], z["values"]
    n_out = len(plan.outputs)
    dp = DevicePlan(plan, csr_layout=args.layout == "csr")
    x = dp.new_values(inputs)
    out = torch.empty(n_out, dtype=torch.float64, device=x.device)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=x.device)  # 512 MB > L2
    for _ in range(args.warmup):
        dp.run_csr(x, out)
    torch.cuda.synchronize()
    want = ref_values[np.asarray(plan.outputs, np.int64)]
    parity = "bitwise vs reference interpret_plan" if np.array_equal(out.cpu().numpy().view(np.uint64),
                                                                     want.view(np.uint64)) else "MISMATCH"
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(0)
    graph = dp.capture_csr(x, out)  # launch-bound: one graph launch per evaluation
    with sampler:
        for e0, e1 in evs:
            flush.fill_(1.0)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
        torch.cuda.synchronize()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps
    inp_h = torch.from_numpy(inputs).pin_memory().numpy()
    out_h = torch.empty(n_out, dtype=torch.float64).pin_memory().numpy()
    dp.run_outputs_host(inp_h, out_h)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps * 20):
        dp.run_outputs_host(inp_h, out_h)
    serial_s = (time.perf_counter() - t0) / (args.e2e_steps * 20)
    # a small plan is launch-bound per value set: the e2e stream carries value sets in batched chunks
    # (sgb_run_batch_csr per chunk, copies of neighbouring chunks overlapping)
    n_chunks, cb = 8, max(1, args.e2e_steps * 20 // 8)
    k_sets = n_chunks * cb
    hin = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(inputs[None, :, None],
                                                                (n_chunks, inputs.size, cb)))).pin_memory()
    hout = torch.empty((n_chunks, n_out, cb), dtype=torch.float64).pin_memory()
    dp.run_batch_outputs_host(hin, hout)  # warm
    t0 = time.perf_counter()
    dp.run_batch_outputs_host(hin, hout)
    e2e_s = (time.perf_counter() - t0) / k_sets
    e2e_ok = bool(np.all(hout.numpy().view(np.uint64) == out.cpu().numpy().view(np.uint64)[None, :, None]))
    cpu = None
    if not args.no_cpu_baseline:
        res = cpu_reference(plan, inputs, 200, 5, key="spgemm_n2000_k10")
        cpu = {"value": n_out / res["seconds_per_eval"], "unit": UNIT, "cores": res["cores"], "kind": res["kind"],
               "sample": f"{res['evals']} sg_run evaluations ({res['what']}, cc -O3 -ffp-contract=off -fopenmp); "
                         f"the reference's plan build (trace 0.94 s + build_plan 2.85 s, SURVEY 6.3) is not included"}
    peak, peak_src = _peak_gbs()
    from paper_2110_12865_b200.metrics import plan_balg

    bal = plan_balg(plan)
    line = {
        "metric": METRIC, "value": n_out / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C1 spgemm C=A.B, random CSR 2000x2000 10 nnz/row, {n_out} out nnz (reference plan)",
                   "l2": "flushed (512 MB write) before every timed evaluation", "parity": parity,
                   "launch": "CUDA graph of one sgb_run_csr evaluation, replayed per step"},
        "roofline": {"bound": "hbm", "achieved": bal / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": bal / (ms * 1e-3) / 1e9 / peak, "traffic": None, "kernel": "whole evaluation",
                     "algorithmic_bytes": bal, "peak_source": peak_src},
        "e2e": {"value": n_out / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * int(plan.input_count),
                "d2h_bytes_per_step": 8 * n_out,
                "api": (f"DevicePlan.run_batch_outputs_host: {k_sets} value sets from pinned host memory in "
                        f"{n_chunks} chunks of {cb} (sgb_run_batch_csr per chunk), copy in / evaluate / copy out "
                        "pipelined on three streams, wall clock over the call"),
                "serial_value": n_out / serial_s,
                "serial_api": "DevicePlan.run_outputs_host -> sgb_run_outputs_host, one synchronous call per step",
                "matches_device_run": e2e_ok},
        "gpu_launches": dp.csr_units, "clocks": sampler.summary(), "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--w", type=int, default=1000, help="grid width (1000 -> 10^6 vertices, config C2)")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=20)
    ap.add_argument("--config", choices=("c1", "c2", "c3", "c4", "c5"), default="c2",
                    help="BASELINE.json config: c2 (default, configs[1]), c1 spgemm, c3 FEM, c4 ARAP, c5 batched")
    ap.add_argument("--m", type=int, default=55, help="C3 cubes per axis (55 -> 998,250 tets)")
    ap.add_argument("--w4", type=int, default=708, help="C4 grid width (708 -> 501,264 vertices)")
    ap.add_argument("--w5", type=int, default=200, help="C5 grid width")
    ap.add_argument("--batch", type=int, default=256, help="C5 value sets (whole job)")
    ap.add_argument("--gather", action="store_true", help="C5: also time the NCCL gather to rank 0")
    ap.add_argument("--split", choices=("replicas", "outputs"), default="replicas",
                    help="N>1: replicas (one evaluation per rank) or one evaluation with its CSR outputs split")
    ap.add_argument("--split-world", type=int, default=0, help="outputs split: ways (default = world size)")
    ap.add_argument("--split-rank", type=int, default=None, help="outputs split: this process's slice")
    ap.add_argument("--layout", choices=("csr", "reference"), default="csr",
                    help="csr: multi-root groups whose readers gather across roots store instance-major "
                         "(lower.choose_relayout); reference: the plan's own value-array layout")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c5":
        return run_batched(args)
    if args.config == "c1":
        return run_spgemm(args)

    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        barrier = dist.barrier
    else:
        barrier = None

    from paper_2110_12865_b200 import DevicePlan
    from paper_2110_12865_b200.metrics import csr_wave_traffic, plan_balg, wave_traffic

    key, plan, row_ptr, col_idx = build_workload(args, rank, world, barrier)
    n_total = len(plan.outputs)
    split = None
    if args.split == "outputs":
        # one evaluation, CSR outputs partitioned: this rank computes its slice's producer cone
        from paper_2110_12865_b200 import lower_plan
        from paper_2110_12865_b200.shard import shard_device_plan, shard_outputs

        s_world = args.split_world or world
        s_rank = rank if args.split_rank is None else args.split_rank
        lo, hi = shard_outputs(n_total, s_world, s_rank)
        lw_full = lower_plan(plan, relayout=False)
        full_tiles = lw_full.units[:, 6] - lw_full.units[:, 5]
        plan, lw_s = shard_device_plan(plan, lw_full, lo, hi)
        split = {"world": s_world, "rank": s_rank, "outputs": [lo, hi],
                 "tiles_kept": int(len(lw_s.tiles)), "tiles_full": int(len(lw_full.tiles)),
                 "unit_tile_frac": [(int(k), int(f)) for k, f in zip(lw_s.units[:, 6] - lw_s.units[:, 5], full_tiles)]}
        dp = DevicePlan(plan, device=local, lowered=lw_s)
        inputs = workload_inputs(args, seed=0)  # every rank: the same value set
        args.no_cpu_baseline = True  # the CPU reference evaluates whole plans (the N=1 line carries it)
    else:
        inputs = workload_inputs(args, seed=rank)
        dp = DevicePlan(plan, device=local, csr_layout=args.layout == "csr")
    n_out = len(plan.outputs)
    x = dp.new_values(inputs)
    out = torch.empty(n_out, dtype=torch.float64, device=x.device)
    stream = torch.cuda.current_stream()

    if dp.lowered.needs_zero == 2:
        raise SystemExit("bench: plan reads slots later waves write; re-zeroing per step is not implemented")

    # warm-up, then parity of this rank's evaluation against the oracle (rank 0)
    for _ in range(args.warmup):
        dp.run_csr(x, out)
    torch.cuda.synchronize()
    parity = None
    if rank == 0:
        from oracle import oracle

        want = oracle.run_outputs(getattr(plan, "_plan", plan), inputs)
        if split:
            want = want[split["outputs"][0]: split["outputs"][1]]
        got = out.cpu().numpy()
        parity = "bitwise" if np.array_equal(got.view(np.uint64), want.view(np.uint64)) else "MISMATCH"
        if parity == "MISMATCH" and not dp.lowered.exact:  # LOG / EXP / ...: CUDA libm vs glibc
            rel = np.abs(got - want) / np.maximum(1.0, np.maximum(np.abs(got), np.abs(want)))
            if float(rel.max()) <= 1e-12:
                parity = f"within 1e-12 (max rel {float(rel.max()):.2e}; transcendental ops, CUDA libm vs glibc)"
        log(f"[bench] parity vs oracle: {parity}")

    # settle clocks for ~1 s of real work (untimed), sampling clocks throughout
    n_w = dp.csr_launches
    sampler = ClockSampler(local)
    with sampler:
        t_end = time.perf_counter() + 1.0
        while time.perf_counter() < t_end:
            for _ in range(20):
                dp.run_csr(x, out)
            torch.cuda.synchronize()
        # ---- timed region: one step = one CSR-mode evaluation (inputs -> CSR values), replayed
        #      as a CUDA graph of every wave's launches and the output gather ----
        graph = dp.capture_csr(x, out)
        steps_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    for _ in range(args.steps)]
        if barrier:
            barrier()
        torch.cuda.synchronize()
        for e0, e1 in steps_ev:
            e0.record(stream)
            graph.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        if barrier:
            barrier()
        # per-launch breakdown (separate pass, wave by wave with events between launches)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n_w + 1)] for _ in range(args.steps)]
        for k in range(args.steps):
            e = evs[k]
            for w in range(n_w):
                e[w].record(stream)
                dp.run_wave(x, w, out=out)
            e[n_w].record(stream)
        torch.cuda.synchronize()
    total_ms = steps_ev[0][0].elapsed_time(steps_ev[-1][1])  # whole timed region, K replays
    per_launch = np.zeros(n_w)
    for e in evs:
        for j in range(n_w):
            per_launch[j] += e[j].elapsed_time(e[j + 1])
    per_launch /= args.steps
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=x.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    job_out = n_total if split and split["world"] == world else world * n_out  # outputs the whole job produces
    value = job_out / (ms_per_step * 1e-3)

    # ---- end to end through the public host-buffer API (pinned host memory) ----
    # (a) one synchronous call per step (sgb_run_outputs_host): copy in, evaluate, copy out
    inp_h = torch.from_numpy(inputs).pin_memory().numpy()
    out_h = torch.empty(n_out, dtype=torch.float64).pin_memory().numpy()
    dp.run_outputs_host(inp_h, out_h)  # warm
    if barrier:
        barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        dp.run_outputs_host(inp_h, out_h)
    serial_s = (time.perf_counter() - t0) / args.e2e_steps
    want_bits = out.cpu().numpy().view(np.uint64)
    e2e_ok = bool(np.array_equal(out_h.view(np.uint64), want_bits))
    # (b) the headline: a stream of K value sets through sgb_run_outputs_host_many, each step's
    # inputs copied in and CSR values copied out inside the timed region, copies of neighbouring
    # steps overlapping the evaluation (PCIe is full duplex)
    k_sets = max(args.e2e_steps, 2)
    ins_h = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(inputs, (k_sets, inputs.size)))).pin_memory()
    outs_h = torch.empty((k_sets, n_out), dtype=torch.float64).pin_memory()
    dp.run_outputs_host_many(ins_h.numpy()[:2], outs_h.numpy()[:2])  # warm (second workspace)
    if barrier:
        barrier()
    t0 = time.perf_counter()
    dp.run_outputs_host_many(ins_h.numpy(), outs_h.numpy())
    e2e_s = (time.perf_counter() - t0) / k_sets
    if world > 1:
        t = torch.tensor([e2e_s, serial_s], dtype=torch.float64, device=x.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s, serial_s = float(t[0].item()), float(t[1].item())
    e2e_ok = e2e_ok and bool(all(np.array_equal(outs_h[k].numpy().view(np.uint64), want_bits)
                                 for k in range(k_sets)))
    del ins_h, outs_h

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant launch ----
    direct = bool(np.any(dp.lowered.groups["flags"] & (384 | 4096)))  # FLAG_OPOS16 | FLAG_OPOS32 | FLAG_WPOS16
    traffic = csr_wave_traffic(plan, dp.lowered) if direct else wave_traffic(plan, dp.lowered)
    assert len(traffic) == n_w, (len(traffic), n_w)
    if split:  # full-plan bytes scaled by the share of each wave's tiles the shard keeps (approximate)
        units = dp.lowered.units
        for w_, t in enumerate(traffic):
            sel = [j for j in range(len(units)) if int(units[j, 0]) == w_]
            kept = sum(split["unit_tile_frac"][j][0] for j in sel)
            full = sum(split["unit_tile_frac"][j][1] for j in sel)
            if full:
                f = kept / full
                traffic[w_] = dataclasses.replace(t, index_bytes=int(t.index_bytes * f), const_bytes=int(t.const_bytes * f),
                                                  read_bytes=int(t.read_bytes * f), write_bytes=int(t.write_bytes * f))
    dom = int(np.argmax(per_launch))
    dom_bytes = traffic[dom].bytes
    achieved = dom_bytes / (per_launch[dom] * 1e-3) / 1e9
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    if peaks_path.exists():
        peak = float(json.loads(peaks_path.read_text())["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    step_bytes = sum(t.bytes for t in traffic)
    ncu_traffic = None
    tpath = ROOT / "profiles" / f"traffic_{key}.json"
    if tpath.exists():
        try:
            ncu_traffic = json.loads(tpath.read_text()).get(traffic[dom].name)
        except Exception:
            ncu_traffic = None

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        res = cpu_reference(plan, inputs, args.cpu_steps, 1, key=key)
        cpu_ok = bool(np.array_equal(res["x"][np.asarray(plan.outputs)].view(np.uint64),
                                     out.cpu().numpy().view(np.uint64)))
        cpu = {"value": n_out / res["seconds_per_eval"], "unit": UNIT, "cores": res["cores"], "kind": res["kind"],
               "sample": f"full plan ({n_out} nnz), {res['evals']} sg_run evaluations; {res['what']}, "
                         f"cc -O3 -ffp-contract=off -fopenmp on {res['cores']} threads of {cpu_model()}; "
                         f"GPU==CPU bitwise: {cpu_ok}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if split else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {
            "workload": workload_name(args, n_out), "w": args.w, "out_nnz": n_out,
            "value_array": int(plan.value_array_size), "kernels": len(plan.kernels),
            "waves": n_w, "index_entries": int(np.asarray(plan.positions).size),
            "parallelism": (f"replicas x{world}: one full evaluation per GPU per step (independent value sets)"
                            if not split else
                            f"one evaluation, CSR outputs split {split['world']} ways (shard.shard_device_plan): "
                            f"this rank computes outputs {split['outputs']} from its producer cone "
                            f"({split['tiles_kept']} of {split['tiles_full']} tiles); no collective in the step"),
            "split": split,
            "l2": "no flush: value array + tables exceed the 126 MB L2",
            "clock_settle": "1 s of untimed evaluations before the timed region",
            "parity": parity, "mode": ("CSR, direct stores (sgb_run_csr)" if direct else
                                       "CSR (sgb_run_csr: value-array waves + u32-indexed output gather)"),
            "launch": "CUDA graph of one sgb_run_csr evaluation replayed per step; per-launch times from a "
                      "separate wave-by-wave pass",
            "layout": (f"CSR layout: plan groups {dp.lowered.csr_layout} store instance-major"
                       if dp.csr_layout else "reference value-array layout"),
            "tile_schedule": ({str(w): {"kept": o, **{k: round(v, 4) for k, v in dp.tile_timings[w].items()}}
                               for w, o in dp.tile_order.items()} if dp.tile_order else "no specialised units"),
            "achieved_hbm_gbs_step": step_bytes / (ms_per_step * 1e-3) / 1e9,
            "balg_bytes_step": step_bytes, "balg_bytes_single_pass": plan_balg(plan),
            "balg_gbs_single_pass": plan_balg(plan) / (ms_per_step * 1e-3) / 1e9,
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic, "kernel": traffic[dom].name,
                     "algorithmic_bytes": dom_bytes,
                     "avg_launch_ms": float(per_launch[dom]), "peak_source": peak_src},
        "launches": [{"name": t.name, "ms": float(ms), "alg_bytes": t.bytes,
                      "gbs": t.bytes / (ms * 1e-3) / 1e9 if ms > 0 else None}
                     for t, ms in zip(traffic, per_launch)],
        "e2e": {"value": job_out / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * int(plan.input_count),
                "d2h_bytes_per_step": 8 * n_out,
                "api": (f"DevicePlan.run_outputs_host_many -> sgb_run_outputs_host_many: {k_sets} value sets "
                        "from pinned host memory, per-set copy in / evaluate / copy out pipelined on "
                        "three streams, wall clock over the whole call"),
                "serial_value": job_out / serial_s,
                "serial_api": "DevicePlan.run_outputs_host -> sgb_run_outputs_host, one synchronous call per step",
                "matches_device_run": e2e_ok},
        "gpu_launches": args.steps * dp.csr_units,
        "clocks": sampler.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
