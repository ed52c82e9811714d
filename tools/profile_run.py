"""Short evaluation loop for ncu captures (not a benchmark: numbers under a profiler are not bench values).

Uses bench.py's plan cache, so a capture after a bench run on the same box skips the plan build.
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--w", type=int, default=1000)
ap.add_argument("--evals", type=int, default=3)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--mode", choices=("csr", "val"), default="csr")
ap.add_argument("--config", choices=("c2", "c3", "c4"), default="c2")
ap.add_argument("--m", type=int, default=55)
ap.add_argument("--w4", type=int, default=708)
ap.add_argument("--layout", choices=("csr", "reference"), default="csr")
ap.add_argument("--schedule", choices=("auto", "inst", "frac"), default="inst",
                help="tile schedule: auto = DevicePlan.autotune (its timing launches distort a capture)")
ap.add_argument("--grid", choices=("persistent", "tiles"), default="persistent",
                help="specialised-unit grid when --schedule is not auto")
args = ap.parse_args()
if args.schedule != "auto":
    import os

    os.environ["SGB_AUTOTUNE"] = "0"

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2110_12865_b200 import DevicePlan  # noqa: E402

t0 = time.time()
key, plan, _, _ = bench.build_workload(args, 0, 1)
print(f"plan {key} ready in {time.time() - t0:.1f}s: {len(plan.kernels)} kernels, {len(plan.outputs)} outputs",
      flush=True)
dp = DevicePlan(plan, csr_layout=args.layout == "csr" and args.mode == "csr")
if args.schedule == "frac" and dp.lowered.tiles_alt is not None:
    dp.set_tiles(dp.lowered.tiles_alt)
if args.schedule != "auto" and args.grid == "tiles":
    for w in range(dp.csr_launches):
        dp.set_wave_grid(w, True)
print("waves", dp.launches, "units", dp.units, "csr units", dp.csr_units, flush=True)
if args.batch:
    X = torch.zeros((plan.value_array_size, args.batch), dtype=torch.float64, device="cuda")
    X[: plan.input_count] = torch.from_numpy(bench.workload_inputs(args, 0)).cuda()[:, None]
    out = torch.empty((len(plan.outputs), args.batch), dtype=torch.float64, device="cuda")
    for _ in range(args.evals):
        dp.run_batch_csr(X, out)
else:
    x = dp.new_values(bench.workload_inputs(args, 0))
    out = torch.empty(len(plan.outputs), dtype=torch.float64, device="cuda")
    for _ in range(args.evals):
        if args.mode == "csr":
            dp.run_csr(x, out)
        else:
            dp.run_values(x)
torch.cuda.synchronize()
print("done", flush=True)
