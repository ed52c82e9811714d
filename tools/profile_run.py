"""Short evaluation loop for ncu captures (not a benchmark: numbers under a profiler are not bench values).

Uses bench.py's plan cache, so a capture after a bench run on the same box skips the plan build.

    ncu --set full -k regex:sgb_wbulk -c 1 python tools/profile_run.py --config c2 --evals 3
"""
import argparse
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--config", choices=("c1", "c2", "c3", "c4"), default="c2")
ap.add_argument("--evals", type=int, default=3)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--wbulk", choices=("auto", "on", "off"), default="auto", help="bulk-fed CSR windows")
ap.add_argument("--schedule", choices=("auto", "inst", "frac"), default="inst",
                help="tile schedule: auto = DevicePlan.autotune (its timing launches distort a capture)")
ap.add_argument("--grid", choices=("persistent", "tiles"), default="persistent",
                help="specialised-unit grid when --schedule is not auto")
args, rest = ap.parse_known_args()
if args.schedule != "auto":
    os.environ["SGB_AUTOTUNE"] = "0"

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2110_12865_b200 import DevicePlan, lower_plan  # noqa: E402

ns = bench.parse_args(rest)
t0 = time.time()
key, plan = bench.build_workload(args.config, ns)
print(f"plan {key} ready in {time.time() - t0:.1f}s: {len(plan.kernels)} kernels, {len(plan.outputs)} outputs",
      flush=True)
kw = {} if args.wbulk == "auto" else {"wbulk": args.wbulk == "on"}
dp = DevicePlan(plan, lowered=lower_plan(plan, relayout=os.environ.get("SGB_RELAYOUT", "auto"), **kw))
if args.schedule == "frac" and dp.lowered.tiles_alt is not None:
    dp.set_tiles(dp.lowered.tiles_alt)
if args.schedule != "auto" and args.grid == "tiles":
    for w in range(dp.csr_launches):
        dp.set_wave_grid(w, True)
print("csr launches", dp.csr_launches, "bulk windows", dp.lowered.wbulk is not None, flush=True)
inputs = bench.workload_inputs(args.config, ns, 0, plan)
if args.batch:
    X = torch.zeros((plan.value_array_size, args.batch), dtype=torch.float64, device="cuda")
    X[: plan.input_count] = torch.from_numpy(inputs).cuda()[:, None]
    out = torch.empty((len(plan.outputs), args.batch), dtype=torch.float64, device="cuda")
    for _ in range(args.evals):
        dp.run_batch_csr(X, out)
else:
    x = dp.new_values(inputs)
    out = torch.empty(len(plan.outputs), dtype=torch.float64, device="cuda")
    for _ in range(args.evals):
        dp.run_csr(x, out)
torch.cuda.synchronize()
print("done", flush=True)
