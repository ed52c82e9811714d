"""Time the batched CSR step (C5 plan) for JIT variants (dev tool; env set per variant in-process)."""
import argparse
import importlib
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for var in sys.argv[2].split(","):
    env = dict(kv.split("=") for kv in var.split(";") if kv)
    for k_, e_ in (("bvec", "SGB_BATCH_VEC"), ("jitvec", "SGB_JIT_VEC")):
        if k_ in env:
            os.environ[e_] = env[k_]
        else:
            os.environ.pop(e_, None)
    import paper_2110_12865_b200.jit as J
    importlib.reload(J)
    from paper_2110_12865_b200 import DevicePlan
    from paper_2110_12865_b200.lower import lower_plan
    ns = argparse.Namespace(config="c2", w=200)
    _, plan, _, _ = bench.build_workload(ns, 0, 1)
    dp = DevicePlan(plan, lowered=lower_plan(plan))
    X = torch.zeros((plan.value_array_size, B), dtype=torch.float64, device="cuda")
    X[: plan.input_count] = torch.from_numpy(bench.workload_inputs(ns, 0)).cuda()[:, None]
    out = torch.empty((len(plan.outputs), B), dtype=torch.float64, device="cuda")
    for _ in range(3):
        dp.run_batch_csr(X, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nw = dp.launches
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(nw + 2)]
    ev[0].record()
    for w in range(nw):
        pass
    dp.run_batch(X)
    ev[1].record()
    dp.gather_outputs_batch(X, out)
    ev[2].record()
    e0.record()
    for _ in range(5):
        dp.run_batch_csr(X, out)
    e1.record()
    torch.cuda.synchronize()
    print(f"{var}: step {e0.elapsed_time(e1) / 5:.3f} ms (waves {ev[0].elapsed_time(ev[1]):.3f} + gather "
          f"{ev[1].elapsed_time(ev[2]):.3f})", flush=True)
