"""A few batched C5 evaluations for an ncu launch list (lower.BATCH_DIRECT from argv[1])."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import os  # noqa: E402

os.environ["SGB_AUTOTUNE"] = "0"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2110_12865_b200 import DevicePlan, lower  # noqa: E402

lower.BATCH_DIRECT = sys.argv[1] == "1"
args = bench.parse_args(["--config", "c5"])
key, plan = bench.build_workload("c5", args)
dp = DevicePlan(plan, csr_layout=True)
b = 256
X = torch.zeros((plan.value_array_size, b), dtype=torch.float64, device="cuda")
X[: plan.input_count] = torch.from_numpy(np.stack([bench.workload_inputs("c5", args, seed=s) for s in range(4)] * 64,
                                                   axis=1)).cuda()
out = torch.empty((len(plan.outputs), b), dtype=torch.float64, device="cuda")
for _ in range(3):
    dp.run_batch_csr(X, out)
torch.cuda.synchronize()
print("done")
