"""Time every launch of one evaluation for builder / lowering variants (dev tool)."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_12865_b200 import DevicePlan  # noqa: E402
from paper_2110_12865_b200.lower import lower_plan  # noqa: E402
from paper_2110_12865_b200.programs.mesh import build_lmlt_plan, lmlt_inputs  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
inputs = lmlt_inputs(w)
ref = None
for split in ("0",):
    os.environ["SGB_SPLIT"] = split
    t0 = time.time()
    plan, _, _ = build_lmlt_plan(w)
    print(f"split={split}: built in {time.time() - t0:.1f}s, {len(plan.kernels)} kernels", flush=True)
    for comp, vec in ((True, "1"), (True, "2"), (True, "4"), (True, "0")):
        os.environ["SGB_TAPE_VEC"] = vec
        dp = DevicePlan(plan, lowered=lower_plan(plan, compress=comp))
        x = dp.new_values(inputs)
        out = torch.empty(len(plan.outputs), dtype=torch.float64, device="cuda")
        for _ in range(5):
            dp.run_values(x)
            dp.gather_outputs(x, out)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        if ref is None:
            ref = got
        same = np.array_equal(got.view(np.uint64), ref.view(np.uint64))
        R = 20
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(dp.units + 2)] for _ in range(R)]
        for r in range(R):
            k = 0
            for wv in range(dp.launches):
                for u in range(dp.units):
                    pass
            # one event per wave
            for wv in range(dp.launches):
                ev[r][wv].record()
                dp.run_wave(x, wv)
            ev[r][dp.launches].record()
            dp.gather_outputs(x, out)
            ev[r][dp.launches + 1].record()
        torch.cuda.synchronize()
        per = np.zeros(dp.launches + 1)
        for r in range(R):
            for j in range(dp.launches + 1):
                per[j] += ev[r][j].elapsed_time(ev[r][j + 1]) / R
        print(f"  compress={comp} vec={vec} same={same} total={per.sum():.3f} ms waves={np.round(per, 4).tolist()} "
              f"units={dp.units}", flush=True)
        dp.close()
