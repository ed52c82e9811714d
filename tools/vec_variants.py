"""Instances per thread of the specialised value-wave kernels (SGB_JIT_VEC) on C2 / C4: per-wave
times and the bits, one GPU.      python tools/vec_variants.py"""
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    from paper_2110_12865_b200 import DevicePlan
    from paper_2110_12865_b200.lower import lower_plan

    ns = bench.parse_args([])
    for cfg in ("c2", "c4"):
        key, plan = bench.build_workload(cfg, ns)
        ins = bench.workload_inputs(cfg, ns, 0, plan)
        want = None
        for vec in ("", "1", "2", "4"):
            if vec:
                os.environ["SGB_JIT_VEC"] = vec
            else:
                os.environ.pop("SGB_JIT_VEC", None)
            t0 = time.perf_counter()
            dp = DevicePlan(plan, lowered=lower_plan(plan, relayout="auto"))
            x = dp.new_values(ins)
            out = torch.empty(len(plan.outputs), dtype=torch.float64, device="cuda")
            dp.run_csr(x, out)
            got = out.cpu().numpy()
            want = got if want is None else want
            same = np.array_equal(got.view(np.uint64), want.view(np.uint64))
            per = []
            for w in range(dp.csr_launches):
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
                for e0, e1 in evs:
                    e0.record()
                    dp.run_wave(x, w, out)
                    e1.record()
                torch.cuda.synchronize()
                tw = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
                per.append(round(tw[10], 4))
            print(f"{cfg} vec={vec or 'auto'} same_bits={same} waves {per} ({time.perf_counter() - t0:.0f}s)", flush=True)
            del dp
    os.environ.pop("SGB_JIT_VEC", None)


if __name__ == "__main__":
    main()
