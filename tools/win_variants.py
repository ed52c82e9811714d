"""Window-kernel variants on the C2 plan (one GPU): time the CSR-window wave and check the bits.

    python tools/win_variants.py [--w 1000]
"""
import argparse
import itertools
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    from paper_2110_12865_b200 import DevicePlan, jit, lower
    from paper_2110_12865_b200.lower import lower_plan

    ap = argparse.ArgumentParser()
    ap.add_argument("--w", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    ns = bench.parse_args(["--w", str(args.w)])
    key, plan = bench.build_workload("c2", ns)
    ins = bench.workload_inputs("c2", ns, 0)
    ref = DevicePlan(plan, lowered=lower_plan(plan, csr_window=False))
    want = ref.run_csr(ref.new_values(ins)).cpu().numpy()
    variants = [dict(cut=c_, wbulk=False) for c_ in (1, 0, 2, 4, 8, 1)]
    for v in variants:
        lower.WIN_GRID_CUT = v["cut"]
        t0 = time.perf_counter()
        lw = lower_plan(plan, csr_window=True, wbulk=v["wbulk"])
        if lw.wbulk is not None:
            wb = lw.wbulk
            v = dict(v, ring=wb.ring, smem_kb=round(wb.smem / 1024, 1), iv=int(wb.iv.shape[0]))
        t_low = time.perf_counter() - t0
        import os
        os.environ["SGB_AUTOTUNE"] = "0"
        dp = DevicePlan(plan, lowered=lw)
        x = dp.new_values(ins)
        out = torch.empty(len(plan.outputs), dtype=torch.float64, device="cuda")
        dp.run_csr(x, out)
        ok = np.array_equal(out.cpu().numpy().view(np.uint64), want.view(np.uint64))
        w = dp.csr_launches - 1
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
        for _ in range(3):
            dp.run_csr(x, out)
        for e0, e1 in evs:
            e0.record()
            dp.run_wave(x, w, out)
            e1.record()
        torch.cuda.synchronize()
        tw = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
        for e0, e1 in evs:
            e0.record()
            dp.run_csr(x, out)
            e1.record()
        torch.cuda.synchronize()
        tt = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
        print(f"{v} bitwise={ok} window_wave median {tw[len(tw)//2]:.4f} ms  whole {tt[len(tt)//2]:.4f} ms "
              f"(lower {t_low:.0f}s)", flush=True)
        del dp


if __name__ == "__main__":
    main()
