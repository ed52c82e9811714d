"""C3 element-kernel variants (one GPU): time each wave of the fem plan under code-generation knobs.

    python tools/c3_variants.py [--m 55]

Knob: lower.JIT_SPLIT (the element template's root set split over k x 256 threads per tile).
Autotune on, as in bench.py.
"""
import argparse
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
    ap.add_argument("--m", type=int, default=55)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    ns = bench.parse_args(["--m", str(args.m)])
    key, plan = bench.build_workload("c3", ns)
    ins = bench.workload_inputs("c3", ns, 0)
    want = None
    for split, early in ((1, False), (1, True), (2, True), (1, False)):
        lower.JIT_SPLIT, lower.STORE_ROOTS_EARLY = split, early
        t0 = time.perf_counter()
        lw = lower_plan(plan, relayout="auto")
        t_low = time.perf_counter() - t0
        dp = DevicePlan(plan, lowered=lw)
        x = dp.new_values(ins)
        out = torch.empty(len(plan.outputs), dtype=torch.float64, device="cuda")
        dp.run_csr(x, out)
        got = out.cpu().numpy()
        if want is None:
            want = got
        ok = np.array_equal(got.view(np.uint64), want.view(np.uint64))
        per = []
        for w in range(dp.csr_launches):
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.reps)]
            for e0, e1 in evs:
                e0.record()
                dp.run_wave(x, w, out)
                e1.record()
            torch.cuda.synchronize()
            tw = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
            per.append(round(tw[len(tw) // 2], 4))
        print(f"split={split} early={early} same_bits_as_first={ok} waves {per} tiles {dp.tile_order} "
              f"(lower {t_low:.0f}s)", flush=True)
        del dp


if __name__ == "__main__":
    main()
