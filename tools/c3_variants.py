"""C3 element-kernel variants (one GPU): time each wave of the fem plan under code-generation knobs.

    python tools/c3_variants.py [--m 55]

Knobs: lower.STORE_ROOTS_EARLY (roots stored as computed vs at the end of the tape) and the LOG
restatement (jit._SLOW[3]: the glibc restatement ``sgb_log`` vs CUDA's ``log``, timing only --
CUDA's log is not bit-exact).  Autotune on, as in bench.py.
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
    ap.add_argument("--m", type=int, default=55)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    ns = bench.parse_args(["--m", str(args.m)])
    key, plan = bench.build_workload("c3", ns)
    ins = bench.workload_inputs("c3", ns, 0)
    want = None
    for early, log in itertools.product((True, False), ("sgb_log({a})", "log({a})")):
        lower.STORE_ROOTS_EARLY = early
        jit._SLOW[3] = log
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
        print(f"early={early} log={log} same_bits_as_first={ok} waves {per} tiles {dp.tile_order} "
              f"(lower {t_low:.0f}s)", flush=True)
        del dp


if __name__ == "__main__":
    main()
