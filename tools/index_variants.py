"""Index arithmetic of the specialised kernels (jit.INDEX64) on the bench configs: per-wave times and
the bits, one GPU.      python tools/index_variants.py [--configs c2,c3,c4]
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
    from paper_2110_12865_b200 import DevicePlan, jit
    from paper_2110_12865_b200.lower import lower_plan

    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3,c4")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    ns = bench.parse_args([])
    for cfg in args.configs.split(","):
        key, plan = bench.build_workload(cfg, ns)
        ins = bench.workload_inputs(cfg, ns, 0, plan)
        want = None
        for idx64 in (True, False, True):
            jit.INDEX64 = idx64
            t0 = time.perf_counter()
            lw = lower_plan(plan, relayout="auto")
            dp = DevicePlan(plan, lowered=lw)
            x = dp.new_values(ins)
            out = torch.empty(len(plan.outputs), dtype=torch.float64, device="cuda")
            dp.run_csr(x, out)
            got = out.cpu().numpy()
            want = got if want is None else want
            same = np.array_equal(got.view(np.uint64), want.view(np.uint64))
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
            g = dp.capture_csr(x, out)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
            for e0, e1 in evs:
                e0.record()
                g.replay()
                e1.record()
            torch.cuda.synchronize()
            tt = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
            print(f"{cfg} index64={idx64} same_bits={same} waves {per} graph {tt[len(tt) // 2]:.4f} ms "
                  f"tiles {dp.tile_order} ({time.perf_counter() - t0:.0f}s)", flush=True)
            del dp, g


if __name__ == "__main__":
    main()
