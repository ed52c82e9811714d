"""Time every CSR-mode launch of one evaluation for lowering variants (dev tool, not the bench)."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import argparse  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2110_12865_b200 import DevicePlan  # noqa: E402
from paper_2110_12865_b200.lower import lower_plan  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["vec=0"]
plans = {}


def get_plan(cfg):
    if cfg not in plans:
        ns = argparse.Namespace(config=cfg, w=w, m=55, w4=708)
        plans[cfg] = (bench.build_workload(ns, 0, 1)[1], bench.workload_inputs(ns, 0))
    return plans[cfg]



refs = {}
for var in variants:
    env = dict(kv.split("=") for kv in var.split(";") if kv)
    os.environ["SGB_TAPE_VEC"] = env.get("vec", "0")
    os.environ["SGB_COMPRESS"] = env.get("compress", "1")
    os.environ["SGB_TILE_ORDER"] = env.get("order", "csr")
    os.environ["SGB_TAPE_JIT"] = env.get("jit", "1")
    os.environ["SGB_CSR_WINDOW"] = env.get("window", "0")
    os.environ["SGB_DIRECT_CSR"] = env.get("direct", "0")
    os.environ["SGB_JIT_MINBLOCKS"] = env.get("minblocks", "")
    if not os.environ["SGB_JIT_MINBLOCKS"]:
        del os.environ["SGB_JIT_MINBLOCKS"]
    cfg = env.get("config", "c2")
    for k_, e_ in (("jitvec", "SGB_JIT_VEC"), ("bvec", "SGB_BATCH_VEC")):
        if k_ in env:
            os.environ[e_] = env[k_]
        else:
            os.environ.pop(e_, None)
    mode = env.get("mode", "csr")
    plan, inputs = get_plan(cfg)
    ref = refs.get(cfg)
    t0 = time.time()
    dp = DevicePlan(plan, lowered=lower_plan(plan))
    x = dp.new_values(inputs)
    out = torch.empty(len(plan.outputs), dtype=torch.float64, device="cuda")
    for _ in range(5):
        dp.run_csr(x, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    if ref is None:
        ref = refs[cfg] = got
    same = np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    R = 20
    nw = dp.csr_launches if mode == "csr" else dp.launches
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nw + 1)] for _ in range(R)]
    for r in range(R):
        for wv in range(nw):
            ev[r][wv].record()
            dp.run_wave(x, wv, out=out if mode == "csr" else None)
        ev[r][nw].record()
    torch.cuda.synchronize()
    per = np.zeros(nw)
    for r in range(R):
        for j in range(nw):
            per[j] += ev[r][j].elapsed_time(ev[r][j + 1]) / R
    print(f"{var}: same={same} total={per.sum():.4f} ms waves={np.round(per, 4).tolist()} "
          f"(lower+upload {time.time() - t0:.1f}s)", flush=True)
    dp.close()
