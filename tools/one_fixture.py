"""Run golden fixtures through the GPU path (debug aid)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

from conftest import Golden, bits  # noqa: E402
from paper_2110_12865_b200 import compile_plan  # noqa: E402

for name in sys.argv[1:]:
    g = Golden(name)
    run = compile_plan(g.plan)
    x = run(g.inputs)
    bad = np.nonzero(bits(x) != bits(g.values))[0]
    u = run.device_plan.lowered.units
    print(name, "units", u.tolist(), "bitwise" if bad.size == 0 else f"MISMATCH {bad.size} first {bad[:6].tolist()} "
          f"got {x[bad[:3]].tolist()} want {g.values[bad[:3]].tolist()}", flush=True)
