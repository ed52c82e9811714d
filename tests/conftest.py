import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

GOLDEN = ROOT / "tests" / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_names():
    return sorted(d.name for d in GOLDEN.iterdir() if (d / "manifest.json").exists())


class Golden:
    def __init__(self, name):
        self.name = name
        self.dir = GOLDEN / name
        self.meta = json.loads((self.dir / "meta.json").read_text())
        with np.load(self.dir / "vectors.npz") as z:
            self.vec = {k: z[k] for k in z.files}
        self._plan = None

    @property
    def plan(self):
        if self._plan is None:
            from paper_2110_12865_b200.plan import load_plan

            self._plan = load_plan(self.dir)
        return self._plan

    @property
    def inputs(self):
        return self.vec["inputs"]

    @property
    def values(self):
        return self.vec["values"]

    @property
    def outputs(self):
        return self.values[np.asarray(self.plan.outputs, dtype=np.int64)]

    @property
    def oracle(self):
        """eval_numeric of the traced outputs (expr.py:423-484)."""
        return self.vec["oracle"] if "oracle" in self.vec else self.outputs

    @property
    def exact(self):
        from paper_2110_12865_b200.lower import lower_plan

        return lower_plan(self.plan, jit=False).exact


@pytest.fixture(params=golden_names())
def golden(request):
    return Golden(request.param)


def bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.uint64)


def have_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
