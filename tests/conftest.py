import json
import os
import sys
from pathlib import Path

# tests time the kernels' results, not the launch configurations: the per-wave autotune
# (runtime.DevicePlan.autotune) has its own test (test_gpu_parity.test_autotune_keeps_bits)
os.environ.setdefault("SGB_AUTOTUNE", "0")

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


import pytest  # noqa: E402


@pytest.hookimpl(trylast=True)  # after -m deselection
def pytest_collection_modifyitems(session, config, items):
    """A GPU run without a GPU, libsgb.so or NVRTC fails once, up front, instead of per test."""
    if not any(item.get_closest_marker("gpu") for item in items):
        return
    try:
        import torch

        from paper_2110_12865_b200 import jit, load_library

        problems = []
        if not torch.cuda.is_available():
            problems.append("no CUDA device")
        load_library()  # raises when libsgb.so is missing
        if not jit.available():
            problems.append("NVRTC (libnvrtc.so.12) not found")
    except Exception as e:  # noqa: BLE001
        problems = [f"{type(e).__name__}: {e}"]
    if problems:
        pytest.exit("GPU suite cannot run: " + "; ".join(problems) + " (build with __graft_entry__.build())",
                    returncode=3)


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
        if getattr(self, "_exact", None) is None:
            from paper_2110_12865_b200.lower import lower_plan

            self._exact = lower_plan(self.plan, jit=False).exact
        return self._exact


@pytest.fixture(params=golden_names())
def golden(request):
    return golden_case(request.param)


_LOWERED: dict = {}
_DEVICE_PLANS: dict = {}


def lowered(name: str, **kw):
    """lower_plan of a fixture, memoised per (fixture, keyword arguments)."""
    key = (name, tuple(sorted(kw.items())))
    if key not in _LOWERED:
        from paper_2110_12865_b200.lower import lower_plan

        _LOWERED[key] = lower_plan(golden_case(name).plan, **kw)
    return _LOWERED[key]


def device_plan(name: str, **kw):
    """A shared DevicePlan of a fixture (tests that change tiles or grids make their own)."""
    key = (name, tuple(sorted(kw.items())))
    if key not in _DEVICE_PLANS:
        from paper_2110_12865_b200 import DevicePlan

        _DEVICE_PLANS[key] = DevicePlan(golden_case(name).plan, lowered=lowered(name, **kw))
    return _DEVICE_PLANS[key]


_GOLDEN: dict = {}


def golden_case(name: str) -> "Golden":
    if name not in _GOLDEN:
        _GOLDEN[name] = Golden(name)
    return _GOLDEN[name]


def bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64)).view(np.uint64)


def have_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
