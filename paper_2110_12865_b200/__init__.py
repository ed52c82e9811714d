"""B200-native evaluation backend for sparsity-specific expression plans.

Reference: arXiv 2110.12865 / the ``sparsegen`` package at /root/reference.
The hot path is the numeric evaluation of an ``ExecutionPlan``
(codegen.py:404-446, emit.py:153-245); this package evaluates such plans on a
B200 through hand-written sm_100a kernels behind the C ABI in include/sgb.h.
"""

from .plan import ExecutionPlan, KernelPlan, OpKind, Template, load_plan, save_plan, slot_addresses
from .lower import lower_plan
from .runtime import DevicePlan, InterpretResult, SgbError, compile_plan, interpret_plan, load_library
from .individual import evaluate_outputs_individually

__all__ = [
    "ExecutionPlan", "KernelPlan", "OpKind", "Template", "load_plan", "save_plan", "slot_addresses",
    "lower_plan", "DevicePlan", "InterpretResult", "SgbError", "compile_plan", "interpret_plan",
    "load_library", "evaluate_outputs_individually",
]
