"""Execution-plan data model and the plan wire format, restated for the device.

The device backend consumes the reference's ``ExecutionPlan`` unchanged: any
object with the fields of ``sparsegen.codegen.ExecutionPlan`` /
``KernelPlan`` (codegen.py:56-98) works, so plans built in-process by the
reference pipeline plug straight in.  Plans that were built elsewhere arrive
through the reference's own wire format -- ``manifest.json`` + ``data.blob``
(codegen.py:619-798) -- which this module reads and writes without importing
the reference package (the GPU host does not have it).

Layout facts the device relies on (codegen.py:244-314):

* value array ``x``: inputs at ``[0, input_count)`` (variable id == offset),
  then per kernel ``dest_base = align(cursor, vector_width)``; result ``r`` of
  instance ``i`` lives at ``dest_base + r*N + i``; padding is zero;
* ``positions`` (u32): per kernel, retained position slots, slot-major
  ("coalesced", ``p[p_base + r*N + i]``) or instance-major ("interleaved",
  ``p[p_base + i*R + r]``); non-retained slots are ``p[slot0] + delta``;
* ``constants`` (f64): per kernel, varying constant slots, same two layouts.
"""

from __future__ import annotations

import json
import struct as _struct
from dataclasses import dataclass, field
from enum import IntEnum
from pathlib import Path

import numpy as np

BLOB_MAGIC = b"SGEN"  # codegen.py:37
BLOB_VERSION = 1  # codegen.py:38
SEC_POSITIONS = 1  # codegen.py:39
SEC_CONSTANTS = 2  # codegen.py:40


class OpKind(IntEnum):
    """Op codes of the expression arena (expr.py:55-69); the tape's op space."""

    VAR = 0
    CONST = 1
    ADD = 2
    SUB = 3
    MUL = 4
    DIV = 5
    NEG = 6
    SQRT = 7
    SIN = 8
    COS = 9
    EXP = 10
    LOG = 11
    POW = 12
    SELECT = 13


# ops a lane-parallel IEEE evaluation reproduces bit-exactly (codegen.py:43-53)
EXACT_OPS = frozenset(
    int(o)
    for o in (
        OpKind.VAR, OpKind.CONST, OpKind.ADD, OpKind.SUB, OpKind.MUL,
        OpKind.DIV, OpKind.NEG, OpKind.SQRT, OpKind.SELECT,
    )
)

_OP_NAMES = {int(op): op.name.lower() for op in OpKind}
_OP_FROM_NAME = {name: code for code, name in _OP_NAMES.items()}


class Template:
    """Minimal append-only node store for a kernel template.

    Mirrors the fields of ``ExprArena`` that evaluation reads (``ops``,
    ``args``, ``payload``; expr.py:141-143).  Nodes are appended in
    topological order (children before parents) and are *not* re-sorted, the
    same guarantee ``_template_from_json`` gets from ``apply(sort=False)``
    (codegen.py:646-659): child order is the evaluation order.
    """

    def __init__(self):
        self.ops: list[int] = []
        self.args: list[tuple[int, ...]] = []
        self.payload: list = []
        self._cons: dict = {}

    def __len__(self) -> int:
        return len(self.ops)

    def _push(self, op, args, payload):
        key = (op, args, payload if op != OpKind.CONST else _f64_bits(payload))
        hit = self._cons.get(key)
        if hit is not None:
            return hit
        ref = len(self.ops)
        self.ops.append(int(op))
        self.args.append(tuple(args))
        self.payload.append(payload)
        self._cons[key] = ref
        return ref

    def var(self, vid: int) -> int:
        return self._push(OpKind.VAR, (), int(vid))

    def const(self, value: float) -> int:
        return self._push(OpKind.CONST, (), float(value))

    def apply(self, op, children) -> int:
        op = int(op)
        cs = tuple(int(c) for c in children)
        n = len(self.ops)
        for c in cs:
            if not 0 <= c < n:
                raise ValueError(f"child {c} is not a node of this template")
        if op in (OpKind.ADD, OpKind.MUL) and len(cs) < 2:
            raise ValueError("n-ary ops need at least two children")
        if op == OpKind.POW:
            ev = self.payload[cs[1]]
            if self.ops[cs[1]] != OpKind.CONST or not float(ev).is_integer() or ev < 2:
                raise ValueError("pow requires a constant integer exponent >= 2")
        return self._push(op, cs, None)


def _f64_bits(v) -> int:
    return _struct.unpack("<Q", _struct.pack("<d", float(v)))[0]


def reachable(tmpl, roots) -> list[int]:
    """Nodes reachable from ``roots`` in ascending (topological) order.

    Restates expr.py:408-420 / 608-611 (reverse sweep marking children; every
    child index is smaller than its parent's).
    """
    n = len(tmpl.ops)
    need = bytearray(n)
    for r in roots:
        if not 0 <= r < n:
            raise ValueError(f"root {r} is not a node of this template")
        need[r] = 1
    args = tmpl.args
    for i in range(n - 1, -1, -1):
        if need[i]:
            for c in args[i]:
                need[c] = 1
    return [i for i in range(n) if need[i]]


@dataclass
class KernelPlan:
    """Field-for-field mirror of codegen.py:56-85."""

    name: str
    level: int
    dest_kind: str
    instances: int
    n_roots: int
    dest_base: int
    template_arena: Template
    template_roots: list[int]
    template_locals: list[int]
    pos_vars: list[int]
    const_vars: list[int]
    coherence: list
    retained: list[int]
    p_base: int
    c_base: int
    layout: str
    self_referencing: bool = False
    uniform_consts: int = 0
    dup_slots: int = 0
    entity_ids: list[int] = field(default_factory=list)

    @property
    def pos_entries(self) -> int:
        return len(self.retained) * self.instances

    @property
    def const_entries(self) -> int:
        return len(self.const_vars) * self.instances


@dataclass
class ExecutionPlan:
    """Field-for-field mirror of codegen.py:88-98."""

    value_array_size: int
    input_count: int
    vector_width: int
    outputs: list[int]
    kernels: list[KernelPlan]
    positions: np.ndarray
    constants: np.ndarray
    metadata: dict
    stats: dict = field(default_factory=dict)


def align(n: int, to: int) -> int:
    """codegen.py:123-124"""
    return ((n + to - 1) // to) * to


# -- index decode (the canonical per-slot address definition) -----------------------


def slot_addresses(plan, kp) -> list[np.ndarray]:
    """Per active position slot, the int64 load address of every instance.

    Restates codegen.py:373-388: retained slots read their column of the
    position table; coherent slots are ``column(slot 0) + delta``.
    """
    n = kp.instances
    r = len(kp.retained)
    seg = np.asarray(plan.positions[kp.p_base: kp.p_base + r * n])
    per = seg.reshape(r, n) if kp.layout == "coalesced" else seg.reshape(n, r).T
    ridx = {s: k for k, s in enumerate(kp.retained)}
    cols = []
    for s, coh in enumerate(kp.coherence):
        if s in ridx:
            cols.append(per[ridx[s]].astype(np.int64))
        else:
            cols.append(per[0].astype(np.int64) + int(coh))
    return cols


def const_columns(plan, kp) -> list[np.ndarray]:
    """codegen.py:391-395"""
    n = kp.instances
    c = len(kp.const_vars)
    seg = np.asarray(plan.constants[kp.c_base: kp.c_base + c * n])
    return list(seg.reshape(c, n) if kp.layout == "coalesced" else seg.reshape(n, c).T)


# -- wire format (codegen.py:619-798) ------------------------------------------------


def _template_json(kp) -> dict:
    """codegen.py:626-643 (live nodes only, renumbered ascending)."""
    tmpl = kp.template_arena
    live = reachable(tmpl, kp.template_roots)
    index = {ref: k for k, ref in enumerate(live)}
    nodes = []
    for ref in live:
        op = int(tmpl.ops[ref])
        if op == OpKind.VAR:
            nodes.append(["var", tmpl.payload[ref]])
        elif op == OpKind.CONST:
            nodes.append(["const", tmpl.payload[ref]])
        else:
            nodes.append([_OP_NAMES[op], [index[c] for c in tmpl.args[ref]]])
    return {
        "nodes": nodes,
        "roots": [index[r] for r in kp.template_roots],
        "locals": [index[r] for r in kp.template_locals if r in index],
    }


def _template_from_json(spec: dict):
    """codegen.py:646-659; children keep their stored order."""
    tmpl = Template()
    refs: list[int] = []
    for node in spec["nodes"]:
        kind = node[0]
        if kind == "var":
            refs.append(tmpl.var(int(node[1])))
        elif kind == "const":
            refs.append(tmpl.const(float(node[1])))
        else:
            if kind not in _OP_FROM_NAME:
                raise ValueError(f"unknown template op {kind!r}")
            refs.append(tmpl.apply(_OP_FROM_NAME[kind], [refs[c] for c in node[1]]))
    return tmpl, [refs[i] for i in spec["roots"]], [refs[i] for i in spec["locals"]]


def plan_manifest(plan) -> dict:
    """codegen.py:662-694"""
    kernels = []
    for kp in plan.kernels:
        kernels.append({
            "name": kp.name, "level": kp.level, "dest_kind": kp.dest_kind,
            "instances": kp.instances, "n_roots": kp.n_roots, "dest_base": kp.dest_base,
            "layout": kp.layout, "template": _template_json(kp),
            "pos_vars": list(kp.pos_vars), "const_vars": list(kp.const_vars),
            "coherence": list(kp.coherence), "retained": list(kp.retained),
            "p_base": kp.p_base, "c_base": kp.c_base,
            "self_referencing": bool(kp.self_referencing),
            "uniform_consts": kp.uniform_consts, "dup_slots": kp.dup_slots,
        })
    return {
        "format": 1,
        "value_array_size": plan.value_array_size,
        "input_count": plan.input_count,
        "vector_width": plan.vector_width,
        "outputs": np.asarray(plan.outputs, dtype=np.int64).tolist(),
        "metadata": plan.metadata,
        "kernels": kernels,
    }


def blob_bytes(plan) -> bytes:
    """codegen.py:697-705: ``SGEN``, u32 version, then (u32 tag, u64 len, payload)."""
    pos = np.ascontiguousarray(plan.positions, dtype="<u4").tobytes()
    con = np.ascontiguousarray(plan.constants, dtype="<f8").tobytes()
    return b"".join([
        BLOB_MAGIC, _struct.pack("<I", BLOB_VERSION),
        _struct.pack("<IQ", SEC_POSITIONS, len(pos)), pos,
        _struct.pack("<IQ", SEC_CONSTANTS, len(con)), con,
    ])


def save_plan(plan, out_dir) -> None:
    """codegen.py:708-717 (byte-compatible manifest and blob)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    (out / "manifest.json").write_text(
        json.dumps(plan_manifest(plan), sort_keys=True, separators=(",", ":")) + "\n"
    )
    (out / "data.blob").write_bytes(blob_bytes(plan))


def parse_blob(raw: bytes, src="blob") -> tuple[np.ndarray, np.ndarray]:
    """Validate and split a data blob (codegen.py:726-745)."""
    if raw[:4] != BLOB_MAGIC:
        raise ValueError(f"{src}: bad data blob magic")
    if len(raw) < 8:
        raise ValueError(f"{src}: truncated blob header")
    (version,) = _struct.unpack_from("<I", raw, 4)
    if version != BLOB_VERSION:
        raise ValueError(f"{src}: unsupported blob version {version}")
    off = 8
    sections: dict[int, bytes] = {}
    while off < len(raw):
        if off + 12 > len(raw):
            raise ValueError(f"{src}: truncated section header")
        tag, length = _struct.unpack_from("<IQ", raw, off)
        off += 12
        if off + length > len(raw):
            raise ValueError(f"{src}: section {tag} overruns the blob")
        sections[tag] = raw[off: off + length]
        off += length
    if SEC_POSITIONS not in sections or SEC_CONSTANTS not in sections:
        raise ValueError(f"{src}: missing blob sections")
    if len(sections[SEC_POSITIONS]) % 4 or len(sections[SEC_CONSTANTS]) % 8:
        raise ValueError(f"{src}: section length is not a whole number of entries")
    positions = np.frombuffer(sections[SEC_POSITIONS], dtype="<u4").astype(np.uint32)
    constants = np.frombuffer(sections[SEC_CONSTANTS], dtype="<f8").astype(np.float64)
    return positions, constants


def load_plan(plan_dir) -> ExecutionPlan:
    """codegen.py:720-784 + _validate_plan (787-798); ValueError on any defect."""
    src = Path(plan_dir)
    manifest = json.loads((src / "manifest.json").read_text())
    if manifest.get("format") != 1:
        raise ValueError(f"{src}: unsupported manifest format {manifest.get('format')!r}")
    positions, constants = parse_blob((src / "data.blob").read_bytes(), src)
    kernels = []
    for kj in manifest["kernels"]:
        tmpl, roots, locals_ = _template_from_json(kj["template"])
        kernels.append(KernelPlan(
            name=kj["name"], level=kj["level"], dest_kind=kj["dest_kind"],
            instances=kj["instances"], n_roots=kj["n_roots"], dest_base=kj["dest_base"],
            template_arena=tmpl, template_roots=roots, template_locals=locals_,
            pos_vars=list(kj["pos_vars"]), const_vars=list(kj["const_vars"]),
            coherence=[None if c is None else int(c) for c in kj["coherence"]],
            retained=list(kj["retained"]), p_base=kj["p_base"], c_base=kj["c_base"],
            layout=kj["layout"], self_referencing=kj["self_referencing"],
            uniform_consts=kj["uniform_consts"], dup_slots=kj["dup_slots"],
        ))
    plan = ExecutionPlan(
        value_array_size=manifest["value_array_size"],
        input_count=manifest["input_count"],
        vector_width=manifest["vector_width"],
        outputs=list(manifest["outputs"]),
        kernels=kernels,
        positions=positions,
        constants=constants,
        metadata=manifest["metadata"],
    )
    validate_plan(plan, src)
    return plan


def validate_plan(plan, src="plan") -> None:
    """codegen.py:787-798, plus the per-kernel bounds the device relies on."""
    expected_p = sum(len(kp.retained) * kp.instances for kp in plan.kernels)
    expected_c = sum(len(kp.const_vars) * kp.instances for kp in plan.kernels)
    if len(plan.positions) != expected_p:
        raise ValueError(f"{src}: position array has {len(plan.positions)} entries, expected {expected_p}")
    if len(plan.constants) != expected_c:
        raise ValueError(f"{src}: constant array has {len(plan.constants)} entries, expected {expected_c}")
    if len(plan.positions) and int(np.max(plan.positions)) >= plan.value_array_size:
        raise ValueError(f"{src}: position index outside the value array")
    outs = np.asarray(plan.outputs, dtype=np.int64)
    if outs.size and (outs.min() < 0 or outs.max() >= plan.value_array_size):
        raise ValueError(f"{src}: output offset outside the value array")
    for kp in plan.kernels:
        if kp.dest_base < plan.input_count or kp.dest_base + kp.n_roots * kp.instances > plan.value_array_size:
            raise ValueError(f"{src}: {kp.name} result range outside the value array")
        if len(kp.coherence) != len(kp.pos_vars):
            raise ValueError(f"{src}: {kp.name} coherence/pos_vars length mismatch")
        if kp.pos_vars and (not kp.retained or kp.retained[0] != 0):
            raise ValueError(f"{src}: {kp.name} slot 0 must be retained")
        if kp.layout not in ("coalesced", "interleaved"):
            raise ValueError(f"{src}: {kp.name} unknown layout {kp.layout!r}")


def unique_addresses(a) -> np.ndarray:
    """Sorted unique non-negative addresses (np.unique through a bitmap: O(n), no hash or sort)."""
    a = np.asarray(a)
    if a.size == 0:
        return np.zeros(0, np.int64)
    hi = int(a.max()) + 1
    if hi > 64 * a.size + (1 << 20):  # sparse: the bitmap would cost more than a sort
        return np.unique(a.astype(np.int64))
    mark = np.zeros(hi, dtype=bool)
    mark[a] = True
    return np.flatnonzero(mark).astype(np.int64)
