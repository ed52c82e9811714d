"""Incremental ExecutionPlan assembly for the scalable (template-instancing) builders.

A builder adds kernel groups in schedule order -- template + one int64
address column per position slot -- and gets each group's result addresses
back immediately, so consumers can be wired to producers with numpy index
arithmetic instead of a symbolic trace.  Memory planning follows the
reference exactly (codegen.py:244-314): ``dest_base = align(cursor,
vector_width)``, result r of instance i at ``dest_base + r*N + i``, slot-major
u32 position table, offset coherence against slot 0 (codegen.py:317-327) so
coherent slots leave the table.
"""

from __future__ import annotations

import numpy as np

from ..plan import ExecutionPlan, KernelPlan, Template, align


def detect_offset_coherence(cols: list[np.ndarray]) -> list:
    """codegen.py:317-327: per slot, fixed delta from slot 0 across instances, else None."""
    if not cols:
        return []
    base = cols[0].astype(np.int64)
    out: list = [0]
    for col in cols[1:]:
        delta = col.astype(np.int64) - base
        first = int(delta[0]) if delta.size else 0
        out.append(first if bool(np.all(delta == first)) else None)
    return out


class PlanBuilder:
    def __init__(self, input_count: int, vector_width: int = 4, coherence: bool = True):
        self.input_count = int(input_count)
        self.vector_width = vector_width
        self.coherence = coherence
        self.cursor = self.input_count
        self.kernels: list[KernelPlan] = []
        self._pos: list[np.ndarray] = []
        self._con: list[np.ndarray] = []
        self._p = 0
        self._c = 0

    def add_group(self, name: str, level: int, template: Template, roots: list[int],
                  slot_addrs: list[np.ndarray], const_cols: list[np.ndarray] | None = None,
                  dest_kind: str = "intermediate") -> np.ndarray:
        """Append one group; returns its result addresses, shape (n_roots, N)."""
        const_cols = const_cols or []
        n = int(len(slot_addrs[0]) if slot_addrs else len(const_cols[0]))
        for col in list(slot_addrs) + list(const_cols):
            if len(col) != n:
                raise ValueError(f"{name}: ragged slot columns")
        dest = align(self.cursor, self.vector_width)
        self.cursor = dest + len(roots) * n
        cols = [np.asarray(c, dtype=np.int64) for c in slot_addrs]
        for c in cols:
            if c.size and (c.min() < 0 or c.max() >= dest):
                raise ValueError(f"{name}: loads outside the values written before it")
        coh = detect_offset_coherence(cols) if self.coherence else ([0] + [None] * (len(cols) - 1) if cols else [])
        retained = [s for s, c in enumerate(coh) if s == 0 or c is None]
        p_base = self._p
        if cols:
            block = np.stack([cols[s] for s in retained])
            if block.max(initial=0) > 0xFFFFFFFF:
                raise ValueError(f"{name}: address exceeds u32")
            block = block.astype(np.uint32)
            self._pos.append(block.reshape(-1))
            self._p += block.size
        c_base = self._c
        if const_cols:
            cb = np.stack([np.asarray(c, np.float64) for c in const_cols])
            self._con.append(cb.reshape(-1))
            self._c += cb.size
        n_pos = len(cols)
        kp = KernelPlan(
            name=name, level=level, dest_kind=dest_kind, instances=n, n_roots=len(roots),
            dest_base=dest, template_arena=template, template_roots=list(roots),
            template_locals=[], pos_vars=list(range(n_pos)),
            const_vars=list(range(n_pos, n_pos + len(const_cols))),
            coherence=coh, retained=retained, p_base=p_base, c_base=c_base, layout="coalesced",
        )
        self.kernels.append(kp)
        return dest + np.arange(len(roots), dtype=np.int64)[:, None] * n + np.arange(n, dtype=np.int64)[None, :]

    def finish(self, outputs: np.ndarray, metadata: dict) -> ExecutionPlan:
        outputs = np.asarray(outputs, dtype=np.int64)
        return ExecutionPlan(
            value_array_size=self.cursor,
            input_count=self.input_count,
            vector_width=self.vector_width,
            outputs=outputs,
            kernels=self.kernels,
            positions=np.concatenate(self._pos) if self._pos else np.zeros(0, np.uint32),
            constants=np.concatenate(self._con) if self._con else np.zeros(0, np.float64),
            metadata=dict(metadata),
        )
