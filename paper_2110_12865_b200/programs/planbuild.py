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

    def producer_ids(self, addrs: np.ndarray) -> np.ndarray:
        """Group index whose result range holds each address (-1 = input value)."""
        starts = np.array([kp.dest_base for kp in self.kernels], dtype=np.int64)
        gid = np.searchsorted(starts, addrs, side="right") - 1
        return np.where(addrs < self.input_count, -1, gid)

    def add_group_split(self, name: str, level: int, template: Template, roots: list[int],
                        slot_addrs: list[np.ndarray], const_cols: list[np.ndarray] | None = None,
                        dest_kind: str = "intermediate", min_class: int = 1024,
                        min_source_class: int = 64, keep_cols: tuple = ()) -> np.ndarray:
        """``add_group`` split so every sub-group gathers from fixed sources.

        1. Instances are partitioned by *source signature* -- which producer
           group (or the input range) each slot reads -- so a slot of a
           sub-group walks one producer's result range in step with the
           instances: compact per-chunk index windows (lower.compress_columns).
        2. Inside a source class, instances with identical offsets from slot 0
           (the reference's coherence test, codegen.py:317-327) form their own
           sub-group with a single index column when the class has at least
           ``min_class`` members.
        Small classes fall into one residual sub-group.  Slots in ``keep_cols``
        stay out of the offset signature.  Sub-groups keep the original
        relative instance order; result addresses come back in original order.
        """
        cols = [np.asarray(c, dtype=np.int64) for c in slot_addrs]
        n = len(cols[0]) if cols else 0
        if n == 0 or not cols:
            return self.add_group(name, level, template, roots, slot_addrs, const_cols, dest_kind)
        src = np.stack([self.producer_ids(c) for c in cols], axis=1)
        _, sinv, scnt = np.unique(src, axis=0, return_inverse=True, return_counts=True)
        sinv = sinv.reshape(-1)
        sinv = np.where(scnt[sinv] >= min_source_class, sinv, -1)
        sig_slots = [s for s in range(1, len(cols)) if s not in keep_cols]
        label = np.full(n, -1, dtype=np.int64)
        next_label = 0
        for sc in np.unique(sinv).tolist():
            members = np.flatnonzero(sinv == sc)
            if sc < 0 or not sig_slots:
                label[members] = next_label
                next_label += 1
                continue
            D = np.stack([cols[s][members] - cols[0][members] for s in sig_slots], axis=1)
            _, inv, counts = np.unique(D, axis=0, return_inverse=True, return_counts=True)
            inv = inv.reshape(-1)
            big = counts >= min_class
            uniq_big = {c: next_label + k for k, c in enumerate(np.flatnonzero(big).tolist())}
            next_label += len(uniq_big)
            rest = next_label
            next_label += 1
            label[members] = np.array([uniq_big.get(c, rest) for c in inv.tolist()], dtype=np.int64) \
                if len(uniq_big) else rest
        out = np.empty((len(roots), n), dtype=np.int64)
        order = np.argsort(label, kind="stable")
        keys, starts = np.unique(label[order], return_index=True)
        ends = np.append(starts[1:], n)
        for k, (a, b) in enumerate(zip(starts.tolist(), ends.tolist())):
            sel = order[a:b]
            sub_const = [np.asarray(c)[sel] for c in (const_cols or [])]
            out[:, sel] = self.add_group(f"{name}_{k}", level, template, roots, [c[sel] for c in cols],
                                         sub_const, dest_kind)
        return out

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
