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

import os

import numpy as np

from ..plan import ExecutionPlan, KernelPlan, Template, align


def _row_classes(M: np.ndarray):
    """np.unique(M, axis=0, return_inverse, return_counts) via a 64-bit row hash (fast)."""
    M = np.ascontiguousarray(M, dtype=np.int64)
    h = np.zeros(M.shape[0], dtype=np.uint64)
    for j in range(M.shape[1]):
        h = (h ^ M[:, j].astype(np.uint64)) * np.uint64(0x9E3779B97F4A7C15)
        h ^= h >> np.uint64(29)
    _, inv, cnt = np.unique(h, return_inverse=True, return_counts=True)
    return inv.reshape(-1), cnt


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
                  dest_kind: str = "intermediate", gap: int = 0, locals_: list[int] | None = None) -> np.ndarray:
        """Append one group; returns its result addresses, shape (n_roots, N).

        ``gap`` reserves zero padding after the result range (room for the
        over-reach of padded structured consumers, see add_structured)."""
        const_cols = const_cols or []
        n = int(len(slot_addrs[0]) if slot_addrs else len(const_cols[0]))
        for col in list(slot_addrs) + list(const_cols):
            if len(col) != n:
                raise ValueError(f"{name}: ragged slot columns")
        dest = align(self.cursor, self.vector_width)
        self.cursor = dest + len(roots) * n + gap
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
            template_locals=list(locals_ or []), pos_vars=list(range(n_pos)),
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
        if n == 0 or not cols or os.environ.get("SGB_SPLIT", "0") == "0":
            return self.add_group(name, level, template, roots, slot_addrs, const_cols, dest_kind)
        src = np.stack([self.producer_ids(c) for c in cols], axis=1)
        sinv, scnt = _row_classes(src)
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
            inv, counts = _row_classes(D)
            big = counts >= min_class
            remap = np.full(counts.size, next_label + int(big.sum()), dtype=np.int64)
            remap[big] = next_label + np.arange(int(big.sum()))
            label[members] = remap[inv]
            next_label += int(big.sum()) + 1
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

    def add_structured(self, name: str, level: int, template: Template, roots: list[int],
                       slot_addrs: list[np.ndarray], anchor: np.ndarray, n_anchor: int,
                       scales=None, min_frac: float = 0.2, gap: int = 0,
                       dest_kind: str = "intermediate") -> np.ndarray:
        """Anchor-rate layout for the regular interior of a structured mesh.

        Every entity (one instance of ``template``) has an anchor vertex.
        Entities whose slot addresses are ``scale_s * anchor + rel_s`` with
        the same ``rel`` vector form a class; every class holding at least
        ``min_frac * n_anchor`` entities becomes one group with ``n_anchor``
        instances, instance a = anchor a (anchors outside the class compute
        the same formula on neighbouring values: padding nobody reads).  In
        such a group consecutive lanes read consecutive addresses of every
        slot (whole 128-byte lines per warp instead of one line per lane) and
        all slots with the slot-0 scale are offset-coherent, i.e. leave the
        index table.  The remaining entities (mesh boundary) go through
        ``add_group_split``.  ``gap`` pads each structured group's range so
        consumers reaching a few anchors past the end stay inside it.
        """
        cols = [np.asarray(c, dtype=np.int64) for c in slot_addrs]
        anchor = np.asarray(anchor, dtype=np.int64)
        E = len(anchor)
        scales = [1] * len(cols) if scales is None else list(scales)
        out = np.empty((len(roots), E), dtype=np.int64)
        if E == 0:
            return out
        rel = np.stack([c - sc * anchor for c, sc in zip(cols, scales)], axis=1)
        inv, counts = _row_classes(rel)
        done = np.zeros(E, dtype=bool)
        big = np.flatnonzero(counts >= max(1, int(min_frac * n_anchor)))
        for k, cls in enumerate(big.tolist()):
            members = np.flatnonzero(inv == cls)
            a = anchor[members]
            if np.unique(a).size != a.size:
                continue  # anchors must be unique inside a structured group
            r = rel[members[0]]
            grid = np.arange(n_anchor, dtype=np.int64)
            sub = [sc * grid + int(rv) for sc, rv in zip(scales, r.tolist())]
            lo = min(int(c.min()) for c in sub)
            hi = max(int(c.max()) for c in sub)
            if lo < 0 or hi >= align(self.cursor, self.vector_width):
                continue  # padding would reach outside the values written so far
            res = self.add_group(f"{name}_s{k}", level, template, roots, sub, None, dest_kind, gap=gap)
            out[:, members] = res[:, a]
            done[members] = True
        rest = np.flatnonzero(~done)
        if rest.size:
            order = rest[np.argsort(anchor[rest], kind="stable")]
            out[:, order] = self.add_group_split(f"{name}_b", level, template, roots,
                                                 [c[order] for c in cols], None, dest_kind)
        return out

    def add_affine_classes(self, name: str, level: int, template: Template, roots: list[int],
                           slot_addrs: list[np.ndarray], anchor: np.ndarray, scales, min_members: int = 4096,
                           min_fill: float = 0.5, dest_kind: str = "intermediate") -> np.ndarray:
        """Groups whose every index column is affine in the instance.

        Entities with the same offset vector ``addr_s - scale_s * anchor`` form
        a class; a class with at least ``min_members`` entities filling at
        least ``min_fill`` of its anchor range [a_lo, a_hi] becomes one group
        of a_hi - a_lo + 1 instances, instance k = anchor a_lo + k (anchors of
        the range outside the class compute the same formula on in-range
        neighbour values: results nobody reads).  Every slot is then
        ``scale_s * (a_lo + k) + rel_s``: affine column 0, coherent rest (one
        index column, lane-contiguous gathers).  The rest goes to add_group.
        """
        cols = [np.asarray(c, dtype=np.int64) for c in slot_addrs]
        anchor = np.asarray(anchor, dtype=np.int64)
        E = len(anchor)
        out = np.empty((len(roots), E), dtype=np.int64)
        if E == 0:
            return out
        sc = np.asarray(list(scales), dtype=np.int64)
        rel = np.stack([c - s_ * anchor for c, s_ in zip(cols, sc.tolist())], axis=1)
        inv, counts = _row_classes(rel)
        done = np.zeros(E, dtype=bool)
        for k, cls in enumerate(np.flatnonzero(counts >= min_members).tolist()):
            members = np.flatnonzero(inv == cls)
            a = anchor[members]
            a_lo, a_hi = int(a.min()), int(a.max())
            if np.unique(a).size != a.size or a.size < min_fill * (a_hi - a_lo + 1):
                continue
            r = rel[members[0]]
            grid = np.arange(a_lo, a_hi + 1, dtype=np.int64)
            sub = [s_ * grid + int(rv) for s_, rv in zip(sc.tolist(), r.tolist())]
            res = self.add_group(f"{name}_a{k}", level, template, roots, sub, None, dest_kind)
            out[:, members] = res[:, a - a_lo]
            done[members] = True
        rest = np.flatnonzero(~done)
        if rest.size:
            out[:, rest] = self.add_group(f"{name}_r", level, template, roots, [c[rest] for c in cols], None,
                                          dest_kind)
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
