"""A minimal restatement of the reference expression arena for plan builders.

Builders trace ONE entity (a finite element) and instance its template for
every entity with numpy.  For the instanced plan to compute exactly what the
reference trace computes, the traced template must have the reference's node
structure: hash-consing on ``(op, children)`` and commutative children in
ascending ``(struct_hash, arena index)`` order (expr.py:214-276,
``ExprArena.apply``), variables and constants consed by id / bit pattern
(expr.py:177-210), and ``Sym`` operator semantics (expr.py:788-847).  Element
programs are written once against the ``Sym`` protocol and run unchanged with
the reference's ``Sym`` (golden fixtures, tests/golden/make_fem_golden.py) and
with this one (the builders, which must run where the reference is absent).
"""

from __future__ import annotations

import struct

from ..plan import OpKind, Template
from . import structhash as S


def _bits(v: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", float(v)))[0]


class Arena:
    def __init__(self):
        self.ops: list[int] = []
        self.args: list[tuple] = []
        self.payload: list = []
        self.sh: list[int] = []
        self.cons: dict = {}

    def _push(self, op, args, payload, sh):
        ref = len(self.ops)
        self.ops.append(int(op))
        self.args.append(tuple(args))
        self.payload.append(payload)
        self.sh.append(sh)
        return ref

    def make_var(self, vid: int) -> int:
        key = (0, int(vid))
        ref = self.cons.get(key)
        if ref is None:
            ref = self._push(OpKind.VAR, (), int(vid), S.SH_VAR)
            self.cons[key] = ref
        return ref

    def make_const(self, v: float) -> int:
        key = (1, _bits(v))
        ref = self.cons.get(key)
        if ref is None:
            ref = self._push(OpKind.CONST, (), float(v), S.SH_CONST)
            self.cons[key] = ref
        return ref

    def apply(self, op, children) -> int:
        op = int(op)
        cs = tuple(int(c) for c in children)
        if op in (OpKind.ADD, OpKind.MUL):
            cs = tuple(sorted(cs, key=lambda c: (self.sh[c], c)))  # expr.py:245-251
        key = (op, cs)
        ref = self.cons.get(key)
        if ref is not None:
            return ref
        pow_k = int(self.payload[cs[1]]) if op == OpKind.POW else None
        sh = S.sh_apply(op, [self.sh[c] for c in cs], pow_k)
        ref = self._push(op, cs, None, sh)
        self.cons[key] = ref
        return ref

    def var(self, vid: int) -> "Sym":
        return Sym(self, self.make_var(vid))

    def to_template(self, roots):
        """Reachable nodes -> plan.Template (ascending order keeps the structure); new root refs."""
        need = bytearray(len(self.ops))
        for r in roots:
            need[r] = 1
        for i in range(len(self.ops) - 1, -1, -1):
            if need[i]:
                for c in self.args[i]:
                    need[c] = 1
        T = Template()
        m = {}
        for i in range(len(self.ops)):
            if not need[i]:
                continue
            op = self.ops[i]
            if op == OpKind.VAR:
                m[i] = T.var(self.payload[i])
            elif op == OpKind.CONST:
                m[i] = T.const(self.payload[i])
            else:
                m[i] = T.apply(op, [m[c] for c in self.args[i]])
        return T, [m[r] for r in roots]


class Sym:
    """expr.py:788-847, operator for operator."""

    __slots__ = ("arena", "ref")

    def __init__(self, arena: Arena, ref: int):
        self.arena = arena
        self.ref = ref

    def _lift(self, other) -> int:
        if isinstance(other, Sym):
            return other.ref
        return self.arena.make_const(other)

    def __add__(self, other):
        return Sym(self.arena, self.arena.apply(OpKind.ADD, (self.ref, self._lift(other))))

    __radd__ = __add__

    def __mul__(self, other):
        return Sym(self.arena, self.arena.apply(OpKind.MUL, (self.ref, self._lift(other))))

    __rmul__ = __mul__

    def __sub__(self, other):
        return Sym(self.arena, self.arena.apply(OpKind.SUB, (self.ref, self._lift(other))))

    def __rsub__(self, other):
        return Sym(self.arena, self.arena.apply(OpKind.SUB, (self._lift(other), self.ref)))

    def __truediv__(self, other):
        return Sym(self.arena, self.arena.apply(OpKind.DIV, (self.ref, self._lift(other))))

    def __rtruediv__(self, other):
        return Sym(self.arena, self.arena.apply(OpKind.DIV, (self._lift(other), self.ref)))

    def __neg__(self):
        return Sym(self.arena, self.arena.apply(OpKind.NEG, (self.ref,)))


def sym_log(x: Sym) -> Sym:
    return Sym(x.arena, x.arena.apply(OpKind.LOG, (x.ref,)))


def sym_sqrt(x: Sym) -> Sym:
    return Sym(x.arena, x.arena.apply(OpKind.SQRT, (x.ref,)))
