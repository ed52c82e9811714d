"""Structural hashes of the reference arena, restated for plan builders.

The reference puts the children of every commutative node (n-ary ADD / MUL)
into canonical order: ascending ``(struct_hash, arena index)``
(expr.py:230-251).  That order is the left-fold order of every sparse-product
entry (sp_mul -> apply(ADD, terms), sparse.py:102-139) and of every assembled
cell (from_triplets, sparse.py:73-99), so a builder that wants bit-identical
sums must reproduce the hashes.  Only the structure matters (any VAR hashes
like any VAR, any CONST like any CONST), so the builders compute hashes per
structural *class*, not per node.

Restated: ``mix64`` / ``mix2`` (expr.py:41-52), the leaf seeds
(expr.py:34-35, 152-153) and the operation chain of ``ExprArena.apply``
(expr.py:257-276, POW exponent folding :271-273).
"""

from __future__ import annotations

MASK64 = (1 << 64) - 1
_VAR_SEED = 0x243F6A8885A308D3  # expr.py:34
_CONST_SEED = 0x13198A2E03707344  # expr.py:35

VAR, CONST, ADD, SUB, MUL, DIV, NEG, SQRT, SIN, COS, EXP, LOG, POW, SELECT = range(14)
COMMUTATIVE = (ADD, MUL)


def mix64(z: int) -> int:
    """SplitMix64 finalizer (expr.py:41-46)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def mix2(a: int, b: int) -> int:
    """mix(a xor rotl(b, 31)) (expr.py:49-52)."""
    b &= MASK64
    return mix64(a ^ (((b << 31) | (b >> 33)) & MASK64))


SH_VAR = mix2(mix64(VAR), _VAR_SEED)  # expr.py:152
SH_CONST = mix2(mix64(CONST), _CONST_SEED)  # expr.py:153


def sh_apply(op: int, child_hashes, pow_k: int | None = None) -> int:
    """Struct hash of ``apply(op, children)``; commutative children sorted.

    Equal child hashes tie-break by arena index in the reference, which does
    not change the hash chain, so sorting the hashes alone is exact.
    """
    hs = list(child_hashes)
    if op in COMMUTATIVE:
        hs.sort()
    h = 0
    for c in hs:
        h = mix2(c, h)
    if op == POW:
        h = mix2(h, mix64(int(pow_k)))
    return mix2(mix64(op), h)
