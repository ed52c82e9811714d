"""Template-instancing plan builders for the full-size configs (C2/C5 mesh.py, C3 fem.py, C4 arap.py)."""

from __future__ import annotations

import hashlib
from pathlib import Path

_HERE = Path(__file__).resolve().parent
BUILDER_SOURCES = ("mesh.py", "planbuild.py", "structhash.py", "fem.py", "arap.py", "symtrace.py", "../plan.py")


def builder_hash() -> str:
    """Identity of the builder sources: plans cached or emitted under another hash are stale."""
    h = hashlib.sha1()
    for f in BUILDER_SOURCES:
        h.update((_HERE / f).read_bytes())
    return h.hexdigest()
