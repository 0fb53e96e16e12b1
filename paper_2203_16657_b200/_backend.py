"""Backend switch, API-compatible with commdyn/_backend.py:19-56.

The reference selects "numba" or "numpy" from COMMDYN_BACKEND at import and
lets callers flip it at runtime.  This build adds the "cuda" backend and is
the only backend it ships: the CPU kernels stay in the reference package (and
in oracle/, as the test checker).  ``set_backend`` therefore accepts only
"cuda"; asking for a CPU backend raises ValueError exactly where the reference
raises for an unknown/unavailable backend (_backend.py:50-56).
"""

from __future__ import annotations

import os

_env = os.environ.get("COMMDYN_BACKEND", "").strip().lower()
if _env not in ("", "cuda"):
    raise ValueError(f"COMMDYN_BACKEND must be 'cuda' for this build, got {_env!r}")

USE_NUMBA = False  # kept for code that reads the reference flag
HAVE_NUMBA = False
USE_CUDA = True


def backend() -> str:
    """Name of the active kernel backend (_backend.py:41-43)."""
    return "cuda"


def set_backend(name: str) -> None:
    """Switch the kernel backend (_backend.py:46-56); only 'cuda' exists here."""
    if name != "cuda":
        raise ValueError(f"unknown backend {name!r} (this build ships only 'cuda')")
