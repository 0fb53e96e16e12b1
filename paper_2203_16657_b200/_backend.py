"""Backend switch of this package, API-compatible with commdyn/_backend.py:19-56.

The reference picks "numba" or "numpy" from COMMDYN_BACKEND at import and lets
callers flip ``USE_NUMBA`` at run time; every dispatcher reads the flag per
call (``_kernels.py:71-73``).  This package ships ONE backend, "cuda"
(libcommdyn_cuda.so): its dispatchers never run CPU code, so there is nothing
to flip to here.  The CPU kernels stay in the reference package, and the
switch between them and this backend lives where a maintainer would put it —
in the reference's own ``_backend`` (``commdyn_hook.install``: ``USE_CUDA``,
``set_backend("cuda" | "numba" | "numpy")``).

Here ``set_backend`` accepts "cuda"; "numba"/"numpy" raise ``ValueError``
naming that binding, as the reference raises for an unknown or unavailable
backend (``_backend.py:50-56``).  ``available()`` reports whether the library
loads and a device is present (the condition under which
``commdyn_hook.set_backend("cuda")`` succeeds), ``info()`` what was loaded.
"""

from __future__ import annotations

import os

_env = os.environ.get("COMMDYN_BACKEND", "").strip().lower()
if _env not in ("", "cuda", "numba", "numpy"):
    raise ValueError(f"COMMDYN_BACKEND must be 'cuda', 'numba' or 'numpy', got {_env!r}")

USE_NUMBA = False  # read by code written against the reference flag
HAVE_NUMBA = False  # this package carries no numba kernels
USE_CUDA = True


def backend() -> str:
    """Name of the active kernel backend (_backend.py:41-43)."""
    return "cuda"


def set_backend(name: str) -> None:
    """Switch the kernel backend (_backend.py:46-56).  Only "cuda" exists in this
    package; the reference's CPU backends are selected in the reference itself
    (``paper_2203_16657_b200.commdyn_hook``)."""
    if name == "cuda":
        from . import _lib

        _lib.lib()  # DeviceError when the library or a GPU is missing
        return
    if name in ("numba", "numpy"):
        raise ValueError(f"backend {name!r} lives in the reference package: install the "
                         "binding with paper_2203_16657_b200.commdyn_hook.import_commdyn() and "
                         "call commdyn._backend.set_backend")
    raise ValueError(f"unknown backend {name!r}")


def available() -> bool:
    """True when libcommdyn_cuda.so loads with the expected ABI and a CUDA
    device is visible."""
    try:
        from . import _lib

        _lib.lib()
        return True
    except Exception:  # noqa: BLE001 - any load/device failure means "not available"
        return False


def info() -> dict:
    """Library path, ABI version and (when present) the device."""
    from . import _lib

    d = {"library": _lib.LIB_PATH, "abi_version": _lib.ABI_VERSION, "device": None}
    try:
        import torch

        if torch.cuda.is_available():
            p = torch.cuda.get_device_properties(0)
            d["device"] = f"{p.name} ({p.multi_processor_count} SMs, sm_{p.major}{p.minor})"
    except Exception:  # noqa: BLE001
        pass
    return d
