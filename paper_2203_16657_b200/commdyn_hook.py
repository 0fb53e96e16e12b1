"""The INTEGRATION.md §2 binding, applied to a live reference package.

A ``commdyn`` maintainer adds a third backend, ``cuda``, to the reference's
switch (``commdyn/_backend.py:19-56``) and one branch to every dispatcher in
``commdyn/_kernels.py`` (e.g. ``:68-73``).  ``install()`` makes exactly that
change at runtime on an imported, UNMODIFIED ``commdyn`` so the drop-in can be
exercised without editing the reference's files:

* ``_backend.USE_CUDA`` (new flag, read per call like ``USE_NUMBA``);
* ``_backend.set_backend("cuda")`` loads libcommdyn_cuda.so (raising
  ``DeviceError`` when it is missing), ``set_backend("numba"|"numpy")`` flips
  back through the reference's own switch (its ValueError for unknown names
  is kept); ``backend()`` reports the active one;
* each dispatcher with a device twin (``DISPATCHERS``) gets the branch
  ``if _backend.USE_CUDA: return paper_2203_16657_b200._kernels.<name>(...)``
  in front of the reference body, same positional signature.
  ``pairs_callable`` (a Python callable per pair) has no device form and
  stays on the reference's numpy path.

``import_commdyn()`` additionally honours ``COMMDYN_BACKEND=cuda`` at import,
which the unmodified reference would reject (``_backend.py:37``).
"""

from __future__ import annotations

import functools
import os
import sys

DISPATCHERS = (
    "order_params_blocks",  # _kernels.py:68-73
    "moments_blocks",       # :109-113
    "dense_complex",        # :165-169
    "dense_real",           # :199-204
    "dense_poly",           # :231-235
    "pairs_trig",           # :353-362
    "pairs_poly",           # :365-369
    "pairs_cs",             # :372-376
    "ho_naive_block",       # :424-428
    "nn_recurrence",        # :472-477
    "spin_field_sums",      # :505-509
)


def install(backend_mod, kernels_mod) -> None:
    """Add the 'cuda' backend to ``commdyn._backend`` and branch every
    dispatcher of ``commdyn._kernels`` that has a device twin.  Idempotent."""
    if getattr(backend_mod, "_cdk_installed", False):
        return
    from . import _kernels as cuda_kernels

    ref_set_backend = backend_mod.set_backend
    backend_mod.USE_CUDA = False

    def set_backend(name: str) -> None:
        if name == "cuda":
            from . import _lib

            _lib.lib()  # raises DeviceError if libcommdyn_cuda.so is absent
            backend_mod.USE_CUDA = True
            return
        ref_set_backend(name)  # the reference's own validation and flag
        backend_mod.USE_CUDA = False

    def backend() -> str:
        if backend_mod.USE_CUDA:
            return "cuda"
        return "numba" if backend_mod.USE_NUMBA else "numpy"

    set_backend.__doc__ = "Switch the kernel backend at runtime ('cuda', 'numba' or 'numpy')."
    backend_mod.set_backend = set_backend
    backend_mod.backend = backend

    for name in DISPATCHERS:
        ref_fn = getattr(kernels_mod, name, None)
        if ref_fn is None:
            continue
        dev_fn = getattr(cuda_kernels, name)

        def make(ref_fn, dev_fn):
            @functools.wraps(ref_fn)
            def dispatch(*args, **kwargs):
                if backend_mod.USE_CUDA:
                    return dev_fn(*args, **kwargs)
                return ref_fn(*args, **kwargs)

            dispatch.__wrapped_reference__ = ref_fn
            return dispatch

        setattr(kernels_mod, name, make(ref_fn, dev_fn))
    backend_mod._cdk_installed = True


def import_commdyn(path: str | None = None):
    """Import the reference package (optionally from ``path``, e.g.
    baseline/_ref), install the binding and apply ``COMMDYN_BACKEND=cuda``.
    Returns (commdyn._backend, commdyn._kernels)."""
    if path is not None and path not in sys.path:
        sys.path.insert(0, path)
    env = os.environ.get("COMMDYN_BACKEND")
    want_cuda = env is not None and env.strip().lower() == "cuda"
    if want_cuda:
        del os.environ["COMMDYN_BACKEND"]  # the unmodified switch only knows numba/numpy
    try:
        from commdyn import _backend, _kernels
    finally:
        if want_cuda:
            os.environ["COMMDYN_BACKEND"] = env
    install(_backend, _kernels)
    if want_cuda:
        _backend.set_backend("cuda")
    return _backend, _kernels
