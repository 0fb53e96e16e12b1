"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes bindings to ``oracle/_build/liboracle.so`` (the plain-C restatement of
``/root/reference/pkg/src/commdyn/_kernels.py``).  The functions below carry
exactly the reference dispatchers' positional signatures, so the SPEC
orchestration in ``oracle/cia.py`` can run on either this module or the real
reference ``_kernels`` module (that is how the fixtures in tests/golden pin
this restatement).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module.  ``set_threads(n)`` selects the per-thread-private OpenMP variant
of the pair kernels (reduced in thread order; n == 1 is the reference's exact
sequential order).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")

IMAG_TOL = 1e-9  # _kernels.py:26

_lib = None
_threads = 1


def build(force: bool = False) -> str:
    """Compile the C restatement (make -C oracle)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
        os.path.join(_HERE, "kernels.c")
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        I = ctypes.c_int
        lib.or_order_params_blocks.argtypes = [P, P, I64, I, D, D, P]
        lib.or_dense_complex.argtypes = [P, P, I64, P, I, D, P, P, P]
        lib.or_dense_real.argtypes = [P, P, I64, P, P, I, D, P]
        lib.or_pairs_trig.argtypes = [P, P, I64, P, I64, D, P, P, I, D, P, P, I]
        lib.or_pairs_cs.argtypes = [P, P, I64, P, P, I64, I, D, D, D, D, P, P, I]
        lib.or_moments_blocks.argtypes = [P, P, I64, I, D, D, P]
        lib.or_dense_poly.argtypes = [P, P, I64, P, I, D, D, P]
        lib.or_ho_naive_block.argtypes = [P, I64, D, D, D, D, P]
        lib.or_pairs_poly.argtypes = [P, P, I64, P, D, P, I, D, P, P]
        lib.or_nn_recurrence.argtypes = [P, I64, I64, D, I64, P]
        lib.or_spin_field_sums.argtypes = [P, I64, P]
        lib.or_num_threads.restype = I
        _lib = lib
    return _lib


def set_threads(n: int) -> None:
    global _threads
    _threads = max(1, int(n))


def max_threads() -> int:
    return int(_load().or_num_threads())


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data


def _check_out(out, dtype=np.float64):
    if out.dtype != dtype or not out.flags.c_contiguous:
        raise TypeError("out must be a C-contiguous float64 array (reference contract)")
    return out.ctypes.data


def order_params_blocks(x, offsets, p, half_width, norm):
    """_kernels.py:68-73 -> :34-51."""
    lib = _load()
    x, xp = _f64(x)
    offsets, op = _i64(offsets)
    m = offsets.shape[0] - 1
    r = np.empty((m, 2 * p + 1), dtype=np.complex128)
    lib.or_order_params_blocks(xp, op, m, int(p), math.pi / half_width, float(norm), r.ctypes.data)
    return r


def dense_complex(x, offsets, tbl, half_width, out):
    """_kernels.py:165-169 -> :124-149; returns (n_viol, max_imag)."""
    lib = _load()
    x, xp = _f64(x)
    offsets, op = _i64(offsets)
    tbl = np.ascontiguousarray(tbl, dtype=np.complex128)
    p = (tbl.shape[1] - 1) // 2
    nv = ctypes.c_int64(0)
    mi = ctypes.c_double(0.0)
    lib.or_dense_complex(xp, op, offsets.shape[0] - 1, tbl.ctypes.data, p, math.pi / half_width,
                         _check_out(out), ctypes.byref(nv), ctypes.byref(mi))
    return int(nv.value), float(mi.value)


def dense_real(x, offsets, tbl_cos, tbl_sin, half_width, out):
    """_kernels.py:199-204 -> :172-187."""
    lib = _load()
    x, xp = _f64(x)
    offsets, op = _i64(offsets)
    tc, tcp = _f64(tbl_cos)
    ts, tsp = _f64(tbl_sin)
    lib.or_dense_real(xp, op, offsets.shape[0] - 1, tcp, tsp, tc.shape[1] - 1,
                      math.pi / half_width, _check_out(out))


def pairs_trig(iu, iv, x, inv_n, d_cos, d_sin, half_width, sgn, out):
    """_kernels.py:353-362 -> :274-283 (+ :246-261)."""
    lib = _load()
    iu, iup = _i64(iu)
    iv, ivp = _i64(iv)
    x, xp = _f64(x)
    dc, dcp = _f64(d_cos)
    ds, dsp = _f64(d_sin)
    sg, sgp = _f64(sgn)
    lib.or_pairs_trig(iup, ivp, iu.shape[0], xp, out.shape[0], float(inv_n), dcp, dsp,
                      dc.shape[0] - 1, math.pi / half_width, sgp, _check_out(out), _threads)


def pairs_cs(iu, iv, pos, vel, inv_n, amp, sigma2, beta, sgn, out):
    """_kernels.py:372-376 -> :297-314."""
    lib = _load()
    iu, iup = _i64(iu)
    iv, ivp = _i64(iv)
    pos, pp = _f64(pos)
    vel, vp = _f64(vel)
    sg, sgp = _f64(sgn)
    lib.or_pairs_cs(iup, ivp, iu.shape[0], pp, vp, out.shape[0], pos.shape[1], float(inv_n),
                    float(amp), float(sigma2), float(beta), sgp, _check_out(out), _threads)


def moments_blocks(x, offsets, p, x0, norm):
    """_kernels.py:109-113 -> :81-93."""
    lib = _load()
    x, xp = _f64(x)
    offsets, op = _i64(offsets)
    m = offsets.shape[0] - 1
    w = np.empty((m, p + 1), dtype=np.float64)
    lib.or_moments_blocks(xp, op, m, int(p), float(x0), float(norm), w.ctypes.data)
    return w


def dense_poly(x, offsets, tbl, scale, shift, out):
    """_kernels.py:231-235 -> :207-217."""
    lib = _load()
    x, xp = _f64(x)
    offsets, op = _i64(offsets)
    t, tp = _f64(tbl)
    lib.or_dense_poly(xp, op, offsets.shape[0] - 1, tp, t.shape[1] - 1, float(scale),
                      float(shift), _check_out(out))


def ho_naive_block(theta, lambdas):
    """_kernels.py:424-428 -> :398-410."""
    lib = _load()
    th, thp = _f64(theta)
    l1, l2, l3, l4 = (float(v) for v in lambdas)
    out = np.empty(th.shape[0], dtype=np.float64)
    lib.or_ho_naive_block(thp, th.shape[0], l1, l2, l3, l4, out.ctypes.data)
    return out


def pairs_poly(iu, iv, x, inv_n, coef, x0, sgn, out):
    """_kernels.py:365-369 -> :286-294 (+ :264-271)."""
    lib = _load()
    iu, iup = _i64(iu)
    iv, ivp = _i64(iv)
    x, xp = _f64(x)
    c, cp = _f64(coef)
    sg, sgp = _f64(sgn)
    lib.or_pairs_poly(iup, ivp, iu.shape[0], xp, float(inv_n), cp, c.shape[0] - 1, float(x0),
                      sgp, _check_out(out))


def nn_recurrence(ph, k, inv_n, anchor_every=1024):
    """_kernels.py:472-477 -> :436-456."""
    lib = _load()
    ph = np.ascontiguousarray(ph, dtype=np.complex128)
    f = np.empty_like(ph)
    lib.or_nn_recurrence(ph.ctypes.data, ph.shape[0], int(k), float(inv_n), int(anchor_every),
                         f.ctypes.data)
    return f


def spin_field_sums(spins):
    """_kernels.py:505-509 -> :485-495."""
    lib = _load()
    s, sp = _i64(spins)
    f = np.empty(s.shape[0], dtype=np.int64)
    lib.or_spin_field_sums(sp, s.shape[0], f.ctypes.data)
    return f
