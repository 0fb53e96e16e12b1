"""Drop-in twins of the reference dispatchers (commdyn/_kernels.py) on the GPU.

Same names, positional signatures and array contracts as the reference
(SURVEY §8b).  Arguments may be numpy arrays (copied to the device; ``out``
is updated in place on return, as the reference mutates it) or CUDA torch
tensors (worked on in place, stream-ordered, no host sync except where the
reference returns host values).  Each call runs a kernel from
libcommdyn_cuda.so; there is no CPU path.

The trajectory hot path does not go through these one-kernel-per-call twins:
it runs the fused stage kernels (engine.py / cdk_kuramoto_rk4).
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib

IMAG_TOL = 1e-9  # _kernels.py:26


def _dev(a, dtype):
    import torch

    if torch.is_tensor(a):
        if not a.is_cuda:
            a = a.cuda()
        return a.to(dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


class _Out:
    """Device view of a caller-owned ``out`` (numpy or tensor) + write-back."""

    def __init__(self, out):
        import torch

        self.host = None
        if torch.is_tensor(out) and out.is_cuda and out.dtype == torch.float64 \
                and out.is_contiguous():
            self.t = out
        else:
            if not torch.is_tensor(out) and (out.dtype != np.float64
                                             or not out.flags.c_contiguous):
                raise TypeError("out must be a C-contiguous float64 array")
            self.host = out
            self.t = _dev(out, torch.float64)

    def finish(self):
        import torch

        if self.host is not None:
            res = self.t.cpu()
            if torch.is_tensor(self.host):
                self.host.copy_(res)
            else:
                self.host[...] = res.numpy()


def order_params_blocks(x, offsets, p, half_width, norm):
    """replaces _kernels.py:68-73.  Returns complex128 [M, 2p+1] (numpy if x is numpy)."""
    import torch

    L = _lib.lib()
    xt = _dev(x, torch.float64)
    ot = _dev(offsets, torch.int64)
    m = ot.shape[0] - 1
    r = torch.empty((m, 2 * p + 1), dtype=torch.complex128, device="cuda")
    _lib.check(L.cdk_order_params_blocks(xt.data_ptr(), ot.data_ptr(), m, int(p),
                                         math.pi / half_width, float(norm), r.data_ptr(),
                                         _lib.stream_ptr()), "order_params_blocks")
    return r if torch.is_tensor(x) else r.cpu().numpy()


def dense_complex(x, offsets, tbl, half_width, out):
    """replaces _kernels.py:165-169; returns (n_viol, max_imag)."""
    import torch

    L = _lib.lib()
    xt = _dev(x, torch.float64)
    ot = _dev(offsets, torch.int64)
    tt = _dev(tbl, torch.complex128)
    p = (tt.shape[1] - 1) // 2
    o = _Out(out)
    guard = torch.zeros(2, dtype=torch.int64, device="cuda")
    _lib.check(L.cdk_dense_complex(xt.data_ptr(), ot.data_ptr(), ot.shape[0] - 1, tt.data_ptr(),
                                   p, math.pi / half_width, o.t.data_ptr(), guard.data_ptr(),
                                   _lib.stream_ptr()), "dense_complex")
    o.finish()
    g = guard.cpu().numpy()
    return int(g[0]), float(g[1:2].view(np.float64)[0])


def dense_real(x, offsets, tbl_cos, tbl_sin, half_width, out):
    """replaces _kernels.py:199-204."""
    import torch

    L = _lib.lib()
    xt = _dev(x, torch.float64)
    ot = _dev(offsets, torch.int64)
    tc = _dev(tbl_cos, torch.float64)
    ts = _dev(tbl_sin, torch.float64)
    o = _Out(out)
    _lib.check(L.cdk_dense_real(xt.data_ptr(), ot.data_ptr(), ot.shape[0] - 1, tc.data_ptr(),
                                ts.data_ptr(), tc.shape[1] - 1, math.pi / half_width,
                                o.t.data_ptr(), _lib.stream_ptr()), "dense_real")
    o.finish()


def pairs_trig(iu, iv, x, inv_n, d_cos, d_sin, half_width, sgn, out):
    """replaces _kernels.py:353-362."""
    import torch

    L = _lib.lib()
    it, vt = _dev(iu, torch.int64), _dev(iv, torch.int64)
    xt = _dev(x, torch.float64)
    dc, ds = _dev(d_cos, torch.float64), _dev(d_sin, torch.float64)
    st = _dev(sgn, torch.float64)
    o = _Out(out)
    _lib.check(L.cdk_pairs_trig(it.data_ptr(), vt.data_ptr(), it.shape[0], xt.data_ptr(),
                                float(inv_n), dc.data_ptr(), ds.data_ptr(), dc.shape[0] - 1,
                                math.pi / half_width, st.data_ptr(), o.t.data_ptr(),
                                _lib.stream_ptr()), "pairs_trig")
    o.finish()


def pairs_cs(iu, iv, pos, vel, inv_n, amp, sigma2, beta, sgn, out):
    """replaces _kernels.py:372-376."""
    import torch

    L = _lib.lib()
    it, vt = _dev(iu, torch.int64), _dev(iv, torch.int64)
    pt, vl = _dev(pos, torch.float64), _dev(vel, torch.float64)
    st = _dev(sgn, torch.float64)
    o = _Out(out)
    _lib.check(L.cdk_pairs_cs(it.data_ptr(), vt.data_ptr(), it.shape[0], pt.data_ptr(),
                              vl.data_ptr(), pt.shape[1], float(inv_n), float(amp), float(sigma2),
                              float(beta), st.data_ptr(), o.t.data_ptr(), _lib.stream_ptr()),
               "pairs_cs")
    o.finish()


def moments_blocks(x, offsets, p, x0, norm):
    """replaces _kernels.py:109-113."""
    import torch

    L = _lib.lib()
    xt = _dev(x, torch.float64)
    ot = _dev(offsets, torch.int64)
    m = ot.shape[0] - 1
    w = torch.empty((m, p + 1), dtype=torch.float64, device="cuda")
    _lib.check(L.cdk_moments_blocks(xt.data_ptr(), ot.data_ptr(), m, int(p), float(x0),
                                    float(norm), w.data_ptr(), _lib.stream_ptr()),
               "moments_blocks")
    return w if torch.is_tensor(x) else w.cpu().numpy()


def dense_poly(x, offsets, tbl, scale, shift, out):
    """replaces _kernels.py:231-235."""
    import torch

    L = _lib.lib()
    xt = _dev(x, torch.float64)
    ot = _dev(offsets, torch.int64)
    tt = _dev(tbl, torch.float64)
    o = _Out(out)
    _lib.check(L.cdk_dense_poly(xt.data_ptr(), ot.data_ptr(), ot.shape[0] - 1, tt.data_ptr(),
                                tt.shape[1] - 1, float(scale), float(shift), o.t.data_ptr(),
                                _lib.stream_ptr()), "dense_poly")
    o.finish()


def pairs_poly(iu, iv, x, inv_n, coef, x0, sgn, out):
    """replaces _kernels.py:365-369 (Desai-Zwanzig polynomial coupling)."""
    import torch

    L = _lib.lib()
    it, vt = _dev(iu, torch.int64), _dev(iv, torch.int64)
    xt = _dev(x, torch.float64)
    ct = _dev(coef, torch.float64)
    st = _dev(sgn, torch.float64)
    o = _Out(out)
    _lib.check(L.cdk_pairs_poly(it.data_ptr(), vt.data_ptr(), it.shape[0], xt.data_ptr(),
                                float(inv_n), ct.data_ptr(), ct.shape[0] - 1, float(x0),
                                st.data_ptr(), o.t.data_ptr(), _lib.stream_ptr()), "pairs_poly")
    o.finish()


def ho_naive_block(theta, lambdas):
    """replaces _kernels.py:424-428 (literal quadruple loop; lam <= 4096)."""
    import torch

    L = _lib.lib()
    l1, l2, l3, l4 = (float(v) for v in lambdas)
    tt = _dev(theta, torch.float64)
    out = torch.empty_like(tt)
    _lib.check(L.cdk_ho_naive_block(tt.data_ptr(), tt.shape[0], l1, l2, l3, l4, out.data_ptr(),
                                    _lib.stream_ptr()), "ho_naive_block")
    return out if torch.is_tensor(theta) else out.cpu().numpy()


def nn_recurrence(ph, k, inv_n, anchor_every=1024):
    """replaces _kernels.py:472-477 (window sums, re-anchored recurrence)."""
    import torch

    L = _lib.lib()
    pt = _dev(ph, torch.complex128)
    f = torch.empty_like(pt)
    _lib.check(L.cdk_nn_recurrence(pt.data_ptr(), pt.shape[0], int(k), float(inv_n),
                                   int(anchor_every), f.data_ptr(), _lib.stream_ptr()),
               "nn_recurrence")
    return f if torch.is_tensor(ph) else f.cpu().numpy()


def spin_field_sums(spins):
    """replaces _kernels.py:505-509 (per-node sum over all spins, int64)."""
    import torch

    L = _lib.lib()
    st = _dev(spins, torch.int64)
    f = torch.empty_like(st)
    scratch = torch.empty(1, dtype=torch.int64, device=st.device)
    _lib.check(L.cdk_spin_field_sums(st.data_ptr(), st.shape[0], f.data_ptr(),
                                     scratch.data_ptr(), _lib.stream_ptr()), "spin_field_sums")
    return f if torch.is_tensor(spins) else f.cpu().numpy()
