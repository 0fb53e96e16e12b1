"""Higher-harmonics Kuramoto: the p > 1
generalisation of the classical model through the fused device path
(csrc/harmonics.cu, C ABI ``cdk_hh_*``):

    theta'_m = omega_m + (1/N) sum_l a_ml h(theta_l - theta_m),
    h(x) = sum_{a=0..p} d_cos[a] cos(a x) + d_sin[a] sin(a x),   p <= 8.

The coefficients come either directly (the SPEC's HigherHarmonicsKuramoto
{d^sin_{1..p}, d^cos_{0..p}}) or from the host P2 fitter
(``expansion.fit_real_fourier_diff`` of an arbitrary coupling function:
``harmonics_model_from_coupling``).  E1 uses 2p+1 Fourier modes per
community; E2 evaluates the exact h on the sparse correction.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BlowUpError, InputError
from .graph import Decomposition
from .plan import build_layout

MAX_P = 8


@dataclass(frozen=True)
class HigherHarmonicsKuramoto:
    omega: np.ndarray
    d_cos: np.ndarray  # [p+1]
    d_sin: np.ndarray  # [p+1] (d_sin[0] unused: sin 0 = 0)
    norm: float | None = None
    state_space: str = "circle"

    def n(self) -> int:
        return int(np.asarray(self.omega).shape[0])

    def norm_value(self) -> float:
        return float(self.norm if self.norm is not None else self.n())

    @property
    def p(self) -> int:
        return int(np.asarray(self.d_cos).shape[0]) - 1


def higher_harmonics_model(omega, d_cos, d_sin, norm=None) -> HigherHarmonicsKuramoto:
    d_cos = np.asarray(d_cos, dtype=np.float64).copy()
    d_sin = np.asarray(d_sin, dtype=np.float64).copy()
    if d_cos.shape != d_sin.shape or d_cos.ndim != 1:
        raise InputError("d_cos and d_sin must be 1-D arrays of the same length p+1")
    if not 1 <= d_cos.shape[0] - 1 <= MAX_P:
        raise InputError(f"higher harmonics: need 1 <= p <= {MAX_P}")
    d_sin[0] = 0.0
    return HigherHarmonicsKuramoto(np.asarray(omega, dtype=np.float64), d_cos, d_sin, norm)


def harmonics_model_from_coupling(omega, h, p: int, norm=None) -> HigherHarmonicsKuramoto:
    """Fit h on [-pi, pi] with p harmonics and build the model."""
    from .expansion import fit_real_fourier_diff

    e = fit_real_fourier_diff(h, p, math.pi)
    return higher_harmonics_model(omega, e.d_cos, e.d_sin, norm)


class HhDeviceGraph:
    """rblocks + the directed correction as two plain CSRs (missing intra,
    sign -1; inter and pool, sign +1), device-resident."""

    def __init__(self, dec: Decomposition, device=None):
        import torch

        from .ho import inter_csr, missing_csr

        dev = torch.device(device if device is not None else "cuda")
        lay = build_layout(dec)
        mptr, mcol = missing_csr(dec)
        xptr, xcol = inter_csr(dec)

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        self._t = {
            "rblk_row0": up(lay.rblk_row0), "rblk_comm": up(lay.rblk_comm),
            "comm_rblk_off": up(lay.comm_rblk_off), "comm_off": up(lay.comm_off),
            "miss_ptr": up(mptr), "miss_col": up(mcol if mcol.size else np.zeros(1, np.int32)),
            "inter_ptr": up(xptr), "inter_col": up(xcol if xcol.size else np.zeros(1, np.int32)),
        }
        self.n_rows = int(dec.n_nodes)
        self.n_rblk = int(lay.n_rblk)
        self.n_comm = int(lay.n_comm)
        self.device = dev

    def struct(self, p: int, d_cos_dev, d_sin_dev) -> "_lib.CdkHhGraph":
        t = self._t
        return _lib.CdkHhGraph(
            n_rows=self.n_rows, n_rblk=self.n_rblk, n_comm=self.n_comm, p=int(p), reserved=0,
            rblk_row0=t["rblk_row0"].data_ptr(), rblk_comm=t["rblk_comm"].data_ptr(),
            comm_rblk_off=t["comm_rblk_off"].data_ptr(), comm_off=t["comm_off"].data_ptr(),
            miss_ptr=t["miss_ptr"].data_ptr(), miss_col=t["miss_col"].data_ptr(),
            inter_ptr=t["inter_ptr"].data_ptr(), inter_col=t["inter_col"].data_ptr(),
            d_cos=d_cos_dev.data_ptr(), d_sin=d_sin_dev.data_ptr())


class HhEngine:
    """Device-resident higher-harmonics CIA engine (permuted order)."""

    def __init__(self, dec: Decomposition, omega, d_cos, d_sin, norm=None, device=None,
                 graph: HhDeviceGraph | None = None):
        import torch

        self.lib = _lib.lib()
        self.graph = graph if graph is not None else HhDeviceGraph(dec, device)
        self.device = self.graph.device
        n = self.graph.n_rows
        self.n = n
        self.p = int(np.asarray(d_cos).shape[0]) - 1
        if not 1 <= self.p <= MAX_P:
            raise InputError(f"higher harmonics: need 1 <= p <= {MAX_P}")
        self.inv_n = 1.0 / float(norm if norm is not None else n)
        self.d_cos = torch.as_tensor(np.asarray(d_cos, np.float64), device=self.device)
        self.d_sin = torch.as_tensor(np.asarray(d_sin, np.float64), device=self.device)
        self.omega = torch.as_tensor(np.asarray(omega, np.float64), device=self.device)
        if self.omega.shape != (n,):
            raise InputError(f"omega must have shape ({n},)")
        self.theta = torch.zeros(n, dtype=torch.float64, device=self.device)
        self.struct = self.graph.struct(self.p, self.d_cos, self.d_sin)
        self._gp = ctypes.byref(self.struct)
        nb = int(self.lib.cdk_hh_workspace_bytes(self._gp))
        self.workspace = torch.empty(max(nb, 256), dtype=torch.uint8, device=self.device)
        self._rhs_ws = None

    def set_state(self, theta, stream=None):
        import torch

        t = theta if torch.is_tensor(theta) else torch.from_numpy(np.ascontiguousarray(theta,
                                                                                   np.float64))
        if t.shape != (self.n,):
            raise InputError(f"state must have shape ({self.n},)")
        self.theta.copy_(t.to(self.device, torch.float64))
        _lib.check(self.lib.cdk_hh_prepare(self._gp, self.theta.data_ptr(),
                                           self.workspace.data_ptr(), _lib.stream_ptr(stream)),
                   "hh_prepare")

    def rhs(self, theta, stream=None):
        import torch

        th = torch.as_tensor(theta, dtype=torch.float64).to(self.device).contiguous()
        out = torch.empty(self.n, dtype=torch.float64, device=self.device)
        if self._rhs_ws is None:
            self._rhs_ws = torch.empty_like(self.workspace)
        _lib.check(self.lib.cdk_hh_rhs(self._gp, th.data_ptr(), self.omega.data_ptr(), self.inv_n,
                                       out.data_ptr(), self._rhs_ws.data_ptr(),
                                       _lib.stream_ptr(stream)), "hh_rhs")
        return out

    def rk4(self, dt: float, n_steps: int, stream=None):
        _lib.check(self.lib.cdk_hh_rk4(self._gp, self.theta.data_ptr(), self.omega.data_ptr(),
                                       self.inv_n, float(dt), int(n_steps),
                                       self.workspace.data_ptr(), _lib.stream_ptr(stream)),
                   "hh_rk4")

    def check(self, stream=None):
        st = _lib.CdkRunStatus()
        _lib.check(self.lib.cdk_hh_status(self._gp, self.workspace.data_ptr(), ctypes.byref(st),
                                          _lib.stream_ptr(stream)), "hh_status")
        if st.nonfinite:
            raise BlowUpError(int(st.first_bad_step))
