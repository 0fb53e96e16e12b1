"""Device-resident CIA engine for the Kuramoto family (the fused hot path).

``KuramotoEngine`` owns the DeviceGraph, the workspace and the device state
(theta, omega in permuted order) and drives the C ABI:

    eng = KuramotoEngine(dec, omega_perm, coupling=K, norm=N)
    eng.set_state(theta_perm)      # prepare: z = exp(i theta), community sums
    eng.rk4(dt, n_steps)           # 4 fused stage kernels per step
    eng.status()                   # -> BlowUpError on non-finite state

No CPU fallback: every method calls libcommdyn_cuda.so.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import BlowUpError, InputError
from .plan import DeviceGraph


class KuramotoEngine:
    def __init__(self, dec, omega, coupling: float = 1.0, norm: float | None = None,
                 device=None, graph: DeviceGraph | None = None):
        import torch

        self.lib = _lib.lib()
        self.graph = graph if graph is not None else DeviceGraph(dec, device=device)
        self.device = self.graph.device
        n = self.graph.n_rows
        self.n = n
        self.coupling = float(coupling)
        self.norm = float(norm if norm is not None else n)
        self.k_over_n = self.coupling / self.norm
        omega = torch.as_tensor(np.asarray(omega, dtype=np.float64) if not torch.is_tensor(omega)
                                else omega, dtype=torch.float64)
        if omega.shape != (n,):
            raise InputError(f"omega must have shape ({n},)")
        # bulk copies read theta/omega in 16-byte units: keep a 4-element tail
        self._omega_buf = torch.zeros(n + 4, dtype=torch.float64, device=self.device)
        self._omega_buf[:n].copy_(omega)
        self.omega = self._omega_buf[:n]
        self._theta_buf = torch.zeros(n + 4, dtype=torch.float64, device=self.device)
        self.theta = self._theta_buf[:n]
        self._rhs_theta = None
        nbytes = int(self.lib.cdk_kuramoto_workspace_bytes(ctypes.byref(self.graph.struct)))
        self.workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        self._gp = ctypes.byref(self.graph.struct)
        self._rhs_ws = None
        self._pinned = None  # host staging buffer for uploads from numpy
        self._stage_dev = None  # device staging buffer for permuted uploads

    def upload_permuted(self, dst, host, perm_dev) -> None:
        """dst = host[perm] with the gather on the device: the host array goes up
        in its own (original) order through the pinned staging buffer."""
        import torch

        if self._stage_dev is None:
            self._stage_dev = torch.empty(self.n, dtype=torch.float64, device=self.device)
        self._upload(self._stage_dev, host, key=dst.data_ptr())
        torch.index_select(self._stage_dev, 0, perm_dev, out=dst)

    def _upload(self, dst, host, key=None) -> None:
        """numpy (or host tensor) -> device view ``dst`` through a pinned staging
        buffer (an async copy at full PCIe/C2C rate instead of a pageable one)."""
        import torch

        if torch.is_tensor(host):
            dst.copy_(host.to(torch.float64), non_blocking=True)
            return
        if self._pinned is None:
            # both usual destinations get their buffer now: a pinned allocation
            # (~1.5 ms) should not land in a later call's timed path
            self._pinned = {t.data_ptr(): [torch.empty(self.n, dtype=torch.float64,
                                                       pin_memory=True), torch.cuda.Event()]
                            for t in (self.omega, self.theta)}
        key = dst.data_ptr() if key is None else key
        slot = self._pinned.get(key)  # one staging buffer per (final) destination
        if slot is None:
            slot = [torch.empty(self.n, dtype=torch.float64, pin_memory=True),
                    torch.cuda.Event()]
            self._pinned[key] = slot
        slot[1].synchronize()  # its last copy has left the buffer (no stream-wide wait)
        slot[0].numpy()[:] = np.asarray(host, dtype=np.float64)
        dst.copy_(slot[0], non_blocking=True)
        slot[1].record(torch.cuda.current_stream(self.device))

    def set_params(self, omega, coupling: float, norm: float) -> None:
        """New model parameters on the same graph and workspace (the public API
        reuses one engine per decomposition across model objects)."""
        import torch

        if tuple(np.shape(omega)) != (self.n,):
            raise InputError(f"omega must have shape ({self.n},)")
        self._upload(self.omega, omega)
        self.coupling = float(coupling)
        self.norm = float(norm)
        self.k_over_n = self.coupling / self.norm

    # -- state --------------------------------------------------------------
    def set_state(self, theta, stream=None) -> None:
        import torch

        if tuple(np.shape(theta)) != (self.n,):
            raise InputError(f"state must have shape ({self.n},)")
        if torch.is_tensor(theta):
            self.theta.copy_(theta.to(self.device, torch.float64), non_blocking=True)
        else:
            self._upload(self.theta, theta)
        self.prepare(stream)

    def prepare(self, stream=None) -> None:
        _lib.check(self.lib.cdk_kuramoto_prepare(self._gp, self.theta.data_ptr(),
                                                 self.workspace.data_ptr(),
                                                 _lib.stream_ptr(stream)), "prepare")

    # -- evaluation ---------------------------------------------------------
    def rhs(self, theta=None, out=None, stream=None):
        """One CIA RHS at ``theta`` (default: current state).  Returns a device tensor."""
        import torch

        if theta is None:
            th = self.theta
        else:
            if self._rhs_theta is None:
                self._rhs_theta = torch.zeros(self.n + 4, dtype=torch.float64, device=self.device)
            th = self._rhs_theta[: self.n]
            th.copy_(torch.as_tensor(theta, dtype=torch.float64).to(self.device))
        if out is None:
            out = torch.empty(self.n, dtype=torch.float64, device=self.device)
        if self._rhs_ws is None:  # separate workspace: never disturbs a running trajectory
            self._rhs_ws = torch.empty_like(self.workspace)
        _lib.check(self.lib.cdk_kuramoto_rhs(self._gp, th.data_ptr(), self.omega.data_ptr(),
                                             self.k_over_n, out.data_ptr(),
                                             self._rhs_ws.data_ptr(), _lib.stream_ptr(stream)),
                   "kuramoto_rhs")
        return out

    def rk4(self, dt: float, n_steps: int, stream=None) -> None:
        _lib.check(self.lib.cdk_kuramoto_rk4(self._gp, self.theta.data_ptr(),
                                             self.omega.data_ptr(), self.k_over_n, float(dt),
                                             int(n_steps), self.workspace.data_ptr(),
                                             _lib.stream_ptr(stream)), "kuramoto_rk4")

    def rk4_stage(self, dt: float, stage: int, stream=None) -> None:
        _lib.check(self.lib.cdk_kuramoto_rk4_stage(self._gp, self.theta.data_ptr(),
                                                   self.omega.data_ptr(), self.k_over_n,
                                                   float(dt), int(stage),
                                                   self.workspace.data_ptr(),
                                                   _lib.stream_ptr(stream)), "rk4_stage")

    def euler(self, dt: float, n_steps: int, stream=None) -> None:
        _lib.check(self.lib.cdk_kuramoto_euler(self._gp, self.theta.data_ptr(),
                                               self.omega.data_ptr(), self.k_over_n, float(dt),
                                               int(n_steps), self.workspace.data_ptr(),
                                               _lib.stream_ptr(stream)), "kuramoto_euler")

    def status(self, stream=None) -> _lib.CdkRunStatus:
        st = _lib.CdkRunStatus()
        _lib.check(self.lib.cdk_kuramoto_status(self._gp, self.workspace.data_ptr(),
                                                ctypes.byref(st), _lib.stream_ptr(stream)),
                   "status")
        return st

    def check(self, step_offset: int = 0, stream=None) -> None:
        st = self.status(stream)
        if st.nonfinite:
            raise BlowUpError(int(st.first_bad_step) + step_offset)
