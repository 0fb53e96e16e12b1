"""Integrator: fixed-step explicit Euler / RK4 trajectories.

``integrate(model, dec, x0, plan)`` runs the whole trajectory on the device
through the fused CIA kernels: 4 stage kernels per RK4 step, state resident
in HBM, host involvement only at record points.  Steps = ceil(T/dt); the last
step is truncated to land exactly on T.  Phases are wrapped to
(-pi, pi] after every full step; a non-finite state raises
BlowUpError(step).  Records every ``record_every``-th state plus
the initial and final state.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import InputError
from .evaluator import engine_for
from .graph import Decomposition


@dataclass(frozen=True)
class IntegrationPlan:
    t_end: float
    dt: float
    scheme: str = "rk4"
    record_every: int = 0
    mode: str = "cia"

    def n_steps(self) -> int:
        if self.dt <= 0 or self.t_end < 0:
            raise InputError("need dt > 0 and t_end >= 0")
        return int(math.ceil(self.t_end / self.dt - 1e-12))

    def step_sizes(self):
        n = self.n_steps()
        last = self.t_end - (n - 1) * self.dt if n else 0.0
        if abs(last - self.dt) <= 1e-9 * self.dt:  # T an integer multiple of dt up to rounding
            last = self.dt
        return n, self.dt, last


@dataclass
class Trajectory:
    times: np.ndarray
    states: np.ndarray  # [n_records, N] original node order
    wall_seconds: float = 0.0
    kernel_launches: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def final(self) -> np.ndarray:
        return self.states[-1]


def integrate(model, dec: Decomposition, x0, plan: IntegrationPlan) -> Trajectory:
    if plan.mode != "cia":
        raise InputError("integrate: only mode='cia' runs on the device path")
    if plan.scheme not in ("rk4", "euler"):
        raise InputError(f"unknown scheme {plan.scheme!r}")
    from .cs import CuckerSmale

    x0 = np.asarray(x0, dtype=np.float64)
    if isinstance(model, CuckerSmale):
        return _integrate_cs(model, dec, x0, plan)
    if x0.shape != (dec.n_nodes,):
        raise InputError("x0 shape does not match the decomposition")
    n_steps, dt, dt_last = plan.step_sizes()
    perm = dec.partition.perm
    eng = engine_for(model, dec)
    if plan.scheme == "euler" and not hasattr(eng, "euler"):
        raise InputError("Euler is implemented for the classical Kuramoto engine only")
    lib = eng.lib
    launches0 = int(lib.cdk_launch_count())
    t0 = time.perf_counter()
    eng.set_state(x0[perm])
    stride = plan.record_every if plan.record_every > 0 else n_steps
    advance = eng.rk4 if plan.scheme == "rk4" else eng.euler

    times = [0.0]
    snaps = [eng.theta.clone()]
    done = 0
    while done < n_steps:
        chunk = min(stride, n_steps - done)
        full = chunk if done + chunk < n_steps else chunk - 1
        if full > 0:
            advance(dt, full)
        if done + chunk == n_steps:
            advance(dt_last, 1)
        done += chunk
        times.append(min(done * dt, plan.t_end) if done < n_steps else plan.t_end)
        snaps.append(eng.theta.clone())
    eng.check()
    states_perm = np.stack([s.cpu().numpy() for s in snaps]) if n_steps else snaps[0].cpu().numpy()[None]
    states = np.empty_like(states_perm)
    states[:, perm] = states_perm
    wall = time.perf_counter() - t0
    return Trajectory(np.asarray(times), states, wall, int(lib.cdk_launch_count()) - launches0,
                      {"n_steps": n_steps, "dt": dt, "dt_last": dt_last})


def _integrate_cs(model, dec: Decomposition, x0, plan: IntegrationPlan) -> Trajectory:
    """Cucker-Smale trajectory: state [N, 4] = (s_x, s_y, v_x, v_y), no wrap.
    The P2 fit domain covers [0, t_end] (cs.cs_plan)."""
    from .evaluator import _cs_engine

    if plan.scheme != "rk4":
        raise InputError("Cucker-Smale integrates with rk4")
    if x0.shape != (dec.n_nodes, 4):
        raise InputError("Cucker-Smale state must have shape (N, 4)")
    n_steps, dt, dt_last = plan.step_sizes()
    perm = dec.partition.perm
    xp = x0[perm]
    t0 = time.perf_counter()
    eng = _cs_engine(model, dec, xp[:, :2], xp[:, 2:], t_end=plan.t_end)
    launches0 = int(eng.lib.cdk_launch_count())
    stride = plan.record_every if plan.record_every > 0 else n_steps
    import torch

    snaps = [torch.cat([eng.pos, eng.vel], 1).clone()]
    times = [0.0]
    done = 0
    while done < n_steps:
        chunk = min(stride, n_steps - done)
        full = chunk if done + chunk < n_steps else chunk - 1
        if full > 0:
            eng.rk4(dt, full)
        if done + chunk == n_steps:
            eng.rk4(dt_last, 1)
        done += chunk
        times.append(min(done * dt, plan.t_end) if done < n_steps else plan.t_end)
        snaps.append(torch.cat([eng.pos, eng.vel], 1).clone())
    eng.check()
    sp = np.stack([s.cpu().numpy() for s in snaps])
    states = np.empty_like(sp)
    states[:, perm] = sp
    return Trajectory(np.asarray(times), states, time.perf_counter() - t0,
                      int(eng.lib.cdk_launch_count()) - launches0,
                      {"n_steps": n_steps, "dt": dt, "sup_err": float(eng.plan.sup_err.max())})


__all__ = ["IntegrationPlan", "Trajectory", "integrate", "_lib"]
