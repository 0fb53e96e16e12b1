"""Integrator: fixed-step explicit Euler / RK4 trajectories.

``integrate(model, dec, x0, plan)`` runs the whole trajectory on the device.

* mode "cia" (default): the fused CIA kernels — 4 stage kernels per RK4 step
  (one persistent launch per recording chunk), state resident in HBM, host
  involvement only at record points;
* mode "naive": the direct sum over the full edge list (naive.NaiveEngine,
  SPEC.md:368-374), the paper's accuracy check; ``dec`` may then also be a
  Graph (original node order).

Steps = ceil(T/dt); the last step is truncated to land exactly on T
(SPEC.md:519).  Phases are wrapped to (-pi, pi] after every full step
(SPEC.md:428,552); a non-finite state raises BlowUpError(step).
Records every ``record_every``-th state plus the initial and final state
(SPEC.md:518,531).

``Trajectory`` carries what SPEC.md:522-525 asks for besides the states:
per-step device wall time (``step_seconds``: CUDA events around every
recording chunk, the chunk's time spread evenly over its steps — one chunk is
one persistent launch) and the coupling-kernel evaluation count
(``kernel_evals``, the machine-independent complexity witness of
SPEC.md:585-591: per CIA RHS one mean-field evaluation per community node plus
one exact coupling per directed sparse correction [plus one per triangle
incidence for the triadic model]; per naive RHS one per directed edge [plus
6 per triangle]).  ``to_csv`` writes the long-form export of SPEC.md:560.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import InputError
from .evaluator import engine_for
from .graph import Decomposition, Graph


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
    states: np.ndarray  # [n_records, N] (or [n_records, N, 4]) original node order
    wall_seconds: float = 0.0
    kernel_launches: int = 0
    meta: dict = field(default_factory=dict)
    step_seconds: np.ndarray = field(default_factory=lambda: np.zeros(0))
    kernel_evals: int = 0

    @property
    def final(self) -> np.ndarray:
        return self.states[-1]

    def to_csv(self, path: str) -> None:
        """Long-form export ``t,node,component,value`` followed by
        a summary block ``step,seconds`` (per-step timings) and the totals."""
        st = self.states if self.states.ndim == 3 else self.states[:, :, None]
        n_rec, n, d = st.shape
        with open(path, "w") as f:
            f.write("t,node,component,value\n")
            node = np.repeat(np.arange(n), d)
            comp = np.tile(np.arange(d), n)
            for r in range(n_rec):
                vals = st[r].reshape(-1)
                f.writelines(f"{float(self.times[r])!r},{a},{b},{v!r}\n"
                             for a, b, v in zip(node.tolist(), comp.tolist(), vals.tolist()))
            f.write("\nstep,seconds\n")
            f.writelines(f"{k + 1},{s!r}\n" for k, s in enumerate(self.step_seconds.tolist()))
            f.write(f"\ntotal_wall_seconds,{self.wall_seconds!r}\n"
                    f"kernel_evals,{self.kernel_evals}\n")


def cia_kernel_evals_per_rhs(model, dec: Decomposition) -> int:
    """Coupling-kernel evaluations of one CIA RHS (see the module docstring)."""
    from .ho import HigherOrderKuramoto

    n = int(dec.partition.offsets[-1]) + int(dec.nnz_dir)
    if isinstance(model, HigherOrderKuramoto):
        from .evaluator import _ho_engine

        n += int(_ho_engine(model, dec).graph.tri_pairs)
    return n


_WARMED = set()  # readback sizes with a spare pinned block on the free list


def _to_host(snaps, first=None) -> np.ndarray:
    """Stack the recorded device states into one pinned host buffer (async
    copies, one synchronisation) and return it as the trajectory's array;
    ``first`` (a host array) becomes record 0.  The pinned block comes from
    torch's caching host allocator: once an earlier trajectory has been
    dropped the allocation is a free-list hit, and handing the buffer itself
    to the caller saves a pageable copy of every record."""
    import torch

    k0 = 0 if first is None else 1
    shape = (len(snaps) + k0,) + tuple(snaps[0].shape if snaps else np.shape(first))
    dtype = snaps[0].dtype if snaps else torch.float64
    buf = torch.empty(shape, dtype=dtype, pin_memory=True)
    nbytes = buf.numel() * buf.element_size()
    if nbytes not in _WARMED and nbytes <= 64 << 20:
        # a caller usually still holds the previous trajectory while the next
        # one is computed: leave one spare block of this size on the
        # allocator's free list so the second call does not pin fresh memory
        _WARMED.add(nbytes)
        del_me = torch.empty(shape, dtype=dtype, pin_memory=True)
        del del_me
    for k, sn in enumerate(snaps):
        buf[k + k0].copy_(sn, non_blocking=True)
    out = buf.numpy()
    if first is not None:
        out[0] = first  # host copy while the device copies are in flight
    torch.cuda.current_stream().synchronize()
    return out


class _ChunkTimer:
    """CUDA events around each recording chunk (one persistent launch)."""

    def __init__(self):
        import torch

        self.torch = torch
        self.ev = []

    def start(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def stop(self, e0, steps: int):
        e1 = self.torch.cuda.Event(enable_timing=True)
        e1.record()
        self.ev.append((e0, e1, steps))

    def per_step(self) -> np.ndarray:
        self.torch.cuda.synchronize()
        out = []
        for e0, e1, k in self.ev:
            out.extend([e0.elapsed_time(e1) / 1e3 / k] * k)
        return np.asarray(out)


def integrate(model, dec, x0, plan: IntegrationPlan) -> Trajectory:
    if plan.scheme not in ("rk4", "euler"):
        raise InputError(f"unknown scheme {plan.scheme!r}")
    x0 = np.asarray(x0, dtype=np.float64)
    if plan.mode == "naive":
        return _integrate_naive(model, dec, x0, plan)
    if plan.mode != "cia":
        raise InputError(f"unknown rhs mode {plan.mode!r} (cia | naive)")
    if not isinstance(dec, Decomposition):
        raise InputError("mode='cia' needs a Decomposition")
    from .cs import CuckerSmale

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
    fast = hasattr(eng, "upload_permuted")  # classical engine: permutations on the device
    if fast:
        from .evaluator import perm_device

        p_dev, inv_dev = perm_device(dec)
        eng.upload_permuted(eng.theta, x0, p_dev)
        eng.prepare()
    else:
        eng.set_state(x0[perm])
    stride = plan.record_every if plan.record_every > 0 else n_steps
    advance = eng.rk4 if plan.scheme == "rk4" else eng.euler
    timer = _ChunkTimer()

    times = [0.0]
    snaps = [] if fast else [eng.theta.clone()]  # fast: the initial record is x0 itself
    done = 0
    while done < n_steps:
        chunk = min(stride, n_steps - done)
        # the last step has its own size unless T is a multiple of dt (then
        # the whole chunk is one persistent launch)
        short_last = done + chunk == n_steps and dt_last != dt
        full = chunk - 1 if short_last else chunk
        e0 = timer.start()
        if full > 0:
            advance(dt, full)
        if short_last:
            advance(dt_last, 1)
        timer.stop(e0, chunk)
        done += chunk
        times.append(min(done * dt, plan.t_end) if done < n_steps else plan.t_end)
        snaps.append(eng.theta.clone())
    if fast:  # records back in original order, gathered on the device
        import torch

        states = _to_host([torch.index_select(sn, 0, inv_dev) for sn in snaps], first=x0)
    else:
        states_perm = _to_host(snaps)  # one pinned D2H of all records
        states = np.empty_like(states_perm)
        states[:, perm] = states_perm
    eng.check()
    wall = time.perf_counter() - t0
    stages = 4 if plan.scheme == "rk4" else 1
    return Trajectory(np.asarray(times), states, wall, int(lib.cdk_launch_count()) - launches0,
                      {"n_steps": n_steps, "dt": dt, "dt_last": dt_last, "mode": "cia"},
                      timer.per_step(),
                      cia_kernel_evals_per_rhs(model, dec) * stages * n_steps)


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

    timer = _ChunkTimer()
    snaps = [torch.cat([eng.pos, eng.vel], 1).clone()]
    times = [0.0]
    done = 0
    while done < n_steps:
        chunk = min(stride, n_steps - done)
        full = chunk if done + chunk < n_steps else chunk - 1
        e0 = timer.start()
        if full > 0:
            eng.rk4(dt, full)
        if done + chunk == n_steps:
            eng.rk4(dt_last, 1)
        timer.stop(e0, chunk)
        done += chunk
        times.append(min(done * dt, plan.t_end) if done < n_steps else plan.t_end)
        snaps.append(torch.cat([eng.pos, eng.vel], 1).clone())
    eng.check()
    sp = np.stack([s.cpu().numpy() for s in snaps])
    states = np.empty_like(sp)
    states[:, perm] = sp
    return Trajectory(np.asarray(times), states, time.perf_counter() - t0,
                      int(eng.lib.cdk_launch_count()) - launches0,
                      {"n_steps": n_steps, "dt": dt, "sup_err": float(eng.plan.sup_err.max()),
                       "mode": "cia"},
                      timer.per_step(), cia_kernel_evals_per_rhs(model, dec) * 4 * n_steps)


def _integrate_naive(model, dec, x0, plan: IntegrationPlan) -> Trajectory:
    """Direct-sum trajectory (naive.NaiveEngine).  ``dec``: a Graph in the
    state's (original) node order, or a Decomposition (its reconstructed graph,
    states mapped through the partition's permutation)."""
    import torch

    from .cs import CuckerSmale
    from .naive import NaiveEngine

    if isinstance(dec, Decomposition):
        graph, perm = dec.graph(), dec.partition.perm
    elif isinstance(dec, Graph):
        graph, perm = dec, None
    else:
        raise InputError("mode='naive' needs a Graph or a Decomposition")
    d = 4 if isinstance(model, CuckerSmale) else 1
    if x0.shape != ((graph.n_nodes, 4) if d == 4 else (graph.n_nodes,)):
        raise InputError("x0 shape does not match the graph")
    if d == 4 and plan.scheme != "rk4":
        raise InputError("Cucker-Smale integrates with rk4")
    if perm is not None:  # engine in the decomposition's permuted order
        from dataclasses import replace

        if d == 1:
            model = replace(model, omega=np.asarray(model.omega)[perm])
        x0 = x0[perm]
    n_steps, dt, dt_last = plan.step_sizes()
    t0 = time.perf_counter()
    eng = NaiveEngine(model, graph)
    launches0 = int(_lib.lib().cdk_launch_count())
    stride = plan.record_every if plan.record_every > 0 else n_steps
    advance = eng.rk4 if plan.scheme == "rk4" else eng.euler
    timer = _ChunkTimer()
    x = torch.as_tensor(x0, device=eng.device)
    snaps, times, done = [x.clone()], [0.0], 0
    while done < n_steps:
        chunk = min(stride, n_steps - done)
        full = chunk if done + chunk < n_steps else chunk - 1
        e0 = timer.start()
        if full > 0:
            x = advance(x, dt, full, step0=done)
        if done + chunk == n_steps:
            x = advance(x, dt_last, 1, step0=done + full)
        timer.stop(e0, chunk)
        done += chunk
        times.append(min(done * dt, plan.t_end) if done < n_steps else plan.t_end)
        snaps.append(x.clone())
    sp = np.stack([s.cpu().numpy() for s in snaps])
    if perm is not None:
        states = np.empty_like(sp)
        states[:, perm] = sp
    else:
        states = sp
    stages = 4 if plan.scheme == "rk4" else 1
    return Trajectory(np.asarray(times), states, time.perf_counter() - t0,
                      int(_lib.lib().cdk_launch_count()) - launches0,
                      {"n_steps": n_steps, "dt": dt, "dt_last": dt_last, "mode": "naive"},
                      timer.per_step(), eng.kernel_evals_per_rhs * stages * n_steps)


__all__ = ["IntegrationPlan", "Trajectory", "integrate", "_lib"]
