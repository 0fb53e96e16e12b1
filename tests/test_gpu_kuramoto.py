"""Fused CIA Kuramoto path (RHS + RK4 stage kernels) vs the oracle and the
golden fixtures of the real reference.  Bar: RHS within 1e-13 abs, trajectories
within 1e-9 max circular error (BASELINE north_star tolerance)."""

import math
import os

import numpy as np
import pytest

from oracle import cia
from oracle import kernels as K
from paper_2203_16657_b200 import configs
from paper_2203_16657_b200 import graph as G

pytestmark = pytest.mark.gpu

TRAJ_TOL = 1e-9
RHS_TOL = 1e-13


def _engine(dec, omega, coupling, norm, **kw):
    from paper_2203_16657_b200.engine import KuramotoEngine

    return KuramotoEngine(dec, omega, coupling=coupling, norm=norm, **kw)


def _oracle_rhs(dec, omega, coupling, norm):
    s = dec.correction

    def rhs(x):
        return cia.kuramoto_rhs_cia(K, x, omega, dec.offsets, s.iu, s.iv, s.sgn, coupling, norm)
    return rhs


@pytest.fixture(params=["ell", "legacy"])
def kernel_path(request, monkeypatch):
    """Both stage-kernel families: the lane-per-row ELL kernels (default for
    graphs without the inter sweep) and the row-group kernels (CDK_ELL=0)."""
    monkeypatch.setenv("CDK_ELL", "1" if request.param == "ell" else "0")
    return request.param


def _assert_path(eng, path):
    assert bool(eng.graph.struct.ell_off) == (path == "ell")


@pytest.fixture(scope="module")
def cfg1():
    c = configs.config1()
    dec = c.decomposition()
    omega, theta0 = c.state()
    return c, dec, omega, theta0


def test_cfg1_rhs_vs_golden(cfg1, golden_dir):
    import torch

    c, dec, omega, theta0 = cfg1
    g = np.load(os.path.join(golden_dir, "cfg1.npz"))
    eng = _engine(dec, omega, c.coupling, c.n)
    k = eng.rhs(torch.from_numpy(theta0).cuda()).cpu().numpy()
    assert np.abs(k - g["rhs0_cia"]).max() <= RHS_TOL
    assert np.abs(k - g["rhs0_naive"]).max() <= 1e-12


def test_cfg1_trajectory_vs_golden(cfg1, golden_dir, kernel_path):
    c, dec, omega, theta0 = cfg1
    g = np.load(os.path.join(golden_dir, "cfg1.npz"))
    eng = _engine(dec, omega, c.coupling, c.n)
    _assert_path(eng, kernel_path)
    eng.set_state(theta0)
    snaps = []
    for _ in range(c.steps // 100):
        eng.rk4(c.dt, 100)
        snaps.append(eng.theta.cpu().numpy())
    eng.check()
    fin = snaps[-1]
    e_cia = cia.circ_dist(fin, g["final_cia"]).max()
    e_naive = cia.circ_dist(fin, g["final_naive"]).max()
    print(f"cfg1 1000 steps: vs reference CIA {e_cia:.3e}, vs direct sum {e_naive:.3e}")
    assert e_cia <= TRAJ_TOL and e_naive <= TRAJ_TOL
    for x, gx in zip(snaps, g["snaps"]):
        assert cia.circ_dist(x, gx).max() <= TRAJ_TOL
    assert np.all(fin > -math.pi) and np.all(fin <= math.pi)


def test_public_integrate_api(cfg1, golden_dir):
    from paper_2203_16657_b200 import IntegrationPlan, integrate, kuramoto_model

    c, dec, omega, theta0 = cfg1
    g = np.load(os.path.join(golden_dir, "cfg1.npz"))
    model = kuramoto_model(omega, c.coupling, c.n)
    tr = integrate(model, dec, theta0, IntegrationPlan(t_end=c.steps * c.dt, dt=c.dt,
                                                         record_every=100))
    assert tr.states.shape == (c.steps // 100 + 1, c.n)
    assert cia.circ_dist(tr.final, g["final_cia"]).max() <= TRAJ_TOL
    assert tr.kernel_launches >= 1  # persistent RK4 kernel: one launch per recorded chunk


def test_trajectories_do_not_alias(cfg1):
    """integrate() hands its pinned readback buffer to the caller: a later
    call (same shapes, other data) must leave an earlier trajectory intact,
    a chunk whose last step keeps dt is one launch, and a short last step
    still lands on t_end."""
    from paper_2203_16657_b200 import IntegrationPlan, integrate, kuramoto_model

    c, dec, omega, theta0 = cfg1
    model = kuramoto_model(omega, c.coupling, c.n)
    plan = IntegrationPlan(t_end=30 * c.dt, dt=c.dt, record_every=10)
    tr1 = integrate(model, dec, theta0, plan)
    keep = tr1.states.copy()
    assert np.array_equal(tr1.states[0], theta0) and tr1.states.shape == (4, c.n)
    tr2 = integrate(model, dec, theta0 + 0.25, plan)
    tr3 = integrate(model, dec, theta0 - 0.25, plan)
    assert np.array_equal(tr1.states, keep)
    assert not np.array_equal(tr2.states[-1], tr1.states[-1])
    assert not np.array_equal(tr3.states[-1], tr2.states[-1])
    # T not a multiple of dt: the last step is shorter and has its own launch
    tr4 = integrate(model, dec, theta0, IntegrationPlan(t_end=29.5 * c.dt, dt=c.dt))
    assert tr4.times[-1] == pytest.approx(29.5 * c.dt) and tr4.meta["n_steps"] == 30
    ref, _ = cia.rk4_integrate(_oracle_rhs(dec, omega, c.coupling, c.n), theta0, c.dt, 29)
    ref, _ = cia.rk4_integrate(_oracle_rhs(dec, omega, c.coupling, c.n), ref, 0.5 * c.dt, 1)
    assert cia.circ_dist(tr4.final, ref).max() <= TRAJ_TOL


def _random_case(seed, sizes, p_in, p_out, pool=0):
    rng = np.random.default_rng(seed)
    g, part = G.planted_partition_graph(sizes, p_in, p_out, seed)
    if pool:
        # move `pool` random nodes of the planted partition into the NONE pool
        a = part.assignment.copy()
        a[rng.choice(a.shape[0], pool, replace=False)] = -1
        used = np.unique(a[a >= 0])
        remap = -np.ones(a.max() + 2, dtype=np.int64)
        remap[used] = np.arange(used.size)
        a = np.where(a >= 0, remap[a], -1)
        part = G.Partition.from_assignment(a)
    dec = G.decompose(g, part)
    n = g.n_nodes
    omega = rng.standard_normal(n)
    theta = rng.uniform(-math.pi, math.pi, n)
    return g, dec, omega, theta


@pytest.mark.parametrize("case", [
    dict(seed=1, sizes=[40, 3, 1, 77, 200], p_in=0.9, p_out=0.05, pool=0),
    dict(seed=2, sizes=[60, 60, 60], p_in=0.7, p_out=0.1, pool=25),   # NONE pool
    dict(seed=3, sizes=[1, 1, 1, 2], p_in=1.0, p_out=0.5, pool=0),    # tiny communities
    dict(seed=4, sizes=[300], p_in=1.0, p_out=0.0, pool=0),            # empty S
    dict(seed=5, sizes=[33, 31, 32, 64, 65], p_in=0.2, p_out=0.3, pool=7),  # ragged rblocks
])
def test_rhs_edge_cases_vs_oracle_and_naive(case, kernel_path):
    import torch

    g, dec, omega_o, theta_o = _random_case(**case)
    perm = dec.partition.perm
    omega, theta = omega_o[perm], theta_o[perm]
    n = g.n_nodes
    eng = _engine(dec, omega, 2.5, n)
    k = eng.rhs(torch.from_numpy(theta).cuda()).cpu().numpy()
    k_or = _oracle_rhs(dec, omega, 2.5, n)(theta)
    assert np.abs(k - k_or).max() <= RHS_TOL
    # direct sum on the original graph
    kn = cia.kuramoto_rhs_dense(theta_o, omega_o, g.dense().astype(float), 2.5, n)
    assert np.abs(k - kn[perm]).max() <= 1e-12


def test_unstaged_large_community(kernel_path):
    """A community above the shared-memory cap gathers from global memory."""
    import torch

    from paper_2203_16657_b200 import plan as PL

    sizes = [15000, 500]
    dec = G.planted_partition_decomposition(sizes, 0.998, 1e-4, 11)
    lay = PL.build_layout(dec)
    sch = PL.build_schedule(lay)
    assert sch.smem_nodes < 15000
    rng = np.random.default_rng(0)
    n = dec.n_nodes
    omega = rng.standard_normal(n)
    theta = rng.uniform(-math.pi, math.pi, n)
    eng = _engine(dec, omega, 5.0, n)
    _assert_path(eng, kernel_path)
    k = eng.rhs(torch.from_numpy(theta).cuda()).cpu().numpy()
    k_or = _oracle_rhs(dec, omega, 5.0, n)(theta)
    assert np.abs(k - k_or).max() <= RHS_TOL


def test_schedule_independent_bitwise(cfg1, kernel_path):
    """Row-owned fixed-order accumulation: results are bitwise identical for
    any CTA schedule (the property the multi-GPU partition relies on)."""
    import torch

    from paper_2203_16657_b200 import plan as PL

    c, dec, omega, theta0 = cfg1
    outs = []
    for sm in (148, 7, 1):
        g = PL.DeviceGraph(dec, sm_count=sm)
        eng = _engine(dec, omega, c.coupling, c.n, graph=g)
        eng.set_state(theta0)
        eng.rk4(c.dt, 50)
        outs.append(eng.theta.cpu().numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_euler_and_blowup(cfg1, kernel_path):
    c, dec, omega, theta0 = cfg1
    eng = _engine(dec, omega, c.coupling, c.n)
    eng.set_state(theta0)
    eng.euler(c.dt, 7)
    eng.check()
    x = theta0.copy()
    rhs = _oracle_rhs(dec, omega, c.coupling, c.n)
    x = cia.euler_integrate(rhs, x, c.dt, 7)
    assert cia.circ_dist(eng.theta.cpu().numpy(), x).max() <= 1e-12
    # blow-up: a non-finite frequency poisons node 3 at the first step
    from paper_2203_16657_b200.errors import BlowUpError

    om = omega.copy()
    om[3] = np.inf
    eng2 = _engine(dec, om, c.coupling, c.n)
    eng2.set_state(theta0)
    eng2.rk4(c.dt, 5)
    with pytest.raises(BlowUpError) as ei:
        eng2.check()
    assert ei.value.step == 1


def test_cfg2_rhs_and_steps_vs_golden(golden_dir, kernel_path):
    import torch

    g = np.load(os.path.join(golden_dir, "cfg2_sample.npz"))
    c = configs.config2()
    dec = c.decomposition()
    omega, theta0 = c.state()
    eng = _engine(dec, omega, c.coupling, c.n)
    _assert_path(eng, kernel_path)
    k = eng.rhs(torch.from_numpy(theta0).cuda()).cpu().numpy()
    idx = g["idx"]
    assert np.abs(k[idx] - g["rhs0"]).max() <= RHS_TOL
    assert abs(k.sum() - float(g["rhs0_sum"])) <= 1e-8
    # size-independent property: sum of the coupling terms vanishes (odd h)
    assert abs(k.sum() - omega.sum()) <= 1e-8
    eng.set_state(theta0)
    eng.rk4(c.dt, int(g["steps"]))
    eng.check()
    fin = eng.theta.cpu().numpy()
    assert cia.circ_dist(fin[idx], g["final"]).max() <= TRAJ_TOL
    assert abs(np.cos(fin).sum() - float(g["final_cos_sum"])) <= 1e-8
    # determinism: a second run is bitwise identical
    eng.set_state(theta0)
    eng.rk4(c.dt, int(g["steps"]))
    assert np.array_equal(fin, eng.theta.cpu().numpy())


def test_calibrated_cuts_bitwise(monkeypatch):
    """The measured re-cut of the ELL CTA ranges moves rblocks between CTAs
    only: trajectories are bitwise equal with and without it."""
    c = configs.scaled_config2(20000, 24, seed=5)
    dec = c.decomposition()
    omega, theta0 = c.state()
    outs = []
    for cal in ("0", "3"):
        monkeypatch.setenv("CDK_ELL_CALIBRATE", cal)
        eng = _engine(dec, omega, c.coupling, c.n)
        assert bool(eng.graph.struct.ell_off)
        assert hasattr(eng.graph, "calibration") == (cal != "0")
        eng.set_state(theta0)
        eng.rk4(c.dt, 10)
        eng.check()
        outs.append(eng.theta.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
