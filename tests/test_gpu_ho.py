"""Higher-order (triadic) Kuramoto on the GPU (csrc/ho.cu) vs the CPU oracle
(CIA restatement and literal triangle sum, oracle/ho.py)."""

import math

import numpy as np
import pytest

from oracle import cia
from oracle import ho as oh
from paper_2203_16657_b200 import configs
from paper_2203_16657_b200 import graph as G
from paper_2203_16657_b200 import ho

pytestmark = pytest.mark.gpu


def _engine(dec, omega, k1, k2, norm=None):
    return ho.HOEngine(dec, omega, k1, k2, norm=norm)


@pytest.mark.parametrize("seed,pool", [(0, 0), (3, 15)])
def test_ho_rhs_vs_triangle_sum(seed, pool):
    import torch

    rng = np.random.default_rng(seed)
    g, part = G.planted_partition_graph([40, 25, 60, 3, 1], 0.8, 0.06, seed)
    if pool:
        a = part.assignment.copy()
        a[rng.choice(a.shape[0], pool, replace=False)] = -1
        used = np.unique(a[a >= 0])
        remap = -np.ones(a.max() + 2, dtype=np.int64)
        remap[used] = np.arange(used.size)
        part = G.Partition.from_assignment(np.where(a >= 0, remap[a], -1))
    dec = G.decompose(g, part)
    A = g.dense()[np.ix_(part.perm, part.perm)]
    th = rng.uniform(-math.pi, math.pi, g.n_nodes)
    om = rng.standard_normal(g.n_nodes)
    kd = oh.ho_rhs_direct(th, om, A, 1.0, 0.5)
    eng = _engine(dec, om, 1.0, 0.5)
    k = eng.rhs(torch.from_numpy(th)).cpu().numpy()
    assert np.abs(k - kd).max() <= 1e-12


def test_ho_trajectory_scaled_config3():
    c = configs.scaled_config3(m=6, lam=100, p_out=3e-3)
    dec = c.decomposition()
    omega, theta0 = c.state()
    span = ho.spanning_triangles(dec)
    eng = _engine(dec, omega, c.k1, c.k2)
    eng.set_state(theta0)
    eng.rk4(c.dt, 40)
    eng.check()

    def rhs(x):
        return oh.ho_rhs_cia(x, omega, dec, c.k1, c.k2, inter_triangles=span)

    ref, _ = cia.rk4_integrate(rhs, theta0, c.dt, 40)
    assert cia.circ_dist(eng.theta.cpu().numpy(), ref).max() <= 1e-9


def test_ho_config3_full_rhs_and_steps():
    import torch

    c = configs.config3()
    dec = c.decomposition()
    omega, theta0 = c.state()
    eng = _engine(dec, omega, c.k1, c.k2)
    span = eng.graph.span_tri
    k = eng.rhs(torch.from_numpy(theta0)).cpu().numpy()
    kc = oh.ho_rhs_cia(theta0, omega, dec, c.k1, c.k2, inter_triangles=span)
    assert np.abs(k - kc).max() <= 1e-12
    eng.set_state(theta0)
    eng.rk4(c.dt, 2)
    eng.check()

    def rhs(x):
        return oh.ho_rhs_cia(x, omega, dec, c.k1, c.k2, inter_triangles=span)

    ref, _ = cia.rk4_integrate(rhs, theta0, c.dt, 2)
    assert cia.circ_dist(eng.theta.cpu().numpy(), ref).max() <= 1e-9
    # determinism
    eng.set_state(theta0)
    eng.rk4(c.dt, 2)
    th1 = eng.theta.cpu().numpy()
    eng.set_state(theta0)
    eng.rk4(c.dt, 2)
    assert np.array_equal(th1, eng.theta.cpu().numpy())


def test_ho_public_api():
    from paper_2203_16657_b200 import IntegrationPlan, eval_rhs_cia, integrate
    from paper_2203_16657_b200.ho import ho_kuramoto_model

    c = configs.scaled_config3(m=4, lam=80, p_out=4e-3, seed=77)
    dec = c.decomposition()
    omega, theta0 = c.state()
    model = ho_kuramoto_model(omega, c.k1, c.k2)
    span = ho.spanning_triangles(dec)
    k = eval_rhs_cia(model, dec, theta0)
    kc = oh.ho_rhs_cia(theta0, omega, dec, c.k1, c.k2, inter_triangles=span)
    assert np.abs(k - kc).max() <= 1e-12
    tr = integrate(model, dec, theta0, IntegrationPlan(t_end=10 * c.dt, dt=c.dt))
    assert tr.states.shape == (2, c.n)
