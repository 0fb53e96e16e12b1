"""Cucker-Smale on the GPU (csrc/cs.cu) vs the same-basis CPU restatement
(oracle/cs.py) and the direct sum (reference kernel pairs_cs)."""

import numpy as np
import pytest

from oracle import cia
from oracle import cs as ocs
from oracle import kernels as K
from paper_2203_16657_b200 import configs, cs

pytestmark = pytest.mark.gpu


def _rk4_oracle(dec, plan, pos, vel, model, n, dt, steps):
    def f(x):
        p, v = x[:, :2], x[:, 2:]
        a = ocs.cs_rhs_cia(K, p, v, dec, plan, model.K, model.sigma**2, model.beta, n)
        return np.concatenate([v, a], 1)

    x = np.concatenate([pos, vel], 1)
    out, _ = cia.rk4_integrate(f, x, dt, steps, wrap=False)
    return out[:, :2], out[:, 2:]


def test_cs_rhs_and_rk4_scaled():
    c = configs.scaled_config4()
    dec = c.decomposition()
    pos, vel = c.state()
    model = cs.CuckerSmale(c.K, c.sigma, c.beta)
    eng = cs.CSEngine(dec, model, pos, vel, t_end=c.t_end)
    _, a = eng.rhs(pos, vel)
    ac = ocs.cs_rhs_cia(K, pos, vel, dec, eng.plan, c.K, c.sigma**2, c.beta, c.n)
    assert np.abs(a.cpu().numpy() - ac).max() <= 1e-12 * max(1.0, np.abs(ac).max())
    eng.rk4(c.dt, 20)
    eng.check()
    ps, vs = _rk4_oracle(dec, eng.plan, pos, vel, model, c.n, c.dt, 20)
    assert np.abs(eng.pos.cpu().numpy() - ps).max() <= 1e-9
    assert np.abs(eng.vel.cpu().numpy() - vs).max() <= 1e-9


def test_cs_config4_full_rhs():
    c = configs.config4()
    dec = c.decomposition()
    pos, vel = c.state()
    model = cs.CuckerSmale(c.K, c.sigma, c.beta)
    eng = cs.CSEngine(dec, model, pos, vel, t_end=c.t_end)
    _, a = eng.rhs(pos, vel)
    ac = ocs.cs_rhs_cia(K, pos, vel, dec, eng.plan, c.K, c.sigma**2, c.beta, c.n)
    assert np.abs(a.cpu().numpy() - ac).max() <= 1e-11 * max(1.0, np.abs(ac).max())
    eng.rk4(c.dt, 2)
    eng.check()
    assert np.all(np.isfinite(eng.pos.cpu().numpy()))


def test_cs_domain_guard():
    from paper_2203_16657_b200.errors import DomainViolationError

    c = configs.scaled_config4(m=2, lam=40)
    dec = c.decomposition()
    pos, vel = c.state()
    model = cs.CuckerSmale(c.K, c.sigma, c.beta)
    eng = cs.CSEngine(dec, model, pos, vel, t_end=0.01)  # domain sized for a tiny horizon
    far = pos.copy()
    far[0] += 1e3
    with pytest.raises(DomainViolationError):
        eng.rhs(far, vel)


def test_cs_public_api():
    from paper_2203_16657_b200 import IntegrationPlan, eval_rhs_cia, integrate

    c = configs.scaled_config4(m=3, lam=50, seed=9)
    dec = c.decomposition()
    pos, vel = c.state()
    model = cs.CuckerSmale(c.K, c.sigma, c.beta)
    x0 = np.concatenate([pos, vel], 1)
    d = eval_rhs_cia(model, dec, x0)
    assert d.shape == (c.n, 4)
    np.testing.assert_array_equal(d[:, :2], vel)
    tr = integrate(model, dec, x0, IntegrationPlan(t_end=0.05, dt=0.01))
    assert tr.states.shape == (2, c.n, 4) and np.all(np.isfinite(tr.final))
