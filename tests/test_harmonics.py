"""Higher-harmonics Kuramoto: p = 4
random coefficients on a planted graph with a NONE pool.  The fixture
tests/golden/harmonics.npz comes from the REAL reference kernels
(order_params_blocks / dense_complex / pairs_trig with 4 harmonics, composed
by oracle/cia.harmonics_rhs_cia; make_golden.py harmonics).

CPU: the oracle C port against the fixture.  GPU (csrc/harmonics.cu through
the C ABI): the fused CIA RHS (1e-12), 200 fused RK4 steps (1e-9), the
direct-sum mode, the p = 1 reduction to the classical engine, the public API
and the host fitter feeding the fused path."""

import math
import os

import numpy as np
import pytest

from oracle import cia
from oracle import kernels as K
from paper_2203_16657_b200 import graph as G


@pytest.fixture(scope="module")
def hh(golden_dir):
    f = dict(np.load(os.path.join(golden_dir, "harmonics.npz")))
    g, part = G.planted_partition_graph([125, 125, 125, 125], 0.9, 0.01, 44)
    part = G.Partition.from_assignment(f["assignment"])
    dec = G.decompose(g, part)
    s = dec.correction
    import hashlib

    h = hashlib.sha256()
    for a in (s.iu, s.iv, s.sgn, dec.offsets):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(f["dec_sha256"])
    return f, g, dec


def test_oracle_harmonics_vs_reference(hh):
    f, g, dec = hh
    s = dec.correction
    perm = dec.partition.perm
    om, th = f["omega"][perm], f["theta0"][perm]

    def rhs(x):
        return cia.harmonics_rhs_cia(K, x, om, dec.offsets, s.iu, s.iv, s.sgn, f["d_cos"],
                                     f["d_sin"], g.n_nodes)

    assert np.abs(rhs(th) - f["rhs_cia"]).max() <= 1e-13
    fin, _ = cia.rk4_integrate(rhs, th, float(f["dt"]), int(f["steps"]))
    assert cia.circ_dist(fin, f["final"]).max() <= 1e-12


@pytest.mark.gpu
def test_fused_rhs_and_rk4_vs_reference(hh):
    from paper_2203_16657_b200.harmonics import HhEngine

    f, g, dec = hh
    perm = dec.partition.perm
    eng = HhEngine(dec, f["omega"][perm], f["d_cos"], f["d_sin"])
    k = eng.rhs(f["theta0"][perm]).cpu().numpy()
    scale = max(1.0, float(np.abs(f["rhs_cia"]).max()))
    assert np.abs(k - f["rhs_cia"]).max() <= 1e-12 * scale
    assert np.abs(k - f["rhs_naive"]).max() <= 1e-12 * scale
    eng.set_state(f["theta0"][perm])
    eng.rk4(float(f["dt"]), int(f["steps"]))
    eng.check()
    assert cia.circ_dist(eng.theta.cpu().numpy(), f["final"]).max() <= 1e-9
    # determinism
    th1 = eng.theta.cpu().numpy()
    eng.set_state(f["theta0"][perm])
    eng.rk4(float(f["dt"]), int(f["steps"]))
    assert np.array_equal(th1, eng.theta.cpu().numpy())


@pytest.mark.gpu
def test_public_api_cia_and_naive(hh):
    from paper_2203_16657_b200 import IntegrationPlan, eval_rhs_cia, eval_rhs_naive, integrate
    from paper_2203_16657_b200.harmonics import higher_harmonics_model

    f, g, dec = hh
    perm = dec.partition.perm
    model = higher_harmonics_model(f["omega"], f["d_cos"], f["d_sin"])
    kc = eval_rhs_cia(model, dec, f["theta0"])
    kn = eval_rhs_naive(model, g, f["theta0"])
    want = np.empty_like(kc)
    want[perm] = f["rhs_cia"]
    assert np.abs(kc - want).max() <= 1e-11
    assert np.abs(kn - want).max() <= 1e-11
    tr = integrate(model, dec, f["theta0"], IntegrationPlan(2.0, 0.01, record_every=100))
    fin = np.empty_like(tr.final)
    fin[:] = tr.final
    assert cia.circ_dist(fin[perm], f["final"]).max() <= 1e-9
    assert tr.states.shape == (3, g.n_nodes) and tr.kernel_evals > 0


@pytest.mark.gpu
def test_p1_reduces_to_classical_and_fitted_coupling():
    from paper_2203_16657_b200 import configs
    from paper_2203_16657_b200.engine import KuramotoEngine
    from paper_2203_16657_b200.harmonics import HhEngine, harmonics_model_from_coupling

    c = configs.config1()
    dec = c.decomposition()
    omega, theta0 = c.state()
    hh = HhEngine(dec, omega, np.array([0.0, 0.0]), np.array([0.0, c.coupling]), norm=c.n)
    ku = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
    import torch

    k1 = hh.rhs(theta0).cpu().numpy()
    k2 = ku.rhs(torch.from_numpy(theta0).cuda()).cpu().numpy()
    assert np.abs(k1 - k2).max() <= 1e-12
    # an arbitrary coupling through the host fitter: exact for trig polynomials
    h = lambda x: 2.0 * np.sin(x) - 0.7 * np.cos(3 * x) + 0.25  # noqa: E731
    model = harmonics_model_from_coupling(omega, h, 3, norm=c.n)
    eng = HhEngine(dec, omega, model.d_cos, model.d_sin, norm=c.n)
    s = dec.correction
    want = cia.harmonics_rhs_cia(K, theta0, omega, dec.offsets, s.iu, s.iv, s.sgn, model.d_cos,
                                 model.d_sin, c.n)
    assert np.abs(eng.rhs(theta0).cpu().numpy() - want).max() <= 1e-12
