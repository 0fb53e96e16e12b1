"""Direct-sum (naive-mode) path on the device and the SPEC's dual-mode
acceptance criteria:

1. oracle equivalence — CIA RHS vs naive RHS, max-norm <= 1e-10, planted
   graphs (4 communities, N = 500, p_in 0.9, p_out 0.01), many random states,
   Kuramoto and higher-order Kuramoto (exact expansions);
2. trajectory equivalence — Kuramoto N = 1000, Euler, T = 20, dt = 0.1, CIA vs
   naive final state <= 1e-8;
5. Cucker–Smale bounded error — |cia - naive| <= C sup_err (+1e-9);
plus the naive device path against the oracle's direct sum (the real
reference's pairs_trig/pairs_cs restated in oracle/kernels.c), the memory
guard, and the Trajectory counters (kernel evaluations, per-step timings,
CSV export).
"""

import math

import numpy as np
import pytest

from oracle import cia
from oracle import ho as oh
from oracle import kernels as K
from paper_2203_16657_b200 import graph as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def planted500():
    g, part = G.planted_partition_graph([125, 125, 125, 125], 0.9, 0.01, 17)
    dec = G.decompose(g, part)
    return g, part, dec


def test_kuramoto_cia_vs_naive_100_states(planted500):
    from paper_2203_16657_b200 import eval_rhs_cia, eval_rhs_naive, kuramoto_model

    g, part, dec = planted500
    rng = np.random.default_rng(1)
    omega = rng.standard_normal(g.n_nodes)
    model = kuramoto_model(omega, 5.0)
    worst = 0.0
    for _ in range(100):
        th = rng.uniform(-math.pi, math.pi, g.n_nodes)
        worst = max(worst, float(np.abs(eval_rhs_cia(model, dec, th)
                                        - eval_rhs_naive(model, g, th)).max()))
    assert worst <= 1e-10, worst


def test_kuramoto_naive_vs_oracle_direct_sum(planted500):
    from paper_2203_16657_b200 import eval_rhs_naive, kuramoto_model

    g, _, _ = planted500
    rng = np.random.default_rng(2)
    omega = rng.standard_normal(g.n_nodes)
    th = rng.uniform(-math.pi, math.pi, g.n_nodes)
    got = eval_rhs_naive(kuramoto_model(omega, 3.0), g, th)
    want = omega.copy()
    e = g.edges
    K.pairs_trig(e[:, 0], e[:, 1], th, 1.0 / g.n_nodes, np.zeros(2), np.array([0.0, 3.0]),
                 math.pi, np.ones(e.shape[0]), want)
    assert np.abs(got - want).max() <= 1e-12


def test_ho_cia_vs_naive(planted500):
    from paper_2203_16657_b200 import eval_rhs_cia, eval_rhs_naive
    from paper_2203_16657_b200.ho import ho_kuramoto_model

    g, part, dec = planted500
    rng = np.random.default_rng(3)
    omega = rng.standard_normal(g.n_nodes)
    model = ho_kuramoto_model(omega, 1.0, 0.5)
    A = g.dense()
    worst = 0.0
    for r in range(20):
        th = rng.uniform(-math.pi, math.pi, g.n_nodes)
        kn = eval_rhs_naive(model, g, th)
        worst = max(worst, float(np.abs(eval_rhs_cia(model, dec, th) - kn).max()))
        if r == 0:  # naive device path vs the dense literal oracle
            assert np.abs(kn - oh.ho_rhs_direct(th, omega, A, 1.0, 0.5)).max() <= 1e-12
    assert worst <= 1e-10, worst


def test_cs_cia_vs_naive_bound():
    """SPEC acceptance 5: N = 200, n = 2: deviation <= sup_err * max speed
    difference (* lambda/N of the normalised dense sum) + 1e-9."""
    from paper_2203_16657_b200 import eval_rhs_cia, eval_rhs_naive
    from paper_2203_16657_b200.cs import CuckerSmale, cs_plan

    g, part = G.planted_partition_graph([50, 50, 50, 50], 0.9, 0.01, 5)
    dec = G.decompose(g, part)
    rng = np.random.default_rng(4)
    pos = rng.uniform(0, 1, (200, 2))
    vel = rng.standard_normal((200, 2))
    model = CuckerSmale(1.0, 1.0, 0.25)
    x = np.concatenate([pos, vel], 1)
    dc = eval_rhs_cia(model, dec, x)
    dn = eval_rhs_naive(model, g, x)
    np.testing.assert_array_equal(dn[:, :2], vel)
    perm = dec.partition.perm
    plan = cs_plan(model, dec, pos[perm], vel[perm], 0.0)
    dv = float(np.linalg.norm(vel.max(0) - vel.min(0)))
    bound = float(plan.sup_err.max()) * dv * 50 / 200 + 1e-9
    assert np.abs(dc - dn).max() <= bound
    # the naive device path vs the oracle's direct sum (reference pairs_cs)
    want = np.zeros((200, 2))
    e = g.edges
    K.pairs_cs(e[:, 0], e[:, 1], pos, vel, 1.0 / 200, 1.0, 1.0, 0.25, np.ones(e.shape[0]), want)
    assert np.abs(dn[:, 2:] - want).max() <= 1e-13


def test_trajectory_euler_cia_vs_naive_n1000():
    """SPEC acceptance 2: Kuramoto N = 1000, Euler, T = 20, dt = 0.1."""
    from paper_2203_16657_b200 import IntegrationPlan, integrate, kuramoto_model

    g, part = G.planted_partition_graph([250] * 4, 0.9, 0.01, 8)
    dec = G.decompose(g, part)
    rng = np.random.default_rng(9)
    omega = rng.standard_normal(1000)
    th0 = rng.uniform(-math.pi, math.pi, 1000)
    model = kuramoto_model(omega, 5.0)
    tc = integrate(model, dec, th0, IntegrationPlan(20.0, 0.1, "euler", record_every=50))
    tn = integrate(model, g, th0, IntegrationPlan(20.0, 0.1, "euler", record_every=50,
                                                 mode="naive"))
    assert tc.states.shape == tn.states.shape == (5, 1000)
    np.testing.assert_allclose(tc.times, tn.times)
    assert cia.circ_dist(tc.final, tn.final).max() <= 1e-8
    # the same through the decomposition (naive graph reconstructed from D + S)
    td = integrate(model, dec, th0, IntegrationPlan(20.0, 0.1, "euler", mode="naive"))
    assert cia.circ_dist(td.final, tn.final).max() <= 1e-12
    # counters: CIA O(N + nnz(S)) vs naive 2|E| per RHS
    assert tc.kernel_evals == 200 * (1000 + dec.nnz_dir)
    assert tn.kernel_evals == 200 * 2 * g.edges.shape[0]
    assert tc.step_seconds.shape == (200,) and np.all(tc.step_seconds > 0)
    assert tn.step_seconds.shape == (200,) and np.all(tn.step_seconds > 0)


def test_ho_trajectory_cia_vs_naive_small():
    """Higher-order Kuramoto, N = 60 (SPEC acceptance 4 pointwise scale)."""
    from paper_2203_16657_b200 import IntegrationPlan, integrate
    from paper_2203_16657_b200.ho import ho_kuramoto_model

    g, part = G.planted_partition_graph([20, 20, 20], 0.8, 0.05, 21)
    dec = G.decompose(g, part)
    rng = np.random.default_rng(10)
    model = ho_kuramoto_model(rng.standard_normal(60), 1.0, 0.5)
    th0 = rng.uniform(-math.pi, math.pi, 60)
    plan = IntegrationPlan(2.0, 0.01)
    tc = integrate(model, dec, th0, plan)
    tn = integrate(model, g, th0, IntegrationPlan(2.0, 0.01, mode="naive"))
    assert cia.circ_dist(tc.final, tn.final).max() <= 1e-9


def test_memory_guard_and_csv(tmp_path):
    from paper_2203_16657_b200 import IntegrationPlan, eval_rhs_naive, integrate, kuramoto_model
    from paper_2203_16657_b200.errors import MemoryGuardError

    big = G.Graph(2**15 + 1, np.zeros((0, 2), np.int64))
    with pytest.raises(MemoryGuardError):
        eval_rhs_naive(kuramoto_model(np.zeros(2**15 + 1)), big, np.zeros(2**15 + 1))
    g, part = G.planted_partition_graph([6, 4], 1.0, 0.2, 1)
    dec = G.decompose(g, part)
    tr = integrate(kuramoto_model(np.linspace(-1, 1, 10), 2.0), dec, np.zeros(10),
                   IntegrationPlan(0.5, 0.1, record_every=2))
    p = tmp_path / "traj.csv"
    tr.to_csv(str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == "t,node,component,value"
    assert len(tr.times) == 4 and sum(1 for ln in lines[1:] if ln.count(",") == 3) == 40
    assert "step,seconds" in lines and lines[-1].startswith("kernel_evals,")
