"""Stated-horizon trajectory parity (BASELINE north_star: max abs/circular
error <= 1e-9 "after the stated number of steps" on every config).

Fixtures: tests/golden/long_cfg*.npz, made in the build container by
tests/golden/make_long.py (the script documents which are the REAL reference
kernels and which are builder restatements):

* config 2 — full size (N = 200 000), 2000 RK4 steps, SPEC orchestration over
  the real ``commdyn._kernels`` (numba, as shipped);
* config 3 — full size (N = 50 000), 1000 RK4 steps of the CIA restatement
  ``oracle.ho.HoCia`` (pinned to the literal triangle sum and to the reference
  ``ho_naive_block`` in tests/test_ho_oracle.py);
* config 4 — full size (N = 100 000), 500 RK4 steps of the same-basis CIA
  restatement whose exact sparse correction is the real ``pairs_cs``, plus one
  direct-sum RHS (real ``pairs_cs`` over the full edge list) for the
  SPEC.md:396,635 bound;
* config 5 — a scaled generated instance (N = 60 000, communities wider than
  the shared-memory window), 200 RK4 steps over the real reference kernels;
  plus a FULL-SIZE (N = 8e6) row-subset RHS check against rows regenerated on
  the host.

Every fixture carries a sha256 of its inputs, recomputed here, so generator
drift fails loudly instead of comparing different problems.
"""

import hashlib
import math
import os

import numpy as np
import pytest

from oracle import cia
from paper_2203_16657_b200 import configs

pytestmark = pytest.mark.gpu

TRAJ_TOL = 1e-9  # BASELINE north_star, fp64


def _sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _load(golden_dir, name):
    path = os.path.join(golden_dir, name)
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {name}: run tests/golden/make_long.py in the build container")
    return np.load(path)


@pytest.mark.parametrize("ell", ["1", "0"])
def test_cfg2_2000_steps_vs_reference(golden_dir, ell, monkeypatch):
    from paper_2203_16657_b200.engine import KuramotoEngine

    monkeypatch.setenv("CDK_ELL", ell)
    g = _load(golden_dir, "long_cfg2.npz")
    c = configs.config2()
    dec = c.decomposition()
    omega, theta0 = c.state()
    s = dec.correction
    assert _sha(s.iu, s.iv, s.sgn, dec.offsets, omega, theta0) == str(g["input_sha256"])
    eng = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
    assert bool(eng.graph.struct.ell_off) == (ell == "1")
    eng.set_state(theta0)
    done = 0
    idx = g["idx"]
    for k, snap in zip(g["snap_steps"].tolist(), g["snaps"]):
        eng.rk4(c.dt, k - done)
        done = k
        eng.check()
        got = eng.theta.cpu().numpy()
        assert cia.circ_dist(got[idx], snap).max() <= TRAJ_TOL, k
    assert done == int(g["steps"]) == c.steps == 2000
    err = float(cia.circ_dist(eng.theta.cpu().numpy(), g["final"]).max())
    assert err <= TRAJ_TOL, err


def test_cfg3_1000_steps_vs_cia_restatement(golden_dir):
    from paper_2203_16657_b200 import ho

    g = _load(golden_dir, "long_cfg3.npz")
    c = configs.config3()
    dec = c.decomposition()
    omega, theta0 = c.state()
    s = dec.correction
    assert _sha(s.iu, s.iv, s.sgn, dec.offsets, omega, theta0) == str(g["input_sha256"])
    eng = ho.HOEngine(dec, omega, c.k1, c.k2)
    assert eng.graph.span_tri.shape[0] == int(g["n_span"])
    eng.set_state(theta0)
    done = 0
    idx = g["idx"]
    for k, snap in zip(g["snap_steps"].tolist(), g["snaps"]):
        eng.rk4(c.dt, k - done)
        done = k
        eng.check()
        assert cia.circ_dist(eng.theta.cpu().numpy()[idx], snap).max() <= TRAJ_TOL, k
    assert done == int(g["steps"]) == c.steps == 1000
    err = float(cia.circ_dist(eng.theta.cpu().numpy(), g["final"]).max())
    assert err <= TRAJ_TOL, err


def test_cfg4_500_steps_and_direct_sum_bound(golden_dir):
    from paper_2203_16657_b200 import cs

    g = _load(golden_dir, "long_cfg4.npz")
    c = configs.config4()
    dec = c.decomposition()
    pos, vel = c.state()
    s = dec.correction
    assert _sha(s.iu, s.iv, s.sgn, dec.offsets, pos, vel) == str(g["input_sha256"])
    model = cs.CuckerSmale(c.K, c.sigma, c.beta)
    eng = cs.CSEngine(dec, model, pos, vel, t_end=c.t_end)
    np.testing.assert_allclose(eng.plan.sup_err, g["sup_err"], rtol=0, atol=0)
    # RHS at t = 0: vs the same-basis CIA, and vs the DIRECT SUM of the real
    # reference pairs_cs within the SPEC bound C * sup_err (C = max pairwise
    # |v_l - v_m|, scaled by the largest community's share lambda/N of the
    # 1/N-normalised dense sum)
    _, a = eng.rhs(pos, vel)
    a = a.cpu().numpy()
    amax = np.abs(g["rhs0_cia"]).max()
    assert np.abs(a - g["rhs0_cia"]).max() <= 1e-11 * max(1.0, amax)
    dv = float(np.linalg.norm(vel.max(0) - vel.min(0)))
    lam = int(np.diff(dec.offsets).max())
    bound = float(g["sup_err"].max()) * dv * lam / c.n + 1e-9
    dev = float(np.abs(a - g["rhs0_direct"]).max())
    assert dev <= bound, (dev, bound)
    eng.set_state(pos, vel)
    done = 0
    idx = g["idx"]
    for k, snap in zip(g["snap_steps"].tolist(), g["snaps"]):
        eng.rk4(c.dt, k - done)
        done = k
        eng.check()
        x = np.concatenate([eng.pos.cpu().numpy(), eng.vel.cpu().numpy()], 1)
        assert np.abs(x[idx] - snap).max() <= TRAJ_TOL, k
    assert done == int(g["steps"]) == c.steps == 500
    x = np.concatenate([eng.pos.cpu().numpy(), eng.vel.cpu().numpy()], 1)
    err = float(np.abs(x - g["final"]).max())
    assert err <= TRAJ_TOL, err


CFG5_SCALED = dict(n=60000, lo=600, hi=12000, seed=55)  # = make_long.CFG5_SCALED


def test_cfg5_scaled_200_steps_vs_reference(golden_dir):
    from oracle import gen as OG
    from paper_2203_16657_b200 import gen
    from paper_2203_16657_b200.engine import KuramotoEngine

    g = _load(golden_dir, "long_cfg5.npz")
    c = gen.scaled_config5(**CFG5_SCALED)
    off, cdf, n_edges, thr = c.gen_inputs()
    _, (iu, iv, sg) = OG.generate_csr(c.graph_seed, off, cdf, n_edges, thr)
    omega, theta0 = c.state()
    assert _sha(iu, iv, sg, off, omega, theta0) == str(g["input_sha256"])
    dg, _ = gen.device_graph(c, "cuda")
    eng = KuramotoEngine(None, omega, coupling=c.coupling, norm=c.n, graph=dg)
    eng.set_state(theta0)
    done = 0
    idx = g["idx"]
    for k, snap in zip(g["snap_steps"].tolist(), g["snaps"]):
        eng.rk4(c.dt, k - done)
        done = k
        eng.check()
        assert cia.circ_dist(eng.theta.cpu().numpy()[idx], snap).max() <= TRAJ_TOL, k
    assert done == int(g["steps"]) == c.steps == 200
    err = float(cia.circ_dist(eng.theta.cpu().numpy(), g["final"]).max())
    assert err <= TRAJ_TOL, err


def test_cfg5_full_size_rhs_row_subset():
    """BASELINE-size config 5 (N = 8e6, ~1e10 corrections): the device RHS on
    sampled rows vs the CIA formula evaluated on the host from the row's
    regenerated intra pattern (counter hash, oracle/gen.py) and its inter
    columns; community sums R_c over the host state.  Bar: 1e-12 + 64 ulp(|k|)
    (omega ~ Cauchy reaches |k| ~ 1e3; the reference accumulates one rounding
    per pair)."""
    import torch

    from oracle import gen as OG
    from paper_2203_16657_b200 import gen
    from paper_2203_16657_b200.engine import KuramotoEngine

    c = gen.config5()
    off, cdf, n_edges, thr = c.gen_inputs()
    omega, theta0 = c.state()
    dg, csr = gen.device_graph(c, "cuda")
    eng = KuramotoEngine(None, omega, coupling=c.coupling, norm=c.n, graph=dg)
    k = eng.rhs(torch.from_numpy(theta0).cuda()).cpu().numpy()
    assert np.all(np.isfinite(k))
    lam = np.diff(off)
    rng = np.random.default_rng(5)
    rows = np.concatenate([rng.integers(0, c.n, 12), [0, c.n - 1]])
    xptr = csr.inter_ptr
    xcol_dev = dg._t["inter_col"]
    z = np.exp(1j * theta0)
    scale = c.coupling / c.n
    for i in rows.tolist():
        cc = int(np.searchsorted(off, i, side="right") - 1)
        a = i - off[cc]
        b = np.arange(lam[cc], dtype=np.uint32)
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        h = OG.hash4(c.graph_seed, np.full_like(b, cc), lo.astype(np.uint32), hi.astype(np.uint32))
        miss = off[cc] + np.nonzero((h < np.uint32(thr)) & (b != a))[0]
        xc = xcol_dev[int(xptr[i]): int(xptr[i + 1])].cpu().numpy().astype(np.int64)
        xc = xc[xc >= 0]
        rc = z[off[cc]: off[cc + 1]].sum()
        coup = ((rc * np.conj(z[i])).imag - np.sin(theta0[miss] - theta0[i]).sum()
                + np.sin(theta0[xc] - theta0[i]).sum())
        want = omega[i] + scale * coup
        tol = 1e-12 + 64 * 2.2e-16 * abs(want)
        assert abs(k[i] - want) <= tol, (i, k[i], want)
    # size-independent property: the coupling is odd, so sum k = sum omega up to
    # rounding of 8e6 terms of |omega| (Cauchy tails)
    assert abs(math.fsum(k) - math.fsum(omega)) <= 1e-9 * np.abs(omega).sum()
    del eng, dg, csr
    torch.cuda.empty_cache()
