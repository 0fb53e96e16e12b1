"""Config-5 device generator (csrc/gen.cu) vs its numpy restatement (bit-exact
CSR), then the fused CIA RHS / RK4 on the generated graph vs the oracle
(BASELINE configs[4]).  Bars: CSR bit-exact; RHS coupling 1e-13 abs (full RHS
1e-13 + 64 ulp(|k|), see below);
trajectories 1e-9 max circular error."""

import numpy as np
import pytest

from oracle import cia
from oracle import gen as OG
from oracle import kernels as K
from paper_2203_16657_b200 import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def case():
    c = gen.scaled_config5(n=6000, lo=60, hi=900, seed=51)
    off, cdf, n_edges, thr = c.gen_inputs()
    ref = OG.generate_csr(c.graph_seed, off, cdf, n_edges, thr)
    return c, ref


def test_device_csr_bit_exact(case):
    c, ((iptr, icol, xptr, xcol, split), _) = case
    csr = gen.generate(c, "cuda")
    dptr, dcol, dxptr, dxcol = csr.to_host()
    assert np.array_equal(csr.split_host(), split)
    assert np.array_equal(dptr, iptr)
    assert np.array_equal(dcol, icol)
    assert np.array_equal(dxptr, xptr)
    assert np.array_equal(dxcol, xcol)
    # deterministic: a second run is identical
    csr2 = gen.generate(c, "cuda")
    assert np.array_equal(csr2.to_host()[1], dcol) and np.array_equal(csr2.to_host()[3], dxcol)


def test_generated_graph_rhs_and_rk4_vs_oracle(case):
    import torch

    from paper_2203_16657_b200.engine import KuramotoEngine

    c, (_, (iu, iv, sg)) = case
    off = c.offsets()
    omega, theta0 = c.state()
    dg, _ = gen.device_graph(c, "cuda")
    eng = KuramotoEngine(None, omega, coupling=c.coupling, norm=c.n, graph=dg)
    th = torch.from_numpy(theta0).cuda()
    # coupling part alone (omega = 0): 1e-13 abs
    eng0 = KuramotoEngine(None, np.zeros_like(omega), coupling=c.coupling, norm=c.n, graph=dg)
    k0 = eng0.rhs(th).cpu().numpy()
    ko0 = cia.kuramoto_rhs_cia(K, theta0, np.zeros_like(omega), off, iu, iv, sg, c.coupling, c.n)
    assert np.abs(k0 - ko0).max() <= 1e-13
    # full RHS: omega ~ Cauchy reaches |k| ~ 1e3 and the reference accumulates
    # every pair into out[] (one rounding at ulp(|k|) per pair), so the bar is
    # 1e-13 + 64 ulp(|k|); ours is omega + coupling rounded once
    k = eng.rhs(th).cpu().numpy()
    ko = cia.kuramoto_rhs_cia(K, theta0, omega, off, iu, iv, sg, c.coupling, c.n)
    assert np.all(np.abs(k - ko) <= 1e-13 + 64 * 2.2e-16 * np.abs(ko))
    assert np.all(np.abs(k - (omega + k0)) <= 2.3e-16 * np.abs(k) + 1e-16)

    def rhs(x):
        return cia.kuramoto_rhs_cia(K, x, omega, off, iu, iv, sg, c.coupling, c.n)

    steps = 40
    ref, _ = cia.rk4_integrate(rhs, theta0, c.dt, steps)
    eng.set_state(theta0)
    eng.rk4(c.dt, steps)
    eng.check()
    err = cia.circ_dist(eng.theta.cpu().numpy(), ref).max()
    assert err <= 1e-9, err


def _small_window_case():
    c = gen.scaled_config5(n=5000, lo=100, hi=1400, seed=58)
    from paper_2203_16657_b200 import plan

    budget = plan.stage_smem_bytes(192) - 128  # 192-node window: 3 gather modes present
    return c, budget, plan.window_nodes(plan.ROWS_CAP, budget)


@pytest.mark.parametrize("blocks", ["0", "3"])
def test_multipass_generated_graph_vs_oracle(blocks, monkeypatch):
    """Communities wider than the window, staged in passes (cdk_graph.intra_split):
    generator CSR bit-exact, RHS and 30 RK4 steps vs the oracle."""
    import torch

    from paper_2203_16657_b200 import plan
    from paper_2203_16657_b200.engine import KuramotoEngine

    monkeypatch.setenv("CDK_INTER_BLOCKS", blocks)
    c, budget, wn = _small_window_case()
    off, cdf, n_edges, thr = c.gen_inputs()
    npass = plan.community_passes(off, wn)
    assert (npass == 1).any() and (npass > 1).any() and (npass == 0).any()
    (iptr, icol, xptr, xcol, split), (iu, iv, sg) = OG.generate_csr(c.graph_seed, off, cdf,
                                                                     n_edges, thr, wn)
    csr = gen.generate(c, "cuda", pass_nodes=wn)
    dptr, dcol, dxptr, dxcol = csr.to_host()
    assert np.array_equal(dptr, iptr) and np.array_equal(dcol, icol)
    assert np.array_equal(csr.split_host(), split)
    assert np.array_equal(dxptr, xptr) and np.array_equal(dxcol, xcol)

    omega, theta0 = c.state()
    omega = np.clip(omega, -20, 20)
    dg, _ = gen.device_graph(c, "cuda", smem_budget=budget)
    segw = dg.schedule.seg_win
    assert ((segw[:, 1] - segw[:, 0]) > wn).any()  # multi-pass segments scheduled
    eng = KuramotoEngine(None, omega, coupling=c.coupling, norm=c.n, graph=dg)
    k = eng.rhs(torch.from_numpy(theta0).cuda()).cpu().numpy()
    ko = cia.kuramoto_rhs_cia(K, theta0, omega, off, iu, iv, sg, c.coupling, c.n)
    assert np.abs(k - ko).max() <= 1e-13

    def rhs(x):
        return cia.kuramoto_rhs_cia(K, x, omega, off, iu, iv, sg, c.coupling, c.n)

    ref, _ = cia.rk4_integrate(rhs, theta0, c.dt, 30)
    eng.set_state(theta0)
    eng.rk4(c.dt, 30)
    eng.check()
    assert cia.circ_dist(eng.theta.cpu().numpy(), ref).max() <= 1e-9


def test_multipass_host_layout_vs_oracle():
    """The same pass machinery through plan.build_layout (Decomposition input,
    bank-ordered sub-runs): config-2 family with a 192-node window."""
    import torch

    from paper_2203_16657_b200 import configs, plan
    from paper_2203_16657_b200.engine import KuramotoEngine

    cs = configs.scaled_config2(20000, 24, seed=9)
    dec = cs.decomposition()
    omega, theta0 = cs.state()
    budget = plan.stage_smem_bytes(192) - 128
    dg = plan.DeviceGraph(dec, smem_budget=budget)
    assert dg.layout.intra_split is not None
    eng = KuramotoEngine(dec, omega, coupling=cs.coupling, norm=cs.n, graph=dg)
    s = dec.correction
    k = eng.rhs(torch.from_numpy(theta0).cuda()).cpu().numpy()
    ko = cia.kuramoto_rhs_cia(K, theta0, omega, dec.offsets, s.iu, s.iv, s.sgn, cs.coupling, cs.n)
    assert np.abs(k - ko).max() <= 1e-13

    def rhs(x):
        return cia.kuramoto_rhs_cia(K, x, omega, dec.offsets, s.iu, s.iv, s.sgn, cs.coupling,
                                    cs.n)

    ref, _ = cia.rk4_integrate(rhs, theta0, cs.dt, 20)
    eng.set_state(theta0)
    eng.rk4(cs.dt, 20)
    eng.check()
    assert cia.circ_dist(eng.theta.cpu().numpy(), ref).max() <= 1e-9


def test_full_size_row_regeneration():
    """BASELINE-size config 5: sampled intra rows regenerated by the numpy
    restatement; inter symmetry on sampled rows; totals near SURVEY App. A.4."""
    import torch

    c = gen.config5()
    off, cdf, n_edges, thr = c.gen_inputs()
    csr = gen.generate(c, "cuda")
    lam = np.diff(off)
    rng = np.random.default_rng(0)
    comm_of = lambda i: int(np.searchsorted(off, i, side="right") - 1)  # noqa: E731
    for i in rng.integers(0, c.n, 6).tolist():
        cc = comm_of(i)
        a = i - off[cc]
        b = np.arange(lam[cc], dtype=np.uint32)
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        h = OG.hash4(c.graph_seed, np.full_like(b, cc), lo.astype(np.uint32), hi.astype(np.uint32))
        want = np.nonzero((h < np.uint32(thr)) & (b != a))[0]
        s, e = int(csr.intra_ptr[i]), int(csr.intra_ptr[i + 1])
        got = csr.intra_col[s:e].cpu().numpy().view(np.uint16)  # ascending across sub-runs
        got = got[got != 0xFFFF].astype(np.int64)
        assert np.array_equal(got, want)
    xptr = csr.inter_ptr
    for i in rng.integers(0, c.n, 6).tolist():
        cols = csr.inter_col[int(xptr[i]): int(xptr[i + 1])].cpu().numpy()
        assert np.all(np.diff(cols) > 0)
        for j in cols[:50].tolist():
            row = csr.inter_col[int(xptr[j]): int(xptr[j + 1])]
            assert bool((row == i).any())
    nnz_dir = csr.nnz_intra + int(xptr[-1])
    assert 0.8e10 < nnz_dir < 1.25e10, nnz_dir
    del csr
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", ["0", "1", "sweep1", "sweep2", "sweep4"])
def test_inter_phase_modes_cfg1_golden(mode, monkeypatch, golden_dir):
    """Every inter-entry path (inline in the row pipeline / separate phase per
    segment / block-phased sweep, plan._seg_lanes and plan.inter_blocking)
    reproduces the reference's config-1 trajectory."""
    import os

    import torch

    from paper_2203_16657_b200 import configs
    from paper_2203_16657_b200.engine import KuramotoEngine

    if mode.startswith("sweep"):
        monkeypatch.setenv("CDK_INTER_BLOCKS", mode[-1])
    else:
        monkeypatch.setenv("CDK_INTER_PHASE", mode)
        monkeypatch.setenv("CDK_INTER_BLOCKS", "0")
    c = configs.config1()
    dec = c.decomposition()
    omega, theta0 = c.state()
    g = np.load(os.path.join(golden_dir, "cfg1.npz"))
    eng = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
    if mode.startswith("sweep"):
        assert eng.graph.inter_blocks == int(mode[-1])
    else:
        assert bool(eng.graph.schedule.seg_lpr[0] & 256) == (mode == "1")
    k = eng.rhs(torch.from_numpy(theta0).cuda()).cpu().numpy()
    assert np.abs(k - g["rhs0_cia"]).max() <= 1e-13
    eng.set_state(theta0)
    eng.rk4(c.dt, c.steps)
    eng.check()
    assert cia.circ_dist(eng.theta.cpu().numpy(), g["final_cia"]).max() <= 1e-9


def test_device_bank_order_matches_host():
    """cdk_bank_order (device, out of place) == cdk_host_bank_order on the same
    rebased runs, including pass sub-runs (192-node window)."""
    from paper_2203_16657_b200 import plan

    c, budget, wn = _small_window_case()
    csr = gen.generate(c, "cuda", pass_nodes=wn)
    iptr, icol, _, _ = csr.to_host()
    lay = csr.layout()
    dg, _ = gen.device_graph(c, "cuda", smem_budget=budget)
    delta = np.repeat(dg.schedule.row_delta.astype(np.int64), np.diff(iptr))
    col = icol.copy()
    m = col != 0xFFFF
    col[m] = (col[m].astype(np.int64) + delta[m]).astype(np.uint16)
    plan._bank_order(col, plan._sub_run_ptr(lay), dg.schedule.smem_nodes)
    got = dg._t["intra_col"][: col.shape[0]].cpu().numpy().view(np.uint16)
    assert np.array_equal(got, col)
