"""Config-5 generator: host-side inputs and the numpy restatement
(oracle/gen.py) — structural properties, no GPU."""

import numpy as np

from oracle import gen as OG
from paper_2203_16657_b200 import gen


def _case():
    return gen.scaled_config5(n=3000, lo=40, hi=500, seed=57)


def test_sizes_cover_n_and_power_law_bounds():
    c = gen.config5()
    s = c.sizes()
    assert s.sum() == c.n
    assert 1500 <= s.shape[0] <= 2200  # ~1808 expected
    assert s.min() >= 900 and s.max() <= 22000


def test_gen_inputs():
    c = _case()
    off, cdf, n_edges, thr = c.gen_inputs()
    assert off[-1] == c.n and np.all(np.diff(off) > 0)
    assert cdf.shape == (c.n,) and cdf[-1] == 1.0 and np.all(np.diff(cdf) >= 0)
    assert abs(thr / 2**32 - (1 - c.p_in)) < 1e-9
    assert n_edges > 0


def test_hash_matches_known_values():
    # fixed vectors of the mix32/hash4 restatement (pinned against the device
    # in tests/test_gpu_gen.py through whole-CSR equality)
    assert int(OG.mix32(np.uint32(0))) == 0
    h = OG.hash4(5001, np.uint32(3), np.uint32(1), np.uint32(2))
    assert h.dtype == np.uint32


def test_oracle_csr_properties():
    c = _case()
    off, cdf, n_edges, thr = c.gen_inputs()
    (iptr, icol, xptr, xcol, _), (iu, iv, sg) = OG.generate_csr(c.graph_seed, off, cdf, n_edges,
                                                                  thr)
    n = c.n
    comm = np.repeat(np.arange(off.shape[0] - 1), np.diff(off))
    # intra: padded to 8, ascending local columns, symmetric, density ~ 1 - p_in
    assert np.all(np.diff(iptr) % 8 == 0)
    rows = np.repeat(np.arange(n), np.diff(iptr))
    real = icol != 0xFFFF
    r, q = rows[real], icol[real].astype(np.int64) + off[comm[rows[real]]]
    pairs = set(zip(r.tolist(), q.tolist()))
    assert all((b, a) in pairs for a, b in list(pairs)[:5000])
    lam = np.diff(off)
    frac = real.sum() / float((lam * (lam - 1)).sum())
    assert abs(frac - (1 - c.p_in)) < 0.01
    # inter: sorted unique per row, symmetric, never inside one community
    xr = np.repeat(np.arange(n), np.diff(xptr))
    assert np.all(comm[xr] != comm[xcol])
    key = xr * n + xcol
    assert np.all(np.diff(key) > 0)
    assert np.array_equal(np.sort(xcol.astype(np.int64) * n + xr), key)
    mean_deg = xcol.shape[0] / n
    target = (c.mu / (1 - c.mu) * c.p_in * (np.repeat(lam, lam) - 1)).mean()
    assert 0.85 * target < mean_deg < 1.1 * target
    # triples: sorted, diagonal once per in-community node
    assert np.all((iu < iv) | (iu == iv))
    assert (iu == iv).sum() == off[-1]
    assert np.all(np.diff(iu * n + iv) > 0)
    assert 2 * (iu != iv).sum() == real.sum() + xcol.shape[0]


def _dec_from_triples(off, n, iu, iv, sg):
    from paper_2203_16657_b200 import graph as G

    part = G.Partition.from_assignment(np.repeat(np.arange(off.shape[0] - 1), np.diff(off)))
    return G.Decomposition(part, G.SparseCorrection(iu, iv, sg), n)


def test_host_layout_matches_generator_layout_with_passes():
    """plan.build_layout on the generator's triples reproduces the generator's
    CSR bit for bit, including the per-pass sub-runs (window of
    192 nodes: staged, multi-pass and unstaged communities all present)."""
    from paper_2203_16657_b200 import plan

    c = gen.scaled_config5(n=5000, lo=100, hi=1400, seed=58)
    off, cdf, n_edges, thr = c.gen_inputs()
    wn = 192
    npass = plan.community_passes(off, wn)
    assert (npass == 1).any() and (npass > 1).any() and (npass == 0).any()
    (iptr, icol, xptr, xcol, split), (iu, iv, sg) = OG.generate_csr(c.graph_seed, off, cdf,
                                                                     n_edges, thr, wn)
    lay = plan.build_layout(_dec_from_triples(off, c.n, iu, iv, sg), pass_nodes=wn)
    assert np.array_equal(lay.intra_ptr, iptr)
    assert np.array_equal(lay.intra_col, icol)
    assert np.array_equal(lay.intra_split, split)
    assert np.array_equal(lay.inter_ptr, xptr)
    assert np.array_equal(lay.inter_col, xcol)


def test_schedule_multipass_segments():
    from paper_2203_16657_b200 import plan

    c = gen.scaled_config5(n=5000, lo=100, hi=1400, seed=58)
    off, cdf, n_edges, thr = c.gen_inputs()
    _, (iu, iv, sg) = OG.generate_csr(c.graph_seed, off, cdf, n_edges, thr)
    budget = plan.stage_smem_bytes(192) - 128
    wn = plan.window_nodes(plan.ROWS_CAP, budget)
    lay = plan.build_layout(_dec_from_triples(off, c.n, iu, iv, sg), pass_nodes=wn)
    sch = plan.build_schedule(lay, sm_count=16, smem_budget=budget)
    npass = plan.community_passes(off, wn)
    rows = lay.rblk_row0
    for s_ in range(sch.n_seg):
        rb0, rb1 = sch.seg_rblk[s_], sch.seg_rblk[s_ + 1]
        comms = set(lay.rblk_comm[rb0:rb1].tolist())
        w0, w1 = sch.seg_win[s_]
        if w1 > w0 and (w1 - w0) > wn:  # multi-pass: one community, its whole window
            assert len(comms) == 1
            cc = comms.pop()
            assert npass[cc] > 1 and w0 == off[cc] // 8 * 8
            assert rows[rb1] - rows[rb0] <= sch.seg_rows_cap
        # every rebased real column of pass q lies in [q wn, (q+1) wn)
        multi = w1 > w0 and (w1 - w0) > wn
        for i in range(rows[rb0], min(rows[rb1], rows[rb0] + 40)):
            e0, e1 = lay.intra_ptr[i], lay.intra_ptr[i + 1]
            col = sch.intra_col[e0:e1].astype(np.int64)
            if not multi:
                if w1 > w0:
                    assert np.all(col[col != 0xFFFF] < w1 - w0)
                continue
            np_ = int((w1 - w0 + wn - 1) // wn)
            sp = int(lay.intra_split[i])
            cuts = [0] + [8 * ((sp >> (16 * q)) & 0xFFFF) for q in range(np_ - 1)] + [e1 - e0]
            for q in range(np_):
                sub = col[cuts[q]:cuts[q + 1]]
                assert (cuts[q + 1] - cuts[q]) % 8 == 0
                sub = sub[sub != 0xFFFF]
                assert np.all((sub >= q * wn) & (sub < (q + 1) * wn))
