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
    (iptr, icol, xptr, xcol), (iu, iv, sg) = OG.generate_csr(c.graph_seed, off, cdf, n_edges, thr)
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
