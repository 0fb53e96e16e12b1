"""Host-side logic (CPU): decomposition exactness (SPEC acceptance 6), planted
generator moments, the device layout/schedule built by plan.py."""

import numpy as np
import pytest

from paper_2203_16657_b200 import graph as G
from paper_2203_16657_b200 import plan as PL
from paper_2203_16657_b200.errors import InputError


def _random_graph_partition(rng, n):
    p = rng.uniform(0.05, 0.6)
    a = rng.random((n, n)) < p
    a = np.triu(a, 1)
    e = np.argwhere(a)
    g = G.Graph.from_pairs(n, e)
    m = int(rng.integers(1, 6))
    assign = rng.integers(-1, m, n)  # -1 = NONE pool
    # make ids dense
    used = np.unique(assign[assign >= 0])
    remap = {int(u): i for i, u in enumerate(used)}
    assign = np.array([remap.get(int(x), -1) for x in assign])
    return g, G.Partition.from_assignment(assign)


def test_decomposition_exactness_random():
    """D + S = P A P^T entrywise, 50 random graphs, N <= 200."""
    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(2, 200))
        g, part = _random_graph_partition(rng, n)
        dec = G.decompose(g, part)
        a = g.dense()
        assert np.array_equal(dec.dense_matrix(), a[np.ix_(part.perm, part.perm)])
        s = dec.correction
        assert np.all(s.iu <= s.iv)
        key = s.iu * n + s.iv
        assert np.all(np.diff(key) > 0)  # sorted, unique


def test_spec_decompose_examples():
    # two 3-cliques + cross edge (0,3) -> S = {(0,3,+1)} plus the diagonal
    e = [(0, 1), (0, 2), (1, 2), (3, 4), (3, 5), (4, 5), (0, 3)]
    g = G.Graph.from_pairs(6, e)
    dec = G.decompose(g, G.Partition.from_assignment([0, 0, 0, 1, 1, 1]))
    s = dec.correction
    off = s.iu != s.iv
    assert list(zip(s.iu[off], s.iv[off], s.sgn[off])) == [(0, 3, 1.0)]
    assert np.all(s.sgn[~off] == -1)
    # K4 minus (1,2), one community -> S = {(1,2,-1)}
    e = [(0, 1), (0, 2), (0, 3), (1, 3), (2, 3)]
    dec = G.decompose(G.Graph.from_pairs(4, e), G.Partition.from_assignment([0] * 4))
    s = dec.correction
    off = s.iu != s.iv
    assert list(zip(s.iu[off], s.iv[off], s.sgn[off])) == [(1, 2, -1.0)]
    # p_in = 1, p_out = 0: only the diagonal
    for seed in range(5):
        d = G.planted_partition_decomposition([3, 3], 1.0, 0.0, seed)
        assert np.all(d.correction.iu == d.correction.iv)


def test_planted_graph_matches_direct_decomposition():
    for seed in range(6):
        g, p = G.planted_partition_graph([9, 4, 13, 1], 0.8, 0.15, seed)
        assert G.decompose(g, p).dense_matrix().tolist() == \
            G.planted_partition_decomposition([9, 4, 13, 1], 0.8, 0.15, seed).dense_matrix().tolist()


def test_planted_binomial_moments():
    """intra edge count within 5 sigma of the binomial expectation."""
    g, p = G.planted_partition_graph([50, 50], 0.9, 0.01, 7)
    comm = p.assignment
    intra = np.sum(comm[g.edges[:, 0]] == comm[g.edges[:, 1]])
    n_pairs = 2 * 50 * 49 // 2
    mu, sd = 0.9 * n_pairs, np.sqrt(n_pairs * 0.9 * 0.1)
    assert abs(intra - mu) < 5 * sd
    with pytest.raises(InputError):
        G.planted_partition_graph([3, 0], 0.5, 0.1, 1)


def _layout_to_directed(lay):
    rows, cols = [], []
    off = lay.comm_off
    comm_of_row = np.full(lay.n_rows, -1)
    for c in range(lay.n_comm):
        comm_of_row[off[c]:off[c + 1]] = c
    for i in range(lay.n_rows):
        a, b = lay.intra_ptr[i], lay.intra_ptr[i + 1]
        assert a % 8 == 0 and b % 8 == 0
        loc = lay.intra_col[a:b]
        loc = loc[loc != PL.INTRA_PAD].astype(np.int64)
        if loc.size:
            assert comm_of_row[i] >= 0
            rows += [i] * loc.size
            cols += list(off[comm_of_row[i]] + loc)
        x0, x1 = lay.inter_ptr[i], lay.inter_ptr[i + 1]
        rows += [i] * (x1 - x0)
        cols += list(lay.inter_col[x0:x1])
    return np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_layout_roundtrip(seed):
    rng = np.random.default_rng(seed)
    g, part = _random_graph_partition(rng, 150)
    dec = G.decompose(g, part)
    lay = PL.build_layout(dec)
    r, c = _layout_to_directed(lay)
    rows, cols, _ = dec.directed()
    k1 = np.sort(r * 1000 + c)
    k2 = np.sort(rows * 1000 + cols)
    assert np.array_equal(k1, k2)
    assert lay.nnz_dir == dec.nnz_dir


def test_bank_order_permutes_within_rows_and_spreads_banks():
    dec = G.planted_partition_decomposition([900, 700], 0.7, 0.01, 9)
    lay = PL.build_layout(dec)
    sch = PL.build_schedule(lay, sm_count=4)
    ip = lay.intra_ptr
    conflicts_before = conflicts_after = 0
    for i in range(0, lay.n_rows, 37):
        a, b = ip[i], ip[i + 1]
        before = np.sort(lay.intra_col[a:b])
        after = sch.intra_col[a:b]
        # same multiset up to the (row-constant) rebasing
        d = before[before != PL.INTRA_PAD].astype(np.int64)
        e = np.sort(after[after != PL.INTRA_PAD].astype(np.int64))
        assert d.size == e.size and np.all(np.diff(e - d) == 0)
        for blk in range(0, b - a, 64):
            for k in range(8):
                pos = [a + blk + 8 * t + k for t in range(8) if blk + 8 * t + k < b - a]
                for arr, tag in ((lay.intra_col, 0), (sch.intra_col, 1)):
                    res = [int(arr[p_]) & 7 for p_ in pos]
                    c = len(res) - len(set(res))
                    if tag:
                        conflicts_after += c
                    else:
                        conflicts_before += c
    assert conflicts_after < 0.2 * conflicts_before


def _schedule_to_directed(lay, sch):
    """Directed S reconstructed from the device columns (rebased to segment bases)."""
    rows_rb = lay.rblk_row0
    seg_rows = rows_rb[sch.seg_rblk]
    rows, cols = [], []
    for s in range(sch.n_seg):
        for i in range(seg_rows[s], seg_rows[s + 1]):
            a, b = lay.intra_ptr[i], lay.intra_ptr[i + 1]
            loc = sch.intra_col[a:b]
            loc = loc[loc != PL.INTRA_PAD].astype(np.int64)
            rows += [i] * loc.size
            cols += list(sch.seg_base[s] + loc)
            x0, x1 = lay.inter_ptr[i], lay.inter_ptr[i + 1]
            rows += [i] * (x1 - x0)
            cols += list(lay.inter_col[x0:x1])
    return np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)


@pytest.mark.parametrize("sm_count,seed,rows_cap", [(1, 0, 1536), (3, 1, 64), (148, 2, 1024),
                                                    (7, 3, 32)])
def test_schedule_invariants(sm_count, seed, rows_cap):
    rng = np.random.default_rng(seed)
    g, part = _random_graph_partition(rng, 190)
    dec = G.decompose(g, part)
    lay = PL.build_layout(dec)
    sch = PL.build_schedule(lay, sm_count=sm_count, rows_cap=rows_cap)
    nrb = lay.n_rblk
    seg = sch.seg_rblk
    assert seg[0] == 0 and seg[-1] == nrb and np.all(np.diff(seg) > 0)
    rows_rb = lay.rblk_row0
    off = lay.comm_off
    for s in range(sch.n_seg):
        cs = lay.rblk_comm[seg[s]:seg[s + 1]]
        w0, w1 = sch.seg_win[s]
        assert rows_rb[seg[s + 1]] - rows_rb[seg[s]] <= max(rows_cap // 8 * 8, 32)
        if w1 > w0:  # staged: every community of the segment inside the window
            assert np.all(cs >= 0) and cs.max() - cs.min() < PL.SEG_MAX_COMM
            assert w1 - w0 <= sch.smem_nodes and sch.seg_base[s] == w0
            assert np.all(off[cs] >= w0) and np.all(off[cs + 1] <= w1)
        else:
            assert np.all(cs == cs[0])
    cta = sch.cta_seg
    assert cta[0] == 0 and cta[-1] == sch.n_seg and np.all(np.diff(cta) >= 0)
    assert sch.n_cta == cta.shape[0] - 1
    # rblocks: <= 32 rows, never straddle communities, cover all rows once
    ends = rows_rb[1:]
    assert np.all(ends - rows_rb[:-1] <= 32) and np.all(ends > rows_rb[:-1])
    assert rows_rb[-1] == lay.n_rows
    # rebased device columns still encode exactly the directed S
    r, c = _schedule_to_directed(lay, sch)
    rows, cols, _ = dec.directed()
    assert np.array_equal(np.sort(r * 1000 + c), np.sort(rows * 1000 + cols))


def test_schedule_small_window_forces_unstaged():
    dec = G.planted_partition_decomposition([300, 40, 40, 500], 0.9, 0.05, 5)
    lay = PL.build_layout(dec)
    # a tiny per-CTA budget: windows of <= ~100 nodes, big communities unstaged
    sch = PL.build_schedule(lay, sm_count=2, rows_cap=64,
                            smem_budget=PL.stage_smem_bytes(0, 64) + 16 * 200)
    assert sch.smem_nodes >= 0
    r, c = _schedule_to_directed(lay, sch)
    rows, cols, _ = dec.directed()
    assert np.array_equal(np.sort(r * 10**6 + c), np.sort(rows * 10**6 + cols))


def test_layout_rejects_inconsistent_signs():
    dec = G.planted_partition_decomposition([5, 5], 0.5, 0.3, 3)
    s = dec.correction
    bad = G.SparseCorrection(s.iu, s.iv, -s.sgn)
    with pytest.raises(InputError):
        PL.build_layout(G.Decomposition(dec.partition, bad, dec.n_nodes))
