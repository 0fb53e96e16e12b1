"""ELL (lane-per-row sliced) layout built by the host planner (CPU): every
row's intra and inter entries appear exactly once in its lane's slots, and
every quarter-warp step of a window-staged rblock hits 8 distinct shared-memory
bank groups (padding included) — the property the ELL stage kernels rely on
for conflict-free LDS.128 gathers (plan.build_ell, cdk_host_ell_intra)."""

import numpy as np
import pytest

from paper_2203_16657_b200 import configs
from paper_2203_16657_b200 import graph as G
from paper_2203_16657_b200 import plan as PL

PAD = 0xFFFF


def _ell_schedule(dec, sm_count=148, window=None, monkeypatch=None):
    if window is not None:
        monkeypatch.setenv("CDK_ELL_WINDOW", str(window))
    lay = PL.build_layout(dec, pass_nodes=1 << 30)
    sch = PL.build_schedule(lay, sm_count=sm_count, ell=True)
    return lay, sch


def _check(lay, sch):
    e = sch.ell
    assert e is not None
    rows = lay.rblk_row0
    nrb = lay.n_rblk
    seg_of_rb = np.repeat(np.arange(sch.n_seg), np.diff(sch.seg_rblk))
    col = sch.intra_col
    wn = sch.smem_nodes
    slots = 0
    for b in range(nrb):
        r0, r1 = int(rows[b]), int(rows[b + 1])
        assert 0 < r1 - r0 <= 32
        nch = (e.ell_off[b + 1] - e.ell_off[b]) // 32
        blk = e.ell_col[8 * e.ell_off[b]: 8 * e.ell_off[b + 1]].reshape(nch, 32, 8)
        seq = blk.transpose(1, 0, 2).reshape(32, nch * 8)  # lane -> its step sequence
        s = int(seg_of_rb[b])
        staged = sch.seg_win[s, 1] > sch.seg_win[s, 0]
        for lane in range(32):
            r = r0 + lane
            want = col[lay.intra_ptr[r]:lay.intra_ptr[r + 1]] if r < r1 else col[:0]
            want = np.sort(want[want != PAD])
            got = seq[lane]
            real = got[got < wn] if staged else got[got != PAD]
            assert np.array_equal(np.sort(real), want), (b, lane)
            if staged:
                assert np.all((got < wn) | ((got >= wn) & (got < wn + 8)))
        if staged and nch:
            for q in range(4):
                banks = seq[8 * q: 8 * q + 8] & 7  # [8 lanes, steps]
                for k in range(banks.shape[1]):
                    assert len(set(banks[:, k].tolist())) == 8, (b, q, k)
        slots += nch * 256
        # inter
        nx = (e.xell_off[b + 1] - e.xell_off[b]) // 32
        xb = e.xell_col[e.xell_off[b]: e.xell_off[b + 1]].reshape(nx, 32)
        for lane in range(32):
            r = r0 + lane
            want = lay.inter_col[lay.inter_ptr[r]:lay.inter_ptr[r + 1]] if r < r1 else []
            got = xb[:, lane]
            assert np.array_equal(got[got >= 0], np.asarray(want, np.int32))
            assert np.all(got[len(want):] == -1)
    assert slots == e.slots()
    # work units: every rblock of a segment exactly once, longest first
    nch = np.diff(e.ell_off) // 32
    nxs = np.diff(e.xell_off) // 32
    units = e.ell_units
    for si in range(sch.n_seg):
        a, z = int(sch.seg_rblk[si]), int(sch.seg_rblk[si + 1])
        u = units[e.seg_unit[si]:e.seg_unit[si + 1]]
        assert sorted(u.tolist()) == list(range(a, z))
        work = nch[u] * 8 + nxs[u]
        assert np.all(np.diff(work) <= 0)
    if e.ell_meta is not None:  # packed unit metadata agrees with the arrays
        m = e.ell_meta.reshape(-1, 8)
        assert m.shape[0] == units.shape[0]
        for k in range(m.shape[0]):
            b = int(units[k])
            assert m[k, 3] == b and m[k, 2] == rows[b] and m[k, 6] == rows[b + 1] - rows[b]
            assert m[k, 0] == e.ell_off[b]
            assert m[k, 4] == nch[b]
            assert m[k, 5] == nxs[b]


def test_ell_layout_config1():
    c = configs.config1()
    lay, sch = _ell_schedule(c.decomposition())
    _check(lay, sch)
    # real entries vs slots: the schedule pads each bundle to its Delta
    assert lay.nnz_intra <= sch.ell.slots() <= 2 * lay.nnz_intra + 256 * lay.n_rblk


def test_ell_layout_edge_cases(monkeypatch):
    """NONE pool, tiny communities, a community wider than the window
    (unstaged: global gathers, pads skipped), empty S."""
    rng = np.random.default_rng(3)
    g, part = G.planted_partition_graph([1, 3, 40, 300, 700], 0.8, 0.02, 5)
    a = part.assignment.copy()
    a[rng.choice(a.shape[0], 37, replace=False)] = -1  # NONE pool
    used = np.unique(a[a >= 0])
    remap = -np.ones(a.max() + 2, dtype=np.int64)
    remap[used] = np.arange(used.size)
    dec = G.decompose(g, G.Partition.from_assignment(np.where(a >= 0, remap[a], -1)))
    lay, sch = _ell_schedule(dec, sm_count=7, window=512, monkeypatch=monkeypatch)
    assert np.any(sch.seg_win[:, 1] == sch.seg_win[:, 0])  # some unstaged segments
    _check(lay, sch)
    dec = G.planted_partition_decomposition([5, 9], 1.0, 0.0, 1)
    lay, sch = _ell_schedule(dec, sm_count=3)
    _check(lay, sch)
    assert sch.ell.slots() == 0


def test_rb_scale_recuts_keep_layout():
    """build_schedule(rb_scale=...) (the calibration's re-cut) changes only the
    CTA ranges: every layout invariant still holds and the per-rblock
    schedules (chunk columns) are unchanged for unchanged segment windows."""
    c = configs.config1()
    lay = PL.build_layout(c.decomposition(), pass_nodes=1 << 30)
    sch0 = PL.build_schedule(lay, sm_count=7, ell=True)
    scale = np.linspace(0.5, 2.0, lay.n_rblk)
    sch1 = PL.build_schedule(lay, sm_count=7, ell=True, rb_scale=scale)
    _check(lay, sch1)
    assert not np.array_equal(sch0.cta_seg, sch1.cta_seg) or not np.array_equal(
        sch0.seg_rblk, sch1.seg_rblk)
