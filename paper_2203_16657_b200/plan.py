"""Host planner: Decomposition -> device CSR layout + static work schedule.

Turns the reference's wire format (sorted unordered COO triples (iu, iv, sgn)
with the diagonal) into the layout the fused kernels
stream (include/commdyn_cuda.h, struct cdk_graph):

* directed CSR without the diagonal (sin(0) = 0 for the Kuramoto family;
  for general h the diagonal is a per-node constant);
* the sign is implied by the column's community, so no sign bytes are
  stored: intra (-1) entries as uint16 community-local columns, each row's
  run padded to a multiple of 8 (one 16-byte vector load per lane), inter
  (+1) entries as int32 global columns;
* 32-row "rblocks" (never straddling a community), cost-balanced contiguous
  CTA ranges, and "segments" = a CTA's run of rblocks whose intra neighbours
  lie in one node window that fits shared memory (the unit of staging), with
  the intra columns rebased to that window.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InputError
from .graph import NONE, Decomposition

RB = 32
INTRA_PAD = 0xFFFF
# Cost model in units of one padded intra entry, fitted to per-CTA cycle
# counts of the stage kernel (tools/prof_cta.py; profiles/r01_v9_cta_phase_profile.txt):
# cycles ~ 16.3 rows + 0.224 entries + 1.9 inter + 8.7e3 segments
ROW_COST = 73.0  # per-row overhead (pipeline, reduction, epilogue, sincos)
INTER_COST = 8.4  # an inter entry: 4-byte index + a random 16-byte L2 gather
DEFAULT_SMS = 148
SMEM_OPTIN = 232448  # max dynamic + static shared memory per block (227 KB)


@dataclass
class HostLayout:
    n_rows: int
    n_comm: int
    comm_off: np.ndarray
    intra_ptr: np.ndarray
    intra_col: np.ndarray
    inter_ptr: np.ndarray
    inter_col: np.ndarray
    rblk_row0: np.ndarray
    rblk_comm: np.ndarray
    comm_rblk_off: np.ndarray
    row_cost: np.ndarray
    nnz_intra: int
    nnz_inter: int
    intra_split: np.ndarray | None = None  # uint64[n] sub-run starts (cdk_graph.intra_split)
    pass_nodes: int = 0  # window capacity the sub-runs were cut for

    @property
    def nnz_dir(self) -> int:
        return self.nnz_intra + self.nnz_inter

    @property
    def n_rblk(self) -> int:
        return int(self.rblk_row0.shape[0] - 1)

    def nbytes(self) -> int:
        return int(sum(a.nbytes for a in (self.comm_off, self.intra_ptr, self.intra_col,
                                           self.inter_ptr, self.inter_col)))


@dataclass
class Schedule:
    n_cta: int
    cta_threads: int
    smem_nodes: int  # staged window capacity (nodes)
    seg_rows_cap: int  # rows per segment (shared-memory row buffers)
    seg_rblk: np.ndarray  # int32[n_seg+1]
    seg_win: np.ndarray  # int64[n_seg, 2]
    seg_base: np.ndarray  # int64[n_seg]
    cta_seg: np.ndarray  # int32[n_cta+1]
    seg_lpr: np.ndarray  # int32[n_seg] lanes per row (4 | 8 | 16 | 32)
    intra_col: np.ndarray  # uint16, rebased to each row's segment base, bank-ordered
    xs_cap: int = 0  # staged inter-column capacity (cdk_graph.xs_cap)
    seg_xr: np.ndarray | None = None  # int64[2*n_seg] inter_ptr at segment bounds
    ell: "EllLayout | None" = None  # lane-per-row sliced layout (ELL kernels)
    rb_cost: np.ndarray | None = None  # the cost model the CTA cuts balanced

    @property
    def n_seg(self) -> int:
        return int(self.seg_rblk.shape[0] - 1)

    def smem_bytes(self) -> int:
        return stage_smem_bytes(self.smem_nodes, self.seg_rows_cap, self.xs_cap)


def _row_runs(rows_sorted: np.ndarray, n_rows: int):
    counts = np.bincount(rows_sorted, minlength=n_rows).astype(np.int64)
    start = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=start[1:])
    return counts, start


# rblocks: <= 32 rows of one community and at most RB_MAX_E padded intra /
# RB_MAX_X inter entries (bounds the work of one warp-level epilogue unit)
RB_MAX_E = 8192
RB_MAX_X = 1016


def _split_heavy_rblocks(row0, row_end, intra_ptr, inter_ptr):
    nxt = np.minimum(row0 + RB, row_end)
    e = intra_ptr[nxt] - intra_ptr[row0]
    x = inter_ptr[nxt] - inter_ptr[row0]
    heavy = np.nonzero((e > RB_MAX_E) | (x > RB_MAX_X))[0]
    if heavy.size == 0:
        return row0
    extra = []
    for b in heavy.tolist():
        r, end = int(row0[b]), int(nxt[b])
        start = r
        while r < end:
            ne = intra_ptr[r + 1] - intra_ptr[start]
            nx = inter_ptr[r + 1] - inter_ptr[start]
            if r > start and (ne > RB_MAX_E or nx > RB_MAX_X):
                extra.append(r)
                start = r
            r += 1
    return np.sort(np.concatenate([row0, np.asarray(extra, dtype=np.int64)]))


WIN_ALIGN = 8  # staged windows start/end on 8-node (128-byte) boundaries (bulk-copy alignment)
CTA_THREADS = 896  # default; the library's value wins (stage_threads())


def stage_threads() -> int:
    """threads per CTA the stage kernels were built for (cdk_kuramoto_stage_threads)"""
    from ._lib import load_library

    return int(load_library().cdk_kuramoto_stage_threads())


def ell_threads() -> int:
    """threads per CTA of the ELL stage kernels (cdk_kuramoto_ell_threads)"""
    from ._lib import load_library

    return int(load_library().cdk_kuramoto_ell_threads())


def ell_ctas_per_sm() -> int:
    """resident ELL CTAs per SM the library was built for"""
    from ._lib import load_library

    return int(load_library().cdk_kuramoto_ell_ctas_per_sm())


def ell_window_nodes() -> int:
    """window capacity of the ELL kernels (CDK_ELL_WINDOW may lower it)"""
    from ._lib import load_library

    cap = int(load_library().cdk_kuramoto_ell_window_nodes())
    w = settings().ell_window
    return min(cap, w // WIN_ALIGN * WIN_ALIGN) if w > 0 else cap


def ell_enabled() -> bool:
    """lane-per-row ELL kernels for graphs without the inter sweep (CDK_ELL=0: off)"""
    return settings().ell


def ell_calibrate_iters() -> int:
    """measured re-cuts of the ELL CTA ranges at DeviceGraph construction
    (CDK_ELL_CALIBRATE, 0 = off)"""
    return settings().ell_calibrate


def ctas_per_sm() -> int:
    """resident stage CTAs per SM the library was built for
    (cdk_kuramoto_stage_ctas_per_sm): the schedule has SMs x this many CTAs"""
    from ._lib import load_library

    return int(load_library().cdk_kuramoto_stage_ctas_per_sm())


from .settings import settings

ROWS_CAP = settings().rows_cap  # rows per segment (multiple of 8)
# shared-memory budget of the stage kernel (CDK_SMEM_BUDGET: experiments with
# a smaller carve-out, which leaves more L1 for in-flight global loads)
SMEM_BUDGET = settings().smem_budget
SEG_MAX_COMM = 64  # communities per staged segment (csrc/kuramoto.cu SEG_MAX_COMM)
MAX_PASS = 4  # window passes per community (cdk_graph.intra_split packs 3 sub-run starts)
XS_MAX = 16384  # staged inter columns per segment (cdk_graph.xs_cap), upper bound
# fixed cost of a segment in cost-model units (~9k cycles per segment in the
# per-CTA profile fit at ~0.22 cycles per unit); SCHED_ITERS re-cuts with it
SEG_COST = settings().seg_cost
SCHED_ITERS = 6
XS_MIN = 1024


def stage_smem_bytes(smem_nodes: int, rows_cap: int = ROWS_CAP, xs_cap: int = 0) -> int:
    """dynamic shared memory of the stage kernel (csrc/kuramoto.cu:stage_smem_bytes):
    row accumulators + pointer slices + epilogue inputs + window (+8 spare)
    + staged inter columns (+4 spare)"""
    return ((rows_cap + 4) * (16 + 5 * 8) + 16 * (smem_nodes + 8)
            + (4 * (xs_cap + 4) if xs_cap > 0 else 0))


def window_nodes(rows_cap: int = ROWS_CAP, smem_budget: int = SMEM_BUDGET) -> int:
    """staged window capacity (nodes, multiple of 8) of the stage kernel"""
    rows_cap = int(rows_cap) // 8 * 8
    return max(0, (smem_budget - stage_smem_bytes(0, rows_cap)) // 16) // WIN_ALIGN * WIN_ALIGN


def community_passes(off: np.ndarray, wn: int) -> np.ndarray:
    """window passes per community: 1 = fits, 2..MAX_PASS = staged in passes,
    0 = wider (gathered from global memory, one run)"""
    off = np.asarray(off, dtype=np.int64)
    width = (off[1:] + WIN_ALIGN - 1) // WIN_ALIGN * WIN_ALIGN - off[:-1] // WIN_ALIGN * WIN_ALIGN
    q = (width + max(wn, 1) - 1) // max(wn, 1) if wn > 0 else np.zeros_like(width)
    return np.where(q <= MAX_PASS, np.maximum(q, 1), 0).astype(np.int64)


def _rblocks(off, n, intra_ptr, inter_ptr, row_range=None, split_heavy=True):
    """rblocks (<= 32 rows of one community, capped entries unless
    ``split_heavy`` is off) of the rows in row_range, then the NONE pool;
    returns (rblk_row0 [+sentinel], rblk_comm, comm_rblk_off)."""
    lo, hi = (0, n) if row_range is None else (int(row_range[0]), int(row_range[1]))
    m = off.shape[0] - 1
    n_in = int(off[-1])
    sizes = np.diff(off)
    owned = (off[:-1] >= lo) & (off[1:] <= hi)
    if row_range is not None and np.any((off[:-1] < hi) & (off[1:] > lo) & ~owned):
        raise InputError("a shard's row range must not split a community")
    nb = np.where(owned, (sizes + RB - 1) // RB, 0)
    comm_rblk_off = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(nb, out=comm_rblk_off[1:])
    rc = np.repeat(np.arange(m, dtype=np.int64), nb)
    within = np.arange(rc.shape[0], dtype=np.int64) - comm_rblk_off[rc]
    row0 = off[rc] + RB * within
    if split_heavy:
        row0 = _split_heavy_rblocks(row0, off[rc + 1] if rc.size else row0, intra_ptr, inter_ptr)
    rc = np.searchsorted(off, row0, side="right").astype(np.int64) - 1
    comm_rblk_off = np.searchsorted(row0, off).astype(np.int64)
    pool_row0 = np.arange(max(n_in, lo), max(min(n, hi), max(n_in, lo)), RB, dtype=np.int64)
    end = min(n, hi) if row_range is not None else n
    rblk_row0 = np.concatenate([row0, pool_row0, [end]]).astype(np.int64)
    rblk_comm = np.concatenate([rc, np.full(pool_row0.shape[0], -1, np.int64)]).astype(np.int32)
    return rblk_row0, rblk_comm, comm_rblk_off.astype(np.int32)


def build_layout(dec: Decomposition, row_range=None, pass_nodes: int | None = None,
                 split_heavy: bool = True) -> HostLayout:
    """Device layout of the directed S.  ``row_range=(lo, hi)`` keeps only rows
    in [lo, hi) (a rank's shard: whole communities; other rows are present but
    empty, columns stay global).  ``pass_nodes``: window capacity the
    multi-pass sub-runs are cut for (default: the stage kernel's).
    ``split_heavy=False`` (ELL kernels): rblocks stay 32 rows however long the
    rows are — a lane-per-row warp with a half-size rblock idles half its
    lanes on every chunk (config 2: 31.4 M -> 26.5 M gather slots)."""
    part = dec.partition
    n = int(dec.n_nodes)
    off = part.offsets
    m = part.n_comm
    if m and int(part.sizes.max()) > INTRA_PAD - 1:
        raise InputError("community larger than 65534 nodes: uint16 intra columns do not fit")
    comm = part.comm_of_permuted()
    rows, cols, sg = dec.directed()
    lo, hi = (0, n) if row_range is None else (int(row_range[0]), int(row_range[1]))
    if row_range is not None:
        keep = (rows >= lo) & (rows < hi)
        rows, cols, sg = rows[keep], cols[keep], sg[keep]
    cr = comm[rows]
    intra = (cr == comm[cols]) & (cr != NONE)
    if np.any(sg[intra] != -1) or np.any(sg[~intra] != 1):
        raise InputError("sparse correction signs inconsistent with the partition "
                         "(-1 must be intra-community, +1 inter-community)")

    # intra: uint16 local columns, rows padded to multiples of 8; rows of
    # communities wider than the window: one padded sub-run per pass
    key = (rows[intra].astype(np.int64) << 16) | (cols[intra] - off[cr[intra]])
    key.sort()
    ri = key >> 16
    ci = (key & 0xFFFF).astype(np.int64)
    wn = window_nodes() if pass_nodes is None else int(pass_nodes)
    npass_c = community_passes(off, wn)
    multi_c = npass_c > 1
    split = None
    if not multi_c.any():
        counts, start = _row_runs(ri, n)
        padded = (counts + 7) // 8 * 8
        intra_ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(padded, out=intra_ptr[1:])
        pos = intra_ptr[ri] + np.arange(ri.shape[0], dtype=np.int64) - start[ri]
    else:
        ce = comm[ri]
        ps = np.where(multi_c[ce], (ci + off[ce] - (off[ce] // 8 * 8)) // wn, 0)
        gid = ri * MAX_PASS + ps
        cnt4 = np.bincount(gid, minlength=n * MAX_PASS).reshape(n, MAX_PASS)
        pad4 = (cnt4 + 7) // 8 * 8
        padded = pad4.sum(axis=1)
        intra_ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(padded, out=intra_ptr[1:])
        sub = np.cumsum(pad4, axis=1) - pad4  # sub-run starts within the row
        np_row = np.ones(n, dtype=np.int64)
        np_row[: off[-1]] = np.repeat(npass_c, np.diff(off))
        split = np.zeros(n, dtype=np.uint64)
        for q in range(1, MAX_PASS):
            on = np_row > q
            split[on] |= (sub[on, q] // 8).astype(np.uint64) << np.uint64(16 * (q - 1))
        gstart = np.zeros(n * MAX_PASS + 1, dtype=np.int64)
        np.cumsum(cnt4.reshape(-1), out=gstart[1:])
        pos = intra_ptr[ri] + sub[ri, ps] + np.arange(ri.shape[0], dtype=np.int64) - gstart[gid]
        counts = cnt4.sum(axis=1)
    intra_col = np.full(int(intra_ptr[-1]), INTRA_PAD, dtype=np.uint16)
    intra_col[pos] = ci.astype(np.uint16)
    nnz_intra = int(ri.shape[0])
    del key, ri, ci, pos

    # inter: int32 global columns
    rx = rows[~intra]
    cx = cols[~intra]
    order = np.lexsort((cx, rx))
    rx = rx[order]
    inter_col = cx[order].astype(np.int32)
    xcounts, inter_ptr = _row_runs(rx, n)
    nnz_inter = int(rx.shape[0])

    rblk_row0, rblk_comm, comm_rblk_off = _rblocks(off, n, intra_ptr, inter_ptr, row_range,
                                                   split_heavy)
    row_cost = padded.astype(np.float64) + INTER_COST * xcounts + ROW_COST
    return HostLayout(n, m, off.astype(np.int64), intra_ptr, intra_col, inter_ptr, inter_col,
                      rblk_row0, rblk_comm, comm_rblk_off, row_cost, nnz_intra, nnz_inter,
                      split, wn)




def _rblk_rows(lay: HostLayout) -> np.ndarray:
    return lay.rblk_row0  # n_rblk + 1 entries (sentinel = end of the last rblock)


def build_schedule(lay: HostLayout, sm_count: int = DEFAULT_SMS, rows_cap: int = ROWS_CAP,
                   smem_budget: int = SMEM_BUDGET, ell: bool = False,
                   rb_scale: np.ndarray | None = None) -> Schedule:
    """Cost-balanced contiguous CTA ranges of rblocks (one CTA per SM), split
    into segments of <= rows_cap rows whose intra neighbours fit one
    shared-memory window (or, for communities above the window capacity and
    the NONE pool, gather from global memory)."""
    rows_cap = int(rows_cap) // 8 * 8
    smem_nodes = window_nodes(rows_cap, smem_budget)
    if ell:  # ELL kernels: no per-row shared buffers, the whole carve-out is window
        rows_cap, smem_nodes = 1 << 24, ell_window_nodes()
        if lay.intra_split is not None:
            raise InputError("ELL schedules need a layout without window-pass sub-runs")
    n_cta = max(1, int(sm_count))
    nrb = lay.n_rblk
    rows = _rblk_rows(lay)
    cum = np.concatenate([[0.0], np.cumsum(lay.row_cost)])
    rb_cost = cum[rows[1:]] - cum[rows[:-1]]
    seg_cost = SEG_COST
    if ell:  # ELL kernels: cost of an rblock = its slots (padding included)
        e_off, x_off = _ell_sizes(lay)
        rb_cost = (np.diff(e_off) * 8 * ELL_SLOT_COST + np.diff(x_off) * ELL_XSLOT_COST
                   + ELL_RBLK_COST).astype(np.float64)
        if rb_scale is not None:  # measured calibration (DeviceGraph._calibrate)
            rb_cost = rb_cost * rb_scale
        seg_cost = ELL_SEG_COST

    off = lay.comm_off
    win_lo = off[:-1] // WIN_ALIGN * WIN_ALIGN
    win_hi = (off[1:] + WIN_ALIGN - 1) // WIN_ALIGN * WIN_ALIGN
    npass_c = community_passes(off, smem_nodes)
    if lay.intra_split is not None and lay.pass_nodes != smem_nodes:
        raise InputError("layout sub-runs were cut for another window capacity")
    if lay.intra_split is None:  # a layout without sub-runs: wide communities unstaged
        npass_c = np.where(npass_c == 1, 1, 0)
    stageable = npass_c >= 1
    multi = npass_c > 1
    # staged inter columns: when no community needs window passes, shrink the
    # window to the widest staged community and give the rest of the budget
    # to the segment's inter-column slice (row pipeline reads them from smem)
    xs_cap = 0
    if (not ell and settings().xs and not multi.any()
            and lay.nnz_inter > 0 and stageable.any()):
        need = int((win_hi - win_lo)[stageable].max())
        rem = smem_budget - stage_smem_bytes(need, rows_cap)
        cap = min(rem // 4 - 4, XS_MAX) // 16 * 16
        if cap >= XS_MIN:
            xs_cap, smem_nodes = int(cap), need
    mode_c, mode_pool = _comm_modes(lay)

    def segments(cta_bounds):
        return _build_segments(lay, rows, cta_bounds, n_cta, rows_cap, smem_nodes, win_lo, win_hi,
                               stageable, multi, mode_c, mode_pool)

    # CTA cuts balanced on row cost plus SEG_COST per segment: a segment's
    # fixed cost (staging, community sums, pipeline ramp, barriers) is only
    # known once the cuts are placed, so iterate (damped) and keep the best
    targets_frac = np.arange(1, n_cta) / n_cta
    extra = np.zeros(nrb)
    best = None
    iters = SCHED_ITERS if n_cta > 1 and nrb > n_cta else 1
    if nrb > 50000:  # huge graphs (config 5): segments are long, the fixed cost matters less
        iters = min(iters, 2)
    for _ in range(iters):
        cum_rb = np.concatenate([[0.0], np.cumsum(rb_cost + extra)])
        cuts = np.clip(np.searchsorted(cum_rb, cum_rb[-1] * targets_frac, side="left"), 0, nrb)
        bounds = np.maximum.accumulate(np.concatenate([[0], cuts, [nrb]]).astype(np.int64))
        segs = segments(bounds)
        nseg_b = np.diff(np.asarray(segs[3]))
        cum0 = np.concatenate([[0.0], np.cumsum(rb_cost)])
        cta_cost = cum0[bounds[1:]] - cum0[bounds[:-1]] + seg_cost * nseg_b
        if best is None or cta_cost.max() < best[0]:
            best = (cta_cost.max(), segs)
        share = np.zeros(nrb)
        for b in range(n_cta):
            lo, hi = int(bounds[b]), int(bounds[b + 1])
            if hi > lo:
                w = rb_cost[lo:hi]
                share[lo:hi] = seg_cost * nseg_b[b] * w / max(w.sum(), 1e-9)
        extra = 0.5 * extra + 0.5 * share
    seg_rblk, seg_win, seg_base, cta_seg, seg_lpr = best[1]
    seg_rblk = np.asarray(seg_rblk, dtype=np.int32)
    seg_lpr = np.asarray(seg_lpr, dtype=np.int32)
    seg_win = np.asarray(seg_win, dtype=np.int64).reshape(-1, 2)
    seg_base = np.asarray(seg_base, dtype=np.int64)
    sch = _finish_schedule(lay, rows, n_cta, rows_cap, smem_nodes, xs_cap, seg_rblk, seg_win,
                           seg_base, cta_seg, seg_lpr, off, bank_order=not ell)
    sch.rb_cost = rb_cost
    if ell:
        sch.cta_threads = ell_threads()
        sch.ell = build_ell(lay, sch)
    return sch


def _build_segments(lay, rows, cta_bounds, n_cta, rows_cap, smem_nodes, win_lo, win_hi,
                    stageable, multi, mode_c, mode_pool):
    """segments of every CTA's rblock range (see build_schedule)"""
    off = lay.comm_off
    seg_rblk, seg_win, seg_base, cta_seg, seg_lpr = [0], [], [], [0], []
    for b in range(n_cta):
        rb, rb_end = int(cta_bounds[b]), int(cta_bounds[b + 1])
        while rb < rb_end:
            c = int(lay.rblk_comm[rb])
            start = rb
            if c < 0 or not stageable[c] or multi[c]:  # a run of one community / the pool
                while (rb < rb_end and lay.rblk_comm[rb] == c
                       and rows[rb + 1] - rows[start] <= rows_cap):
                    rb += 1
                if c >= 0 and multi[c]:  # staged in passes over the community's window
                    seg_win.append((int(win_lo[c]), int(win_hi[c])))
                    seg_base.append(int(win_lo[c]))
                else:  # unstaged: global gathers
                    seg_win.append((0, 0))
                    seg_base.append(int(off[c]) if c >= 0 else 0)
                seg_lpr.append(int(mode_c[c]) if c >= 0 else mode_pool)
            else:  # staged window over whole communities, 128-byte aligned
                w0 = int(win_lo[c])
                while rb < rb_end:
                    cc = int(lay.rblk_comm[rb])
                    if cc < 0 or not stageable[cc] or multi[cc] or mode_c[cc] != mode_c[c]:
                        break
                    if (int(win_hi[cc]) - w0 > smem_nodes or rows[rb + 1] - rows[start] > rows_cap
                            or cc - c >= SEG_MAX_COMM):
                        break
                    rb += 1
                seg_win.append((w0, int(win_hi[int(lay.rblk_comm[rb - 1])])))
                seg_base.append(w0)
                seg_lpr.append(int(mode_c[c]))
            seg_rblk.append(rb)
        cta_seg.append(len(seg_rblk) - 1)
    return seg_rblk, seg_win, seg_base, cta_seg, seg_lpr


def _finish_schedule(lay, rows, n_cta, rows_cap, smem_nodes, xs_cap, seg_rblk, seg_win, seg_base,
                     cta_seg, seg_lpr, off, bank_order: bool = True):
    """rebasing, bank ordering, segment inter ranges -> Schedule"""
    nrb = lay.n_rblk

    # rebase intra columns (community-local in the layout) to each row's segment base
    n = lay.n_rows
    delta = np.zeros(n, dtype=np.int64)  # rows outside the rblocks (other shards) stay 0
    if nrb:
        seg_of_row = np.repeat(np.arange(seg_base.shape[0]), np.diff(rows[seg_rblk]))
        comm_row = np.repeat(lay.rblk_comm.astype(np.int64), np.diff(rows))
        cstart = np.where(comm_row >= 0, off[np.maximum(comm_row, 0)], 0)
        delta[rows[0]: rows[-1]] = cstart - seg_base[seg_of_row]
    seg_rows = rows[seg_rblk]
    seg_xr = np.stack([lay.inter_ptr[seg_rows[:-1]], lay.inter_ptr[seg_rows[1:]]], 1).reshape(-1)
    seg_xr = seg_xr.astype(np.int64)
    if lay.intra_col is None:  # columns live on the device: caller rebases (cdk_gen_rebase)
        sch = Schedule(n_cta, stage_threads(), int(smem_nodes), int(rows_cap), seg_rblk, seg_win,
                       seg_base, np.asarray(cta_seg, dtype=np.int32), seg_lpr, None, xs_cap,
                       seg_xr)
        sch.row_delta = delta.astype(np.int32)
        return sch
    col = lay.intra_col.copy()
    if np.any(delta != 0):
        d_ent = np.repeat(delta, np.diff(lay.intra_ptr))
        m = col != INTRA_PAD
        newc = col[m].astype(np.int64) + d_ent[m]
        if newc.size and (newc.min() < 0 or newc.max() >= INTRA_PAD):
            raise InputError("rebased intra column out of uint16 range")
        col[m] = newc.astype(np.uint16)
    if bank_order:
        _bank_order(col, _sub_run_ptr(lay), smem_nodes)
    return Schedule(n_cta, stage_threads(), int(smem_nodes), int(rows_cap), seg_rblk, seg_win,
                    seg_base, np.asarray(cta_seg, dtype=np.int32), seg_lpr, col, xs_cap, seg_xr)


@dataclass
class EllLayout:
    """Lane-per-row sliced layout of the ELL kernels (cdk_graph.ell_off ...):
    per rblock, chunk c of lane l is ell_col[(ell_off[b] + 32 c + l) * 8 ..
    +8) and inter column k of lane l is xell_col[xell_off[b] + 32 k + l]."""
    ell_off: np.ndarray  # int64[n_rblk+1], uint4 units
    ell_col: np.ndarray  # uint16[8 * ell_off[-1]]
    xell_off: np.ndarray  # int64[n_rblk+1], int32 units
    xell_col: np.ndarray  # int32[xell_off[-1]], -1 = none
    ell_units: np.ndarray | None = None  # int32[n_units]: rblock of each unit, claim order
    seg_unit: np.ndarray | None = None  # int32[n_seg+1]
    ell_meta: np.ndarray | None = None  # int32[8*n_units] packed unit metadata (or None)

    def slots(self) -> int:
        """intra gather slots (entries + padding) one RHS issues"""
        return int(self.ell_col.shape[0])


# ELL cost model (cycles per CTA, least-squares fit of per-CTA cycles on
# config 2, tools/prof_ell.py): intra slot (one LDS.128 lane, 1/8 of a
# wavefront), inter slot (a global z gather), per-rblock fixed work
# (pointers, epilogue, sincos, partial) and per-segment staging
ELL_SLOT_COST = settings().ell_slot_cost
ELL_XSLOT_COST = settings().ell_xslot_cost
ELL_RBLK_COST = settings().ell_rblk_cost
ELL_SEG_COST = settings().ell_seg_cost


def _ell_call(lay: HostLayout, col, staged, shift, zero_slot, ell_off, out):
    import ctypes

    from ._lib import load_library

    vp = ctypes.c_void_p
    rows_c = np.ascontiguousarray(lay.rblk_row0, dtype=np.int64)
    ptr = np.ascontiguousarray(lay.intra_ptr, dtype=np.int64)
    rc = load_library().cdk_host_ell_intra(
        rows_c.ctypes.data_as(vp), lay.n_rblk, ptr.ctypes.data_as(vp), col.ctypes.data_as(vp),
        staged.ctypes.data_as(vp), shift.ctypes.data_as(vp), int(zero_slot),
        ell_off.ctypes.data_as(vp),
        out.ctypes.data_as(vp) if out is not None else None)
    if rc != 0:
        raise InputError(f"cdk_host_ell_intra failed ({rc})")


def _ell_sizes(lay: HostLayout):
    """(ell_off, xell_off) of the ELL layout (sizes do not depend on the
    segment windows: bank groups are column mod 8 before and after rebasing)"""
    nrb = lay.n_rblk
    col = np.ascontiguousarray(lay.intra_col if lay.intra_col is not None and lay.intra_col.size
                               else np.full(8, INTRA_PAD, np.uint16))
    ell_off = np.zeros(nrb + 1, dtype=np.int64)
    # layout columns are community-local: bank group of the global column
    shift = np.zeros(max(nrb, 1), np.uint8)
    if nrb:
        c = np.maximum(lay.rblk_comm, 0)
        shift[:nrb] = np.where(lay.rblk_comm >= 0, lay.comm_off[c] & 7, 0).astype(np.uint8)
    _ell_call(lay, col, np.zeros(max(nrb, 1), np.uint8), shift, 0, ell_off, None)
    xcnt = np.diff(lay.inter_ptr)
    nx = np.zeros(nrb, dtype=np.int64)
    if nrb:
        rows = lay.rblk_row0
        rb_of_row = np.repeat(np.arange(nrb), np.diff(rows))
        np.maximum.at(nx, rb_of_row, xcnt[int(rows[0]):int(rows[-1])])
    xell_off = np.zeros(nrb + 1, dtype=np.int64)
    np.cumsum(32 * nx, out=xell_off[1:])
    return ell_off, xell_off


def build_ell(lay: HostLayout, sch: Schedule) -> EllLayout:
    """ELL arrays from the rebased intra columns (cdk_host_ell_intra: each
    quarter-warp step on 8 distinct bank groups) and the inter runs."""
    nrb = lay.n_rblk
    rows = lay.rblk_row0
    seg_of_rb = np.repeat(np.arange(sch.n_seg), np.diff(sch.seg_rblk))
    staged = np.zeros(max(nrb, 1), dtype=np.uint8)
    if nrb:
        staged[:nrb] = (sch.seg_win[seg_of_rb, 1] > sch.seg_win[seg_of_rb, 0]).astype(np.uint8)
    col = np.ascontiguousarray(sch.intra_col if sch.intra_col.size else
                               np.full(8, INTRA_PAD, np.uint16))
    shift = np.zeros(max(nrb, 1), np.uint8)  # rebased columns: base = seg_base
    if nrb:
        shift[:nrb] = (sch.seg_base[seg_of_rb] & 7).astype(np.uint8)
    ell_off, xell_off = _ell_sizes(lay)
    ell_col = np.full(8 * int(ell_off[-1]), INTRA_PAD, dtype=np.uint16)
    if ell_col.size:
        _ell_call(lay, col, staged, shift, sch.smem_nodes, ell_off, ell_col)
    xcnt = np.diff(lay.inter_ptr)
    xell_col = np.full(int(xell_off[-1]), -1, dtype=np.int32)
    if nrb and lay.nnz_inter:
        r = np.repeat(np.arange(lay.n_rows, dtype=np.int64), xcnt)
        k = np.arange(r.shape[0], dtype=np.int64) - lay.inter_ptr[r]
        b = np.searchsorted(rows, r, side="right") - 1
        if np.any((r < rows[0]) | (r >= rows[-1])):
            raise InputError("inter entries outside the rblocks")
        xell_col[xell_off[b] + 32 * k + (r - rows[b])] = lay.inter_col
    units, seg_unit = _ell_units(ell_off, xell_off, sch)
    meta = _ell_meta(lay, sch, ell_off, xell_off, units, seg_unit)
    return EllLayout(ell_off, ell_col, xell_off, xell_col, units, seg_unit, meta)


def _ell_meta(lay: HostLayout, sch: Schedule, ell_off, xell_off, units, seg_unit):
    """packed per-unit metadata (cdk_graph.ell_meta): the kernel reads one
    unit's rblock, rows, chunk and inter ranges and community slot in one
    round trip instead of three dependent lookups; None if offsets overflow
    int32"""
    if ell_off[-1] >= 2**31 or xell_off[-1] >= 2**31 or lay.n_rows >= 2**31:
        return None
    rb = units.astype(np.int64)
    nu = rb.shape[0]
    meta = np.zeros((nu, 8), dtype=np.int64)
    if nu == 0:
        return meta.astype(np.int32).reshape(-1)
    rows = lay.rblk_row0
    seg = np.repeat(np.arange(sch.n_seg), np.diff(seg_unit))
    c = lay.rblk_comm[rb].astype(np.int64)
    cA = lay.rblk_comm[sch.seg_rblk[seg]].astype(np.int64)
    ci = np.where(c >= 0, c - cA, 255)
    if np.any((ci < 0) | ((ci >= SEG_MAX_COMM) & (ci != 255))):
        return None
    meta[:, 0] = ell_off[rb]
    meta[:, 1] = xell_off[rb]
    meta[:, 2] = rows[rb]
    meta[:, 3] = rb
    meta[:, 4] = (ell_off[rb + 1] - ell_off[rb]) // 32
    meta[:, 5] = (xell_off[rb + 1] - xell_off[rb]) // 32
    meta[:, 6] = rows[rb + 1] - rows[rb]
    meta[:, 7] = ci
    return meta.astype(np.int32).reshape(-1)


def _ell_units(ell_off, xell_off, sch: Schedule):
    """Work units of the ELL kernels: one per rblock; each segment's units are
    listed longest first (the warps' claim order), ties by rblock.  (Splitting
    long rblocks into parts that meet through a counter was measured slower on
    config 2 at every part size and removed.)"""
    nch = np.diff(ell_off) // 32
    nx = np.diff(xell_off) // 32
    units, seg_unit = [], [0]
    for si in range(sch.n_seg):
        a, z = int(sch.seg_rblk[si]), int(sch.seg_rblk[si + 1])
        rb = np.arange(a, z)
        work = nch[rb] * 8 + nx[rb]
        units.append(rb[np.lexsort((rb, -work))])
        seg_unit.append(seg_unit[-1] + rb.shape[0])
    units = (np.concatenate(units) if units else np.zeros(0, np.int64)).astype(np.int32)
    return units, np.asarray(seg_unit, dtype=np.int32)


SEG_INTER_PHASE = 256  # include/commdyn_cuda.h CDK_SEG_INTER_PHASE
INTER_PHASE_MIN = 16.0  # mean inter entries per row above which a segment runs the inter phase


def _comm_modes(lay: HostLayout):
    """Gather mode per community (and for the NONE pool): lanes per row (rows
    in flight matter more than lanes per row — measured: 16/32 lanes per row
    double the gather time) | SEG_INTER_PHASE for inter-heavy rows.  Decided per community from its own rows, so every
    shard of a multi-GPU run picks the same mode for the same rows (bitwise
    equal trajectories); segments never mix modes.  CDK_LPR and
    CDK_INTER_PHASE (0/1) override for experiments."""
    import os

    off = lay.comm_off
    lam = np.maximum(np.diff(off), 1)
    lens = (lay.intra_ptr[off[1:]] - lay.intra_ptr[off[:-1]]) / lam
    xl = (lay.inter_ptr[off[1:]] - lay.inter_ptr[off[:-1]]) / lam
    # 8 lanes everywhere: a per-community 4/8 choice split config 2 into 24%
    # more segments and cost 15% (segments cannot mix lane counts)
    st = settings()
    lpr = np.full(lens.shape[0], st.lpr, dtype=np.int32)
    fx = st.inter_phase
    sep = (np.full(lens.shape[0], fx == 1) if fx in (0, 1) else xl > INTER_PHASE_MIN)
    mode = (lpr | np.where(sep, SEG_INTER_PHASE, 0)).astype(np.int32)
    pool = st.lpr | (SEG_INTER_PHASE if fx == 1 else 0)
    return mode, int(pool)


def _sub_run_ptr(lay: HostLayout) -> np.ndarray:
    """run boundaries for the bank ordering: rows, split at pass sub-runs"""
    if lay.intra_split is None:
        return lay.intra_ptr
    sp = lay.intra_split
    extra = [lay.intra_ptr[:-1][sp != 0] + 8 * ((sp[sp != 0] >> np.uint64(16 * q)) &
                                                np.uint64(0xFFFF)).astype(np.int64)
             for q in range(MAX_PASS - 1)]
    return np.unique(np.concatenate([lay.intra_ptr] + extra))


def _bank_order(col: np.ndarray, ptr: np.ndarray, smem_nodes: int) -> None:
    """Native in-place bank-conflict-free ordering of every row's intra run."""
    import ctypes

    from ._lib import load_library

    if col.size == 0:
        return
    lib = load_library()
    col = np.ascontiguousarray(col)
    ptr = np.ascontiguousarray(ptr, dtype=np.int64)
    rc = lib.cdk_host_bank_order(col.ctypes.data_as(ctypes.c_void_p),
                                 ptr.ctypes.data_as(ctypes.c_void_p), ptr.shape[0] - 1,
                                 INTRA_PAD, int(smem_nodes) & 7)
    if rc != 0:
        raise InputError("cdk_host_bank_order failed")


INTER_SWEEP_BYTES = 48 << 20  # z above this: block-phased inter sweep (cdk_graph.inter_blocks)
INTER_BLOCK_BYTES = 40e6  # target z bytes per column block


def inter_blocking(n_rows: int) -> tuple[int, int]:
    """(inter_blocks, inter_block_nodes) for a graph of n_rows (CDK_INTER_BLOCKS
    overrides the block count; 0 disables)."""
    forced = settings().inter_blocks
    if forced is not None:
        nb = forced
    elif n_rows * 16 > INTER_SWEEP_BYTES:
        nb = int(min(4, max(2, np.ceil(n_rows * 16 / INTER_BLOCK_BYTES))))
    else:
        nb = 0
    if nb <= 0 or n_rows < 16:
        return 0, 0
    nb = min(nb, 4)
    return nb, int((n_rows + nb - 1) // nb + 7) // 8 * 8


def _attach_inter_split(self, lay_n_rows: int) -> None:
    """compute cdk_graph.inter_split on the device when the sweep is on"""
    import torch

    from ._lib import check, load_library

    nb, bn = inter_blocking(lay_n_rows)
    self.inter_blocks, self.inter_block_nodes = nb, bn
    if nb < 2:  # 0: off; 1: one block (separate inter launch, no split needed)
        return
    t = self._t
    t["inter_split"] = torch.zeros(lay_n_rows, dtype=torch.int64, device=self.device)
    check(load_library().cdk_inter_split(lay_n_rows, t["inter_ptr"].data_ptr(),
                                         t["inter_col"].data_ptr(), nb, bn,
                                         t["inter_split"].data_ptr(),
                                         torch.cuda.current_stream(self.device).cuda_stream),
          "inter_split")


class DeviceGraph:
    """Device-resident layout + schedule; owns the torch tensors behind the
    cdk_graph struct handed to the C ABI."""

    def __init__(self, dec: Decomposition, device=None, sm_count: int | None = None,
                 row_range=None, smem_budget: int = SMEM_BUDGET):
        import torch

        from ._lib import CdkGraph

        dev = torch.device(device if device is not None else "cuda")
        # ELL kernels unless the graph needs the inter sweep or the caller
        # asked for the row-group kernels' shared-memory budget
        ell = (ell_enabled() and inter_blocking(int(dec.n_nodes))[0] == 0
               and smem_budget == SMEM_BUDGET)
        if sm_count is None:
            sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
            sm_count *= ell_ctas_per_sm() if ell else ctas_per_sm()
        lay = build_layout(dec, row_range=row_range,
                           pass_nodes=(1 << 30) if ell else window_nodes(ROWS_CAP, smem_budget),
                           split_heavy=not ell)
        sch = build_schedule(lay, sm_count=sm_count, smem_budget=smem_budget, ell=ell)
        self.row_range = (0, lay.n_rows) if row_range is None else tuple(int(x) for x in row_range)
        self.layout = lay
        self.n_rows = lay.n_rows
        self.n_comm = lay.n_comm
        self.device = dev
        self._upload(lay, sch)
        if ell and ell_calibrate_iters() > 0 and lay.n_rblk > sch.n_cta:
            self._calibrate(lay, sm_count, smem_budget)

    def _calibrate(self, lay, sm_count, smem_budget):
        """Re-cut the CTA ranges from measured per-CTA cycles: the cost model
        balances the planner's features, but what is left of the CTA spread
        is stable across launches (tools/prof_stab.py), so each rblock's cost
        is rescaled by its CTA's measured/modelled ratio and the cuts are
        redone (ELL_CAL_ITERS times, keeping the fastest schedule)."""
        import ctypes

        import torch

        from ._lib import check, load_library

        lib = load_library()
        n = lay.n_rows
        scale = np.ones(lay.n_rblk)
        dev = self.device
        theta = torch.zeros(n + 4, dtype=torch.float64, device=dev)
        omega = torch.zeros(n + 4, dtype=torch.float64, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream

        def measure():
            nb = int(lib.cdk_kuramoto_workspace_bytes(ctypes.byref(self.struct)))
            ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=dev)
            cyc = torch.zeros(self.schedule.n_cta, dtype=torch.int64, device=dev)
            gp = ctypes.byref(self.struct)
            check(lib.cdk_kuramoto_prepare(gp, theta.data_ptr(), ws.data_ptr(), stream), "prepare")
            best = None
            for _ in range(5):  # min over launches: drops one-off noise
                check(lib.cdk_kuramoto_stage_cycles(gp, theta.data_ptr(), omega.data_ptr(), 0.0,
                                                    0.01, ws.data_ptr(), cyc.data_ptr(), stream),
                      "stage_cycles")
                c = cyc.cpu().numpy().astype(np.float64)
                best = c if best is None else np.minimum(best, c)
            return best

        cur = measure()
        best_max, best = cur.max(), (self.schedule, self._t, self.struct)
        for _ in range(ell_calibrate_iters()):
            sch = self.schedule
            rows_rb = sch.seg_rblk[sch.cta_seg]  # first rblock of each CTA (+ end)
            cta_of_rb = np.repeat(np.arange(sch.n_cta), np.diff(rows_rb))
            model = np.asarray(sch.rb_cost, dtype=np.float64)
            cta_model = np.bincount(cta_of_rb, weights=model[rows_rb[0]:rows_rb[-1]],
                                    minlength=sch.n_cta)
            ratio = np.where(cta_model > 0, cur / np.maximum(cta_model, 1e-9), 0.0)
            ratio = ratio / max(np.mean(ratio[ratio > 0]), 1e-12) if np.any(ratio > 0) else ratio
            r_rb = np.ones(lay.n_rblk)
            r_rb[rows_rb[0]:rows_rb[-1]] = np.where(ratio[cta_of_rb] > 0, ratio[cta_of_rb], 1.0)
            scale = scale * np.sqrt(r_rb)  # damped
            sch2 = build_schedule(lay, sm_count=sm_count, smem_budget=smem_budget, ell=True,
                                  rb_scale=scale)
            self._upload(lay, sch2)
            cur = measure()
            if cur.max() < best_max:
                best_max, best = cur.max(), (self.schedule, self._t, self.struct)
        self.schedule, self._t, self.struct = best
        self.calibration = {"cta_max_cycles": float(best_max)}

    def _upload(self, lay, sch):
        import torch

        from ._lib import CdkGraph

        dev = self.device
        self.schedule = sch

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        # uint16 has no torch dtype with from_numpy in older builds: ship as int16 bits
        pad = np.zeros(4, dtype=np.int64)
        self._t = {
            "comm_off": up(lay.comm_off),
            # bulk copies read the pointer slices in 16-byte units: 4 entries of slack
            "intra_ptr": up(np.concatenate([lay.intra_ptr, pad + lay.intra_ptr[-1]])),
            "intra_col": up(sch.intra_col.view(np.int16)),
            "inter_ptr": up(np.concatenate([lay.inter_ptr, pad + lay.inter_ptr[-1]])),
            "inter_col": up(lay.inter_col),
            "rblk_row0": up(lay.rblk_row0),
            "rblk_comm": up(lay.rblk_comm),
            "comm_rblk_off": up(lay.comm_rblk_off),
            "seg_rblk": up(sch.seg_rblk),
            "seg_win": up(sch.seg_win.reshape(-1)),
            "seg_base": up(sch.seg_base),
            "cta_seg": up(sch.cta_seg),
            "seg_lpr": up(sch.seg_lpr if sch.n_seg else np.zeros(1, np.int32)),
            "seg_xr": up(sch.seg_xr if sch.n_seg else np.zeros(2, np.int64)),
        }
        if lay.intra_split is not None:
            self._t["intra_split"] = up(lay.intra_split.view(np.int64))
        # keep a 16-byte tail on intra_col so uint4 loads never run past the allocation
        if self._t["intra_col"].numel() == 0:
            self._t["intra_col"] = torch.full((8,), -1, dtype=torch.int16, device=dev)
        if self._t["inter_col"].numel() == 0:
            self._t["inter_col"] = torch.zeros(4, dtype=torch.int32, device=dev)
        if sch.ell is not None:
            e = sch.ell
            self._t["ell_off"] = up(e.ell_off)
            self._t["ell_col"] = up(e.ell_col.view(np.int16) if e.ell_col.size
                                    else np.full(8, -1, np.int16))
            self._t["xell_off"] = up(e.xell_off)
            self._t["xell_col"] = up(e.xell_col if e.xell_col.size else np.full(4, -1, np.int32))
            self._t["ell_units"] = up(e.ell_units if e.ell_units.size else np.zeros(2, np.int32))
            self._t["seg_unit"] = up(e.seg_unit)
            if e.ell_meta is not None and settings().ell_meta:
                self._t["ell_meta"] = up(e.ell_meta if e.ell_meta.size else np.zeros(8, np.int32))
        _attach_inter_split(self, lay.n_rows)
        t = self._t
        self.struct = CdkGraph(
            n_rows=lay.n_rows, n_comm=lay.n_comm,
            comm_off=t["comm_off"].data_ptr(), intra_ptr=t["intra_ptr"].data_ptr(),
            intra_col=t["intra_col"].data_ptr(), inter_ptr=t["inter_ptr"].data_ptr(),
            inter_col=t["inter_col"].data_ptr(),
            n_rblk=lay.n_rblk, n_seg=sch.n_seg, n_cta=sch.n_cta, cta_threads=sch.cta_threads,
            smem_nodes=sch.smem_nodes, seg_rows_cap=sch.seg_rows_cap,
            rblk_row0=t["rblk_row0"].data_ptr(), rblk_comm=t["rblk_comm"].data_ptr(),
            comm_rblk_off=t["comm_rblk_off"].data_ptr(), seg_rblk=t["seg_rblk"].data_ptr(),
            seg_win=t["seg_win"].data_ptr(), seg_base=t["seg_base"].data_ptr(),
            cta_seg=t["cta_seg"].data_ptr(), seg_lpr=t["seg_lpr"].data_ptr(),
            intra_split=t["intra_split"].data_ptr() if "intra_split" in t else None,
            inter_blocks=self.inter_blocks, inter_block_nodes=self.inter_block_nodes,
            inter_split=t["inter_split"].data_ptr() if "inter_split" in t else None,
            xs_cap=sch.xs_cap,
            seg_xr=t["seg_xr"].data_ptr(),
            ell_off=t["ell_off"].data_ptr() if "ell_off" in t else None,
            ell_col=t["ell_col"].data_ptr() if "ell_off" in t else None,
            xell_off=t["xell_off"].data_ptr() if "ell_off" in t else None,
            xell_col=t["xell_col"].data_ptr() if "ell_off" in t else None,
            ell_units=t["ell_units"].data_ptr() if "ell_off" in t else None,
            seg_unit=t["seg_unit"].data_ptr() if "ell_off" in t else None,
            ell_meta=t["ell_meta"].data_ptr() if "ell_meta" in t else None,
        )

    def device_bytes(self) -> int:
        return int(sum(v.numel() * v.element_size() for v in self._t.values()))

    @classmethod
    def from_device_csr(cls, lay: "HostLayout", intra_col_dev, inter_col_dev, device,
                        sm_count: int | None = None, split_dev=None,
                        smem_budget: int = SMEM_BUDGET, bank_order: bool = True,
                        row_range=None):
        """Graph whose columns were generated on the device (config 5): the
        schedule is planned from the host copies of the row pointers and the
        intra columns are rebased in place on the device."""
        import torch

        from ._lib import CdkGraph, check, load_library

        self = cls.__new__(cls)
        dev = torch.device(device)
        if sm_count is None:
            sm_count = torch.cuda.get_device_properties(dev).multi_processor_count * ctas_per_sm()
        sch = build_schedule(lay, sm_count=sm_count, smem_budget=smem_budget)
        self.layout, self.schedule = lay, sch
        self.n_rows, self.n_comm, self.device = lay.n_rows, lay.n_comm, dev
        self.row_range = (0, lay.n_rows) if row_range is None else tuple(int(x) for x in row_range)

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        pad = np.zeros(4, dtype=np.int64)
        self._t = {
            "comm_off": up(lay.comm_off),
            "intra_ptr": up(np.concatenate([lay.intra_ptr, pad + lay.intra_ptr[-1]])),
            "intra_col": intra_col_dev,
            "inter_ptr": up(np.concatenate([lay.inter_ptr, pad + lay.inter_ptr[-1]])),
            "inter_col": inter_col_dev,
            "rblk_row0": up(lay.rblk_row0), "rblk_comm": up(lay.rblk_comm),
            "comm_rblk_off": up(lay.comm_rblk_off), "seg_rblk": up(sch.seg_rblk),
            "seg_win": up(sch.seg_win.reshape(-1)), "seg_base": up(sch.seg_base),
            "cta_seg": up(sch.cta_seg), "seg_lpr": up(sch.seg_lpr),
            "seg_xr": up(sch.seg_xr),
        }
        if split_dev is not None:
            self._t["intra_split"] = split_dev
        _attach_inter_split(self, lay.n_rows)
        t = self._t
        delta = up(sch.row_delta)
        lib = load_library()
        stream = torch.cuda.current_stream().cuda_stream
        check(lib.cdk_gen_rebase(lay.n_rows, t["intra_ptr"].data_ptr(), delta.data_ptr(),
                                 t["intra_col"].data_ptr(), stream), "gen_rebase")
        del delta
        if bank_order:  # device twin of the host path's _bank_order (out of place)
            ordered = torch.empty_like(t["intra_col"])
            ordered[-8:].fill_(-1)
            check(lib.cdk_bank_order(lay.n_rows, t["intra_ptr"].data_ptr(),
                                     t["intra_split"].data_ptr() if "intra_split" in t else None,
                                     t["intra_col"].data_ptr(), ordered.data_ptr(),
                                     int(sch.smem_nodes) & 7, stream), "bank_order")
            t["intra_col"] = ordered
        self.struct = CdkGraph(
            n_rows=lay.n_rows, n_comm=lay.n_comm,
            comm_off=t["comm_off"].data_ptr(), intra_ptr=t["intra_ptr"].data_ptr(),
            intra_col=t["intra_col"].data_ptr(), inter_ptr=t["inter_ptr"].data_ptr(),
            inter_col=t["inter_col"].data_ptr(),
            n_rblk=lay.n_rblk, n_seg=sch.n_seg, n_cta=sch.n_cta, cta_threads=sch.cta_threads,
            smem_nodes=sch.smem_nodes, seg_rows_cap=sch.seg_rows_cap,
            rblk_row0=t["rblk_row0"].data_ptr(), rblk_comm=t["rblk_comm"].data_ptr(),
            comm_rblk_off=t["comm_rblk_off"].data_ptr(), seg_rblk=t["seg_rblk"].data_ptr(),
            seg_win=t["seg_win"].data_ptr(), seg_base=t["seg_base"].data_ptr(),
            cta_seg=t["cta_seg"].data_ptr(), seg_lpr=t["seg_lpr"].data_ptr(),
            intra_split=t["intra_split"].data_ptr() if "intra_split" in t else None,
            inter_blocks=self.inter_blocks, inter_block_nodes=self.inter_block_nodes,
            inter_split=t["inter_split"].data_ptr() if "inter_split" in t else None,
            xs_cap=sch.xs_cap,
            seg_xr=t["seg_xr"].data_ptr(),
        )
        return self
