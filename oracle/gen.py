"""TEST INFRASTRUCTURE ONLY — numpy restatement of the device graph generator
(paper_2203_16657_b200/csrc/gen.cu, model in paper_2203_16657_b200/gen.py).

The reference has no large-graph generator (config 5 is specified only by its
parameters, BASELINE.json configs[4]); the generator's contract is this
restatement: the same counter-based hashes evaluated with numpy uint32
arithmetic, producing the CSR bit for bit.  The Kuramoto RHS on the result is
then checked against the reference-derived oracle (oracle/cia.py).
Only tests/ may import this module.
"""

from __future__ import annotations

import numpy as np

M32 = np.uint32(0xFFFFFFFF)


def mix32(x):
    """csrc/gen.cu mix32 (uint32 wrap-around arithmetic)."""
    x = np.asarray(x, dtype=np.uint32)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint32(16))
        x = x * np.uint32(0x7FEB352D)
        x = x ^ (x >> np.uint32(15))
        x = x * np.uint32(0x846CA68B)
        x = x ^ (x >> np.uint32(16))
    return x


def hash4(seed: int, a, b, c):
    """csrc/gen.cu hash4: seed mixed in two halves, then a, b + k1, c + k2."""
    s_lo = np.uint32(seed & 0xFFFFFFFF)
    s_hi = np.uint32((seed >> 32) & 0xFFFFFFFF)
    h = mix32(s_lo ^ np.uint32(0x9E3779B9))
    h = mix32(h ^ s_hi ^ np.uint32(0x85EBCA6B))
    h = mix32(h ^ np.asarray(a, np.uint32))
    with np.errstate(over="ignore"):
        b = np.asarray(b, np.uint32) + np.uint32(0x27D4EB2F)
        c = np.asarray(c, np.uint32) + np.uint32(0x165667B1)
    h = mix32(h ^ b)
    h = mix32(h ^ c)
    return h


def intra_missing(seed: int, c: int, lam: int, thr: int):
    """Boolean [lam, lam] missing-pair matrix of community c (diagonal False)."""
    a = np.arange(lam, dtype=np.uint32)
    lo = np.minimum(a[:, None], a[None, :])
    hi = np.maximum(a[:, None], a[None, :])
    with np.errstate(over="ignore"):
        m = hash4(seed, np.full_like(lo, c), lo, hi) < np.uint32(thr)
    np.fill_diagonal(m, False)
    return m


def inter_endpoints(seed: int, n_edges: int, node_cdf: np.ndarray):
    """(u, v) int64[n_edges] endpoint nodes of the sampled inter edges."""
    e = np.arange(n_edges, dtype=np.uint64)
    lo = (e & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    hi = (e >> np.uint64(32)).astype(np.uint32)
    s = seed ^ 0xABCDEF12345
    out = []
    with np.errstate(over="ignore"):
        for k in (0, 1):
            h = hash4(s, lo, hi, np.full_like(lo, k))
            u = (h.astype(np.float64) + 0.5) * (1.0 / 4294967296.0)
            out.append(np.minimum(np.searchsorted(node_cdf, u, side="right"),
                                  node_cdf.shape[0] - 1).astype(np.int64))
    return out[0], out[1]


def _passes(c0: int, lam: int, wn: int) -> int:
    """window passes of a community (csrc/gen.cu pass_geom): 1, or 2..4"""
    w0 = c0 // 8 * 8
    width = (c0 + lam + 7) // 8 * 8 - w0
    if wn and width > wn:
        q = (width + wn - 1) // wn
        return q if q <= 4 else 1
    return 1


def generate_csr(seed: int, offsets: np.ndarray, node_cdf: np.ndarray, n_edges: int, thr: int,
                 pass_nodes: int = 0):
    """The generator's output: (intra_ptr, intra_col uint16 local ascending,
    padded with 0xFFFF to multiples of 8 per window-pass sub-run; inter_ptr,
    inter_col int32 sorted unique; intra_split uint64) plus the undirected
    triples (iu, iv, sgn) with the in-community diagonal, i.e. the reference's
    sparse-correction wire format."""
    n = int(node_cdf.shape[0])
    off = np.asarray(offsets, np.int64)
    m = off.shape[0] - 1
    rows_i, cols_i = [], []
    intra_len = np.zeros(n, np.int64)
    split = np.zeros(n, np.uint64)
    runs = []  # per community: (rows, [per pass (row-local entries)])
    for c in range(m):
        c0, lam = int(off[c]), int(off[c + 1] - off[c])
        mm = intra_missing(seed, c, lam, thr)
        r, q = np.nonzero(mm)
        rows_i.append(r + c0)
        cols_i.append(q.astype(np.int64))
        np_c = _passes(c0, lam, pass_nodes)
        w0 = c0 // 8 * 8
        bounds = [0] + [min(max(w0 + k * pass_nodes - c0, 0), lam) for k in range(1, np_c)] + [lam]
        cnt = np.stack([np.count_nonzero(mm[:, bounds[k]:bounds[k + 1]], axis=1)
                        for k in range(np_c)], axis=1)
        pad = (cnt + 7) // 8 * 8
        intra_len[c0:c0 + lam] = pad.sum(axis=1)
        sub = np.cumsum(pad, axis=1) - pad
        for k in range(1, np_c):
            split[c0:c0 + lam] |= (sub[:, k] // 8).astype(np.uint64) << np.uint64(16 * (k - 1))
        runs.append((c0, lam, mm, bounds, sub))
    ri = np.concatenate(rows_i) if rows_i else np.zeros(0, np.int64)
    ci = np.concatenate(cols_i) if cols_i else np.zeros(0, np.int64)
    intra_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(intra_len, out=intra_ptr[1:])
    intra_col = np.full(int(intra_ptr[-1]), 0xFFFF, np.uint16)
    for c0, lam, mm, bounds, sub in runs:
        for a in range(lam):
            for k in range(len(bounds) - 1):
                cols = np.nonzero(mm[a, bounds[k]:bounds[k + 1]])[0] + bounds[k]
                s = intra_ptr[c0 + a] + sub[a, k]
                intra_col[s:s + cols.shape[0]] = cols.astype(np.uint16)

    comm = np.full(n, -1, np.int64)
    comm[: off[-1]] = np.repeat(np.arange(m), np.diff(off))
    u, v = inter_endpoints(seed, n_edges, node_cdf)
    cu = np.where(comm[u] >= 0, comm[u], -1 - u)
    cv = np.where(comm[v] >= 0, comm[v], -1 - v)
    keep = cu != cv
    u, v = u[keep], v[keep]
    rx = np.concatenate([u, v])
    cx = np.concatenate([v, u])
    key = np.unique(rx * n + cx)
    rx, cx = key // n, key % n
    inter_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rx, minlength=n), out=inter_ptr[1:])
    inter_col = cx.astype(np.int32)

    # undirected triples: missing pairs (sgn -1) + diagonal, inter pairs (+1)
    up = ri < ci + off[np.maximum(comm[ri], 0)]
    mi_u = ri[up]
    mi_v = ci[up] + off[comm[ri[up]]]
    xu = rx[rx < cx]
    xv = cx[rx < cx]
    diag = np.arange(off[-1], dtype=np.int64)
    iu = np.concatenate([mi_u, diag, xu])
    iv = np.concatenate([mi_v, diag, xv])
    sg = np.concatenate([-np.ones(mi_u.shape[0] + diag.shape[0]), np.ones(xu.shape[0])])
    order = np.lexsort((iv, iu))
    return (intra_ptr, intra_col, inter_ptr, inter_col, split), (iu[order], iv[order], sg[order])
