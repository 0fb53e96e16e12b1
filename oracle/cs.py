"""ORACLE — TEST INFRASTRUCTURE ONLY.

Cucker–Smale (BASELINE config 4), 2-D.

* ``cs_rhs_direct``  direct sum over the graph's edge list with the EXACT
                     coupling, through the reference kernel ``pairs_cs``
                     (_kernels.py:297-314) with sgn = +1.
* ``cs_rhs_cia``     CPU restatement of the CIA with the SAME per-community
                     polynomial coefficients and basis as the device path
                     (moments M^f_ij, contraction H = T M, bivariate
                     evaluation) plus the exact sparse correction via
                     ``pairs_cs`` over S (diagonal entries are skipped by the
                     kernel, _kernels.py:309-310).
Parity at 1e-9 is only meaningful against this same-basis restatement; the
CIA vs direct distance is bounded by sup|eta~ - eta| max|v_l - v_m|.
"""

from __future__ import annotations

import numpy as np


def cs_rhs_direct(kern, pos, vel, eu, ev, K, sigma2, beta, norm):
    out = np.zeros_like(vel)
    kern.pairs_cs(eu, ev, pos, vel, 1.0 / norm, K, sigma2, beta, np.ones(eu.shape[0]), out)
    return out


def cs_rhs_cia(kern, pos, vel, dec, plan, K, sigma2, beta, norm):
    from paper_2203_16657_b200.cs import D2, mono_index

    mon = mono_index()
    I = np.array([m[0] for m in mon])
    J = np.array([m[1] for m in mon])
    off = dec.offsets
    out = np.zeros_like(vel)
    for c in range(dec.partition.n_comm):
        sl = slice(off[c], off[c + 1])
        p = (pos[sl] - plan.mu[c]) / plan.L[c]
        xp = p[:, 0:1] ** np.arange(D2 + 1)
        yp = p[:, 1:2] ** np.arange(D2 + 1)
        mono = xp[:, I] * yp[:, J]  # [lam, NMON]
        F = np.column_stack([np.ones(p.shape[0]), vel[sl]])  # f = 1, vx, vy
        Mf = mono.T @ F  # [NMON, 3]
        H = plan.T[c] @ Mf  # [NMON, 3]
        G = mono @ H  # [lam, 3]  (evaluation at the nodes' own scaled positions)
        out[sl] = (G[:, 1:3] - vel[sl] * G[:, 0:1]) / norm
    s = dec.correction
    kern.pairs_cs(s.iu, s.iv, pos, vel, 1.0 / norm, K, sigma2, beta, s.sgn, out)
    return out


def full_edge_list(dec):
    """(eu, ev) int64: every edge {u < v} of the graph D + S (permuted order):
    the present intra-community pairs plus the inter edges — the direct sum's
    input."""
    s = dec.correction
    off = dec.offsets
    od = s.iu != s.iv
    miss = od & (s.sgn < 0)
    n = dec.n_nodes
    mkey = np.sort(s.iu[miss] * n + s.iv[miss])
    eus, evs = [], []
    for c in range(dec.partition.n_comm):
        idx = np.arange(off[c], off[c + 1], dtype=np.int64)
        u, v = np.triu_indices(idx.shape[0], 1)
        u, v = idx[u], idx[v]
        key = u * n + v
        pos = np.searchsorted(mkey, key)
        pos = np.minimum(pos, max(mkey.shape[0] - 1, 0))
        keep = mkey[pos] != key if mkey.shape[0] else np.ones(key.shape[0], bool)
        eus.append(u[keep])
        evs.append(v[keep])
    inter = od & (s.sgn > 0)
    eus.append(s.iu[inter])
    evs.append(s.iv[inter])
    return np.concatenate(eus), np.concatenate(evs)
