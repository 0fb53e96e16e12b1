"""ORACLE — TEST INFRASTRUCTURE ONLY.

Higher-order (triadic) Kuramoto on the 3-cliques of a graph (BASELINE config
3).  The reference has no triangle model; its only
higher-order kernel is ``ho_naive_block`` (``_kernels.py:398-428``, the
all-to-all block sum), which pins the dense (Z^2) part of the CIA expansion
(tests/test_oracle.py).  Model (open decisions fixed in DESIGN.md §9):

    theta'_i = omega_i + (K1/N) sum_j a_ij sin(theta_j - theta_i)
                       + (K2/N^2) sum_{(j,k) ordered, {i,j,k} triangle}
                                  sin(theta_j + theta_k - 2 theta_i)

* ``ho_rhs_direct``   literal evaluation with dense matrices,
                      S = diag(A Z A Z A) (O(N^3); N <= ~3000).
* ``ho_rhs_cia``      CPU restatement of the CIA inclusion-exclusion over the
                      missing-edge graph (scipy.sparse), O(nnz + triangles).
"""

from __future__ import annotations

import numpy as np


def ho_rhs_direct(theta, omega, adj, k1, k2, norm=None):
    n = theta.shape[0]
    norm = float(norm if norm is not None else n)
    z = np.exp(1j * theta)
    a = np.asarray(adj, dtype=np.float64)
    pair = (a @ z)
    b = a * z[None, :]
    c = b @ b
    s = (c * a.T).sum(axis=1)  # sum_{j,k} a_ij z_j a_jk z_k a_ki
    zc = np.conj(z)
    return omega + (k1 / norm) * np.imag(pair * zc) + (k2 / norm**2) * np.imag(s * zc * zc)


def ho_rhs_cia(theta, omega, dec, k1, k2, norm=None, inter_triangles=None):
    """CIA form.  ``dec`` is a Decomposition; ``inter_triangles`` int64 [T,3]
    (triangles not inside one community)."""
    import scipy.sparse as sp

    n = theta.shape[0]
    norm = float(norm if norm is not None else n)
    z = np.exp(1j * theta)
    rows, cols, sg = dec.directed()
    mi = sg < 0
    M = sp.csr_matrix((np.ones(int(mi.sum())), (rows[mi], cols[mi])), shape=(n, n))
    X = sp.csr_matrix((np.ones(int((~mi).sum())), (rows[~mi], cols[~mi])), shape=(n, n))
    off = dec.offsets
    comm = dec.partition.comm_of_permuted()
    m = dec.partition.n_comm
    Zc = np.zeros(m, complex)
    Z2c = np.zeros(m, complex)
    inc = comm >= 0
    np.add.at(Zc, comm[inc], z[inc])
    np.add.at(Z2c, comm[inc], z[inc] ** 2)
    Y = M @ z            # proper missing neighbours
    V = M @ (z * z)
    P = z * Y
    Wc = np.zeros(m, complex)
    np.add.at(Wc, comm[inc], P[inc])
    U = M @ P
    # ordered missing triangles through i: T_i = sum_{j,k} m_ij m_jk m_ki z_j z_k
    MZ = M @ sp.diags(z)
    T = np.asarray((MZ @ MZ).multiply(M.T).sum(axis=1)).ravel() if M.nnz else np.zeros(n, complex)
    pair = np.where(inc, Zc[np.maximum(comm, 0)], 0) - Y + X @ z
    S = np.zeros(n, complex)
    ci = np.maximum(comm, 0)
    Zi = Zc[ci] - z
    Z2i = Z2c[ci] - z * z
    S_in = Zi * Zi - Z2i - 2 * Y * Zi + V - Wc[ci] + Y * Y + 2 * U - T
    S[inc] = S_in[inc]
    if inter_triangles is not None and len(inter_triangles):
        t = np.asarray(inter_triangles, dtype=np.int64)
        for a_, b_, c_ in ((0, 1, 2), (1, 0, 2), (2, 0, 1)):
            np.add.at(S, t[:, a_], 2 * z[t[:, b_]] * z[t[:, c_]])
    zc = np.conj(z)
    return omega + (k1 / norm) * np.imag(pair * zc) + (k2 / norm**2) * np.imag(S * zc * zc)


def spanning_triangles_ref(dec):
    """Triangles of the graph with at least one inter-community edge (an
    independent enumeration for the oracle: for every inter edge (u, v), the
    common neighbours of u and v in the full adjacency D - M + X).  int64 [T, 3]."""
    import scipy.sparse as sp

    n = dec.n_nodes
    rows, cols, sg = dec.directed()
    comm = dec.partition.comm_of_permuted()
    off = dec.offsets
    parts = []
    for c in range(dec.partition.n_comm):  # D: complete community blocks
        idx = np.arange(off[c], off[c + 1])
        r, q = np.meshgrid(idx, idx, indexing="ij")
        keep = r != q
        parts.append((r[keep], q[keep]))
    dr = np.concatenate([p[0] for p in parts]) if parts else np.zeros(0, np.int64)
    dc = np.concatenate([p[1] for p in parts]) if parts else np.zeros(0, np.int64)
    A = sp.csr_matrix((np.ones(dr.shape[0]), (dr, dc)), shape=(n, n))
    A = A + sp.csr_matrix((sg.astype(np.float64), (rows, cols)), shape=(n, n))
    A.eliminate_zeros()
    A.sort_indices()
    ptr, col = A.indptr, A.indices
    found = set()
    xi = np.nonzero((sg > 0) & (rows < cols))[0]
    for u, v in zip(rows[xi].tolist(), cols[xi].tolist()):
        w = np.intersect1d(col[ptr[u]:ptr[u + 1]], col[ptr[v]:ptr[v + 1]], assume_unique=True)
        for x in w.tolist():
            found.add(tuple(sorted((u, v, x))))
    del comm
    if not found:
        return np.zeros((0, 3), dtype=np.int64)
    return np.array(sorted(found), dtype=np.int64)


def missing_triangles_ref(M):
    """Triangles {i<j<k} of the (symmetric, 0/1 CSR) missing graph M, by
    intersecting upper neighbour lists.  int64 [T, 3]."""
    import scipy.sparse as sp

    U = sp.triu(M, 1).tocsr()
    U.sort_indices()
    ptr, col = U.indptr, U.indices
    n = M.shape[0]
    out = []
    for i in range(n):
        ni = col[ptr[i]:ptr[i + 1]]
        if ni.shape[0] < 2:
            continue
        # for each j in N+(i): k in N+(i) ∩ N+(j)
        js = np.repeat(ni, ptr[ni + 1] - ptr[ni])
        ks = np.concatenate([col[ptr[j]:ptr[j + 1]] for j in ni]) if ni.shape[0] else ni
        hit = np.isin(ks, ni, assume_unique=False)
        if hit.any():
            out.append(np.stack([np.full(int(hit.sum()), i), js[hit], ks[hit]], 1))
    if not out:
        return np.zeros((0, 3), dtype=np.int64)
    return np.concatenate(out).astype(np.int64)


class HoCia:
    """``ho_rhs_cia`` with the graph-dependent pieces precomputed once (for
    long trajectories): the missing-graph triangle term T_i = sum over ordered
    (j, k) of z_j z_k is accumulated from the enumerated missing triangles
    instead of the sparse triple product; spanning triangles from
    ``spanning_triangles_ref``.  Same formula as ``ho_rhs_cia`` otherwise."""

    def __init__(self, dec, span=None):
        import scipy.sparse as sp

        n = dec.n_nodes
        self.n = n
        rows, cols, sg = dec.directed()
        mi = sg < 0
        self.M = sp.csr_matrix((np.ones(int(mi.sum())), (rows[mi], cols[mi])), shape=(n, n))
        self.X = sp.csr_matrix((np.ones(int((~mi).sum())), (rows[~mi], cols[~mi])), shape=(n, n))
        self.comm = dec.partition.comm_of_permuted()
        self.m = dec.partition.n_comm
        self.inc = self.comm >= 0
        self.ci = np.maximum(self.comm, 0)
        self.tri = missing_triangles_ref(self.M)
        self.span = spanning_triangles_ref(dec) if span is None else np.asarray(span, np.int64)

    def _csum(self, v):
        out = np.zeros(self.m, complex)
        np.add.at(out, self.comm[self.inc], v[self.inc])
        return out

    @staticmethod
    def _tri_acc(n, tri, z, scale=2.0):
        out = np.zeros(n, complex)
        if tri.shape[0] == 0:
            return out
        for a_, b_, c_ in ((0, 1, 2), (1, 0, 2), (2, 0, 1)):
            w = scale * z[tri[:, b_]] * z[tri[:, c_]]
            out += np.bincount(tri[:, a_], weights=w.real, minlength=n)
            out += 1j * np.bincount(tri[:, a_], weights=w.imag, minlength=n)
        return out

    def rhs(self, theta, omega, k1, k2, norm=None):
        n = self.n
        norm = float(norm if norm is not None else n)
        z = np.exp(1j * theta)
        ci, inc = self.ci, self.inc
        Zc = self._csum(z)
        Z2c = self._csum(z * z)
        Y = self.M @ z
        V = self.M @ (z * z)
        P = z * Y
        Wc = self._csum(P)
        U = self.M @ P
        T = self._tri_acc(n, self.tri, z)
        pair = np.where(inc, Zc[ci], 0) - Y + self.X @ z
        Zi = Zc[ci] - z
        Z2i = Z2c[ci] - z * z
        S_in = Zi * Zi - Z2i - 2 * Y * Zi + V - Wc[ci] + Y * Y + 2 * U - T
        S = np.where(inc, S_in, 0) + self._tri_acc(n, self.span, z)
        zc = np.conj(z)
        return omega + (k1 / norm) * np.imag(pair * zc) + (k2 / norm**2) * np.imag(S * zc * zc)
