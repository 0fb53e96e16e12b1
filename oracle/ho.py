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
