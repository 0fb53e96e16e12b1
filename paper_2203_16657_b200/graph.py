"""graph_core (P1): Graph, Partition, SparseCorrection, Decomposition.

Host-side setup that builds the hot path's inputs.  Restates the SPEC
operations the reference declares but does not ship:

* types           SPEC.md:23-48 (Graph, Partition, SparseCorrection, Decomposition)
* planted graph   SPEC.md:61-69 (``planted_partition_graph``)
* decompose       SPEC.md:101-109 (S = PAP^T - D; -1 missing intra pairs and the
                  diagonal, +1 inter edges; sorted coordinate triples)

Sampling is exact independent-Bernoulli per pair via geometric skipping over the
pair index space, so a planted graph at N = 2e5 (config 2) is produced without
enumerating its ~4.5e8 intra pairs.  ``planted_partition_graph`` and
``planted_partition_decomposition`` draw from the same streams, so
``decompose(planted_partition_graph(...))`` equals the direct decomposition.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import InputError

NONE = -1


# ---------------------------------------------------------------------------
# types
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Graph:
    """Undirected, unweighted, no self-loops.  edges: int64 [E, 2], u < v."""

    n_nodes: int
    edges: np.ndarray

    @staticmethod
    def from_pairs(n_nodes: int, pairs) -> "Graph":
        e = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
        e = e[e[:, 0] != e[:, 1]]
        e = np.sort(e, axis=1)
        key = np.unique(e[:, 0] * n_nodes + e[:, 1])
        return Graph(int(n_nodes), np.stack([key // n_nodes, key % n_nodes], axis=1))

    def dense(self) -> np.ndarray:
        a = np.zeros((self.n_nodes, self.n_nodes), dtype=np.int64)
        a[self.edges[:, 0], self.edges[:, 1]] = 1
        a[self.edges[:, 1], self.edges[:, 0]] = 1
        return a


@dataclass(frozen=True)
class Partition:
    """SPEC.md:30-35.  perm[m] = kappa(m): original node at permuted index m;
    inv_perm[node] = m.  Communities occupy [offsets[c], offsets[c+1]) in the
    permuted order; the NONE pool sits after offsets[-1]."""

    assignment: np.ndarray  # int64[N], community id or NONE
    perm: np.ndarray  # int64[N]
    inv_perm: np.ndarray  # int64[N]
    sizes: np.ndarray  # int64[M]

    @property
    def offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)

    @property
    def n_comm(self) -> int:
        return int(self.sizes.shape[0])

    @staticmethod
    def from_assignment(assignment) -> "Partition":
        a = np.asarray(assignment, dtype=np.int64)
        m = int(a.max()) + 1 if (a >= 0).any() else 0
        sizes = np.bincount(a[a >= 0], minlength=m).astype(np.int64)
        if m and (sizes == 0).any():
            raise InputError("community ids must be dense 0..M-1 with no empty community")
        key = np.where(a >= 0, a, m)  # NONE pool last
        perm = np.argsort(key, kind="stable").astype(np.int64)
        inv = np.empty_like(perm)
        inv[perm] = np.arange(perm.shape[0], dtype=np.int64)
        return Partition(a, perm, inv, sizes)

    def comm_of_permuted(self) -> np.ndarray:
        """community id per permuted index (NONE for the pool)."""
        n = self.perm.shape[0]
        c = np.full(n, NONE, dtype=np.int64)
        c[: int(self.sizes.sum())] = np.repeat(np.arange(self.n_comm), self.sizes)
        return c


@dataclass(frozen=True)
class SparseCorrection:
    """SPEC.md:37-42.  Stored once per unordered pair (iu <= iv), sorted by
    (iu, iv), permuted indices; the diagonal (m, m, -1) of every in-community
    node is included."""

    iu: np.ndarray  # int64
    iv: np.ndarray  # int64
    sgn: np.ndarray  # float64, +-1

    @property
    def n_pairs(self) -> int:
        return int(self.iu.shape[0])


@dataclass
class Decomposition:
    """partition + sparse correction (+ the source N)."""

    partition: Partition
    correction: SparseCorrection
    n_nodes: int
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def offsets(self) -> np.ndarray:
        return self.partition.offsets

    def dense_matrix(self) -> np.ndarray:
        """D + S reconstructed densely (permuted order).  Small N only."""
        n = self.n_nodes
        b = np.zeros((n, n), dtype=np.int64)
        off = self.offsets
        for c in range(self.partition.n_comm):
            b[off[c] : off[c + 1], off[c] : off[c + 1]] = 1
        s = self.correction
        sg = s.sgn.astype(np.int64)
        np.add.at(b, (s.iu, s.iv), sg)
        off_diag = s.iu != s.iv
        np.add.at(b, (s.iv[off_diag], s.iu[off_diag]), sg[off_diag])
        return b

    def graph(self) -> "Graph":
        """The graph D + S describes, as an edge list in PERMUTED order (the
        direct-sum / naive-mode input; O(sum lambda_c^2) memory: small and
        mid-size N only).  Vectorised: complete intra blocks minus the missing
        pairs, plus the inter pairs."""
        if "graph" not in self._cache:
            n = self.n_nodes
            s = self.correction
            od = s.iu != s.iv
            lo = np.minimum(s.iu[od], s.iv[od])
            hi = np.maximum(s.iu[od], s.iv[od])
            miss = np.sort(lo[s.sgn[od] < 0] * n + hi[s.sgn[od] < 0])
            keys = [lo[s.sgn[od] > 0] * n + hi[s.sgn[od] > 0]]
            off = self.offsets
            for c in range(self.partition.n_comm):
                lam = int(off[c + 1] - off[c])
                if lam < 2:
                    continue
                a, b = np.triu_indices(lam, 1)
                k = (a + off[c]) * n + (b + off[c])
                keys.append(k[~np.isin(k, miss, assume_unique=False)])
            key = np.unique(np.concatenate(keys)) if keys else np.empty(0, np.int64)
            self._cache["graph"] = Graph(int(n), np.stack([key // n, key % n], axis=1))
        return self._cache["graph"]

    def directed(self):
        """Directed S without the diagonal: (rows, cols, sign) int64/int64/int8."""
        if "directed" not in self._cache:
            s = self.correction
            od = s.iu != s.iv
            rows = np.concatenate([s.iu[od], s.iv[od]])
            cols = np.concatenate([s.iv[od], s.iu[od]])
            sg = np.concatenate([s.sgn[od], s.sgn[od]]).astype(np.int8)
            self._cache["directed"] = (rows, cols, sg)
        return self._cache["directed"]

    @property
    def nnz_dir(self) -> int:
        if "nnz_dir" not in self._cache:  # an 11 M-pair scan on config 2: once
            s = self.correction
            self._cache["nnz_dir"] = int(2 * np.count_nonzero(s.iu != s.iv))
        return self._cache["nnz_dir"]


# ---------------------------------------------------------------------------
# sampling helpers
# ---------------------------------------------------------------------------


def _bernoulli_indices(rng: np.random.Generator, n_total: int, q: float) -> np.ndarray:
    """Sorted indices in [0, n_total), each selected independently w.p. q
    (geometric skipping: exact Bernoulli semantics, O(selected) work)."""
    n_total = int(n_total)
    if n_total <= 0 or q <= 0.0:
        return np.empty(0, dtype=np.int64)
    if q >= 1.0:
        return np.arange(n_total, dtype=np.int64)
    out = []
    pos = np.int64(-1)
    expected = n_total * q
    while True:
        remaining = n_total - 1 - int(pos)
        chunk = int(min(remaining, 1.05 * remaining * q + 8 * np.sqrt(remaining * q + 1) + 64))
        chunk = max(chunk, 16)
        gaps = rng.geometric(q, size=chunk).astype(np.int64)
        idx = pos + np.cumsum(gaps)
        done = idx[-1] >= n_total
        idx = idx[idx < n_total]
        out.append(idx)
        if done:
            break
        pos = idx[-1]
    del expected
    return np.concatenate(out) if out else np.empty(0, dtype=np.int64)


def _tri_decode(t: np.ndarray, n: int):
    """Row-major strict-upper-triangle index t -> (a, b), a < b < n."""
    t = np.asarray(t, dtype=np.int64)
    nn = 2 * n - 1
    a = np.floor((nn - np.sqrt(np.maximum(float(nn) * nn - 8.0 * t, 0.0))) / 2.0).astype(np.int64)
    a = np.clip(a, 0, n - 2)

    def start(a_):
        return a_ * n - (a_ * (a_ + 1)) // 2

    for _ in range(3):  # fix float rounding
        hi = start(a) > t
        a = np.where(hi, a - 1, a)
        lo = start(a + 1) <= t
        a = np.where(lo, a + 1, a)
    b = t - start(a) + a + 1
    return a, b


def power_law_sizes(rng, m: int, exponent: float, lo: float, hi: float, total: int | None):
    """m community sizes, density ~ s^-exponent on [lo, hi] (inverse CDF),
    optionally renormalised to sum exactly to ``total`` (floor + largest
    remainders).  Renormalisation may push sizes outside [lo, hi]; that is the
    documented choice."""
    u = rng.random(m)
    if abs(exponent - 1.0) < 1e-12:
        s = lo * (hi / lo) ** u
    else:
        a = 1.0 - exponent
        s = (lo**a + u * (hi**a - lo**a)) ** (1.0 / a)
    if total is None:
        return np.maximum(np.round(s), 1).astype(np.int64)
    scaled = s * (total / s.sum())
    base = np.floor(scaled).astype(np.int64)
    rem = int(total - base.sum())
    order = np.argsort(-(scaled - base), kind="stable")
    base[order[:rem]] += 1
    return base


# ---------------------------------------------------------------------------
# planted partition
# ---------------------------------------------------------------------------


def _streams(seed: int):
    ss = np.random.SeedSequence(int(seed))
    return [np.random.Generator(np.random.PCG64(s)) for s in ss.spawn(2)]


def _sample_planted(sizes, p_in, p_out, seed):
    sizes = np.asarray(sizes, dtype=np.int64)
    if sizes.size == 0:
        raise InputError("sizes must be nonempty")
    if (sizes <= 0).any():
        raise InputError("zero-size community")
    if not (0.0 <= p_in <= 1.0 and 0.0 <= p_out <= 1.0):
        raise InputError("probabilities must lie in [0, 1]")
    rng_in, rng_out = _streams(seed)
    n = int(sizes.sum())
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    # missing intra pairs: each intra pair absent independently w.p. 1 - p_in
    miss_u, miss_v = [], []
    for c in range(sizes.shape[0]):
        lam = int(sizes[c])
        if lam < 2:
            continue
        t = _bernoulli_indices(rng_in, lam * (lam - 1) // 2, 1.0 - p_in)
        a, b = _tri_decode(t, lam)
        miss_u.append(a + off[c])
        miss_v.append(b + off[c])
    miss_u = np.concatenate(miss_u) if miss_u else np.empty(0, np.int64)
    miss_v = np.concatenate(miss_v) if miss_v else np.empty(0, np.int64)
    # inter edges: each inter-community pair present independently w.p. p_out
    comm = np.repeat(np.arange(sizes.shape[0]), sizes)
    t = _bernoulli_indices(rng_out, n * (n - 1) // 2, p_out)
    a, b = _tri_decode(t, n) if t.size else (t, t)
    keep = comm[a] != comm[b]
    return sizes, off, (miss_u, miss_v), (a[keep], b[keep])


def planted_partition_decomposition(sizes, p_in: float, p_out: float, seed: int) -> Decomposition:
    """Decomposition of ``planted_partition_graph(sizes, p_in, p_out, seed)``
    built directly from the sampled missing/extra pairs (O(nnz(S)) work)."""
    sizes, off, (mu, mv), (xu, xv) = _sample_planted(sizes, p_in, p_out, seed)
    n = int(off[-1])
    part = Partition.from_assignment(np.repeat(np.arange(sizes.shape[0]), sizes))
    diag = np.arange(n, dtype=np.int64)
    iu = np.concatenate([mu, diag, xu])
    iv = np.concatenate([mv, diag, xv])
    sg = np.concatenate([-np.ones(mu.size + n), np.ones(xu.size)])
    order = np.lexsort((iv, iu))
    return Decomposition(part, SparseCorrection(iu[order], iv[order], sg[order]), n)


def planted_partition_graph(sizes, p_in: float, p_out: float, seed: int):
    """SPEC.md:61-69.  Returns (Graph, Partition); identity-within-block kappa.
    Enumerates intra pairs: meant for N up to ~1e4."""
    sizes, off, (mu, mv), (xu, xv) = _sample_planted(sizes, p_in, p_out, seed)
    n = int(off[-1])
    edges = []
    missing = set(zip(mu.tolist(), mv.tolist()))
    for c in range(sizes.shape[0]):
        lam = int(sizes[c])
        if lam < 2:
            continue
        a, b = np.triu_indices(lam, 1)
        a = a + off[c]
        b = b + off[c]
        if missing:
            keep = np.array([(x, y) not in missing for x, y in zip(a.tolist(), b.tolist())],
                            dtype=bool)
            a, b = a[keep], b[keep]
        edges.append(np.stack([a, b], 1))
    edges.append(np.stack([xu, xv], 1))
    g = Graph.from_pairs(n, np.concatenate(edges))
    part = Partition.from_assignment(np.repeat(np.arange(sizes.shape[0]), sizes))
    return g, part


def decompose(graph: Graph, partition: Partition) -> Decomposition:
    """S = P A P^T - D, stored once per unordered pair."""
    n = graph.n_nodes
    if partition.perm.shape[0] != n:
        raise InputError("partition size does not match graph")
    inv = partition.inv_perm
    e = np.sort(inv[graph.edges], axis=1) if graph.edges.size else np.empty((0, 2), np.int64)
    comm = partition.comm_of_permuted()
    same = (comm[e[:, 0]] == comm[e[:, 1]]) & (comm[e[:, 0]] != NONE)
    present = set((e[same, 0] * n + e[same, 1]).tolist())
    off = partition.offsets
    mu, mv = [], []
    for c in range(partition.n_comm):
        a, b = np.triu_indices(int(partition.sizes[c]), 1)
        a = a + off[c]
        b = b + off[c]
        k = a * n + b
        miss = np.array([x not in present for x in k.tolist()], dtype=bool)
        mu.append(a[miss])
        mv.append(b[miss])
    mu = np.concatenate(mu) if mu else np.empty(0, np.int64)
    mv = np.concatenate(mv) if mv else np.empty(0, np.int64)
    n_in = int(off[-1])
    diag = np.arange(n_in, dtype=np.int64)
    xu, xv = e[~same, 0], e[~same, 1]
    iu = np.concatenate([mu, diag, xu])
    iv = np.concatenate([mv, diag, xv])
    sg = np.concatenate([-np.ones(mu.size + n_in), np.ones(xu.size)])
    order = np.lexsort((iv, iu))
    return Decomposition(partition, SparseCorrection(iu[order], iv[order], sg[order]), n)
