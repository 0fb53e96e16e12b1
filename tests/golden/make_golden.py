"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the build container only (it reads /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nbcache python tests/golden/make_golden.py

It imports the reference's own kernels (``commdyn._kernels``, numba backend
as shipped, single-threaded) and runs

1. each hot-path kernel on small seeded inputs (a1-a7 of SURVEY §8a);
2. the SPEC orchestration of oracle/cia.py — composed only of those reference
   kernels — for config 1 (CIA RK4 and direct-sum RK4, 1000 steps) and for
   one RHS + 2 RK4 steps of config 2 (subsampled outputs + full checksums).

The outputs pin both the C restatement (oracle/kernels.c) and the CUDA path.
Inputs are regenerated from seeds by the product's generator; the fixture
stores a sha256 of the generated decomposition so drift is detected.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")  # never write into the reference
os.environ["COMMDYN_BACKEND"] = "numba"
sys.path.insert(0, REPO)
sys.path.insert(0, REF_SRC)

from commdyn import _backend, _kernels as ref  # noqa: E402

from oracle import cia  # noqa: E402
from paper_2203_16657_b200 import configs  # noqa: E402

assert _backend.backend() == "numba"


def dec_hash(dec) -> str:
    h = hashlib.sha256()
    s = dec.correction
    for a in (s.iu, s.iv, s.sgn, dec.offsets):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def kernel_fixtures():
    rng = np.random.Generator(np.random.PCG64(12345))
    out = {}
    sizes = np.array([7, 1, 12, 30, 5])
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n_in = int(offsets[-1])
    n = n_in + 4  # NONE pool of 4 nodes
    x = rng.uniform(-math.pi, math.pi, n)
    out["offsets"] = offsets
    out["x"] = x
    for p in (1, 2, 3):
        out[f"op_p{p}"] = ref.order_params_blocks(x, offsets, p, math.pi, n)
        out[f"op_l2_p{p}"] = ref.order_params_blocks(x, offsets, p, 2.0, 13.0)
    # dense_complex with a random conjugate-symmetric table (real series) p=2
    p = 2
    m = sizes.size
    tbl = rng.standard_normal((m, 2 * p + 1)) + 1j * rng.standard_normal((m, 2 * p + 1))
    for j in range(p):
        tbl[:, 2 * p - j] = np.conj(tbl[:, j])
    tbl[:, p] = tbl[:, p].real
    out["dc_tbl"] = tbl
    o = rng.standard_normal(n)
    out["dc_out0"] = o.copy()
    nv, mi = ref.dense_complex(x, offsets, tbl, math.pi, o)
    out["dc_out"] = o
    out["dc_nviol"] = np.array(nv)
    out["dc_maximag"] = np.array(mi)
    # a non-real table: the guard must fire
    tbl_bad = tbl.copy()
    tbl_bad[:, 0] += 0.5
    o2 = np.zeros(n)
    nv2, mi2 = ref.dense_complex(x, offsets, tbl_bad, math.pi, o2)
    out["dcbad_tbl"] = tbl_bad
    out["dcbad_out"] = o2
    out["dcbad_nviol"] = np.array(nv2)
    out["dcbad_maximag"] = np.array(mi2)
    # dense_real p=3
    tc = rng.standard_normal((m, 4))
    ts = rng.standard_normal((m, 4))
    o = np.zeros(n)
    ref.dense_real(x, offsets, tc, ts, math.pi, o)
    out["dr_tc"], out["dr_ts"], out["dr_out"] = tc, ts, o
    # pairs_trig on random pairs incl. diagonal entries, p=2
    P = 300
    iu = rng.integers(0, n, P)
    iv = rng.integers(0, n, P)
    iv[:20] = iu[:20]
    sgn = np.where(rng.random(P) < 0.5, -1.0, 1.0)
    dcos = rng.standard_normal(3)
    dsin = rng.standard_normal(3)
    o = np.zeros(n)
    ref.pairs_trig(iu, iv, x, 1.0 / n, dcos, dsin, math.pi, sgn, o)
    out.update(pt_iu=iu, pt_iv=iv, pt_sgn=sgn, pt_dcos=dcos, pt_dsin=dsin, pt_out=o)
    # pairs_cs 2-D
    pos = rng.uniform(0, 10, (n, 2))
    vel = rng.standard_normal((n, 2))
    o = np.zeros((n, 2))
    ref.pairs_cs(iu, iv, pos, vel, 1.0 / n, 1.0, 1.0, 0.25, sgn, o)
    out.update(cs_pos=pos, cs_vel=vel, cs_out=o)
    # moments / dense_poly
    out["mom"] = ref.moments_blocks(x, offsets, 5, 0.3, n)
    tp = rng.standard_normal((m, 6))
    o = np.zeros(n)
    ref.dense_poly(x, offsets, tp, 0.5, -0.1, o)
    out.update(dp_tbl=tp, dp_out=o)
    # higher-order naive block
    th = rng.uniform(-math.pi, math.pi, 17)
    out["ho_theta"] = th
    out["ho_1102"] = ref.ho_naive_block(th, (1, 1, 0, -2))
    out["ho_11m1m1"] = ref.ho_naive_block(th, (1, 1, -1, -1))
    np.savez_compressed(os.path.join(HERE, "kernels_small.npz"), **out)
    print("kernels_small.npz written")


def cfg1_fixture():
    c = configs.config1()
    dec = c.decomposition()
    omega, theta0 = c.state()
    s = dec.correction
    off = dec.offsets
    # full edge list for the direct sum: S (+1 entries) plus present intra pairs
    adj = dec.dense_matrix()
    np.fill_diagonal(adj, 0)
    eu, ev = np.nonzero(np.triu(adj, 1))

    def rhs_cia(x):
        return cia.kuramoto_rhs_cia(ref, x, omega, off, s.iu, s.iv, s.sgn, c.coupling, c.n)

    def rhs_naive(x):
        return cia.kuramoto_rhs_naive(ref, x, omega, eu, ev, c.coupling, c.n)

    t = time.time()
    k_cia = rhs_cia(theta0)
    k_naive = rhs_naive(theta0)
    fin, snaps = cia.rk4_integrate(rhs_cia, theta0, c.dt, c.steps, record_every=100)
    t_cia = time.time() - t
    fin_naive, _ = cia.rk4_integrate(rhs_naive, theta0, c.dt, c.steps)
    print(f"cfg1 cia traj {t_cia:.2f}s; max circ cia-vs-naive "
          f"{cia.circ_dist(fin, fin_naive).max():.3e}")
    np.savez_compressed(
        os.path.join(HERE, "cfg1.npz"),
        dec_sha256=np.array(dec_hash(dec)), rhs0_cia=k_cia, rhs0_naive=k_naive,
        final_cia=fin, final_naive=fin_naive,
        snap_steps=np.array([st for st, _ in snaps]), snaps=np.stack([x for _, x in snaps]),
    )
    print("cfg1.npz written")


def cfg2_fixture(n_sample=4096, steps=2):
    c = configs.config2()
    dec = c.decomposition()
    omega, theta0 = c.state()
    s = dec.correction
    off = dec.offsets

    def rhs_cia(x):
        return cia.kuramoto_rhs_cia(ref, x, omega, off, s.iu, s.iv, s.sgn, c.coupling, c.n)

    t = time.time()
    k0 = rhs_cia(theta0)
    t_rhs = time.time() - t
    fin, _ = cia.rk4_integrate(rhs_cia, theta0, c.dt, steps)
    print(f"cfg2 one RHS {t_rhs:.2f}s (reference numba, 1 thread)")
    rng = np.random.Generator(np.random.PCG64(99))
    idx = np.sort(rng.choice(c.n, n_sample, replace=False))
    np.savez_compressed(
        os.path.join(HERE, "cfg2_sample.npz"),
        dec_sha256=np.array(dec_hash(dec)), idx=idx, rhs0=k0[idx], rhs0_sum=np.array(k0.sum()),
        rhs0_abs_sum=np.array(np.abs(k0).sum()), steps=np.array(steps), final=fin[idx],
        final_cos_sum=np.array(np.cos(fin).sum()), final_sin_sum=np.array(np.sin(fin).sum()),
        ref_rhs_seconds=np.array(t_rhs),
    )
    print("cfg2_sample.npz written")


def f4_fixtures():
    """SURVEY §8(f) rank 4 kernels: pairs_poly (Desai-Zwanzig coupling),
    nn_recurrence (Appendix B window sums), spin_field_sums (Bornholdt-Rohlf
    oracle) and ho_naive_block at a larger block, all by the real reference."""
    rng = np.random.Generator(np.random.PCG64(424242))
    out = {}
    n = 257
    x = rng.uniform(-2.0, 2.0, n)
    P = 800
    iu = rng.integers(0, n, P)
    iv = rng.integers(0, n, P)
    iv[:40] = iu[:40]  # diagonal entries: counted once
    sgn = np.where(rng.random(P) < 0.5, -1.0, 1.0)
    coef = rng.standard_normal(4)
    o = rng.standard_normal(n)
    out.update(pp_x=x, pp_iu=iu, pp_iv=iv, pp_sgn=sgn, pp_coef=coef, pp_out0=o.copy())
    ref.pairs_poly(iu, iv, x, 1.0 / n, coef, 0.2, sgn, o)
    out["pp_out"] = o
    # window sums: phases on the unit circle; windows narrower than, equal to
    # and wider than the ring; anchor strides that do / do not divide n
    for tag, nn, k, anchor in (("a", 5000, 1, 1024), ("b", 5000, 37, 100), ("c", 5000, 1250, 1024),
                               ("d", 7, 10, 1024), ("e", 3001, 500, 1)):
        ph = np.exp(1j * rng.uniform(-math.pi, math.pi, nn))
        out[f"nn_{tag}_ph"] = ph
        out[f"nn_{tag}_k"] = np.array(k)
        out[f"nn_{tag}_anchor"] = np.array(anchor)
        out[f"nn_{tag}_f"] = ref.nn_recurrence(ph, k, 1.0 / nn, anchor)
    spins = np.where(rng.random(1000) < 0.37, -1, 1).astype(np.int64)
    out["spin"] = spins
    out["spin_f"] = ref.spin_field_sums(spins)
    th = rng.uniform(-math.pi, math.pi, 40)
    out["ho40_theta"] = th
    out["ho40_1102"] = ref.ho_naive_block(th, (1, 1, 0, -2))
    out["ho40_2m11m2"] = ref.ho_naive_block(th, (2, -1, 1, -2))
    np.savez_compressed(os.path.join(HERE, "kernels_f4.npz"), **out)
    print("kernels_f4.npz written")


def harmonics_fixture():
    """Higher-harmonics Kuramoto, p = 4 random coefficients
    on a planted 4 x 125 graph with a NONE pool of 12 nodes: one CIA RHS, one
    direct-sum RHS and 200 CIA RK4 steps (dt 0.01), all over the real
    reference kernels (oracle.cia.harmonics_rhs_cia orchestration)."""
    from paper_2203_16657_b200 import graph as G

    rng = np.random.Generator(np.random.PCG64(4040))
    g, part = G.planted_partition_graph([125, 125, 125, 125], 0.9, 0.01, 44)
    a = part.assignment.copy()
    a[rng.choice(a.shape[0], 12, replace=False)] = -1
    part = G.Partition.from_assignment(a)
    dec = G.decompose(g, part)
    n = g.n_nodes
    d_cos = rng.standard_normal(5)
    d_sin = rng.standard_normal(5)
    d_sin[0] = 0.0
    omega = rng.standard_normal(n)
    theta0 = rng.uniform(-math.pi, math.pi, n)
    s = dec.correction
    perm = dec.partition.perm
    om_p, th_p = omega[perm], theta0[perm]

    def rhs(x):
        return cia.harmonics_rhs_cia(ref, x, om_p, dec.offsets, s.iu, s.iv, s.sgn, d_cos, d_sin,
                                     n)

    k_cia = rhs(th_p)
    eg = dec.graph().edges
    k_naive = om_p.copy()
    ref.pairs_trig(eg[:, 0], eg[:, 1], th_p, 1.0 / n, d_cos, d_sin, math.pi,
                   np.ones(eg.shape[0]), k_naive)
    fin, _ = cia.rk4_integrate(rhs, th_p, 0.01, 200)
    np.savez_compressed(os.path.join(HERE, "harmonics.npz"), dec_sha256=np.array(dec_hash(dec)),
                        assignment=a, d_cos=d_cos, d_sin=d_sin, omega=omega, theta0=theta0,
                        rhs_cia=k_cia, rhs_naive=k_naive, final=fin, steps=np.array(200),
                        dt=np.array(0.01))
    print("harmonics.npz written; |cia - naive| =", np.abs(k_cia - k_naive).max())


if __name__ == "__main__":
    which = sys.argv[1:] or ["kernels", "cfg1", "cfg2", "f4", "harmonics"]
    for w in which:
        {"kernels": kernel_fixtures, "cfg1": cfg1_fixture, "cfg2": cfg2_fixture,
         "f4": f4_fixtures, "harmonics": harmonics_fixture}[w]()
