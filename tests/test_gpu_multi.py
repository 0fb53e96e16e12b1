"""The sharded (multi-GPU) code path on one device: per-rank layouts,
schedules and stage kernels with the exchange done by device copies
(VirtualCluster).  Row-owned fixed-order accumulation => bitwise equal to the
single-rank trajectory for any rank count."""

import numpy as np
import pytest

from paper_2203_16657_b200 import configs
from paper_2203_16657_b200 import graph as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
def test_virtual_cluster_bitwise_equals_single(world):
    from paper_2203_16657_b200.engine import KuramotoEngine
    from paper_2203_16657_b200.multi import VirtualCluster

    c = configs.config1()
    dec = c.decomposition()
    omega, theta0 = c.state()
    single = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
    single.set_state(theta0)
    single.rk4(c.dt, 25)
    vc = VirtualCluster(dec, omega, c.coupling, c.n, world)
    vc.set_state(theta0)
    vc.rk4(c.dt, 25)
    vc.check()
    assert np.array_equal(vc.theta().cpu().numpy(), single.theta.cpu().numpy())


def test_virtual_cluster_with_pool_and_tiny_communities():
    from paper_2203_16657_b200.engine import KuramotoEngine
    from paper_2203_16657_b200.multi import VirtualCluster

    rng = np.random.default_rng(2)
    g, part = G.planted_partition_graph([60, 3, 1, 90, 40], 0.8, 0.05, 4)
    a = part.assignment.copy()
    a[rng.choice(a.shape[0], 30, replace=False)] = -1
    used = np.unique(a[a >= 0])
    remap = -np.ones(a.max() + 2, dtype=np.int64)
    remap[used] = np.arange(used.size)
    part = G.Partition.from_assignment(np.where(a >= 0, remap[a], -1))
    dec = G.decompose(g, part)
    n = g.n_nodes
    omega = rng.standard_normal(n)
    theta = rng.uniform(-3, 3, n)
    single = KuramotoEngine(dec, omega, coupling=2.0, norm=n)
    single.set_state(theta)
    single.rk4(0.01, 10)
    vc = VirtualCluster(dec, omega, 2.0, n, 3)
    vc.set_state(theta)
    vc.rk4(0.01, 10)
    assert np.array_equal(vc.theta().cpu().numpy(), single.theta.cpu().numpy())


@pytest.mark.parametrize("world,blocks", [(2, "0"), (3, "3")])
def test_virtual_cluster_generated_graph_bitwise(world, blocks, monkeypatch):
    """Config-5 family, every rank generating only its own rows (gen.generate
    row_range) with multi-pass windows and (blocks=3) the block-phased inter
    sweep: bitwise equal to the single-rank trajectory."""
    from paper_2203_16657_b200 import gen, plan
    from paper_2203_16657_b200.engine import KuramotoEngine
    from paper_2203_16657_b200.multi import VirtualCluster

    monkeypatch.setenv("CDK_INTER_BLOCKS", blocks)
    c = gen.scaled_config5(n=5000, lo=100, hi=1400, seed=58)
    budget = plan.stage_smem_bytes(192) - 128
    omega, theta0 = c.state()
    omega = np.clip(omega, -20, 20)
    dg, _ = gen.device_graph(c, "cuda", smem_budget=budget)
    single = KuramotoEngine(None, omega, coupling=c.coupling, norm=c.n, graph=dg)
    single.set_state(theta0)
    single.rk4(c.dt, 12)
    vc = VirtualCluster.generated(c, world, "cuda", smem_budget=budget)
    for e, _ in vc.ranks:
        e.omega.copy_(single.omega)
    vc.set_state(theta0)
    vc.rk4(c.dt, 12)
    vc.check()
    assert len({tuple(r) for r in vc.ranges}) == world
    assert np.array_equal(vc.theta().cpu().numpy(), single.theta.cpu().numpy())


@pytest.mark.parametrize("world,gen_case", [(2, False), (3, False), (2, True)])
def test_virtual_cluster_fused_exchange_bitwise(world, gen_case, monkeypatch):
    """Fused exchange (stage epilogues store z rows into every peer's buffer,
    cdk_kuramoto_rk4_stage_peers) on one device: bitwise equal to the
    single-rank trajectory, with no NCCL/copy exchange after any stage."""
    import torch

    from paper_2203_16657_b200 import gen, plan
    from paper_2203_16657_b200.engine import KuramotoEngine
    from paper_2203_16657_b200.multi import VirtualCluster

    if gen_case:
        monkeypatch.setenv("CDK_INTER_BLOCKS", "2")
        c = gen.scaled_config5(n=5000, lo=100, hi=1400, seed=58)
        budget = plan.stage_smem_bytes(192) - 128
        omega, theta0 = c.state()
        omega = np.clip(omega, -20, 20)
        dg, _ = gen.device_graph(c, "cuda", smem_budget=budget)
        single = KuramotoEngine(None, omega, coupling=c.coupling, norm=c.n, graph=dg)
        vc = VirtualCluster.generated(c, world, "cuda", smem_budget=budget, p2p=True)
        for e, _ in vc.ranks:
            e.omega.copy_(single.omega)
    else:
        c = configs.config1()
        dec = c.decomposition()
        omega, theta0 = c.state()
        single = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
        vc = VirtualCluster(dec, omega, c.coupling, c.n, world, p2p=True)
    single.set_state(theta0)
    single.rk4(c.dt, 10)
    vc.set_state(theta0)
    # poison the non-owned rows of every rank's stage buffer 1 (buffer 0 holds
    # the exchanged initial state): only the fused peer stores can refill them
    for (e, views), (lo, hi) in zip(vc.ranks, vc.ranges):
        views[1][:lo].fill_(float("nan"))
        views[1][hi:].fill_(float("nan"))
    vc.rk4(c.dt, 10)
    vc.check()
    assert np.array_equal(vc.theta().cpu().numpy(), single.theta.cpu().numpy())
    from paper_2203_16657_b200.multi import workspace_offsets

    for e, _ in vc.ranks:  # every rank signalled every rank once per stage
        o = workspace_offsets(e)[6]
        assert int(e.workspace[o:o + 4].view(torch.int32).item()) == 10 * 4 * world
