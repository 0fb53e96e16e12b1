import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes
from paper_2203_16657_b200 import configs, _lib
from paper_2203_16657_b200.multi import VirtualCluster, workspace_offsets
c = configs.config1(); dec = c.decomposition(); omega, theta0 = c.state()
vc = VirtualCluster(dec, omega, c.coupling, c.n, 2, p2p=True)
vc.set_state(theta0)
for (e, views), (lo, hi) in zip(vc.ranks, vc.ranges):
    views[1].fill_(float("nan"))
print("ranges", vc.ranges)
for (e, _), pt in zip(vc.ranks, vc.peers):
    print("peers", pt.struct.n_ranks, pt.struct.rank, [hex(int(x)) for x in pt._t[1].cpu().numpy()], hex(e.workspace.data_ptr()), workspace_offsets(e))
    rc = e.lib.cdk_kuramoto_rk4_stage_peers(ctypes.byref(e.graph.struct), e.theta.data_ptr(), e.omega.data_ptr(), e.k_over_n, float(c.dt), 1, e.workspace.data_ptr(), ctypes.byref(pt.struct), None)
    print("rc", rc, e.lib.cdk_last_error())
torch.cuda.synchronize()
for (e, views) in vc.ranks:
    z1 = views[1].cpu().numpy()
    bad = np.nonzero(~np.isfinite(z1[:, 0]))[0]
    print("nan rows", bad.size, bad[:5], bad[-5:] if bad.size else None)
print("--- full step")
vc = VirtualCluster(dec, omega, c.coupling, c.n, 2, p2p=True)
vc.set_state(theta0)
for stg in range(1, 5):
    for (e, _), pt in zip(vc.ranks, vc.peers):
        e.lib.cdk_kuramoto_rk4_stage_peers(ctypes.byref(e.graph.struct), e.theta.data_ptr(), e.omega.data_ptr(), e.k_over_n, float(c.dt), stg, e.workspace.data_ptr(), ctypes.byref(pt.struct), None)
        pt.advance(1)
    torch.cuda.synchronize()
    for r, (e, views) in enumerate(vc.ranks):
        zb = views[stg & 1].cpu().numpy()
        th = e.theta.cpu().numpy()
        print("stage", stg, "rank", r, "nan z", int((~np.isfinite(zb[:, 0])).sum()), "nan theta", int((~np.isfinite(th)).sum()), "st", e.status().nonfinite)
