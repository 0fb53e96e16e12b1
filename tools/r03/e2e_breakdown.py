"""Phase-by-phase wall time of the public integrate() path (config 2, K steps):
each phase is followed by a synchronize so its own cost shows (the real call
overlaps them; the sum is an upper bound)."""
import os, sys, time
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import numpy as np, torch
from paper_2203_16657_b200 import configs, kuramoto_model
from paper_2203_16657_b200.evaluator import engine_for, perm_device
from paper_2203_16657_b200.integrator import _to_host
from paper_2203_16657_b200.plan import DeviceGraph

c = configs.config2(); dec = c.decomposition(); omega, theta0 = c.state()
dec._cache["device_graph"] = DeviceGraph(dec)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
def sync(): torch.cuda.synchronize()
for rep in range(3):
    T = {}
    def lap(name, t0):
        sync(); T[name] = (time.perf_counter() - t0) * 1e3
    model = kuramoto_model(omega.copy(), c.coupling, c.n)
    sync(); t_all = time.perf_counter()
    t = time.perf_counter(); eng = engine_for(model, dec); lap("engine_for (omega upload)", t)
    t = time.perf_counter(); p_dev, inv_dev = perm_device(dec); lap("perm_device", t)
    t = time.perf_counter(); eng.upload_permuted(eng.theta, theta0, p_dev); lap("theta upload + permute", t)
    t = time.perf_counter(); eng.prepare(); lap("prepare", t)
    t = time.perf_counter(); eng.rk4(c.dt, K); lap(f"rk4 x{K}", t)
    t = time.perf_counter(); sn = eng.theta.clone(); rec = torch.index_select(sn, 0, inv_dev); lap("clone + unpermute", t)
    t = time.perf_counter(); h = _to_host([rec]); lap("readback", t)
    t = time.perf_counter(); st = np.concatenate([theta0[None], h]); lap("concatenate", t)
    t = time.perf_counter(); eng.check(); lap("status check", t)
    total = (time.perf_counter() - t_all) * 1e3
    print(f"rep {rep}: total {total:.3f} ms  " + "  ".join(f"{k} {v:.3f}" for k, v in T.items()))
