"""Where a 20-step public integrate() call spends its wall time (config 2):
cProfile of the call with the device graph resident, after warm-up."""
import cProfile, io, os, pstats, sys, time
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import numpy as np, torch
from paper_2203_16657_b200 import IntegrationPlan, configs, integrate, kuramoto_model
from paper_2203_16657_b200.plan import DeviceGraph

c = configs.config2(); dec = c.decomposition(); omega, theta0 = c.state()
inv = dec.partition.inv_perm
omega_o, theta_o = omega[inv], theta0[inv]  # original node order
dec._cache["device_graph"] = DeviceGraph(dec)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
plan = IntegrationPlan(t_end=K * c.dt, dt=c.dt)
for rep in range(3):
    model = kuramoto_model(omega_o.copy(), c.coupling, c.n)
    torch.cuda.synchronize(); t = time.perf_counter()
    tr = integrate(model, dec, theta_o, plan)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"rep {rep}: {dt*1e3:.3f} ms for {K} steps -> {c.n*K/dt:.3e} node-updates/s; device per step "
          f"{tr.step_seconds.mean()*1e6:.1f} us")
model = kuramoto_model(omega_o.copy(), c.coupling, c.n)
pr = cProfile.Profile(); pr.enable()
tr = integrate(model, dec, theta_o, plan); torch.cuda.synchronize()
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(28); print(s.getvalue()[:6000])
