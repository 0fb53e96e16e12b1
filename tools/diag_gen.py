"""Save device vs oracle RHS on the scaled config-5 graph (diagnostics)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import cia, gen as OG, kernels as K
from paper_2203_16657_b200 import gen
from paper_2203_16657_b200.engine import KuramotoEngine

c = gen.scaled_config5(n=6000, lo=60, hi=900, seed=51)
off, cdf, E, thr = c.gen_inputs()
(_, (iu, iv, sg)) = OG.generate_csr(c.graph_seed, off, cdf, E, thr)
omega, theta0 = c.state()
dg, _ = gen.device_graph(c, "cuda")
eng = KuramotoEngine(None, omega, coupling=c.coupling, norm=c.n, graph=dg)
k = eng.rhs(torch.from_numpy(theta0).cuda()).cpu().numpy()
k0 = KuramotoEngine(None, np.zeros_like(omega), coupling=c.coupling, norm=c.n, graph=dg).rhs(
    torch.from_numpy(theta0).cuda()).cpu().numpy()
ko = cia.kuramoto_rhs_cia(K, theta0, omega, off, iu, iv, sg, c.coupling, c.n)
ko0 = cia.kuramoto_rhs_cia(K, theta0, np.zeros_like(omega), off, iu, iv, sg, c.coupling, c.n)
np.savez("gpurun_out/diag_gen.npz", k=k, k0=k0, ko=ko, ko0=ko0, omega=omega)
print("max |k-ko|", np.abs(k - ko).max(), "max |k0-ko0|", np.abs(k0 - ko0).max())
