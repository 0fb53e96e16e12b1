"""Per-CTA cycles of the ELL stage kernel (CDK_PROFILE build) against the
CTA's ELL slots, inter slots, rblocks and segments: least-squares fit for the
planner's ELL cost model (plan.ELL_*_COST)."""
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
os.environ.setdefault("CDK_LIB", os.path.join(REPO, "paper_2203_16657_b200/_build/libcommdyn_cuda_profile.so"))
import numpy as np, torch
from paper_2203_16657_b200 import configs
from paper_2203_16657_b200.engine import KuramotoEngine
c = configs.config2(); dec = c.decomposition(); omega, theta0 = c.state()
eng = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
sch = eng.graph.schedule; lay = eng.graph.layout; e = sch.ell
assert e is not None
prof = torch.zeros(6 * sch.n_cta, dtype=torch.int64, device="cuda")
eng.lib.cdk_debug_set_profile_buffer(prof.data_ptr())
eng.set_state(theta0)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(3):
    ev[0].record(); eng.rk4_stage(c.dt, 1); ev[1].record()
torch.cuda.synchronize()
P6 = prof.view(-1, 6).cpu().numpy()
cyc = P6[:, 0].astype(np.float64)
g0, g1 = P6[:, 4] - P6[:, 4].min(), P6[:, 5] - P6[:, 4].min()
print(f"event-timed stage {ev[0].elapsed_time(ev[1])*1e3:.1f} us; CTA start skew max {g0.max()/1e3:.1f} us; "
      f"CTA end min {g1.min()/1e3:.1f} p50 {np.median(g1)/1e3:.1f} max {g1.max()/1e3:.1f} us")
seg_rb = sch.seg_rblk
F = []
for b in range(sch.n_cta):
    s0, s1 = sch.cta_seg[b], sch.cta_seg[b + 1]
    a, z = seg_rb[s0], seg_rb[s1]
    win = sum(int(sch.seg_win[q, 1] - sch.seg_win[q, 0]) for q in range(s0, s1))
    F.append((8 * (e.ell_off[z] - e.ell_off[a]), e.xell_off[z] - e.xell_off[a], z - a, s1 - s0, win))
F = np.array(F, dtype=np.float64)
print("cycles mean/max/min", cyc.mean(), cyc.max(), cyc.min())
rdy = P6[:, 1].astype(np.float64)
print("first segment ready after (cycles) mean/max/min", rdy.mean(), rdy.max(), rdy.min())
print("slots/xslots/rblocks/segs/window mean", F.mean(0), "max", F.max(0))
X = np.column_stack([F, np.ones(len(F))])
coef, *_ = np.linalg.lstsq(X, cyc, rcond=None)
pred = X @ coef
print("fit slots/xslots/rblocks/segs/window/const", np.round(coef, 4), "R2", round(1 - ((cyc - pred) ** 2).sum() / ((cyc - cyc.mean()) ** 2).sum(), 3))
for b in np.argsort(-cyc)[:6]: print("slow", b, int(cyc[b]), F[b].astype(int))
for b in np.argsort(cyc)[:4]: print("fast", b, int(cyc[b]), F[b].astype(int))
