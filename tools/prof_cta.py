"""Per-CTA phase timing of the stage kernel (needs the CDK_PROFILE build)."""
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
os.environ.setdefault("CDK_LIB", os.path.join(REPO, "paper_2203_16657_b200/_build/libcommdyn_cuda_profile.so"))
import numpy as np, torch
from paper_2203_16657_b200 import configs
from paper_2203_16657_b200.engine import KuramotoEngine
if "--cfg5" in sys.argv:
    from paper_2203_16657_b200 import gen
    c = gen.config5() if "--small" not in sys.argv else gen.scaled_config5(400_000, 1000, 20000)
    omega, theta0 = c.state()
    dg, _ = gen.device_graph(c, "cuda")
    eng = KuramotoEngine(None, omega, coupling=c.coupling, norm=c.n, graph=dg)
else:
    c = configs.config2(); dec = c.decomposition(); omega, theta0 = c.state()
    eng = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
sch = eng.graph.schedule; lay = eng.graph.layout
prof = torch.zeros(6 * sch.n_cta, dtype=torch.int64, device="cuda")
eng.lib.cdk_debug_set_profile_buffer(prof.data_ptr())
eng.set_state(theta0)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(3):
    ev[0].record(); eng.rk4_stage(c.dt, 1); ev[1].record()
torch.cuda.synchronize()
P6 = prof.view(-1, 6).cpu().numpy()
P = P6[:, :4].astype(np.float64)
g0, g1 = P6[:, 4] - P6[:, 4].min(), P6[:, 5] - P6[:, 4].min()
print(f"event-timed stage {ev[0].elapsed_time(ev[1])*1e3:.1f} us; CTA start skew max {g0.max()/1e3:.1f} us "
      f"(p50 {np.median(g0)/1e3:.1f}); CTA end min {g1.min()/1e3:.1f} p50 {np.median(g1)/1e3:.1f} max {g1.max()/1e3:.1f} us")
rows = lay.rblk_row0
seg_rows = rows[sch.seg_rblk]
feat = []
for b in range(sch.n_cta):
    s0, s1 = sch.cta_seg[b], sch.cta_seg[b + 1]
    r0, r1 = seg_rows[s0], seg_rows[s1]
    ent = lay.intra_ptr[r1] - lay.intra_ptr[r0]
    xen = lay.inter_ptr[r1] - lay.inter_ptr[r0]
    un = sum(int(lay.intra_ptr[seg_rows[s + 1]] - lay.intra_ptr[seg_rows[s]])
             for s in range(s0, s1) if sch.seg_win[s][1] == sch.seg_win[s][0])
    feat.append((r1 - r0, ent - un, un, xen, s1 - s0))
F = np.array(feat, dtype=np.float64)
np.set_printoptions(linewidth=150)
print("cycles total/stage/gather/epi: mean", P.mean(0).astype(int), "max", P.max(0).astype(int), "min", P.min(0).astype(int))
print("rows/staged ent/unstaged ent/inter/segs: mean", F.mean(0).astype(int), "max", F.max(0).astype(int), "min", F.min(0).astype(int))
X = np.column_stack([F[:, :5], np.ones(len(F))])
for j, name in enumerate(["total", "stage", "gather", "epi"]):
    coef, *_ = np.linalg.lstsq(X, P[:, j], rcond=None)
    pred = X @ coef
    print(name, "fit rows/staged/unstaged/inter/segs/const", np.round(coef, 3), "R2", round(1 - ((P[:, j] - pred) ** 2).sum() / ((P[:, j] - P[:, j].mean()) ** 2).sum(), 3))
order = np.argsort(-P[:, 0])[:8]
for b in order: print("slow cta", b, P[b].astype(int), F[b].astype(int))
order = np.argsort(P[:, 0])[:4]
for b in order: print("fast cta", b, P[b].astype(int), F[b].astype(int))
