"""probe: D[mu] on the star vs the oracle for several (tol, delta_1, J); errors split by distance to the curve"""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import numpy as np, torch
import paper_2409_11998_b200 as vp
from oracle import layer
from workloads import geometry
rng = np.random.default_rng(1)
th = rng.uniform(0, 2 * np.pi, 300)
rb = geometry.star_radius(th)
rr = rb * rng.uniform(0.0, 0.98, 300)
tg = np.stack([rr * np.cos(th), rr * np.sin(th)], 1)
dist = rb - rr
cv, dcv = layer.star()
muf = lambda t: 1.0 + 0.5 * np.cos(2 * t) + 0.3 * np.sin(3 * t)
ref = layer.double_layer(cv, dcv, muf, tg)
ch = geometry.star_chunks(200, q=16)
thn = np.arctan2(ch[..., 1], ch[..., 0])
nodes = rng.uniform(-0.5, 0.5, (200, 12, 2)); wts = np.full((200, 12), 1.0 / 2400)
for tol, d1, J in [(1e-10, 2.5e-5, 3), (1e-10, 2.5e-5, 0), (1e-10, 1e-4, 3), (1e-12, 2.5e-5, 3), (1e-8, 2.5e-5, 3), (1e-10, 6e-6, 3)]:
    plan = vp.Plan(torch.from_numpy(nodes).cuda(), torch.from_numpy(wts).cuda(), torch.from_numpy(tg).cuda(), tol,
                   boundary=("chunks", ch), parts=vp.PART_HISTORY, delta1_override=d1)
    plan.set_layer_levels(J)
    plan.prepare_dlp()
    D = plan.eval_dlp(torch.from_numpy(muf(thn)).cuda()).cpu().numpy()
    info = plan.info() if hasattr(plan, "info") else None
    plan.destroy()
    err = np.abs(D - ref)
    near = dist < 12 * np.sqrt(d1)
    print(f"tol {tol:.0e} d1 {d1:.1e} J {J}: rel l2 {np.linalg.norm(D-ref)/np.linalg.norm(ref):.2e} near max {err[near].max() if near.any() else 0:.2e} far max {err[~near].max():.2e} (n_near {near.sum()})")
