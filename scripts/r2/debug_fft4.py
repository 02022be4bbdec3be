"""Debug: four-step column pass vs cuFFT 2D vs a numpy direct G_H sum (smooth part, few sources)."""
import sys
import numpy as np
import scipy.special as sp
import torch
sys.path.insert(0, ".")
import paper_2409_11998_b200 as vp
rng = np.random.default_rng(141)
src = rng.uniform(0.0, 1.0, (1200, 2))
wts_np = rng.uniform(0.5, 1.5, (100, 12)) / 1200
f_np = rng.standard_normal((100, 12))
tg_np = rng.uniform(0.0, 1.0, (300, 2))
nodes = torch.from_numpy(src.reshape(100, 12, 2).copy()).cuda()
wts = torch.from_numpy(wts_np).cuda()
fv = torch.from_numpy(f_np).cuda()
tg = torch.from_numpy(tg_np).cuda()
c = (f_np * wts_np).ravel()
keys = ["nf_nh", "nf_fh", "nmode_nh", "nmode_fh", "fft_path_nh", "fft_path_fh"]
for d1, tol in [(6.25e-8, 1e-13), (6.25e-8, 1e-10), (6.25e-8, 1e-13), (3.2e-8, 1e-13), (6.25e-8, 1e-13)]:
    r2 = ((tg_np[:, None, :] - src[None, :, :]) ** 2).sum(-1)
    G = -(np.log(r2) + sp.exp1(r2 / (4 * d1))) / (4 * np.pi)
    ref = G @ c
    for mode in (0, 1, 0, 1):
        p = vp.Plan(nodes, wts, tg, tol, parts=vp.PART_HISTORY, delta1_override=float(d1), fft_mode=mode)
        V = p.eval(fv).cpu().numpy()
        i = p.info()
        e = np.sqrt(np.sum((V - ref) ** 2) / np.sum(ref ** 2))
        print(f"{d1:.3e} {tol:.0e} mode {mode}", [i[k] for k in keys], f"rel l2 vs direct {e:.3e}", flush=True)
        p.destroy()
