"""Small plans through every eval path (strip spread, tile spread, fused FFT, cuFFT, batch, levels) for
compute-sanitizer runs."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_11998_b200 as vp  # noqa: E402
from workloads import configs  # noqa: E402

w = configs.config2(n=40)
dev = "cuda"
nodes = torch.from_numpy(np.ascontiguousarray(w.nodes)).to(dev)
wts = torch.from_numpy(w.weights).to(dev)
tg = torch.from_numpy(np.ascontiguousarray(w.targets)).to(dev)
f = torch.from_numpy(w.f).to(dev)
for kw in [{}, {"spread_tile": 32}, {"fft_mode": 1}, {"deterministic": True}, {"tol": 1e-4}, {"tol": 1e-13}]:
    tol = kw.pop("tol", w.tol)
    plan = vp.Plan(nodes, wts, tg, tol, boundary=w.boundary, targets_are_nodes=True, **kw)
    V = plan.eval(f)
    if not kw:
        F = torch.stack([f, 2 * f, 3 * f]).contiguous()
        plan.eval_batch(F)
    torch.cuda.synchronize()
    print("ok", kw, tol, float(V.abs().max()))
    plan.destroy()
w3 = configs.config3(M_target=20000, lmin=7, lmax=12, g=0.1)  # graded: level bands (strip band spreads)
plan = vp.Plan(torch.from_numpy(np.ascontiguousarray(w3.nodes)).to(dev), torch.from_numpy(w3.weights).to(dev),
               torch.from_numpy(np.ascontiguousarray(w3.targets)).to(dev), w3.tol, boundary=w3.boundary,
               targets_are_nodes=True)
V = plan.eval(torch.from_numpy(w3.f).to(dev))
torch.cuda.synchronize()
print("ok c3 levels", plan.info()["n_levels"], float(V.abs().max()))
print("done")
