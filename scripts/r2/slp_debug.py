"""Per-group error of vp_eval_slp on the star (debugging aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2409_11998_b200 as vp  # noqa: E402
from oracle import layer  # noqa: E402
from workloads import geometry  # noqa: E402
from test_layer import _targets, _plan  # noqa: E402

rng = np.random.default_rng(21)
n_in, n_near, n_on, n_out = 80, 120, 24, 60
tg = _targets(rng, geometry.star_radius, n_in=n_in, n_near=n_near, n_on=n_on, n_out=n_out)
groups = {"in": slice(0, n_in), "near": slice(n_in, n_in + n_near), "on": slice(n_in + n_near, n_in + n_near + n_on),
          "out": slice(n_in + n_near + n_on, None)}
cv, dcv = layer.star()
for nch, d1 in ((200, 1e-4), (400, 1e-4), (200, 2.5e-5), (800, 2.5e-5)):
    ch = geometry.star_chunks(nch, q=16)
    plan, _ = _plan(tg, ch, 1e-9, d1)
    thn = np.arctan2(ch[..., 1], ch[..., 0])
    for name, sigf in (("one", lambda t: np.ones_like(t)), ("smooth", lambda t: 1.0 + 0.5 * np.cos(2 * t) + 0.3 * np.sin(3 * t))):
        S = plan.eval_slp(torch.from_numpy(sigf(thn)).cuda()).cpu().numpy()
        ref = layer.single_layer(cv, dcv, sigf, tg)
        msg = " ".join(f"{g}:{np.max(np.abs(S[s] - ref[s])):.2e}" for g, s in groups.items())
        print(f"chunks {nch} d1 {d1:.1e} sigma {name}: max abs err {msg}; max|S| {np.max(np.abs(ref)):.3f}", flush=True)
    plan.destroy()
