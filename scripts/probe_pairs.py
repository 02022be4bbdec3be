"""Fraction of targets whose NH footprint origin cell holds other targets (interpolation-unit potential)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_11998_b200 as vp  # noqa: E402
from workloads import configs, rule  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = {"c2": configs.config2, "c4": configs.config4, "c5": configs.config5}[name]()
tg = torch.from_numpy(np.ascontiguousarray(w.targets)).cuda()
plan = vp.Plan(torch.from_numpy(np.ascontiguousarray(w.nodes)).cuda(), torch.from_numpy(w.weights).cuda(), tg, w.tol,
               boundary=w.boundary, targets_are_nodes=w.targets_are_nodes, ref_nodes=rule.BARY[:, 1:3],
               levels=-1 if name == "c5" else 0)
info = plan.info()
nf, L, W = info["nf_nh"], info["L_nh"], info["w_es"]
h = L / nf
ox = tg[:, 0].min().item()  # the grid origin is not exported; counts only need a consistent cell lattice
cx = torch.floor((tg[:, 0] - tg[:, 0].mean()) / h).to(torch.int64)
cy = torch.floor((tg[:, 1] - tg[:, 1].mean()) / h).to(torch.int64)
key = (cy - cy.min()) * (cx.max() - cx.min() + 1) + (cx - cx.min())
_, inv, cnt = torch.unique(key, return_inverse=True, return_counts=True)
per_t = cnt[inv]
out = {"config": name, "targets": int(tg.shape[0]), "cells_occupied": int(cnt.numel())}
for g in [2, 4, 8, 32]:
    out[f"frac_targets_in_cells_ge{g}"] = float((per_t >= g).double().mean())
# pairs formed greedily per cell: floor(cnt/2) pairs
out["pairable_frac"] = float((2 * (cnt // 2)).sum().item() / tg.shape[0])
out["units_if_pairs"] = int((cnt - cnt // 2).sum().item())
out["units_if_quads"] = int(((cnt + 3) // 4).sum().item())
print(json.dumps(out))
