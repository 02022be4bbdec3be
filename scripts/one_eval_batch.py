"""Plan one config and run a few vp_eval_batch calls (for ncu captures of the batched kernels)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_11998_b200 as vp  # noqa: E402
from workloads import configs, rule  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = {"c2": configs.config2, "c4": configs.config4, "c5": configs.config5}[name]()
nodes = torch.from_numpy(np.ascontiguousarray(w.nodes)).cuda()
wts = torch.from_numpy(w.weights).cuda()
tg = torch.from_numpy(np.ascontiguousarray(w.targets)).cuda()
f = torch.from_numpy(w.f).cuda()
plan = vp.Plan(nodes, wts, tg, w.tol, boundary=w.boundary, targets_are_nodes=w.targets_are_nodes,
               ref_nodes=rule.BARY[:, 1:3], levels=-1 if name == "c5" else 0)
F = torch.stack([f * (1.0 + 0.25 * k) for k in range(K)]).contiguous()
for _ in range(2):
    plan.eval_batch(F)
torch.cuda.synchronize()
print("ok", name, K)
