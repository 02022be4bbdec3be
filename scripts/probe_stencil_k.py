"""GPU probe: config-2 parity and eval time vs the KNN stencil size K (degree 4, 15 monomials)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2409_11998_b200 as vp  # noqa: E402
from workloads import configs  # noqa: E402

w = configs.config2()
idx = configs.sample_targets(w.T, 192, seed=22)
ref = oracle.workload_potential(w, idx)
dev = "cuda"
nodes = torch.from_numpy(np.ascontiguousarray(w.nodes)).to(dev)
wts = torch.from_numpy(w.weights).to(dev)
tg = torch.from_numpy(np.ascontiguousarray(w.targets)).to(dev)
f = torch.from_numpy(w.f).to(dev)
for K in [30, 24, 20, 17]:
    plan = vp.Plan(nodes, wts, tg, w.tol, boundary=w.boundary, targets_are_nodes=True, deriv_k=K)
    plan.set_profiling(True)
    for _ in range(3):
        V = plan.eval(f)
    ph = plan.phase_times()
    V = V.cpu().numpy()
    e = float(np.sqrt(np.sum((V[idx] - ref) ** 2) / np.sum(ref ** 2)))
    print(json.dumps({"K": K, "rel_l2": e, "eval_ms": sum(ph.values()), "interp_local": ph["interp_local"]}), flush=True)
    plan.destroy()
