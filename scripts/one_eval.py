"""Plan one config and run a few evals (for ncu captures of single kernels)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_11998_b200 as vp  # noqa: E402
from workloads import configs, rule  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
st = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n_eval = int(sys.argv[3]) if len(sys.argv) > 3 else 3
# extra vp_opts fields from the environment, e.g. VP_OPTS="fft_rows=1 spread_pack=2"
import os  # noqa: E402
extra = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in os.environ.get("VP_OPTS", "").split()}
w = {"c2": configs.config2, "c3": configs.config3, "c4": configs.config4, "c5": configs.config5}[name]()
nodes = torch.from_numpy(np.ascontiguousarray(w.nodes)).cuda()
wts = torch.from_numpy(w.weights).cuda()
tg = torch.from_numpy(np.ascontiguousarray(w.targets)).cuda()
f = torch.from_numpy(w.f).cuda()
plan = vp.Plan(nodes, wts, tg, w.tol, boundary=w.boundary, targets_are_nodes=w.targets_are_nodes,
               ref_nodes=rule.BARY[:, 1:3], levels=-1 if name == "c5" else 0, spread_tile=st, **extra)
for _ in range(n_eval):
    plan.eval(f)
torch.cuda.synchronize()
print("ok", name, st)
