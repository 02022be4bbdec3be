"""GPU probe: eval time vs spreading / interpolation tile sizes (config given on the command line)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_11998_b200 as vp  # noqa: E402
from workloads import configs, rule  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = {"c2": configs.config2, "c5": configs.config5, "c4": configs.config4}[name]()
dev = "cuda"
nodes = torch.from_numpy(np.ascontiguousarray(w.nodes)).to(dev)
wts = torch.from_numpy(w.weights).to(dev)
tg = torch.from_numpy(np.ascontiguousarray(w.targets)).to(dev)
f = torch.from_numpy(w.f).to(dev)
ref = None
for st, it in [(32, 64), (24, 64), (48, 64), (64, 64), (32, 48), (32, 96)]:
    plan = vp.Plan(nodes, wts, tg, w.tol, boundary=w.boundary, targets_are_nodes=True, ref_nodes=rule.BARY[:, 1:3],
                   levels=-1 if name == "c5" else 0, spread_tile=st, interp_tile=it)
    plan.set_profiling(True)
    for _ in range(3):
        V = plan.eval(f)
    ph = [plan.phase_times() for _ in range(1)]
    times = []
    for _ in range(3):
        plan.eval(f)
        times.append(plan.phase_times())
    V = plan.eval(f).cpu().numpy()
    if ref is None:
        ref = V
    d = float(np.max(np.abs(V - ref)) / np.max(np.abs(ref)))
    sp = float(np.mean([t["spread"] for t in times]))
    ip = float(np.mean([t["interp_local"] for t in times]))
    print(json.dumps({"spread_tile": st, "interp_tile": it, "spread_ms": sp, "interp_local_ms": ip,
                      "total_ms": float(np.mean([sum(t.values()) for t in times])), "max_rel_diff": d}), flush=True)
    plan.destroy()
    torch.cuda.empty_cache()
