"""GPU probe: fused FFT path (fft_mode=0) vs cuFFT (fft_mode=1): phase times, eval time, max rel diff."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_11998_b200 as vp  # noqa: E402
from workloads import configs, rule  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = {"c1": configs.config1, "c2": configs.config2, "c3": configs.config3, "c4": configs.config4,
     "c5": configs.config5}[name]()
dev = "cuda"
nodes = torch.from_numpy(np.ascontiguousarray(w.nodes)).to(dev)
wts = torch.from_numpy(w.weights).to(dev)
tg = torch.from_numpy(np.ascontiguousarray(w.targets)).to(dev)
f = torch.from_numpy(w.f).to(dev)
ref = None
for mode in [1, 0]:
    plan = vp.Plan(nodes, wts, tg, w.tol, boundary=w.boundary, targets_are_nodes=w.targets_are_nodes,
                   ref_nodes=rule.BARY[:, 1:3], levels=-1 if name == "c5" else 0, fft_mode=mode)
    plan.set_profiling(True)
    for _ in range(3):
        plan.eval(f)
    times = []
    for _ in range(5):
        plan.eval(f)
        times.append(plan.phase_times())
    plan.set_profiling(False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        plan.eval(f)
    e1.record()
    torch.cuda.synchronize()
    V = plan.eval(f).cpu().numpy()
    if ref is None:
        ref = V
    d = float(np.max(np.abs(V - ref)) / np.max(np.abs(ref)))
    info = plan.info()
    print(json.dumps({"config": name, "fft_mode": mode, "nf_nh": info["nf_nh"], "nf_fh": info["nf_fh"],
                      "phases": {k: round(float(np.median([t[k] for t in times])), 4) for k in times[0]},
                      "eval_ms": e0.elapsed_time(e1) / 10, "max_rel_diff_vs_cufft": d}), flush=True)
    plan.destroy()
    torch.cuda.empty_cache()
