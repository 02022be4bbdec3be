"""GPU probe: parity of configs 4/5 (scaled or full) in KNN and TRIANGLE derivative modes vs the oracle."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle
import paper_2409_11998_b200 as vp
from workloads import configs, rule

def run(w, modes=("knn", "triangle"), ntg=48, seed=3, levels=(0,)):
    dev = "cuda"
    nodes = torch.from_numpy(np.ascontiguousarray(w.nodes)).to(dev)
    wts = torch.from_numpy(w.weights).to(dev)
    tg = torch.from_numpy(np.ascontiguousarray(w.targets)).to(dev)
    f = torch.from_numpy(w.f).to(dev)
    idx = configs.sample_targets(w.T, ntg, seed=seed)
    if w.T > w.N:   # include some off-node targets
        idx = np.unique(np.concatenate([idx, w.N + configs.sample_targets(w.T - w.N, ntg // 4, seed=seed + 1)]))
    t0 = time.time()
    ref = oracle.workload_potential(w, idx)
    t_or = time.time() - t0
    out = {"name": w.name, "M": w.M, "N": w.N, "T": w.T, "oracle_s": t_or, "n_idx": len(idx)}
    for m, lev in [(m, l) for m in modes for l in levels]:
        t0 = time.time()
        plan = vp.Plan(nodes, wts, tg, w.tol, boundary=w.boundary, targets_are_nodes=True, deriv=m,
                       ref_nodes=rule.BARY[:, 1:3], levels=lev)
        torch.cuda.synchronize()
        tp = time.time() - t0
        plan.set_profiling(True)
        V = plan.eval(f)
        V = plan.eval(f).cpu().numpy()
        ph = plan.phase_times()
        e = float(np.sqrt(np.sum((V[idx] - ref) ** 2) / np.sum(ref ** 2)))
        eo = None
        if w.T > w.N:
            sel = idx >= w.N
            eo = float(np.sqrt(np.sum((V[idx][sel] - ref[sel]) ** 2) / np.sum(ref[sel] ** 2)))
        inf = plan.info()
        out[f"{m}_lev{lev}"] = {"rel_l2": e, "rel_l2_offnode": eo, "plan_s": tp, "eval_ms": sum(ph.values()),
                                "phases": ph, "n_stencil": inf["n_stencil_targets"], "nf_nh": inf["nf_nh"],
                                "mem_GB": inf["device_bytes"] / 1e9, "levels": inf["n_levels"],
                                "level_targets": inf["level_targets"][:8], "boxes": inf["n_boxes"]}
        print(json.dumps(out[f"{m}_lev{lev}"]), flush=True)
        plan.destroy()
        del plan
        torch.cuda.empty_cache()
    print(json.dumps(out))

if __name__ == "__main__":
    which = sys.argv[1]
    if which == "c4s":
        run(configs.config4(n=int(sys.argv[2]) if len(sys.argv) > 2 else 400))
    elif which == "c5s":
        run(configs.config5(M_target=int(float(sys.argv[2])), lmin=int(sys.argv[3]), lmax=int(sys.argv[4]), n_random=100000))
    elif which == "c5":
        t0 = time.time()
        w = configs.config5()
        print("c5 generated", w.M, w.N, w.T, time.time() - t0, flush=True)
        run(w, modes=("triangle",), ntg=48, levels=(-1, 0))
    elif which == "c4":
        t0 = time.time()
        w = configs.config4()
        print("c4 generated", w.M, w.N, time.time() - t0, flush=True)
        run(w, modes=("triangle",), ntg=48)
