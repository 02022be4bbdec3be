"""GPU probe: config 3 (graded star, nonconforming) with and without the level bands (a12) vs the oracle.

usage: python scripts/probe_c3.py small|full [n_uniform] [n_near]
Reports rel l2 on a seeded uniform node sample (the parity metric) and on a near-source sample
(diagnostic), for levels off (-1) and auto (0) and a few (C_min, rho)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2409_11998_b200 as vp  # noqa: E402
from workloads import configs  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "small"
    nu = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    nn = int(sys.argv[3]) if len(sys.argv) > 3 else 128
    t0 = time.time()
    w = configs.config3() if which == "full" else configs.config3(M_target=60000, lmin=7, lmax=13, g=0.1)
    t_gen = time.time() - t0
    idx_u = configs.sample_targets(w.T, nu, seed=31)
    d = np.hypot(w.targets[:, 0] - 0.3, w.targets[:, 1] + 0.2)
    near = np.nonzero(d < 6e-3)[0]
    idx_n = near[configs.sample_targets(near.size, nn, seed=32)]
    t0 = time.time()
    ref_u = oracle.workload_potential(w, idx_u)
    ref_n = oracle.workload_potential(w, idx_n)
    t_or = time.time() - t0
    dev = "cuda"
    nodes = torch.from_numpy(np.ascontiguousarray(w.nodes)).to(dev)
    wts = torch.from_numpy(w.weights).to(dev)
    tg = torch.from_numpy(np.ascontiguousarray(w.targets)).to(dev)
    f = torch.from_numpy(w.f).to(dev)
    out = {"name": w.name, "M": w.M, "N": w.N, "gen_s": t_gen, "oracle_s": t_or, "n_near_nodes": int(near.size)}
    for lev, cmin, rho in [(-1, 0, 0), (0, 2.0, 4.0), (0, 1.5, 4.0), (0, 3.0, 4.0)]:
        t0 = time.time()
        plan = vp.Plan(nodes, wts, tg, w.tol, boundary=None, targets_are_nodes=True, levels=lev, level_cmin=cmin,
                       level_rho=rho)
        torch.cuda.synchronize()
        tp = time.time() - t0
        plan.set_profiling(True)
        plan.eval(f)
        V = plan.eval(f).cpu().numpy()
        ph = plan.phase_times()
        inf = plan.info()
        eu = float(np.sqrt(np.sum((V[idx_u] - ref_u) ** 2) / np.sum(ref_u ** 2)))
        en = float(np.sqrt(np.sum((V[idx_n] - ref_n) ** 2) / np.sum(ref_n ** 2)))
        out[f"lev{lev}_c{cmin}_r{rho}"] = {
            "rel_l2_uniform": eu, "rel_l2_near": en, "max_abs_near": float(np.max(np.abs(V[idx_n] - ref_n))),
            "plan_s": tp, "eval_ms": sum(ph.values()), "phases": ph,
            "levels": inf["n_levels"], "boxes": inf["n_boxes"], "nf_band": inf["nf_band"],
            "level_targets": inf["level_targets"][:8], "pairs": inf["n_band_pairs"],
            "n_stencil": inf["n_stencil_targets"], "nf_nh": inf["nf_nh"], "delta1": inf["delta1"]}
        print(json.dumps(out[f"lev{lev}_c{cmin}_r{rho}"]), flush=True)
        plan.destroy()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
