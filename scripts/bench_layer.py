#!/usr/bin/env python
"""Measurement of the layer potentials and BIE solves on B200.

Workload: config 3's star domain (BASELINE.json configs[2]: 1M graded triangles, 12M quadrature nodes) with its
boundary r = 1 + 0.3 cos 5 theta as NCH chunks of degree 16 (default 4096 chunks, 69632 boundary nodes).
  eval_slp / eval_dlp : S[sigma], D[mu] at all 12M volume nodes (history on the plan's grids + telescoped local
                        parts), one step = one call, CUDA events on the plan's stream, L2 flushed between steps;
                        pts/s = (boundary nodes + targets) / time.
  bie_solve           : interior Dirichlet (-1/2 + D) mu = g on a plan whose targets are the boundary nodes
                        (same volume nodes -> same grids); ms per solve, GMRES iterations, ms per iteration.
Prints one JSON line per measurement.  Synthetic data (seeded); see DESIGN.md §4 for the inputs.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--nch", type=int, default=4096)
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--skip-bie", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2409_11998_b200 as vp
    from workloads import configs, geometry
    dev = torch.device("cuda", 0)
    w = configs.config3()
    ch = geometry.star_chunks(args.nch, q=16)
    thn = np.arctan2(ch[..., 1], ch[..., 0])
    nb = ch.shape[0] * ch.shape[1]
    nodes = torch.from_numpy(np.ascontiguousarray(w.nodes)).to(dev)
    wts = torch.from_numpy(w.weights).to(dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    dens = torch.from_numpy(1.0 + 0.5 * np.cos(2 * thn) + 0.3 * np.sin(3 * thn)).to(dev)

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for a, b in ev:
            flush.zero_()
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        return float(np.mean([a.elapsed_time(b) for a, b in ev]))

    tg = torch.from_numpy(np.ascontiguousarray(w.targets)).to(dev)
    t0 = time.perf_counter()
    plan = vp.Plan(nodes, wts, tg, w.tol, boundary=("chunks", ch), parts=vp.PART_HISTORY, stream=stream)
    plan.set_layer_levels(args.levels)
    plan.prepare_slp()
    plan.prepare_dlp()
    torch.cuda.synchronize()
    prep_s = time.perf_counter() - t0
    info = plan.info()
    out = torch.empty(w.T, dtype=torch.float64, device=dev)
    base = {"workload": f"c3_star_nodes_{w.T}_chunks_{args.nch}x17", "tol": w.tol, "levels": args.levels,
            "nf_nh": info["nf_nh"], "nf_fh": info["nf_fh"], "plan_and_prepare_s": prep_s,
            "l2": "flushed between steps (256 MiB write outside the step events)"}
    for name, fn in (("eval_slp", lambda: plan.eval_slp(dens, out)), ("eval_dlp", lambda: plan.eval_dlp(dens, out))):
        ms = timed(fn)
        kern, ffts = plan.launch_count()
        print(json.dumps({"metric": f"{name} (boundary + target pts/s)", "value": (nb + w.T) / (ms * 1e-3),
                          "unit": "pts/s", "ms_per_step": ms, "steps": args.steps, "warmup": args.warmup,
                          "dtype": "f64", "data": "synthetic", "gpu_launches": kern + ffts,
                          "config": dict(base, n_boundary=nb, T=w.T)}), flush=True)
    plan.destroy()
    if args.skip_bie:
        return
    bn = torch.from_numpy(np.ascontiguousarray(ch.reshape(-1, 2))).to(dev)
    A = vp.Plan(nodes, wts, bn, w.tol, boundary=("chunks", ch), parts=vp.PART_HISTORY, stream=stream)
    A.set_layer_levels(args.levels)
    A.prepare_dlp()
    x, y = bn[:, 0], bn[:, 1]
    g = x ** 3 - 3 * x * y * y + 0.4 * x + 0.7
    res = {}

    def solve():
        res["r"] = A.bie_solve(vp.BIE_DIRICHLET_INT, g, tol=1e-12)
    ms = timed(solve)
    _, it, rr = res["r"]
    print(json.dumps({"metric": "bie_solve interior Dirichlet (ms per solve)", "value": ms, "unit": "ms",
                      "higher_is_better": False, "iterations": it, "resid": rr, "ms_per_iteration": ms / max(it, 1),
                      "steps": args.steps, "warmup": args.warmup, "dtype": "f64", "data": "synthetic",
                      "config": dict(base, n_boundary=nb, gmres_tol=1e-12, restart=50)}), flush=True)
    A.destroy()


if __name__ == "__main__":
    main()
