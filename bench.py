#!/usr/bin/env python
"""Benchmark: volume-potential evaluations per second (src + tgt points / s) on B200.

One "step" = one vp_eval over the whole workload: spread (NH+FH) -> cuFFT D2Z x2 -> multiply x2 ->
cuFFT Z2D x2 -> interpolation + local part (all of SURVEY §8(a) rows a4-a11; plan-time rows a1-a3
are not timed).  Inputs are resident in HBM when the timed region starts; L2 is flushed (256 MiB
write) between timed steps, outside the per-step CUDA events.

  python bench.py [--gpus N --steps K --warmup W] [--config c5] [--impl ours|reference]

Default workload: config 5 (BASELINE.json configs[4], the 16M-triangle config the north star's roofline target
names; it fits one B200).  --config c1..c4 for the others.

N > 1 (torchrun): every rank evaluates its own replica of the workload (the north star fixes one
GPU per problem), value = total points of all ranks / max-over-ranks time.
--impl reference times the CPU oracle (the method's definition, oracle/) on the host cores.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "volume-potential evals/sec (src+tgt pts/s) at tol 1e-9; % of B200 HBM roofline"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


def make_workload(name):
    from workloads import configs
    if name == "c1":
        return configs.config1(f="gauss")
    if name == "c2":
        return configs.config2()
    if name == "c3":
        return configs.config3()
    if name == "c4":
        return configs.config4()
    if name == "c5":
        return configs.config5()
    if name.startswith("c2n"):
        return configs.config2(n=int(name[3:]))
    raise SystemExit(f"unknown config {name}")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING recipe)."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def wait_first(self, timeout=5.0):
        t0 = time.time()
        while self.proc and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.05)

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, n in enumerate(names):
                if len(r) > 4 + k and r[4 + k].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def oracle_rate(w, budget_s=15.0, seed=99, prep=None):
    """Time the CPU oracle (as it stands) on a bounded seeded target sample: the per-triangle setup once (timed),
    then a target batch sized (by a 4-target probe) to take about budget_s.  Full-job estimate
    t_full = t_setup + t_batch * T / n (direct summation is linear in T up to near-field variation)."""
    import oracle
    from workloads import configs
    t0 = time.perf_counter()
    own = prep is None
    if own:
        prep = oracle.Prepared(w)
    t_setup = time.perf_counter() - t0
    probe = configs.sample_targets(w.T, 4, seed=seed + 7)
    t0 = time.perf_counter()
    prep.eval(w.targets[probe])
    per = (time.perf_counter() - t0) / len(probe)
    n = int(max(4, min(4096, budget_s / max(per, 1e-9))))
    idx = configs.sample_targets(w.T, n, seed=seed)
    t0 = time.perf_counter()
    prep.eval(w.targets[idx])
    dt = time.perf_counter() - t0
    if own:
        prep.close()
    t_full = t_setup + dt * w.T / len(idx)
    return {"value": (w.N + w.T) / t_full, "unit": "pts/s", "cores": oracle.num_threads(), "kind": "oracle",
            "cpu": cpu_model(),
            "sample": f"{len(idx)} of {w.T} targets (seeded uniform) against all {w.M} triangles: {dt:.2f} s, "
                      f"plus the per-triangle setup {t_setup:.2f} s; t_full = setup + batch * T / {len(idx)}",
            "seconds": dt, "setup_s": t_setup, "t_full_s": t_full, "n": len(idx)}


def ncu_traffic(workload, phase):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the phase's kernels, from the committed ncu
    --set full captures (profiles/r2/ncu_traffic.json, else r1's); None if that workload/phase was not captured."""
    for rnd in ("r2", "r1"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "ncu_traffic.json")) as fh:
                tab = json.load(fh)
        except Exception:
            continue
        for prefix, phases in tab.get("workloads", {}).items():
            if workload.startswith(prefix) and phase in phases:
                return phases[phase]["bytes"], phases[phase]["source"]
    return None, None


def max_over_ranks(x, dev=None):
    """Max of a per-rank float over all ranks (identity at world size 1); NCCL on the GPU, gloo in tests."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(world, pts_per_rank, ms_max):
    """Whole-job throughput: replicas (DESIGN.md §7 "replicas only") -> all ranks' points / slowest rank's time."""
    return world * pts_per_rank / (ms_max * 1e-3)


def run_reference(args, rank, world):
    """--impl reference: the oracle (the method's definition, oracle/) timed on the host cores, rank 0 only.  The
    per-triangle setup is paid once; every step evaluates a fresh seeded target batch sized so that the whole
    run stays within a few minutes (per-step budget min(10 s, 120 s / (steps + warmup)))."""
    if rank != 0:
        return
    import oracle
    w = make_workload(args.config)
    t0 = time.perf_counter()
    prep = oracle.Prepared(w)
    t_setup = time.perf_counter() - t0
    budget = args.ref_seconds or min(10.0, 120.0 / max(1, args.steps + args.warmup))
    for s in range(args.warmup):
        oracle_rate(w, budget_s=min(budget, 2.0), seed=500 + s, prep=prep)
    fulls = []
    last = None
    for s in range(args.steps):
        last = oracle_rate(w, budget_s=budget, seed=1000 + s, prep=prep)
        fulls.append(t_setup + last["seconds"] * w.T / last["n"])
    prep.close()
    t_full = float(np.mean(fulls))
    val = (w.N + w.T) / t_full
    cpu = {k: v for k, v in last.items() if k not in ("seconds", "setup_s", "t_full_s", "n")}
    cpu["value"] = val
    cpu["sample"] = (f"per step {last['sample'].split(' against')[0]} against all {w.M} triangles; setup "
                     f"{t_setup:.2f} s once; t_full = setup + batch time * T / n, mean over {args.steps} steps")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "pts/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_full * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "M": w.M, "N_src": w.N, "N_tgt": w.T, "tol": w.tol,
                       "parallelism": "cpu-oracle"},
            "cpu_baseline": cpu,
            "e2e": {"value": val, "unit": "pts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("VP_BENCH_CONFIG", "c5"))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU-baseline sample sized to ~this many seconds")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=None, help="--impl reference: per-step oracle budget (s)")
    ap.add_argument("--opt", action="append", default=[],
                    help="extra vp_opts field for A/B runs, e.g. --opt spread_pack=1 --opt fft_mode=1")
    ap.add_argument("--batch", type=int, default=4,
                    help="also time vp_eval_batch with this many fields (SURVEY §8(f) f3); 0 or 1 to skip")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2409_11998_b200 as vp

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w = make_workload(args.config)
    nodes = torch.from_numpy(np.ascontiguousarray(w.nodes)).to(dev)
    wts = torch.from_numpy(w.weights).to(dev)
    tg = torch.from_numpy(np.ascontiguousarray(w.targets)).to(dev)
    f = torch.from_numpy(w.f).to(dev)
    stream = torch.cuda.current_stream(dev)
    from workloads import rule
    # config 5: level bands off (delta_1 / sigma_min^2 = 0.016; parity 4.9e-10 without them)
    levels = -1 if w.name.startswith("c5") else 0
    extra = {k: int(v) for k, v in (o.split("=") for o in args.opt)}
    levels = extra.pop("levels", levels)  # --opt levels=0: auto level bands on config 5 (A/B of their cost)
    plan = vp.Plan(nodes, wts, tg, w.tol, boundary=w.boundary, targets_are_nodes=w.targets_are_nodes, stream=stream,
                   ref_nodes=rule.BARY[:, 1:3], levels=levels, **extra)
    info = plan.info()
    out = torch.empty(w.T, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    phases = []
    with ClockSampler(local) as clk:
        clk.wait_first()
        # W warm-up evals, then keep the GPU under load for >= 0.5 s so the clock samples (100 ms period)
        # straddle the timed region
        t_w = time.perf_counter()
        nw = 0
        while nw < args.warmup or time.perf_counter() - t_w < 0.5:
            plan.eval(f, out)
            nw += 1
            if nw % 8 == 0:
                torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_wall0 = time.perf_counter()
        for s in range(args.steps):
            flush.zero_()                       # L2 flush outside the timed events
            evs[s][0].record(stream)
            plan.eval(f, out)                   # fork/join across three streams; joined on `stream`
            evs[s][1].record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.mean(step_ms))
    ms_max = max_over_ranks(ms, dev)
    pts = (w.N + w.T)
    value = aggregate_rate(world, pts, ms_max)
    kern, ffts = plan.launch_count()

    # ---- per-phase times: separate profiled evals (serial on one stream so that the CUDA events bracket each
    # phase; the timed steps above overlap the far-history chain and the local part with the near-history FFTs)
    plan.set_profiling(True)
    for s in range(max(3, min(args.steps, 10))):
        flush.zero_()
        plan.eval(f, out)
        phases.append(plan.phase_times())
    plan.set_profiling(False)
    ph = {k: float(np.mean([p[k] for p in phases])) for k in phases[0]}
    serial_ms = float(sum(ph.values()))
    # ---- roofline (SURVEY §8(d) bytes model): per unit, spread reads x, y, w, f (32 B per source)
    # and writes the NH grid once (8 B per cell); interp_local reads x, y and writes out (24 B per target), reads
    # the NH grid once (8 B per cell) and the node target's own f or V_L word (8 B per node target).  KNN
    # stencil entries (8 B each: int32 index + fp32 weight) are reported separately as overhead, not as algorithmic bytes.
    cells = float(info["nf_nh"]) ** 2
    K_st = info["deriv_k"]
    S_st = info["n_stencil_targets"]
    T_node = w.N if w.targets_are_nodes or w.name.startswith("c5") else 0
    alg = {"spread": 32.0 * w.N + 8.0 * cells,
           "interp_local": 24.0 * w.T + 8.0 * cells + 8.0 * T_node}
    peaks, peak_src = load_peaks()
    hbm = peaks["hbm_gbs"]
    kstat = {}
    for k in ("spread", "interp_local"):
        a = alg[k] / (ph[k] * 1e-3) / 1e9
        tr, trs = ncu_traffic(w.name, k)
        kstat[k] = {"ms": ph[k], "algorithmic_bytes": alg[k], "achieved": a, "frac": a / hbm, "traffic": tr,
                    "traffic_source": trs}
    dom = max(kstat, key=lambda k: kstat[k]["ms"])
    both_ms = ph["spread"] + ph["interp_local"]
    roof = {"kernel": dom, "bound": "hbm", "achieved": kstat[dom]["achieved"], "peak": hbm, "unit": "GB/s",
            "frac": kstat[dom]["frac"], "traffic": kstat[dom]["traffic"], "traffic_source": kstat[dom]["traffic_source"],
            "peak_source": peak_src, "algorithmic_bytes": alg[dom], "kernel_ms": ph[dom],
            "kernels": kstat,
            "spread_plus_interp": {"ms": both_ms, "algorithmic_bytes": alg["spread"] + alg["interp_local"],
                                   "frac": (alg["spread"] + alg["interp_local"]) / (both_ms * 1e-3) / 1e9 / hbm,
                                   "north_star_target_frac": 0.5},
            "overhead_bytes": {"knn_stencil": 8.0 * K_st * S_st, "stencil_targets": S_st, "stencil_k": K_st},
            "bytes_model": "SURVEY §8(d): spread 32 B/source + 8 B/NH cell; interp 24 B/target + 8 B/NH cell + "
                           "8 B/node target; phase times from the serial profiled evals (phase_ms)",
            "co_bound": "fp64 issue + shared-memory wavefronts (DESIGN.md §5.1/§5.4, profiles/r2/microbench)"}

    # ---- end-to-end through the public API with host buffers (pinned)
    f_pin = torch.from_numpy(w.f).pin_memory()
    out_pin = torch.empty(w.T, dtype=torch.float64).pin_memory()
    plan.set_profiling(False)
    plan.eval_host(f_pin.numpy(), out_pin.numpy())
    e2e_ms = []
    for s in range(max(3, args.steps // 2)):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan.eval_host(f_pin.numpy(), out_pin.numpy())
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_serial = max_over_ranks(float(np.mean(e2e_ms)), dev)
    # pipelined: K = steps fields through vp_eval_host_many (H2D of field k+1 and D2H of field k-1 overlap the
    # evaluation of field k); every step still copies its f in and its out back.  Device-timed with CUDA events on
    # the plan's stream (the call orders its copy streams after / before it).  Inputs (1.5 GB at config 5) exceed L2.
    nk = max(3, args.steps)
    plan.eval_host_many([f_pin.numpy()] * 2, [out_pin.numpy()] * 2)
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ea.record(stream)
    plan.eval_host_many([f_pin.numpy()] * nk, [out_pin.numpy()] * nk)
    eb.record(stream)
    torch.cuda.synchronize()
    e2e_pipe = max_over_ranks(ea.elapsed_time(eb) / nk, dev)
    e2e = {"value": aggregate_rate(world, pts, e2e_pipe), "unit": "pts/s", "h2d_bytes_per_step": 8 * w.N,
           "d2h_bytes_per_step": 8 * w.T, "ms_per_step": e2e_pipe, "api": "vp_eval_host_many",
           "schedule": f"{nk} fields streamed from pinned host memory; H2D(k+1) and D2H(k-1) overlap eval(k)",
           "serial": {"api": "vp_eval_host", "ms_per_step": e2e_serial,
                      "value": aggregate_rate(world, pts, e2e_serial), "timing": "wall clock per call"}}

    # ---- batched fields (vp_eval_batch): K scaled copies of f, same plan; device-timed like the steps
    batch = None
    if args.batch and args.batch > 1:
        KB = args.batch
        F = torch.stack([f * (1.0 + 0.25 * k) for k in range(KB)]).contiguous()
        OB = torch.empty(KB, w.T, dtype=torch.float64, device=dev)
        plan.eval_batch(F, OB)
        bms = []
        for s in range(max(3, args.steps // 2)):
            flush.zero_()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            b0.record(stream)
            plan.eval_batch(F, OB)
            b1.record(stream)
            torch.cuda.synchronize()
            bms.append(b0.elapsed_time(b1))
        bmax = max_over_ranks(float(np.mean(bms)), dev)
        batch = {"K": KB, "ms_per_batch": bmax, "value": aggregate_rate(world, KB * pts, bmax), "unit": "pts/s",
                 "note": "K fields per vp_eval_batch; value counts K * (N_src + N_tgt) points"}
        del F, OB

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = oracle_rate(w, budget_s=args.cpu_seconds)
            for k in ("seconds", "setup_s", "t_full_s", "n"):
                cpu.pop(k)
        line = {"metric": METRIC, "value": value, "unit": "pts/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": w.name, "M": w.M, "N_src": w.N, "N_tgt": w.T, "tol": w.tol,
                           "parallelism": f"replicas x{world}" if world > 1 else "single-gpu",
                           "l2": "flushed between steps (256 MiB write outside the step events)",
                           "nf_nh": info["nf_nh"], "nf_fh": info["nf_fh"], "w_es": info["w_es"],
                           "deriv": f"{['auto', 'knn', 'triangle'][info['deriv_mode']]} (knn deg {info['deriv_degree']} "
                                    f"K {K_st} on {S_st} targets)", "levels": info["n_levels"], "plan_ms": info["plan_ms"],
                           "spread": ("row-pair strips (k_spread_pair)" if extra.get("spread_pack", 0) == 0 and info["w_es"] <= 12
                                      else "32-column strips (k_spread_strip)"), "spread_items": info["n_batches"],
                           "fft_path": {"nh": ["fused", "cufft2d", "cufftrows+4step", "rows4+4step"][info["fft_path_nh"]],
                                        "fh": ["fused", "cufft2d", "cufftrows+4step", "rows4+4step"][info["fft_path_fh"]]},
                           "opts": extra},
                "phase_ms": ph, "serial_ms_per_step": serial_ms, "wall_ms_per_step": t_wall * 1e3 / args.steps,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "batch": batch,
                "clocks": clk.summary(), "gpu_launches": kern * args.steps,
                "cufft_execs": ffts * args.steps}
        print(json.dumps(line))
    plan.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
