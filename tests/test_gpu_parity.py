"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star):
  * full V vs the oracle's exact integral: relative l2 <= 10 x tol
  * smooth (history) part vs the direct real-space sum of G_H[delta_1] (and the direct DFT of the same
    split): relative l2 <= 1e-12 at eps = 1e-13
"""
import json
import os

import numpy as np
import pytest

import oracle
from strata import extra_square_targets, report, square_strata
from workloads import configs, fields

torch = pytest.importorskip("torch")
import paper_2409_11998_b200 as vp  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda"


def rel_l2(a, b):
    return float(np.sqrt(np.sum((a - b) ** 2) / np.sum(b ** 2)))


def log_result(name, value):
    """Merge one result into the JSON file named by VP_PARITY_LOG (profiles/r2/SUMMARY.md is built from it)."""
    path = os.environ.get("VP_PARITY_LOG")
    print(name, value)
    if not path:
        return
    try:
        with open(path) as fh:
            d = json.load(fh)
    except Exception:
        d = {}
    d[name] = value
    with open(path, "w") as fh:
        json.dump(d, fh, indent=1, default=float)


def check_strata(name, strata, V, prep, targets, bar):
    """oracle at the union of the strata (one prepared oracle), per-stratum rel l2 logged and held to the bar"""
    allidx = np.unique(np.concatenate([v for v in strata.values() if len(v)]))
    ref = prep.eval(targets[allidx])
    by = dict(zip(allidx.tolist(), ref))
    res = report(name, strata, V, by, {})
    log_result(name, {k: {"n": n, "rel_l2": e} for k, (n, e) in res.items()})
    for k, (n, e) in res.items():
        if n:
            assert e <= bar, (name, k, n, e)
    return res


@pytest.fixture(scope="module")
def c2full():
    return configs.config2()


@pytest.fixture(scope="module")
def c2prep(c2full):
    p = oracle.Prepared(c2full)
    yield p
    p.close()


@pytest.fixture(scope="module")
def c5full():
    return configs.config5()


def to_dev(w):
    return (torch.from_numpy(np.ascontiguousarray(w.nodes)).to(DEV), torch.from_numpy(w.weights).to(DEV),
            torch.from_numpy(np.ascontiguousarray(w.targets)).to(DEV), torch.from_numpy(w.f).to(DEV))


def make_plan(w, **kw):
    nodes, wts, tg, f = to_dev(w)
    kw.setdefault("boundary", w.boundary)
    kw.setdefault("targets_are_nodes", w.targets_are_nodes)
    tol = kw.pop("tol", w.tol)
    return vp.Plan(nodes, wts, tg, tol, **kw), f


# ------------------------------------------------------------------------------------ smooth part
@pytest.mark.parametrize("which", ["c1", "c2small"])
def test_smooth_part_vs_direct_GH_sum(which):
    w = configs.config1() if which == "c1" else configs.config2(n=40)
    d1 = 3.0 * w.weights.mean()
    plan, f = make_plan(w, tol=1e-13, parts=vp.PART_HISTORY, delta1_override=d1)
    V = plan.eval(f).cpu().numpy()
    idx = configs.sample_targets(w.T, 1500, seed=21)
    ref = oracle.smooth_direct(w.nodes.reshape(-1, 2), (w.f * w.weights).ravel(), w.targets[idx], d1)
    e = rel_l2(V[idx], ref)
    print(which, "smooth rel l2", e, plan.info()["w_es"])
    assert e < 1e-12


def _smooth_gate(w, n_tg, seed, extra_tg=None, **plan_kw):
    """history part at eps = 1e-13 on the full source set vs oracle.smooth_direct (north star: <= 1e-12)"""
    d1 = 3.0 * float(w.weights.mean())
    idx = configs.sample_targets(w.T, n_tg, seed=seed)
    tg_np = w.targets[idx]
    if extra_tg is not None:
        tg_np = np.concatenate([tg_np, extra_tg])
    nodes = torch.from_numpy(np.ascontiguousarray(w.nodes)).to(DEV)
    wts = torch.from_numpy(w.weights).to(DEV)
    f = torch.from_numpy(w.f).to(DEV)
    plan = vp.Plan(nodes, wts, torch.from_numpy(np.ascontiguousarray(tg_np)).to(DEV), 1e-13,
                   parts=vp.PART_HISTORY, delta1_override=d1, **plan_kw)
    info = plan.info()
    V = plan.eval(f).cpu().numpy()
    plan.destroy()
    del nodes, wts, f
    ref = oracle.smooth_direct(w.nodes.reshape(-1, 2), (w.f * w.weights).ravel(), tg_np, d1)
    e = rel_l2(V, ref)
    log_result(f"smooth_gate_{w.name}", {"rel_l2": e, "targets": int(tg_np.shape[0]), "nf_nh": info["nf_nh"],
                                         "nf_fh": info["nf_fh"], "w_es": info["w_es"],
                                         "transform": ["fused", "cuFFT 2D", "cuFFT rows + four-step",
                                                       "own rows + four-step"][info["fft_path_nh"]]})
    assert e < 1e-12, e


def test_smooth_gate_full_c2(c2full):
    _smooth_gate(c2full, 512, 201)


def test_smooth_gate_full_c4():
    """n_f,NH > 6400 at eps = 1e-13: the cuFFT transform path"""
    _smooth_gate(configs.config4(), 64, 202)


def test_smooth_gate_c5_subsample(c5full):
    """all 192M config-5 sources spread at eps = 1e-13 (w = 14, cuFFT 2D transforms); 64 sampled targets + 16
    near-corner points"""
    _smooth_gate(c5full, 64, 203, extra_tg=extra_square_targets(1e-8, n_edge=0, n_corner=4))


def test_smooth_part_vs_direct_dft():
    rng = np.random.default_rng(31)
    src = rng.uniform(0.1, 0.9, (400, 2))
    c = rng.standard_normal(400)
    # 400 sources as 100 "triangles" of 4 nodes each; weights = c, f = 1 so c_j = f_j w_j
    nodes = torch.from_numpy(src.reshape(100, 4, 2).copy()).to(DEV)
    wts = torch.from_numpy(np.abs(c).reshape(100, 4)).to(DEV)
    fv = torch.from_numpy(np.sign(c).reshape(100, 4)).to(DEV)
    tg_np = np.concatenate([rng.uniform(0.1, 0.9, (60, 2)), src[:10]])
    tg = torch.from_numpy(tg_np).to(DEV)
    d1 = 2e-3
    plan = vp.Plan(nodes, wts, tg, 1e-13, parts=vp.PART_HISTORY, delta1_override=d1)
    V = plan.eval(fv).cpu().numpy()
    p = oracle.dft_params(src, tg_np, d1, 32 * d1, 1e-14)
    ref = oracle.smooth_dft(src, c, tg_np, d1, 32 * d1, **p)
    ref2 = oracle.smooth_direct(src, c, tg_np, d1)
    assert rel_l2(V, ref) < 1e-12
    assert rel_l2(V, ref2) < 1e-12


# ------------------------------------------------------------------------------------ full V
@pytest.mark.parametrize("f", ["const", "gauss"])
def test_config1_full_parity(f):
    w = configs.config1(f=f)
    plan, fd = make_plan(w)
    V = plan.eval(fd).cpu().numpy()
    ref = oracle.workload_potential(w)            # all 24k targets
    e = rel_l2(V, ref)
    print("config1", f, "rel l2 vs oracle", e, plan.info())
    assert e <= 10 * w.tol
    if f == "const":
        ex = (1 - (w.targets ** 2).sum(1)) / 4
        assert rel_l2(V, ex) <= 10 * w.tol


def test_config2_full_size_sampled(c2full, c2prep):
    """Full config 2 in the bench launch configuration: 4096 uniform targets plus edge / corner / sliver strata
    (relative l2 per stratum <= 10 tol)."""
    w = c2full
    plan, fd = make_plan(w)
    info = plan.info()
    V = plan.eval(fd).cpu().numpy()
    st = square_strata(w.targets, info["delta1"], tri=w.tri, n_nodes=w.N)
    check_strata("c2_full", st, V, c2prep, w.targets, 10 * w.tol)


def test_determinism_and_host_path():
    w = configs.config2(n=60)
    plan, fd = make_plan(w)
    a = plan.eval(fd).cpu().numpy()
    b = plan.eval(fd).cpu().numpy()
    assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(a))        # atomics order only
    h = plan.eval_host(w.f)
    assert np.max(np.abs(h - a)) <= 1e-13 * np.max(np.abs(a))


def test_nonfinite_and_degenerate_inputs():
    w = configs.config2(n=20)
    nodes, wts, tg, f = to_dev(w)
    bad = wts.clone()
    bad[3, 2] = float("nan")
    with pytest.raises(vp.VpError) as ei:
        vp.Plan(nodes, bad, tg, 1e-9)
    assert ei.value.status == vp.VP_ERR_NONFINITE
    plan = vp.Plan(nodes, wts, tg, 1e-9, boundary=w.boundary, targets_are_nodes=True)
    fb = f.clone()
    fb[0, 0] = float("inf")
    assert not plan.check_finite(fb)
    assert plan.check_finite(f)
    # zero-weight (degenerate) triangles are accepted and contribute nothing
    w0 = wts.clone()
    w0[:5] = 0.0
    plan0 = vp.Plan(nodes, w0, tg, 1e-9, boundary=w.boundary, targets_are_nodes=True)
    V = plan0.eval(f)
    assert torch.isfinite(V).all()


def test_off_node_targets(c2full, c2prep):
    """Targets that are not quadrature nodes (config 5 style) on the full config-2 mesh (f resolved by the 12-point
    rule): jets from the kNN fit including f itself; 10 x tol, with edge / corner strata."""
    w = c2full
    rng = np.random.default_rng(5)
    tg_np = np.concatenate([rng.uniform(0, 1, (3000, 2)), extra_square_targets(3 * float(w.weights.mean()),
                                                                                n_edge=128, n_corner=32)])
    nodes, wts, _, f = to_dev(w)
    plan = vp.Plan(nodes, wts, torch.from_numpy(tg_np).to(DEV), w.tol, boundary=w.boundary)
    V = plan.eval(f).cpu().numpy()
    st = square_strata(tg_np, plan.info()["delta1"], n_uniform=256, n_edge=128, n_corner=32)
    check_strata("c2_offnode", st, V, c2prep, tg_np, 10 * w.tol)


# ------------------------------------------------------------------------------------ graded meshes (a12)
def _near_source_idx(w, n, seed):
    d = np.hypot(w.targets[:, 0] - 0.3, w.targets[:, 1] + 0.2)
    near = np.nonzero(d < 6e-3)[0]
    return near[configs.sample_targets(near.size, n, seed=seed)]


def test_config3_small_levels():
    """Scaled-down config 3 (graded star, nonconforming patches): the level bands make the parity bar reachable;
    one global delta_1 does not (R15)."""
    w = configs.config3(M_target=60000, lmin=7, lmax=13, g=0.1)
    idx = np.unique(np.concatenate([configs.sample_targets(w.T, 512, seed=33), _near_source_idx(w, 256, 34)]))
    # steeper grading than the full config (g = 0.1): default C_min = 1.5
    ref = oracle.workload_potential(w, idx)
    plan, fd = make_plan(w)
    info = plan.info()
    V = plan.eval(fd).cpu().numpy()
    e = rel_l2(V[idx], ref)
    print("config3 small levels", info["n_levels"], info["level_targets"][:8], "rel l2", e)
    assert info["n_levels"] >= 3
    assert e <= 10 * w.tol
    plan0, _ = make_plan(w, levels=-1)
    e0 = rel_l2(plan0.eval(fd).cpu().numpy()[idx], ref)
    print("config3 small, global delta only:", e0)
    assert e0 > 100 * e


def test_config3_full_size_sampled():
    w = configs.config3()
    st = {"uniform": configs.sample_targets(w.T, 4096, seed=35), "near_source": np.sort(_near_source_idx(w, 256, 36))}
    prep = oracle.Prepared(w)
    plan, fd = make_plan(w)
    V = plan.eval(fd).cpu().numpy()
    print("config3 levels", plan.info()["n_levels"], plan.info()["level_targets"][:8])
    check_strata("c3_full", st, V, prep, w.targets, 10 * w.tol)
    prep.close()


# ------------------------------------------------------------------------------------ configs 4 / 5 (full size)
def test_config4_full_size_sampled():
    """4M uniform triangles, Fourier field |k| <= 64, tol 1e-10; TRIANGLE-mode jets (bench launch configuration)."""
    from workloads import rule
    w = configs.config4()
    plan, fd = make_plan(w, ref_nodes=rule.BARY[:, 1:3])
    info = plan.info()
    V = plan.eval(fd).cpu().numpy()
    plan.destroy()
    st = square_strata(w.targets, info["delta1"], n_uniform=128, seed=41)
    prep = oracle.Prepared(w)
    check_strata("c4_full", st, V, prep, w.targets, 10 * w.tol)
    prep.close()


def test_config5_full_size_sampled(c5full):
    """16M quadtree-graded triangles, 20 Gaussians, 192M node + 4M random targets, tol 1e-9 (bench launch
    configuration) plus 512 extra off-node targets in the edge band and at the corners.  Level bands are off
    (levels=-1): delta_1 / sigma_min^2 = 0.016, so V_L[delta_1] is accurate without them.
    Strata: uniform nodes, edge, corners, slivers, off-node."""
    from workloads import rule
    w = c5full
    d1 = 3.0 * float(w.weights.mean())
    extra = extra_square_targets(d1, n_edge=256, n_corner=64, seed=53)
    tg_np = np.concatenate([w.targets, extra])
    nodes, wts, _, fd = to_dev(w)
    plan = vp.Plan(nodes, wts, torch.from_numpy(tg_np).to(DEV), w.tol, boundary=w.boundary, targets_are_nodes=True,
                   ref_nodes=rule.BARY[:, 1:3], levels=-1)
    info = plan.info()
    V = plan.eval(fd).cpu().numpy()
    plan.destroy()
    del nodes, wts, fd
    T0 = w.T
    st = square_strata(tg_np[:T0], info["delta1"], n_uniform=96, n_edge=128, n_corner=32, tri=w.tri, n_nodes=w.N,
                       n_offnode=64, seed=51)
    ne = len(extra) - 256
    for k in range(4):
        st[f"corner{k}"] = np.concatenate([st[f"corner{k}"], T0 + np.arange(64 * k, 64 * k + 64)])
    st["edge"] = np.concatenate([st["edge"], T0 + ne + np.arange(256)])
    prep = oracle.Prepared(w)
    check_strata("c5_full", st, V, prep, tg_np, 10 * w.tol)
    prep.close()


def test_deterministic_mode_bit_identical(c2full, c2prep):
    """opts.deterministic: colour-separated spreading without atomics -> bit-identical evals, on the
    full config-2 mesh (f resolved by the 12-point rule) and held to the oracle at 10 x tol."""
    w = c2full
    plan, fd = make_plan(w, deterministic=True)
    a = plan.eval(fd).cpu().numpy()
    b = plan.eval(fd).cpu().numpy()
    assert np.array_equal(a, b)
    plan.destroy()
    plan2, _ = make_plan(w)
    c = plan2.eval(fd).cpu().numpy()
    assert np.max(np.abs(a - c)) <= 1e-13 * np.max(np.abs(c))
    idx = configs.sample_targets(w.T, 256, seed=61)
    e = rel_l2(a[idx], c2prep.eval(w.targets[idx]))
    log_result("c2_deterministic", {"n": 256, "rel_l2": e})
    assert e <= 10 * w.tol


def test_tiny_and_ragged_inputs_run():
    """Degenerate sizes: one triangle / one target, a handful of triangles with targets outside the mesh; the
    plan and eval succeed and return finite values (no boundary terms: the local expansion is not meant to be
    accurate at the edges of a one-triangle domain, so only sanity is checked)."""
    from workloads import rule
    tri = np.array([[[0.2, 0.2], [0.7, 0.25], [0.3, 0.8]]])
    nodes = np.einsum("kj,mjd->mkd", rule.BARY, tri)
    area = 0.5 * abs(np.cross(tri[0, 1] - tri[0, 0], tri[0, 2] - tri[0, 0]))
    wts = np.tile(rule.WEIGHTS * area, (1, 1))
    for tg in [np.array([[0.4, 0.4]]), np.array([[0.4, 0.4], [3.0, -2.0], [0.2, 0.2]])]:
        plan = vp.Plan(torch.from_numpy(nodes).to(DEV), torch.from_numpy(wts).to(DEV), torch.from_numpy(tg).to(DEV),
                       1e-8)
        V = plan.eval(torch.ones(1, 12, dtype=torch.float64, device=DEV)).cpu().numpy()
        assert np.all(np.isfinite(V)) and V.shape == (tg.shape[0],)
        if tg.shape[0] == 3:  # the far target sees only the smooth part: exact to the NUFFT tolerance
            far = oracle.volume_potential(tri, None, None, fields.const(1.0), tg[1:2])[0]
            assert abs(V[1] - far) < 1e-7 * abs(far)


def test_loose_tolerance_parity():
    """tol 1e-4 (w = 5): parity at 10 x tol."""
    w = configs.config2(n=60)
    plan, fd = make_plan(w, tol=1e-4)
    assert plan.info()["w_es"] == 5
    V = plan.eval(fd).cpu().numpy()
    idx = configs.sample_targets(w.T, 96, seed=71)
    ref = oracle.workload_potential(w, idx)
    assert rel_l2(V[idx], ref) <= 1e-3


@pytest.mark.parametrize("tol", [1e-4, 1e-7, 1e-9, 1e-11, 1e-13])
def test_strip_spread_matches_tile_spread(tol):
    """Register-strip spreading (default) vs the shared-memory tile batches (spread_tile=32) on the same plan
    inputs: same grid, so the history parts agree to rounding.  Mixed density: a uniform background, a dense
    clump (thousands of nodes in a few NH cells -> strips split into several work items) and nodes along the
    box edge (footprints wrapping around the periodic grid)."""
    rng = np.random.default_rng(91)
    bg = rng.uniform(0.0, 1.0, (3000, 12, 2))
    clump = 0.5 + 1e-4 * rng.standard_normal((800, 12, 2))
    edge = np.stack([rng.uniform(0, 1, (200, 12)), rng.choice([0.0, 1.0], (200, 12))], axis=-1)
    nodes_np = np.concatenate([bg, clump, edge])
    wts_np = rng.uniform(0.5, 1.5, nodes_np.shape[:2]) / nodes_np.shape[0]
    f_np = rng.standard_normal(nodes_np.shape[:2])
    tg_np = rng.uniform(0.0, 1.0, (2000, 2))
    nodes, wts, tg, f = (torch.from_numpy(np.ascontiguousarray(a)).to(DEV) for a in (nodes_np, wts_np, tg_np, f_np))
    out = []
    # spread_pack 0: row-pair strips (w <= 12) / 32-column strips; 1: 32-column packs; 2: 32-column single steps
    for st, pk in ((32, 0), (0, 0), (0, 1), (0, 2)):
        plan = vp.Plan(nodes, wts, tg, tol, parts=vp.PART_HISTORY, spread_tile=st, spread_pack=pk)
        out.append(plan.eval(f).cpu().numpy())
    scale = np.max(np.abs(out[0]))
    for k in range(1, 4):
        assert np.max(np.abs(out[k] - out[0])) <= 1e-13 * scale, k


@pytest.mark.parametrize("which", ["c1", "c2small", "c2loose"])
def test_fused_fft_matches_cufft(which):
    """Fused row/column transforms with the multiply in the column pass (default) vs cuFFT D2Z + k_multiply +
    Z2D (fft_mode=1) on the same plan inputs: the full V agrees to rounding."""
    if which == "c1":
        w, tol = configs.config1(), None
    elif which == "c2small":
        w, tol = configs.config2(n=60), None
    else:
        w, tol = configs.config2(n=60), 1e-4
    out = []
    for mode in (0, 1):
        kw = {"fft_mode": mode}
        if tol:
            kw["tol"] = tol
        plan, f = make_plan(w, **kw)
        out.append(plan.eval(f).cpu().numpy())
    assert np.max(np.abs(out[0] - out[1])) <= 1e-12 * np.max(np.abs(out[1]))


@pytest.mark.parametrize("K", [2, 3, 5])
def test_eval_batch_matches_single_evals(K, c2full):
    """vp_eval_batch: K distinct analytic fields (seeded 5-Gaussian sets) on the full config-2
    mesh through the shared strip pass (pairs / quadruples + a single): the batch equals K separate vp_eval calls
    to rounding, and EVERY field matches the oracle at 10 x tol (linearity in c_j)."""
    w = c2full
    plan, _ = make_plan(w)
    flds = []
    for k in range(K):
        g = np.random.default_rng(900 + 10 * K + k)
        flds.append(fields.gauss(g.standard_normal(5), g.uniform(0, 1, 5), g.uniform(0, 1, 5),
                                 g.uniform(0.02, 0.1, 5) ** 2))
    F = torch.stack([torch.from_numpy(fields.evaluate(fl, w.nodes[..., 0], w.nodes[..., 1])).to(DEV)
                     for fl in flds]).contiguous()
    VB = plan.eval_batch(F).cpu().numpy()
    idx = configs.sample_targets(w.T, 128, seed=111 + K)
    errs = []
    for k in range(K):
        Vk = plan.eval(F[k]).cpu().numpy()
        assert np.max(np.abs(VB[k] - Vk)) <= 1e-13 * np.max(np.abs(Vk)), k
        ref = oracle.volume_potential(w.tri, w.curved, w.circle, flds[k], w.targets[idx])
        errs.append(rel_l2(VB[k][idx], ref))
    log_result(f"c2_batch_K{K}", {"n": 128, "rel_l2_per_field": errs})
    assert max(errs) <= 10 * w.tol, errs


@pytest.mark.parametrize("tol", [1e-4, 1e-6, 1e-8, 1e-9, 1e-11])
def test_eval_batch_pair2_widths(tol):
    """Four- and two-field row-pair spreaders (k_spread_pair4 / k_spread_pair2, w <= 10; w = 12 at 1e-11 falls back
    to one pass per field): K = 2, 3, 4, 7 random fields on clustered random nodes that reach the periodic wrap of
    the grid; the batch equals the single evals, the pairs-only (batch_pair = 2) and the per-field passes
    (batch_pair = 1) to rounding."""
    rng = np.random.default_rng(int(-np.log10(tol)) + 500)
    n = 12 * 700
    pts = np.concatenate([rng.uniform(0.0, 1.0, (n // 2, 2)), 0.5 + 0.02 * rng.standard_normal((n - n // 2, 2))])
    nodes_np = pts.reshape(-1, 12, 2)
    wts_np = rng.uniform(0.5, 1.5, nodes_np.shape[:2]) / n
    tg_np = np.concatenate([pts[::5], rng.uniform(0.0, 1.0, (200, 2))])
    nodes, wts, tg = (torch.from_numpy(np.ascontiguousarray(a)).to(DEV) for a in (nodes_np, wts_np, tg_np))
    d1 = 3.0 * float(wts_np.mean())
    F = torch.from_numpy(rng.standard_normal((7,) + nodes_np.shape[:2])).to(DEV)
    plan = vp.Plan(nodes, wts, tg, tol, parts=vp.PART_HISTORY, delta1_override=d1)
    plan1 = vp.Plan(nodes, wts, tg, tol, parts=vp.PART_HISTORY, delta1_override=d1, batch_pair=1)
    plan2 = vp.Plan(nodes, wts, tg, tol, parts=vp.PART_HISTORY, delta1_override=d1, batch_pair=2)
    Vs = [plan.eval(F[k].contiguous()).cpu().numpy() for k in range(7)]
    for K in (2, 3, 4, 7):  # pair; pair + single; quadruple; quadruple + pair + single
        VB = plan.eval_batch(F[:K].contiguous()).cpu().numpy()
        V1 = plan1.eval_batch(F[:K].contiguous()).cpu().numpy()
        V2 = plan2.eval_batch(F[:K].contiguous()).cpu().numpy()
        for k in range(K):
            sc = np.max(np.abs(Vs[k]))
            assert np.max(np.abs(VB[k] - Vs[k])) <= 1e-13 * sc, (K, k)
            assert np.max(np.abs(V1[k] - Vs[k])) <= 1e-13 * sc, (K, k)
            assert np.max(np.abs(V2[k] - Vs[k])) <= 1e-13 * sc, (K, k)
    w_es = plan.info()["w_es"]
    assert (w_es <= 10) == (tol >= 1e-9), w_es  # the cases cover both the two-field kernel and the fallback


def test_strip_spread_lattice_nodes():
    """Nodes on a dyadic lattice (coordinates k/256, many of them exactly on NH cell boundaries for power-of-two
    related grids): strip spreading (plan-time strip keys and eval-time footprints use the same rounding) agrees
    with the tile batches and with the direct G_H sum of the smooth part."""
    xs = (np.arange(8, 248, 2) / 256.0)
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    pts = np.stack([X.ravel(), Y.ravel()], axis=-1)
    pts = pts[: (len(pts) // 12) * 12]
    nodes_np = pts.reshape(-1, 12, 2)
    rng = np.random.default_rng(121)
    wts_np = rng.uniform(0.5, 1.5, nodes_np.shape[:2]) / pts.shape[0]
    f_np = rng.standard_normal(nodes_np.shape[:2])
    tg_np = np.concatenate([pts[::7], rng.uniform(0.05, 0.95, (300, 2))])
    nodes, wts, tg, f = (torch.from_numpy(np.ascontiguousarray(a)).to(DEV) for a in (nodes_np, wts_np, tg_np, f_np))
    d1 = 3.0 * float(wts_np.mean())
    out = []
    for tol, st, pk in ((1e-13, 32, 0), (1e-13, 0, 0), (1e-13, 0, 1), (1e-11, 32, 0), (1e-11, 0, 0), (1e-11, 0, 2)):
        plan = vp.Plan(nodes, wts, tg, tol, parts=vp.PART_HISTORY, delta1_override=d1, spread_tile=st,
                       spread_pack=pk)
        out.append(plan.eval(f).cpu().numpy())
    for a, b in ((1, 0), (2, 0), (4, 3), (5, 3)):  # same tol: same grid, the spreaders agree to rounding
        assert np.max(np.abs(out[a] - out[b])) <= 1e-13 * np.max(np.abs(out[b])), (a, b)
    ref = oracle.smooth_direct(pts, (f_np * wts_np).ravel(), tg_np, d1)
    assert rel_l2(out[0], ref) < 1e-12


def test_fused_fft_grid_sizes():
    """Fused transforms vs cuFFT over a sweep of grid sizes (delta_1 varied: n_f runs through 2,3,5,7-smooth
    sizes, including ones with odd n_f / 2): the smooth part agrees to rounding for every size."""
    rng = np.random.default_rng(131)
    src = rng.uniform(0.1, 0.9, (600, 2))
    nodes = torch.from_numpy(src.reshape(50, 12, 2).copy()).to(DEV)
    wts = torch.from_numpy(rng.uniform(0.5, 1.5, (50, 12)) / 600).to(DEV)
    fv = torch.from_numpy(rng.standard_normal((50, 12))).to(DEV)
    tg = torch.from_numpy(rng.uniform(0.05, 0.95, (200, 2))).to(DEV)
    sizes = set()
    for d1 in np.geomspace(2e-3, 2e-5, 9):
        out = []
        for mode in (0, 1):
            plan = vp.Plan(nodes, wts, tg, 1e-10, parts=vp.PART_HISTORY, delta1_override=float(d1), fft_mode=mode)
            out.append(plan.eval(fv).cpu().numpy())
            nf = plan.info()["nf_nh"]
            plan.destroy()
        sizes.add(nf)
        assert np.max(np.abs(out[0] - out[1])) <= 1e-12 * np.max(np.abs(out[1])), nf
    assert any((n // 2) % 2 == 1 for n in sizes), sorted(sizes)


@pytest.mark.parametrize("d1", [6e-8, 2.4e-8, 8e-9])
def test_four_step_matches_cufft(d1):
    """Grids above 6400^2 (configs 4 and 5): own pruned row passes + the four-step column pass with the multiply
    on the fly (default, fft_path 3), cuFFT batched row passes + four-step (fft_rows=1, fft_path 2) vs cuFFT 2D
    D2Z + k_multiply + Z2D (fft_mode=1) on the same plan inputs; and the smooth part vs the direct G_H sum."""
    rng = np.random.default_rng(141)
    src = rng.uniform(0.02, 0.98, (1200, 2))
    nodes = torch.from_numpy(src.reshape(100, 12, 2).copy()).to(DEV)
    wts = torch.from_numpy(rng.uniform(0.5, 1.5, (100, 12)) / 1200).to(DEV)
    fv = torch.from_numpy(rng.standard_normal((100, 12))).to(DEV)
    tg_np = np.concatenate([rng.uniform(0.0, 1.0, (300, 2)), src[:20]])
    tg = torch.from_numpy(tg_np).to(DEV)
    out, paths = [], []
    for kw in ({}, {"fft_rows": 1}, {"fft_mode": 1}):  # own rows + four-step, cuFFT rows + four-step, cuFFT 2D
        plan = vp.Plan(nodes, wts, tg, 1e-10, parts=vp.PART_HISTORY, delta1_override=d1, **kw)
        out.append(plan.eval(fv).cpu().numpy())
        info = plan.info()
        paths.append((info["fft_path_nh"], info["fft_path_fh"], info["nf_nh"], info["nf_fh"]))
        plan.destroy()
    print("four-step", d1, paths)
    # own row passes hold a whole row (2 x nf/4 complex values) in shared memory: nf <= 28160;
    # larger grids keep cuFFT's batched rows
    assert paths[0][0] == (3 if paths[0][2] <= 28160 else 2) and paths[1][0] == 2 and paths[2][0] == 1
    for o in out[:2]:
        assert np.max(np.abs(o - out[2])) <= 1e-12 * np.max(np.abs(out[2])), paths
    ref = oracle.smooth_direct(src, (fv.cpu().numpy() * wts.cpu().numpy()).ravel(), tg_np, d1)
    assert rel_l2(out[0], ref) < 1e-9


def test_four_step_fresh_process():
    """A process whose first (and only) plan uses the four-step column pass: the constant-bank DFT roots of the
    odd radices must be uploaded by that path itself (regression: they were uploaded only by the fused path)."""
    import subprocess
    import sys
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2409_11998_b200 as vp
rng = np.random.default_rng(3)
src = rng.uniform(0.0, 1.0, (1200, 2))
nodes = torch.from_numpy(src.reshape(100, 12, 2).copy()).cuda()
wts = torch.from_numpy(rng.uniform(0.5, 1.5, (100, 12)) / 1200).cuda()
fv = torch.from_numpy(rng.standard_normal((100, 12))).cuda()
tg = torch.from_numpy(rng.uniform(0.0, 1.0, (200, 2))).cuda()
out = []
for mode in (0, 1):
    p = vp.Plan(nodes, wts, tg, 1e-13, parts=vp.PART_HISTORY, delta1_override=6.25e-8, fft_mode=mode)
    assert p.info()["fft_path_nh"] in ((2, 3) if mode == 0 else (1,))
    out.append(p.eval(fv).cpu().numpy())
print(np.max(np.abs(out[0] - out[1])) / np.max(np.abs(out[1])))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) < 1e-12, r.stdout
