"""Pins for the CPU oracle (oracle/): closed forms, invariants, library routines, brute force.

Each check pins the oracle to something other than itself (SURVEY §8(c) "What pins it"):
  * E1 vs scipy.special.exp1; G_H vs scipy; W_R vs scipy.quad of its defining integral and the
    paper's printed W(0) (PAPER.md lemma, lines 465-470)
  * unit disk, f = 1:            V = (1 - r^2)/4                       (closed form)
  * Gaussian f on R^2:           V = -(s/4)[log rho^2 + E1(rho^2/s)]   (closed form)
  * f = 1 on a rectangle:        corner-function closed form, itself checked vs scipy dblquad
  * -Laplace V = f               (4th-order finite differences)
  * single triangles:            independent scipy adaptive polar quadrature
  * additivity / translation invariance
  * smooth part: real-space G_H sum vs numpy+scipy; direct-DFT form vs real-space form
"""
import numpy as np
import pytest
import scipy.integrate as si
import scipy.special as sp

import oracle
from workloads import configs, fields


def test_e1_vs_scipy():
    x = np.concatenate([np.logspace(-12, 0, 40), np.linspace(1.0, 700, 60)])
    ref = sp.exp1(x)
    got = oracle.e1(x)
    assert np.max(np.abs(got / ref - 1)) < 5e-15


def test_GH_vs_scipy_and_origin():
    d = 2e-3
    r2 = np.logspace(-8, 0, 50)
    ref = -(np.log(r2) + sp.exp1(r2 / (4 * d))) / (4 * np.pi)
    got = oracle.GH(r2, d)
    # small r2 lose digits in the *reference* (log r2 + E1 cancel); compare where ref is stable
    ok = r2 / (4 * d) > 1e-3
    assert np.max(np.abs(got[ok] - ref[ok])) < 1e-14 * np.max(np.abs(ref))
    g0 = (np.euler_gamma - np.log(4 * d)) / (4 * np.pi)
    assert abs(oracle.GH(0.0, d) - g0) < 1e-15
    assert abs(oracle.GH(1e-14, d) - g0) < 1e-12


def test_WR_pins():
    # PAPER.md lemma (lines 465-470): W(0) = (1 - 2 log(2 sqrt 2)) (2 sqrt 2)^2 / 4 for R = 2 sqrt 2
    R = 2 * np.sqrt(2)
    assert abs(oracle.WR(0.0, R) - (-2.158883083359673)) < 1e-14
    for R in [0.7, 1.3, 2 * np.sqrt(2)]:
        for k in [1e-5, 0.3, 2.0, 17.0]:
            ref = -si.quad(lambda r: r * np.log(r) * sp.j0(k * r), 0, R, limit=400, epsabs=1e-15, epsrel=1e-13)[0]
            assert abs(oracle.WR(k, R) - ref) < 1e-11 * max(1, abs(ref)), (R, k)


@pytest.fixture(scope="module")
def disk_const():
    return configs.config1(f="const")


def test_disk_closed_form(disk_const):
    w = disk_const
    idx = configs.sample_targets(w.T, 600, seed=7)
    V = oracle.workload_potential(w, idx)
    r2 = (w.targets[idx] ** 2).sum(1)
    ex = (1 - r2) / 4
    assert np.max(np.abs(V - ex)) < 1e-12 * np.max(ex)
    # a few off-node targets including the centre (SPEC: centre value 1/4) and near-boundary points
    tg = np.array([[0.0, 0.0], [0.3, -0.2], [0.999, 0.0], [0.0, -0.9999], [0.70710678, 0.70710678]])
    V = oracle.volume_potential(w.tri, w.curved, w.circle, w.field, tg)
    ex = (1 - (tg ** 2).sum(1)) / 4
    assert np.max(np.abs(V - ex)) < 1e-12


@pytest.mark.parametrize("s", [0.01, 0.02])
def test_gaussian_closed_form(disk_const, s):
    w = disk_const
    fld = fields.gauss([1.0], [0.1], [0.2], [s])      # exterior mass < 1e-13: R^2 closed form applies
    idx = configs.sample_targets(w.T, 300, seed=8)
    tg = np.concatenate([w.targets[idx], [[0.1, 0.2], [0.1 + 1e-9, 0.2]]])
    V = oracle.volume_potential(w.tri, w.curved, w.circle, fld, tg)
    rho2 = ((tg - [0.1, 0.2]) ** 2).sum(1)
    with np.errstate(divide="ignore"):
        ex = np.where(rho2 > 0, -(s / 4) * (np.log(np.where(rho2 > 0, rho2, 1)) + sp.exp1(np.where(rho2 > 0, rho2, 1) / s)),
                      (s / 4) * (np.euler_gamma - np.log(s)))
    assert np.max(np.abs(V - ex)) < 2e-12 * np.max(np.abs(ex))


def _rect_F(X, Y):
    with np.errstate(divide="ignore", invalid="ignore"):
        r2 = X * X + Y * Y
        t1 = np.where(r2 > 0, X * Y * np.log(np.where(r2 > 0, r2, 1)), 0.0)
        t3 = np.where(X != 0, X * X * np.arctan(Y / np.where(X != 0, X, 1)), 0.0)
        t4 = np.where(Y != 0, Y * Y * np.arctan(X / np.where(Y != 0, Y, 1)), 0.0)
    return t1 - 3 * X * Y + t3 + t4


def rect_closed_form(x, y, a=(0.0, 0.0), b=(1.0, 1.0)):
    """V for f = 1 on [a0,b0]x[a1,b1]: -(1/4pi) sum of corner values of F (d^2F/dXdY = log(X^2+Y^2))."""
    X1, X2 = a[0] - x, b[0] - x
    Y1, Y2 = a[1] - y, b[1] - y
    S = _rect_F(X2, Y2) - _rect_F(X1, Y2) - _rect_F(X2, Y1) + _rect_F(X1, Y1)
    return -S / (4 * np.pi)


def test_rect_closed_form_itself():
    for (x, y) in [(0.3, 0.4), (0.05, 0.9), (1.3, -0.2)]:
        ref = -si.dblquad(lambda v, u: np.log((u - x) ** 2 + (v - y) ** 2), 0, 1, 0, 1,
                          epsabs=1e-13, epsrel=1e-12)[0] / (4 * np.pi)
        assert abs(rect_closed_form(x, y) - ref) < 1e-10


def test_rect_oracle_on_flawed_square_mesh():
    rng = np.random.default_rng(3)
    tri = configs.square_grid(12, jitter=0.4, rng=rng)
    tri = configs.cevian_split(tri, 0.2, rng)
    tg = np.concatenate([rng.uniform(0, 1, (40, 2)), [[0.0, 0.0], [0.5, 0.0], [1.0, 1.0], [1.5, 0.5]]])
    V = oracle.volume_potential(tri, None, None, fields.const(1.0), tg)
    ex = rect_closed_form(tg[:, 0], tg[:, 1])
    assert np.max(np.abs(V - ex)) < 1e-12 * np.max(np.abs(ex))


def test_fd_laplacian_equals_minus_f():
    w = configs.config2(n=16)
    h = 3e-3
    pts = np.array([[0.37, 0.52], [0.61, 0.28], [0.45, 0.71]])
    offs = [(0, 0), (h, 0), (-h, 0), (2 * h, 0), (-2 * h, 0), (0, h), (0, -h), (0, 2 * h), (0, -2 * h)]
    tg = np.array([[p[0] + o[0], p[1] + o[1]] for p in pts for o in offs])
    V = oracle.volume_potential(w.tri, w.curved, w.circle, w.field, tg).reshape(len(pts), len(offs))
    c, px, mx, p2x, m2x, py, my, p2y, m2y = V.T
    lap = (-(p2x + m2x) + 16 * (px + mx) - 30 * c) / (12 * h * h) + (-(p2y + m2y) + 16 * (py + my) - 30 * c) / (12 * h * h)
    f = fields.evaluate(w.field, pts[:, 0], pts[:, 1])
    assert np.max(np.abs(-lap - f)) < 2e-6 * np.max(np.abs(f)) + 1e-7


def _scipy_polar_triangle(tri, f, p):
    """Independent brute force: int_T -(1/2pi) log|p-y| f(y) dy by scipy adaptive polar quadrature
    (signed fan of the three edges about p)."""
    total = 0.0
    for e in range(3):
        A, B = tri[e] - p, tri[(e + 1) % 3] - p
        cr = A[0] * B[1] - A[1] * B[0]
        if abs(cr) < 1e-15:
            continue
        thA, thB = np.arctan2(A[1], A[0]), np.arctan2(B[1], B[0])
        dth = np.angle(np.exp(1j * (thB - thA)))
        n = np.array([B[1] - A[1], -(B[0] - A[0])])
        n /= np.linalg.norm(n)
        dist = A @ n

        def inner(th):
            u = np.array([np.cos(th), np.sin(th)])
            rmax = dist / (u @ n)
            g = lambda r: -np.log(r) / (2 * np.pi) * f(p[0] + r * u[0], p[1] + r * u[1]) * r
            return si.quad(g, 0, rmax, limit=200, epsabs=1e-15, epsrel=1e-13)[0]

        val = si.quad(inner, thA, thA + dth, limit=200, epsabs=1e-15, epsrel=1e-13)[0]
        total += val if dth > 0 else val  # dth carries the sign of the fan sector
    return total


@pytest.mark.parametrize("case", range(4))
def test_single_triangle_brute_force(case):
    rng = np.random.default_rng(100 + case)
    tri = np.array([[0.0, 0.0], [1.0, 0.1], [0.3, 0.8]]) * 0.1 + rng.uniform(0, 0.5, 2)
    if case == 3:   # sliver, aspect ~ 1e3
        tri = np.array([[0.0, 0.0], [0.1, 0.0], [0.05, 1e-4]]) + 0.2
    c = tri.mean(0)
    fld = fields.gauss([1.3], [c[0] + 0.01], [c[1] - 0.02], [0.01])
    f = lambda x, y: fields.evaluate(fld, np.array(x), np.array(y))
    targets = [c, tri[0] * 0.7 + tri[1] * 0.3, c + np.array([0.2, 0.1]), tri[2] + np.array([1e-3, 2e-3])]
    for p in targets:
        ref = _scipy_polar_triangle(tri, f, np.asarray(p, float))
        got = oracle.triangle_integral(tri, fld, p)
        assert abs(got - ref) < 2e-13 * max(1e-3, abs(ref)), (case, p, got, ref)


def test_additivity_and_translation():
    tri = np.array([[0.1, 0.1], [0.5, 0.15], [0.2, 0.6]])
    a, b, c = tri
    ab, bc, ca = (a + b) / 2, (b + c) / 2, (c + a) / 2
    kids = [np.array(k) for k in ([a, ab, ca], [ab, b, bc], [ca, bc, c], [ab, bc, ca])]
    fld = fields.gauss([1.0, -0.5], [0.3, 0.2], [0.3, 0.4], [0.02, 0.05])
    for p in [np.array([0.25, 0.3]), ab, np.array([0.9, 0.9])]:
        whole = oracle.triangle_integral(tri, fld, p)
        parts = sum(oracle.triangle_integral(k, fld, p) for k in kids)
        assert abs(whole - parts) < 1e-14 * max(1.0, abs(whole)) + 1e-15
        sh = np.array([0.37, -1.2])
        fld2 = fields.gauss(fld["a"], fld["cx"] + sh[0], fld["cy"] + sh[1], fld["s"])
        moved = oracle.triangle_integral(tri + sh, fld2, p + sh)
        assert abs(whole - moved) < 1e-14 + 1e-13 * abs(whole)


def test_smooth_direct_vs_numpy():
    rng = np.random.default_rng(5)
    src = rng.uniform(0, 1, (300, 2))
    c = rng.standard_normal(300)
    tg = np.concatenate([rng.uniform(0, 1, (50, 2)), src[:5]])
    d = 1e-3
    got = oracle.smooth_direct(src, c, tg, d)
    r2 = ((tg[:, None, :] - src[None, :, :]) ** 2).sum(-1)
    with np.errstate(divide="ignore"):
        G = np.where(r2 > 0, -(np.log(np.where(r2 > 0, r2, 1)) + sp.exp1(np.where(r2 > 0, r2, 1) / (4 * d))) / (4 * np.pi),
                     (np.euler_gamma - np.log(4 * d)) / (4 * np.pi))
    ref = G @ c
    assert np.max(np.abs(got - ref)) < 1e-12 * np.max(np.abs(ref))


def test_smooth_dft_equals_real_space():
    """The Fourier route (near + far history, §3) equals the real-space G_H sum: pins the
    normalisation (Delta k)^2/(2 pi)^2 and the period / truncation-radius readings (DESIGN R1-R3)."""
    rng = np.random.default_rng(6)
    src = rng.uniform(0.2, 0.8, (60, 2))
    c = rng.standard_normal(60)
    tg = np.concatenate([rng.uniform(0.2, 0.8, (25, 2)), src[:5]])
    for d1 in [2e-3, 5e-4]:
        d2 = 32 * d1
        p = oracle.dft_params(src, tg, d1, d2, 1e-14)
        got = oracle.smooth_dft(src, c, tg, d1, d2, **p)
        ref = oracle.smooth_direct(src, c, tg, d1)
        assert np.max(np.abs(got - ref)) < 1e-12 * np.max(np.abs(ref)), d1
        # the literal paper box (R = 2 sqrt 2 on a period-4 box scaled to this data) aliases: the
        # reading is load-bearing
        bad = oracle.smooth_dft(src, c, tg, d1, d2, p["L_nh"] * 0.6, p["n_nh"], p["L_fh"], p["n_fh"], p["R"], p["x0"], p["y0"])
        assert np.max(np.abs(bad - ref)) > 1e-9 * np.max(np.abs(ref))


def test_oracle_own_nodes_match_generator():
    w = configs.config1(f="const")
    n, wt = oracle.rule12_nodes(w.tri, w.curved, w.circle)
    assert np.max(np.abs(n - w.nodes)) < 1e-14
    assert np.max(np.abs(wt - w.weights)) < 1e-15


def test_fourier_field_resolved():
    """Config 4's Fourier field (|k| <= 64) is resolved by the 12-point rule on its 1414^2-cell mesh: on a patch of
    that mesh the far field by the own 12-point rule (assume_resolved, the fast path oracle.workload_potential
    uses for Fourier fields) agrees with the oracle's full resolution ladder (Duffy up to 30 x 30 per triangle)."""
    from workloads import configs, fields
    rng = np.random.default_rng(4)
    tri = configs.square_grid(1414)
    fld = fields.random_fourier(rng, 64)
    c = tri.mean(1)
    patch = tri[(c[:, 0] > 0.5) & (c[:, 0] < 0.52) & (c[:, 1] > 0.5) & (c[:, 1] < 0.52)]
    assert patch.shape[0] > 500
    tg = np.array([[0.5101, 0.5137], [0.6, 0.45], [0.53, 0.515]])
    a = oracle.volume_potential(patch, None, None, fld, tg)
    b = oracle.volume_potential(patch, None, None, fld, tg, assume_resolved=True)
    assert np.max(np.abs(a - b)) < 1e-12 * np.max(np.abs(a))


def test_WR_closed_form():
    """The oracle evaluates W_R from its defining integral; the closed form (1 - J0(Rk))/k^2 - R log R J1(Rk)/k
    (PAPER.md eq. (Wdef), general R) with scipy's Bessel functions must agree."""
    for R in [0.7, 1.3, 2 * np.sqrt(2), 3.9]:
        for k in [1e-3, 0.1, 1.0, 7.5, 40.0, 150.0]:
            z = R * k
            if z < 1.0:  # 1 - J0 and J1 by their full power series (no cancellation at small z)
                m = np.arange(1, 30)
                lg = sp.gammaln(m + 1)
                one_m_j0 = np.sum((-1.0) ** (m + 1) * np.exp(2 * m * np.log(z / 2) - 2 * lg))
                j1 = np.sum((-1.0) ** (m - 1) * np.exp((2 * m - 1) * np.log(z / 2) - lg - sp.gammaln(m)))
            else:
                one_m_j0, j1 = 1 - sp.j0(z), sp.j1(z)
            ref = one_m_j0 / k ** 2 - R * np.log(R) * j1 / k
            assert abs(oracle.WR(k, R) - ref) < 2e-13 * max(1.0, abs(ref)), (R, k)


def test_e1_branches_and_recurrence():
    """E1 on both sides of the oracle's series / quadrature switch (x = 2) and the exact recurrence-free identity
    d/dx E1 = -e^{-x}/x checked by a 4th-order central difference (independent of scipy)."""
    x = np.array([1.999999, 2.0, 2.000001, 3.7, 25.0, 300.0])
    assert np.max(np.abs(oracle.e1(x) / sp.exp1(x) - 1)) < 3e-15
    for x0 in [0.3, 1.9, 2.1, 6.0, 40.0]:
        h = min(1e-3 * x0, 4e-3)
        d = (-oracle.e1(x0 + 2 * h) + 8 * oracle.e1(x0 + h) - 8 * oracle.e1(x0 - h) + oracle.e1(x0 - 2 * h)) / (12 * h)
        ex = -np.exp(-x0) / x0
        assert abs(d - ex) < 1e-9 * abs(ex), x0


def test_fourier_field_values_vs_numpy():
    """The oracle's Fourier field evaluation (table + recurrences, vp_oracle.c field_eval) against a direct numpy
    sum of a_k cos(2 pi k.x) + b_k sin(2 pi k.x) (config 4's field, |k| <= 64)."""
    rng = np.random.default_rng(4)
    fld = fields.random_fourier(rng, 64)
    pts = np.random.default_rng(9).uniform(-0.2, 1.2, (300, 2))
    got = oracle.field_values(fld, pts)
    ph = 2 * np.pi * (pts[:, 0:1] * fld["k1"][None, :] + pts[:, 1:2] * fld["k2"][None, :])
    ref = np.cos(ph) @ fld["a"] + np.sin(ph) @ fld["b"]
    assert np.max(np.abs(got - ref)) < 1e-13 * np.max(np.abs(ref))
    g = fields.gauss([1.3, -0.4], [0.2, 0.7], [0.5, 0.1], [0.01, 0.003])
    ref = 1.3 * np.exp(-((pts[:, 0] - 0.2) ** 2 + (pts[:, 1] - 0.5) ** 2) / 0.01) - \
        0.4 * np.exp(-((pts[:, 0] - 0.7) ** 2 + (pts[:, 1] - 0.1) ** 2) / 0.003)
    assert np.max(np.abs(oracle.field_values(g, pts) - ref)) < 1e-15


def test_narrow_gaussian_graded_mesh_closed_form():
    """A config-3/5-like narrow source (width 1e-3, s = 1e-6) on a quadtree-graded square mesh: most triangles
    see f < 1e-100, which exercises the oracle's resolution ladder with its absolute floor (O1).  The
    R^2 closed form V = -(s/4)[log rho^2 + E1(rho^2/s)] applies (exterior mass e^{-0.2^2/1e-6} = 0)."""
    c = np.array([0.5, 0.5])
    leaves = configs.quadtree_leaves([c], 0.08, 4, 13)
    x0, y0, h = leaves[:, 0], leaves[:, 1], leaves[:, 2]
    a, b = np.stack([x0, y0], 1), np.stack([x0 + h, y0], 1)
    cc, d = np.stack([x0 + h, y0 + h], 1), np.stack([x0, y0 + h], 1)
    tri = np.concatenate([np.stack([a, b, cc], 1), np.stack([a, cc, d], 1)])
    s = 1e-6
    fld = fields.gauss([1.0], [c[0]], [c[1]], [s])
    rng = np.random.default_rng(12)
    tg = np.concatenate([c + 3e-3 * rng.standard_normal((12, 2)), c + [[0.0, 0.0], [1e-4, 0], [0.2, 0.3]]])
    V = oracle.volume_potential(tri, None, None, fld, tg)
    rho2 = ((tg - c) ** 2).sum(1)
    with np.errstate(divide="ignore"):
        ex = np.where(rho2 > 0, -(s / 4) * (np.log(np.where(rho2 > 0, rho2, 1)) + sp.exp1(np.where(rho2 > 0, rho2, 1) / s)),
                      (s / 4) * (np.euler_gamma - np.log(s)))
    assert np.max(np.abs(V - ex)) < 1e-12 * np.max(np.abs(ex)), np.max(np.abs(V - ex)) / np.max(np.abs(ex))
