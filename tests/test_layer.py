"""Single-layer potential S[sigma] (§2.3, Lemma slp).

CPU: the oracle (oracle/layer.py) against closed forms on the unit circle and an independent scipy quadrature;
the reading R19 of the local expansion (slplocO5 with its overall sign reversed) against oracle - direct history
sum.  GPU (`-m gpu`): vp_eval_slp through the C ABI against the closed forms (circle) and the oracle (star) at
10 x tol."""
import numpy as np
import pytest
from scipy import integrate
from scipy.special import erfc

import oracle
from oracle import layer
from strata import rel_l2
from workloads import geometry


def _polar(pts):
    return np.hypot(pts[:, 0], pts[:, 1]), np.arctan2(pts[:, 1], pts[:, 0])


def circle_S(pts, m):
    """S[cos(m theta)] (m >= 1) or S[1] (m = 0) for the unit circle: r^{+-m} cos(m theta) / (2m), -log max(r, 1)"""
    r, th = _polar(pts)
    if m == 0:
        return -np.log(np.maximum(r, 1.0))
    return np.where(r <= 1.0, r ** m, r ** (-m)) * np.cos(m * th) / (2 * m)


def test_layer_oracle_circle_closed_forms():
    rng = np.random.default_rng(3)
    r = np.concatenate([rng.uniform(0, 0.99, 20), rng.uniform(1.01, 2, 20), np.ones(8), 1 + 1e-6 * rng.standard_normal(8)])
    th = rng.uniform(0, 2 * np.pi, r.size)
    pts = np.stack([r * np.cos(th), r * np.sin(th)], 1)
    cv, dcv = layer.circle()
    for m in (0, 1, 3):
        got = layer.single_layer(cv, dcv, (lambda t, m=m: np.cos(m * t)), pts)
        assert np.max(np.abs(got - circle_S(pts, m))) < 1e-13, m


def test_layer_oracle_star_vs_scipy_quad():
    """Independent check of the adaptive rule: scipy.integrate.quad over theta (breakpoint at the closest
    parameter) on the star, at targets 1e-3 inside and outside and 0.3 away."""
    cv, dcv = layer.star()
    sig = lambda t: 1.0 + 0.5 * np.cos(2 * t) + 0.3 * np.sin(3 * t)  # noqa: E731
    t0 = 0.9
    p0 = np.array(cv(t0))
    d0 = np.array(dcv(t0))
    nrm = np.array([-d0[1], d0[0]]) / np.hypot(*d0)
    for off in (1e-3, -1e-3, 0.3):
        x = p0 + off * nrm

        def integrand(t):
            px, py = cv(t)
            dx, dy = dcv(t)
            return -np.log((px - x[0]) ** 2 + (py - x[1]) ** 2) / (4 * np.pi) * sig(t) * np.hypot(dx, dy)
        ref = (integrate.quad(integrand, 0.0, t0, limit=400, epsabs=1e-15, epsrel=1e-14)[0]
               + integrate.quad(integrand, t0, 2 * np.pi, limit=400, epsabs=1e-15, epsrel=1e-14)[0])
        got = layer.single_layer(cv, dcv, sig, x[None, :])[0]
        assert abs(got - ref) < 1e-12 * max(1.0, abs(ref)), (off, got, ref)


def test_slp_local_expansion_reading():
    """Reading R19: S_L = -(printed eq. slplocO5), with the curve over its tangent line along the inward normal and
    sgn = +1 inside.  On the circle (kappa = 1, gamma3 = 0, gamma4 = 3 in that frame) the expansion must equal
    S - S_H (oracle minus the direct history sum over a fine boundary rule) to its O(delta^{5/2}) truncation, on
    both sides; the printed sign is off by 2 S_L."""
    d = 1e-4
    sd = np.sqrt(d)
    npan, q = 512, 16
    xg, wg = np.polynomial.legendre.leggauss(q)
    th = ((np.arange(npan)[:, None] + 0.5 * (xg[None, :] + 1)) * 2 * np.pi / npan).ravel()
    W = np.tile(wg, npan) * np.pi / npan
    Y = np.stack([np.cos(th), np.sin(th)], 1)
    m, phi = 3, 0.7
    s0, s1, s2 = np.cos(m * phi), -m * np.sin(m * phi), -m * m * np.cos(m * phi)  # sigma and d/dxi, d2/dxi2 at b
    for side in (1, -1):  # +1: interior
        for c in (0.0, 0.5, 1.5, 3.0, 6.0):
            r = 1 - side * c * sd
            x = np.array([[r * np.cos(phi), r * np.sin(phi)]])
            true = circle_S(x, m)[0] - oracle.smooth_direct(Y, W * np.cos(m * th), x, d)[0]
            e = np.exp(-c * c / 4) / np.sqrt(np.pi)
            E = erfc(c / 2)
            F1, F2, F3, F4 = c * E - 2 * e, 2 * c**3 * E - (4 * c * c + 1) * e, 3 * c**3 * E - (6 * c * c - 2) * e, \
                2 * (c * c - 2) * e - c**3 * E
            kap, g4, sg = 1.0, 3.0, float(side) if c > 0 else 0.0
            printed = (sd * s0 / 2 * F1 + sg * d * c * kap * s0 / 4 * F1 + d**1.5 * s0 * kap**2 / 12 * F2
                       + d**1.5 * s2 / 12 * F4 + d * d * sg * (c * kap**3 * s0 / 16 * F3 + c * kap * s2 / 8 * F4)
                       + d * d * sg * (c * s0 * g4 / 48 * F4))
            assert abs(-printed - true) < 1e-9, (side, c, -printed, true)
            if c < 2:
                assert abs(printed - true) > 1e-4 * abs(true)


# ------------------------------------------------------------------------------------------------- GPU
def _plan(targets, chunks, tol, delta1, levels=None, kind="slp"):
    torch = pytest.importorskip("torch")
    import paper_2409_11998_b200 as vp
    rng = np.random.default_rng(5)
    # the history grids only need nodes / weights for the grid frame and delta_1 (given explicitly here)
    nodes = rng.uniform(-0.5, 0.5, (200, 12, 2))
    wts = np.full((200, 12), 1.0 / 2400)
    dev = "cuda"
    plan = vp.Plan(torch.from_numpy(nodes).to(dev), torch.from_numpy(wts).to(dev),
                   torch.from_numpy(np.ascontiguousarray(targets)).to(dev), tol, boundary=("chunks", chunks),
                   parts=vp.PART_HISTORY, delta1_override=delta1)
    if levels is not None:
        plan.set_layer_levels(levels)
    if kind == "slp":
        plan.prepare_slp()
    else:
        plan.prepare_dlp()
    return plan, torch


def _targets(rng, curve_r, n_in=300, n_near=400, n_on=64, n_out=200):
    th = rng.uniform(0, 2 * np.pi, n_in + n_near + n_on + n_out)
    rb = curve_r(th)
    rr = np.concatenate([rng.uniform(0.05, 0.9, n_in) * rb[:n_in],
                         rb[n_in:n_in + n_near] * (1 + rng.uniform(-0.02, 0.02, n_near)),
                         rb[n_in + n_near:n_in + n_near + n_on],
                         rb[n_in + n_near + n_on:] * rng.uniform(1.05, 1.4, n_out)])
    return np.stack([rr * np.cos(th), rr * np.sin(th)], 1)


@pytest.mark.gpu
@pytest.mark.parametrize("m", [0, 1, 3])
def test_slp_circle_closed_form(m):
    """Unit circle as 96 chunks of degree 16, sigma = cos(m theta) (m = 0: sigma = 1): S at interior, near-boundary
    (both sides), on-boundary and exterior targets equals the closed form to 10 x tol."""
    rng = np.random.default_rng(10 + m)
    tg = _targets(rng, lambda t: np.ones_like(t))
    ch = geometry.circle_chunks(0.0, 0.0, 1.0, 96, q=16, theta0=0.05)
    tol = 1e-9
    plan, torch = _plan(tg, ch, tol, 2e-4)
    thn = np.arctan2(ch[..., 1], ch[..., 0])
    sig = torch.from_numpy(np.cos(m * thn)).cuda()
    S = plan.eval_slp(sig).cpu().numpy()
    plan.destroy()
    ref = circle_S(tg, m)
    e = rel_l2(S, ref)
    print("slp circle m", m, "rel l2", e)
    assert e <= 10 * tol, e


@pytest.mark.gpu
def test_slp_star_vs_oracle():
    """Config 3's star r = 1 + 0.3 cos 5 theta as 200 chunks of degree 16, sigma smooth and non-symmetric:
    S at interior / near / on / exterior targets vs the adaptive-quadrature oracle at 10 x tol (tol 1e-8,
    delta_1 = 1e-4, the default J = 3 levels of the dyadic telescoping, §4.1).  Without telescoping
    (J = 0) the star's tips (radius of curvature 0.19) make the local expansion's O(delta^{5/2}) remainder visible:
    that near-boundary error must fall at least like delta^2 from delta_1 = 1e-4 to 2.5e-5 (the order of eq.
    slplocO5), while the interior error (history part only) stays at the NUFFT level."""
    rng = np.random.default_rng(21)
    n_in, n_near, n_on, n_out = 80, 120, 24, 60
    tg = _targets(rng, geometry.star_radius, n_in=n_in, n_near=n_near, n_on=n_on, n_out=n_out)
    ch = geometry.star_chunks(200, q=16)
    thn = np.arctan2(ch[..., 1], ch[..., 0])
    sigf = lambda t: 1.0 + 0.5 * np.cos(2 * t) + 0.3 * np.sin(3 * t)  # noqa: E731
    cv, dcv = layer.star()
    ref = layer.single_layer(cv, dcv, sigf, tg)
    near = slice(n_in, n_in + n_near + n_on)
    tol = 1e-8
    errs = {}
    for d1, J in ((1e-4, 0), (2.5e-5, 0), (1e-4, None)):
        plan, torch = _plan(tg, ch, tol, d1, J)
        S = plan.eval_slp(torch.from_numpy(sigf(thn)).cuda()).cpu().numpy()
        plan.destroy()
        errs[d1, J] = (rel_l2(S, ref), np.max(np.abs(S[near] - ref[near])), np.max(np.abs(S[:n_in] - ref[:n_in])))
        print("slp star delta_1", d1, "J", J, "rel l2 %.3e, near max %.3e, interior max %.3e" % errs[d1, J])
    assert errs[1e-4, None][0] <= 10 * tol, errs
    assert errs[1e-4, None][1] <= 10 * tol, errs
    assert errs[2.5e-5, 0][0] <= 10 * tol, errs
    assert errs[1e-4, 0][1] / errs[2.5e-5, 0][1] >= 4.0 ** 2, errs
    assert errs[2.5e-5, 0][2] <= 10 * tol, errs


# ------------------------------------------------------------------------------------------------- double layer
def circle_D(pts, m, on=None):
    """D[cos(m theta)] (outward normal) for the unit circle: -r^m cos/2 inside, r^-m cos/2 outside, 0 on it (m >= 1);
    D[1] = -1, -1/2, 0 inside / on / outside (Gauss; the interior limit is D(b) - mu/2)"""
    r, th = _polar(pts)
    on = np.zeros(len(r), bool) if on is None else on
    if m == 0:
        out = np.where(r < 1.0, -1.0, 0.0)
        out[on] = -0.5
        return out
    out = np.where(r < 1.0, -r ** m / 2, r ** (-m) / 2) * np.cos(m * th)
    out[on] = 0.0
    return out


def test_dlp_oracle_circle_closed_forms():
    rng = np.random.default_rng(4)
    r = np.concatenate([rng.uniform(0, 0.99, 12), rng.uniform(1.01, 2, 12), np.ones(8), 1 + 1e-6 * rng.standard_normal(8)])
    th = rng.uniform(0, 2 * np.pi, r.size)
    pts = np.stack([r * np.cos(th), r * np.sin(th)], 1)
    on = np.zeros(r.size, bool)
    on[24:32] = True
    cv, dcv = layer.circle()
    for m in (0, 1, 3):
        got = layer.double_layer(cv, dcv, (lambda t, m=m: np.cos(m * t)), pts, on_curve=on)
        err = np.abs(got - circle_D(pts, m, on))
        assert np.max(err[:32]) < 1e-12, (m, err)
        assert np.max(err[32:]) < 1e-9, (m, err)  # 1e-6 off the curve: the adaptive rule's cancellation floor


def test_dlp_oracle_star_green_identity():
    """Green's representation on the star for the harmonic u = Re((x + i y)^3) + 0.4 x: S[du/dnu] - D[u] = u inside,
    0 outside (PAPER.md eq. neu_rep family, lines 1310-1318) -- pins D against the independently pinned S, with
    the outward normal and the sign convention of the kernel."""
    cv, dcv = layer.star()

    def u_of(t):
        x, y = cv(t)
        return x ** 3 - 3 * x * y * y + 0.4 * x

    def dudn(t):
        x, y = cv(t)
        dx, dy = dcv(t)
        nx, ny = dy / np.hypot(dx, dy), -dx / np.hypot(dx, dy)
        return (3 * x * x - 3 * y * y + 0.4) * nx - 6 * x * y * ny
    rng = np.random.default_rng(8)
    th = rng.uniform(0, 2 * np.pi, 12)
    rb = geometry.star_radius(th)
    rr = np.concatenate([rb[:6] * rng.uniform(0.2, 0.97, 6), rb[6:] * rng.uniform(1.03, 1.6, 6)])
    pts = np.stack([rr * np.cos(th), rr * np.sin(th)], 1)
    rep = layer.single_layer(cv, dcv, dudn, pts) - layer.double_layer(cv, dcv, u_of, pts)
    u = pts[:, 0] ** 3 - 3 * pts[:, 0] * pts[:, 1] ** 2 + 0.4 * pts[:, 0]
    assert np.max(np.abs(rep[:6] - u[:6])) < 1e-11, rep[:6] - u[:6]
    assert np.max(np.abs(rep[6:])) < 1e-11, rep[6:]


def test_dlp_oracle_star_vs_scipy_quad():
    cv, dcv = layer.star()
    mu = lambda t: 1.0 + 0.5 * np.cos(2 * t) + 0.3 * np.sin(3 * t)  # noqa: E731
    t0 = 2.1
    p0 = np.array(cv(t0))
    d0 = np.array(dcv(t0))
    nrm = np.array([d0[1], -d0[0]]) / np.hypot(*d0)
    for off in (2e-3, -2e-3, 0.3):
        x = p0 + off * nrm

        def integrand(t):
            px, py = cv(t)
            dx, dy = dcv(t)
            return ((x[0] - px) * dy - (x[1] - py) * dx) / ((px - x[0]) ** 2 + (py - x[1]) ** 2) / (2 * np.pi) * mu(t)
        ref = (integrate.quad(integrand, 0.0, t0, limit=400, epsabs=1e-15, epsrel=1e-14)[0]
               + integrate.quad(integrand, t0, 2 * np.pi, limit=400, epsabs=1e-15, epsrel=1e-14)[0])
        got = layer.double_layer(cv, dcv, mu, x[None, :])[0]
        assert abs(got - ref) < 1e-11 * max(1.0, abs(ref)), (off, got, ref)


def _dlp_expansion(c, s, d, kap, g3, g4, mu0, mu1, mu2, mu4):
    """eq. dlplocO5 as printed"""
    sd = np.sqrt(d)
    E = np.exp(-c * c / 4) / np.sqrt(np.pi)
    er = erfc(c / 2)
    return (s * mu0 / 2 * er + sd * kap * mu0 / 2 * E + d * s * (3 * c * kap ** 2 * mu0 / 8 * E + c * mu2 / 4 * (2 * E - c * er))
            + d ** 1.5 * (5 * (c * c - 2) * kap ** 3 * mu0 / 16 * E + g4 * mu0 / 4 * E
                          + kap * mu2 / 4 * (2 * (c * c + 1) * E - c ** 3 * er) + g3 * mu1 / 12 * (2 * (c * c + 4) * E - c ** 3 * er))
            + d * d * s * (35 * c * kap ** 4 * mu0 * (c * c - 6) / 128 * E + 5 * c * g3 ** 2 * mu0 / 12 * E + 5 * c * kap * g4 * mu0 / 8 * E)
            + d * d * s * 5 * c * (kap ** 2 * mu2 / 16 * (2 * (c * c + 1) * E - c ** 3 * er)
                                   + kap * g3 * mu1 / 24 * (2 * (c * c + 4) * E - c ** 3 * er))
            + d * d * s * c * mu4 / 48 * (c ** 3 * er - 2 * (c * c - 2) * E))


def test_dlp_local_expansion_reading():
    """Reading R21: eq. dlplocO5 as printed holds for D with the OUTWARD normal when the curve is written over its
    tangent line along the outward normal (unit circle: kappa = -1, gamma3 = 0, gamma4 = -3) and sgn = +1 outside.
    Checked against D - D_H (closed form minus the direct history sum over a fine boundary rule; the D_H kernel
    (1/2 pi)(1 - e^{-|x-y|^2/4 delta}) (x - y).nu / |x - y|^2 is smooth) to the O(delta^{5/2}) truncation; the
    inward-frame reading of R19 (sgn = +1 inside, kappa = +1) is off by O(1)."""
    d = 1e-4
    sd = np.sqrt(d)
    npan, q = 512, 16
    xg, wg = np.polynomial.legendre.leggauss(q)
    th = ((np.arange(npan)[:, None] + 0.5 * (xg[None, :] + 1)) * 2 * np.pi / npan).ravel()
    W = np.tile(wg, npan) * np.pi / npan
    Y = np.stack([np.cos(th), np.sin(th)], 1)
    m, phi = 3, 0.7
    mu_t = np.cos(m * th)

    def DH(x):
        dx, dy = x[0] - Y[:, 0], x[1] - Y[:, 1]
        r2 = dx * dx + dy * dy
        return np.sum(W * mu_t * (1 - np.exp(-r2 / (4 * d))) * (dx * Y[:, 0] + dy * Y[:, 1]) / r2) / (2 * np.pi)
    # mu along the tangent line: theta = phi + asin(xi) = phi + xi + xi^3/6 + ...
    cm, sm = np.cos(m * phi), np.sin(m * phi)
    mu0, mu1, mu2, mu4 = cm, -m * sm, -m * m * cm, (m ** 4 - 4 * m * m) * cm
    for side in (1, -1):  # +1: exterior
        for c in (0.0, 0.5, 1.5, 3.0, 6.0):
            rr = 1 + side * c * sd
            x = np.array([rr * np.cos(phi), rr * np.sin(phi)])
            full = 0.0 if c == 0 else circle_D(x[None, :], m)[0]
            true = full - DH(x)
            s = float(side) if c > 0 else 0.0
            got = _dlp_expansion(c, s, d, -1.0, 0.0, -3.0, mu0, mu1, mu2, mu4)
            assert abs(got - true) < 2e-9, (side, c, got, true)
            if c < 2:
                inward = _dlp_expansion(c, -s, d, 1.0, 0.0, 3.0, mu0, mu1, mu2, mu4)
                assert abs(inward - true) > 1e-5, (side, c)


def _plan_dlp(targets, chunks, tol, delta1, levels=None):
    return _plan(targets, chunks, tol, delta1, levels, kind="dlp")


@pytest.mark.gpu
@pytest.mark.parametrize("m", [0, 1, 3])
def test_dlp_circle_closed_form(m):
    """Unit circle as 96 chunks of degree 16, mu = cos(m theta) (m = 0: mu = 1): D at interior, near-boundary (both
    sides), on-boundary (direct value) and exterior targets equals the closed form to 10 x tol."""
    rng = np.random.default_rng(30 + m)
    n_in, n_near, n_on, n_out = 300, 400, 64, 200
    tg = _targets(rng, lambda t: np.ones_like(t), n_in, n_near, n_on, n_out)
    on = np.zeros(len(tg), bool)
    on[n_in + n_near:n_in + n_near + n_on] = True
    ch = geometry.circle_chunks(0.0, 0.0, 1.0, 96, q=16, theta0=0.05)
    tol = 1e-9
    plan, torch = _plan_dlp(tg, ch, tol, 2e-4)
    thn = np.arctan2(ch[..., 1], ch[..., 0])
    D = plan.eval_dlp(torch.from_numpy(np.cos(m * thn)).cuda()).cpu().numpy()
    plan.destroy()
    ref = circle_D(tg, m, on)
    e = rel_l2(D, ref)
    print("dlp circle m", m, "rel l2", e, "max", np.max(np.abs(D - ref)))
    assert e <= 10 * tol, e


@pytest.mark.gpu
def test_dlp_star_vs_oracle():
    """The star as 200 chunks of degree 16, mu smooth and non-symmetric: D at interior / near / on / exterior targets
    vs the adaptive-quadrature oracle (on-curve targets: direct value) at 10 x tol, tol 1e-8, delta_1 = 1e-4 with
    the default J = 3 telescoping levels; without telescoping (J = 0) the near-boundary error must fall at least
    like delta^2 from delta_1 = 1e-4 to 2.5e-5 (order of eq. dlplocO5)."""
    rng = np.random.default_rng(22)
    n_in, n_near, n_on, n_out = 80, 120, 24, 60
    tg = _targets(rng, geometry.star_radius, n_in=n_in, n_near=n_near, n_on=n_on, n_out=n_out)
    on = np.zeros(len(tg), bool)
    on[n_in + n_near:n_in + n_near + n_on] = True
    ch = geometry.star_chunks(200, q=16)
    thn = np.arctan2(ch[..., 1], ch[..., 0])
    muf = lambda t: 1.0 + 0.5 * np.cos(2 * t) + 0.3 * np.sin(3 * t)  # noqa: E731
    cv, dcv = layer.star()
    ref = layer.double_layer(cv, dcv, muf, tg, on_curve=on)
    near = slice(n_in, n_in + n_near + n_on)
    tol = 1e-8
    errs = {}
    for d1, J in ((1e-4, 0), (2.5e-5, 0), (1e-4, None)):
        plan, torch = _plan_dlp(tg, ch, tol, d1, J)
        D = plan.eval_dlp(torch.from_numpy(muf(thn)).cuda()).cpu().numpy()
        plan.destroy()
        errs[d1, J] = (rel_l2(D, ref), np.max(np.abs(D[near] - ref[near])), np.max(np.abs(D[:n_in] - ref[:n_in])))
        print("dlp star delta_1", d1, "J", J, "rel l2 %.3e, near max %.3e, interior max %.3e" % errs[d1, J])
    assert errs[1e-4, None][0] <= 10 * tol, errs
    assert errs[1e-4, None][1] <= 10 * tol, errs
    assert errs[1e-4, 0][1] / errs[2.5e-5, 0][1] >= 4.0 ** 2, errs
    assert errs[2.5e-5, 0][2] <= 10 * tol, errs
