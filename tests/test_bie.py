"""Boundary integral equations of the Poisson solve (§5 "s:bie", lines 1271-1330):
restarted GMRES (vp_bie_solve) whose product is the GPU double-layer operator, checked against exact solutions.

- interior Dirichlet on the star for a harmonic u (f = 0): (-1/2 + D) mu = g, u = D[mu] inside (eq. dir_inteq);
- exterior Dirichlet on the star for a bounded harmonic u: (1/2 + D + int ds) mu = g, u = D[mu] + int mu ds
  (eq. dir_repext with A = 0);
- interior Neumann on the star: (1/2 + D) u = S[du/dnu] on Gamma (lines 1310-1318), u up to a constant;
- the full Poisson problem -Lap u = f on the unit disk (config 1's curved mesh): u = V[f] + D[mu] with
  (-1/2 + D) mu = g - V[f] -- the volume potential, the layer potential and the solve all on the GPU.
The references are closed-form solutions (no oracle involved): harmonic polynomials / Re(1/z), u = cos 2x sin y."""
import numpy as np
import pytest

from strata import rel_l2
from workloads import configs, geometry

pytestmark = pytest.mark.gpu

NCH, Q = 200, 16


def _star_W(n=NCH, q=Q, a=0.3, m=5):
    """boundary rule weights W_j = w_k |d gamma / ds| of geometry.star_chunks (uniform in theta: ds = (pi / n) dtheta)"""
    s, w = np.polynomial.legendre.leggauss(q + 1)
    th = 2 * np.pi * (np.arange(n)[:, None] + 0.5 * (s[None, :] + 1.0)) / n
    r = 1.0 + a * np.cos(m * th)
    dr = -a * m * np.sin(m * th)
    return (w[None, :] * np.hypot(r, dr) * np.pi / n).ravel(), th.ravel()


def _star_normal(th, a=0.3, m=5):
    r = 1.0 + a * np.cos(m * th)
    dr = -a * m * np.sin(m * th)
    tx, ty = dr * np.cos(th) - r * np.sin(th), dr * np.sin(th) + r * np.cos(th)
    nrm = np.hypot(tx, ty)
    return ty / nrm, -tx / nrm  # outward


def _plan(targets, chunks, tol, delta1=None, nodes=None, wts=None, parts=None):
    import torch

    import paper_2409_11998_b200 as vp
    if nodes is None:  # history grids only: nodes / weights fix the grid frame; delta_1 given
        rng = np.random.default_rng(5)
        nodes = rng.uniform(-0.5, 0.5, (200, 12, 2))
        wts = np.full((200, 12), 1.0 / 2400)
        parts = vp.PART_HISTORY
    kw = {} if delta1 is None else {"delta1_override": delta1}
    if parts is not None:
        kw["parts"] = parts
    plan = vp.Plan(torch.from_numpy(nodes).cuda(), torch.from_numpy(wts).cuda(),
                   torch.from_numpy(np.ascontiguousarray(targets)).cuda(), tol, boundary=("chunks", chunks), **kw)
    return plan, torch, vp


def _inside_outside(rng, n_in=200, n_out=200):
    th = rng.uniform(0, 2 * np.pi, n_in + n_out)
    rb = geometry.star_radius(th)
    rr = np.concatenate([rb[:n_in] * rng.uniform(0.0, 0.98, n_in), rb[n_in:] * rng.uniform(1.02, 2.0, n_out)])
    return np.stack([rr * np.cos(th), rr * np.sin(th)], 1)


def test_bie_dirichlet_interior_star():
    ch = geometry.star_chunks(NCH, Q)
    bn = ch.reshape(-1, 2)
    u = lambda p: p[:, 0] ** 3 - 3 * p[:, 0] * p[:, 1] ** 2 + 0.4 * p[:, 0] + 0.7  # noqa: E731
    tol = 1e-10
    A, torch, vp = _plan(bn, ch, tol, 2.5e-5)
    A.prepare_dlp()
    mu, it, res = A.bie_solve(vp.BIE_DIRICHLET_INT, torch.from_numpy(u(bn)).cuda(), tol=1e-13)
    A.destroy()
    tg = _inside_outside(np.random.default_rng(1), 400, 0)
    Bp, _, _ = _plan(tg, ch, tol, 2.5e-5)
    Bp.prepare_dlp()
    got = Bp.eval_dlp(mu).cpu().numpy()
    Bp.destroy()
    e = rel_l2(got, u(tg))
    print("bie dirichlet interior star: iters", it, "resid %.2e" % res, "rel l2 %.3e" % e)
    assert res <= 1e-13 and it < 60
    assert e <= 1e-8, e


def test_bie_dirichlet_exterior_star():
    ch = geometry.star_chunks(NCH, Q)
    bn = ch.reshape(-1, 2)
    W, _ = _star_W()

    def u(p):  # bounded exterior harmonic: Re(1/z) + 0.3 Im(1/z^2) + 0.5
        z = p[:, 0] + 1j * p[:, 1]
        return np.real(1 / z) + 0.3 * np.imag(1 / z ** 2) + 0.5
    tol = 1e-10
    A, torch, vp = _plan(bn, ch, tol, 2.5e-5)
    A.prepare_dlp()
    mu, it, res = A.bie_solve(vp.BIE_DIRICHLET_EXT, torch.from_numpy(u(bn)).cuda(), tol=1e-13)
    A.destroy()
    tg = _inside_outside(np.random.default_rng(2), 0, 400)
    Bp, _, _ = _plan(tg, ch, tol, 2.5e-5)
    Bp.prepare_dlp()
    mh = mu.cpu().numpy()
    got = Bp.eval_dlp(mu).cpu().numpy() + np.sum(W * mh)
    Bp.destroy()
    e = rel_l2(got, u(tg))
    print("bie dirichlet exterior star: iters", it, "resid %.2e" % res, "rel l2 %.3e" % e)
    assert res <= 1e-13 and it < 60
    assert e <= 1e-8, e


def test_bie_neumann_interior_star():
    ch = geometry.star_chunks(NCH, Q)
    bn = ch.reshape(-1, 2)
    W, th = _star_W()
    nx, ny = _star_normal(th)
    x, y = bn[:, 0], bn[:, 1]
    u = x ** 3 - 3 * x * y * y + 0.4 * x
    dudn = (3 * x * x - 3 * y * y + 0.4) * nx - 6 * x * y * ny
    tol = 1e-10
    A, torch, vp = _plan(bn, ch, tol, 2.5e-5)
    A.prepare_slp()
    A.prepare_dlp()
    rhs = A.eval_slp(torch.from_numpy(dudn).cuda())
    sol, it, res = A.bie_solve(vp.BIE_NEUMANN_INT, rhs, tol=1e-12)
    A.destroy()
    s = sol.cpu().numpy()
    # the solution is defined up to a constant: compare after removing the W-weighted means
    d = (s - np.sum(W * s) / np.sum(W)) - (u - np.sum(W * u) / np.sum(W))
    e = np.sqrt(np.sum(W * d * d) / np.sum(W * u * u))
    print("bie neumann interior star: iters", it, "resid %.2e" % res, "rel l2 %.3e" % e)
    assert res <= 1e-12
    assert e <= 1e-8, e


def test_poisson_dirichlet_disk():
    """-Lap u = f on the unit disk with u = cos(2x) sin(y) (f = 5u): V[f] at the boundary nodes, GMRES for mu,
    u = V[f] + D[mu] at interior targets; the error is the volume potential's (tol 1e-10 on 8000 triangles)."""
    w = configs.config1(M_target=8000, f="const", tol=1e-10)
    ch = geometry.circle_chunks(0.0, 0.0, 1.0, 96, q=Q, theta0=0.05)
    bn = ch.reshape(-1, 2)
    uex = lambda p: np.cos(2 * p[..., 0]) * np.sin(p[..., 1])  # noqa: E731
    f = 5.0 * uex(w.nodes)
    A, torch, vp = _plan(bn, ch, w.tol, nodes=w.nodes, wts=w.weights)
    A.prepare_dlp()
    fd = torch.from_numpy(np.ascontiguousarray(f)).cuda()
    Vb = A.eval(fd)
    rhs = torch.from_numpy(uex(bn)).cuda() - Vb
    mu, it, res = A.bie_solve(vp.BIE_DIRICHLET_INT, rhs, tol=1e-13)
    A.destroy()
    rng = np.random.default_rng(4)
    r = np.sqrt(rng.uniform(0, 0.98 ** 2, 500))
    t = rng.uniform(0, 2 * np.pi, 500)
    tg = np.stack([r * np.cos(t), r * np.sin(t)], 1)
    Bp, _, _ = _plan(tg, ch, w.tol, nodes=w.nodes, wts=w.weights)
    Bp.prepare_dlp()
    got = (Bp.eval(fd) + Bp.eval_dlp(mu)).cpu().numpy()
    Bp.destroy()
    e = rel_l2(got, uex(tg))
    print("poisson dirichlet disk: M", w.M, "iters", it, "resid %.2e" % res, "rel l2 %.3e" % e)
    assert res <= 1e-13
    assert e <= 1e-7, e
