"""Triangle geometry for the synthetic workloads (input description, not method arithmetic).

A triangle is three CCW vertices plus a 3-bit mask saying which edges
e = (v_e, v_{e+1 mod 3}) are circular arcs of one shared circle (config 1's
unit disk).  PAPER.md §2.2 (lines 593-617) describes boundary triangles whose
boundary side is a curve; SURVEY.md §8(c) item "Curved triangles" fixes the
reading used here: a *smooth* blending map from the reference triangle

    x(l) = sum_k l_k v_k + sum_{curved e=(i,j)} l_i l_j q_e(l_j - l_i)

with q_e(s) = D_e(lam) / (lam (1 - lam)), lam = (1 + s)/2 and D_e the
arc-minus-chord deviation of the edge.  On the edge l_i + l_j = 1 the
correction equals D_e(l_j) exactly, and it vanishes on the two straight
edges, so neighbouring straight triangles stay conforming.

Quadrature nodes are the images of the 12-point rule's barycentric points;
weights are w_bary * |det J| / 2 (reference triangle of area 1/2), with the
Jacobian taken by complex-step differentiation (exact to rounding).
The CPU oracle implements the same geometric definition independently in C.
"""
import numpy as np

from . import rule


def _sinc(z):
    z = np.asarray(z)
    small = np.abs(z) < 1e-4
    zs = np.where(small, 1.0, z)
    return np.where(small, 1.0 - z * z / 6.0 + z ** 4 / 120.0, np.sin(zs) / zs)


def arc_q(lam, va, vb, circle):
    """q(lam) = (arc(lam) - chord(lam)) / (lam (1 - lam)) for the arc va -> vb (complex-step safe).

    lam: array (...,), va/vb: (..., 2) arrays, circle = (cx, cy, rho).
    The arc is the shorter one between the two vertices' polar angles.
    """
    cx, cy, rho = circle
    ta = np.arctan2(va[..., 1].real - cy, va[..., 0].real - cx)
    tb = np.arctan2(vb[..., 1].real - cy, vb[..., 0].real - cx)
    dt = np.angle(np.exp(1j * (tb - ta)))            # signed shortest angle in (-pi, pi]
    dvx = vb[..., 0] - va[..., 0]
    dvy = vb[..., 1] - va[..., 1]
    lo = np.real(lam) <= 0.5
    # branch lam <= 1/2, expand from va:  D/lam = rho*dt*sinc(lam dt/2)*(-sin, cos)(ta + lam dt/2) - (vb - va)
    ph = ta + lam * dt / 2.0
    s = rho * dt * _sinc(lam * dt / 2.0)
    dl_x = s * (-np.sin(ph)) - dvx
    dl_y = s * np.cos(ph) - dvy
    qa_x = dl_x / (1.0 - lam)
    qa_y = dl_y / (1.0 - lam)
    # branch lam > 1/2, expand from vb with mu = 1 - lam: D/mu = -rho*dt*sinc(mu dt/2)*(-sin, cos)(tb - mu dt/2) + (vb - va)
    mu = 1.0 - lam
    ph2 = tb - mu * dt / 2.0
    s2 = -rho * dt * _sinc(mu * dt / 2.0)
    dm_x = s2 * (-np.sin(ph2)) + dvx
    dm_y = s2 * np.cos(ph2) + dvy
    qb_x = dm_x / lam
    qb_y = dm_y / lam
    return np.where(lo, qa_x, qb_x), np.where(lo, qa_y, qb_y)


def map_points(tri, curved, circle, xi1, xi2):
    """Map reference points (xi1, xi2) (shape (M, K)) through each triangle's map.

    tri: (M, 3, 2); curved: (M,) int bitmask.  Returns x, y of shape (M, K).
    Complex inputs are propagated (complex-step differentiation).
    """
    l = [1.0 - xi1 - xi2, xi1, xi2]
    x = sum(l[k] * tri[:, k, 0:1] for k in range(3))
    y = sum(l[k] * tri[:, k, 1:2] for k in range(3))
    if circle is None or not np.any(curved):
        return x, y
    x = x.astype(np.result_type(x, xi1))
    y = y.astype(np.result_type(y, xi1))
    for e in range(3):
        sel = (curved & (1 << e)) != 0
        if not np.any(sel):
            continue
        i, j = e, (e + 1) % 3
        li, lj = l[i][sel], l[j][sel]
        s = lj - li
        lam = (1.0 + s) / 2.0
        va = tri[sel, i, None, :]
        vb = tri[sel, j, None, :]
        va = np.broadcast_to(va, lam.shape + (2,))
        vb = np.broadcast_to(vb, lam.shape + (2,))
        qx, qy = arc_q(lam, va, vb, circle)
        x[sel] = x[sel] + li * lj * qx
        y[sel] = y[sel] + li * lj * qy
    return x, y


def nodes_weights(tri, curved=None, circle=None, chunk=1 << 20):
    """Quadrature nodes (M, 12, 2) and weights (M, 12) of the 12-point rule on each triangle."""
    M = tri.shape[0]
    if curved is None:
        curved = np.zeros(M, dtype=np.int8)
    bary = rule.BARY
    xi1 = np.broadcast_to(bary[None, :, 1], (M, rule.P))
    xi2 = np.broadcast_to(bary[None, :, 2], (M, rule.P))
    nodes = np.empty((M, rule.P, 2))
    wts = np.empty((M, rule.P))
    straight = curved == 0
    # affine triangles: exact closed form
    v0, v1, v2 = tri[:, 0], tri[:, 1], tri[:, 2]
    area = 0.5 * ((v1[:, 0] - v0[:, 0]) * (v2[:, 1] - v0[:, 1]) - (v1[:, 1] - v0[:, 1]) * (v2[:, 0] - v0[:, 0]))
    nodes[...] = np.einsum("kj,mjd->mkd", bary, tri, optimize=False)
    np.multiply(rule.WEIGHTS[None, :], np.abs(area)[:, None], out=wts)
    cur = np.nonzero(~straight)[0]
    if cur.size:
        h = 1e-30
        t = tri[cur]
        c = curved[cur]
        a1 = xi1[cur].astype(np.complex128)
        a2 = xi2[cur].astype(np.complex128)
        x, y = map_points(t, c, circle, a1.real, a2.real)
        x1, y1 = map_points(t, c, circle, a1 + 1j * h, a2)
        x2, y2 = map_points(t, c, circle, a1, a2 + 1j * h)
        J11, J21 = x1.imag / h, y1.imag / h
        J12, J22 = x2.imag / h, y2.imag / h
        det = J11 * J22 - J12 * J21
        nodes[cur, :, 0] = x
        nodes[cur, :, 1] = y
        wts[cur] = rule.WEIGHTS[None, :] * 0.5 * np.abs(det)
    return nodes, wts


# --------------------------------------------------------------------------- boundary descriptors
def _gl_nodes(q):
    """q + 1 Gauss-Legendre points of [-1, 1], increasing (numpy's leggauss)."""
    return np.polynomial.legendre.leggauss(q + 1)[0]


def circle_chunks(cx, cy, rho, n, q=16, theta0=0.0):
    """CCW circle as n chunks of degree q: chunk c samples theta in [theta0 + 2 pi c / n, theta0 + 2 pi (c+1) / n]
    at the Gauss-Legendre points (the vp_boundary CHUNKS convention, R17).  -> [n, q+1, 2]"""
    s = _gl_nodes(q)
    th = theta0 + 2 * np.pi * (np.arange(n)[:, None] + 0.5 * (s[None, :] + 1.0)) / n
    return np.stack([cx + rho * np.cos(th), cy + rho * np.sin(th)], -1)


def star_radius(th, a=0.3, m=5):
    return 1.0 + a * np.cos(m * th)


def star_chunks(n, q=16, a=0.3, m=5, cx=0.0, cy=0.0):
    """CCW star r(theta) = 1 + a cos(m theta) (config 3's domain) as n chunks of degree q, uniform in theta."""
    s = _gl_nodes(q)
    th = 2 * np.pi * (np.arange(n)[:, None] + 0.5 * (s[None, :] + 1.0)) / n
    r = star_radius(th, a, m)
    return np.stack([cx + r * np.cos(th), cy + r * np.sin(th)], -1)
