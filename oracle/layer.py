"""CPU fp64 oracle for the layer potentials -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    S[sigma](x) = int_Gamma G(x - y) sigma(y) ds_y,   G(z) = -(1/2 pi) log |z|        (PAPER.md lines 493-510,
                                                                                     eq. sheatdecomp)
    D[mu](x)    = int_Gamma dG(x - y)/dnu_y mu(y) ds_y = (1/2 pi) int_Gamma (x - y).nu_y / |x - y|^2 mu ds_y
                  with nu the OUTWARD unit normal (eq. dheatdecomp; the Dirichlet
                  equation -mu/2 + D[mu] = g of lines 1281-1287 fixes the interior limit D - mu/2)

on a closed curve given by an analytic parametrisation gamma(theta), theta in [0, 2 pi), and an analytic density
sigma(theta).  The integral is the plain definition evaluated by adaptive Gauss-Legendre quadrature in theta: a
panel is accepted when its distance to the target exceeds ETA times its length (the log kernel is then smooth on
it to ~1e-15 with 20 nodes), otherwise it is bisected; a target on the curve makes the recursion refine
geometrically towards the (integrable) logarithmic singularity, down to panels of length 1e-14.  Shares no code
with the CUDA path.  Pinned in tests/test_oracle.py (closed forms on the unit circle: S[1] = -log max(r, 1),
S[cos m theta] = r^{+-m} cos(m theta) / (2m); additivity over densities; a brute-force comparison with
scipy.integrate.quad for one off-curve target).  double_layer uses the same adaptive rule off the curve; for
targets ON the curve (flag on_curve) it takes the direct value (the kernel is smooth along a smooth curve) with a
fixed composite rule, because bisecting towards the target would cancel (x - y).nu catastrophically.  Pinned in
tests/test_layer.py: unit-circle closed forms (D[1] = -1 / -1/2 / 0 inside / on / outside, D[cos m theta] =
-r^m cos(m theta)/2 inside, r^-m cos(m theta)/2 outside, 0 on the circle), Green's representation
u = S[du/dnu] - D[u] (interior) / 0 (exterior) for a harmonic u on the star, and scipy.integrate.quad.
"""
import numpy as np

_NG = 20
_XG, _WG = np.polynomial.legendre.leggauss(_NG)
ETA = 3.0
MIN_LEN = 1e-14


def _panel(curve, dcurve, sigma, a, b):
    """nodes, weights (ds included) and density values of the _NG-point rule on theta in [a, b]"""
    t = 0.5 * (a + b) + 0.5 * (b - a) * _XG
    p = curve(t)
    dp = dcurve(t)
    ds = np.hypot(dp[0], dp[1])
    return p, 0.5 * (b - a) * _WG * ds, sigma(t)


def single_layer(curve, dcurve, sigma, targets, n0=64):
    """S[sigma] at targets [T, 2].  curve(theta) -> (x, y) arrays, dcurve(theta) -> (x', y'), sigma(theta)."""
    targets = np.asarray(targets, dtype=np.float64)
    out = np.zeros(len(targets))
    edges = np.linspace(0.0, 2.0 * np.pi, n0 + 1)
    for i, x in enumerate(targets):
        acc = 0.0
        stack = [(edges[k], edges[k + 1]) for k in range(n0)]
        while stack:
            a, b = stack.pop()
            p, w, s = _panel(curve, dcurve, sigma, a, b)
            length = np.sum(w)  # panel arc length (the weights carry ds)
            dist = np.min(np.hypot(p[0] - x[0], p[1] - x[1]))
            if dist > ETA * length or (b - a) < MIN_LEN:
                r2 = (p[0] - x[0]) ** 2 + (p[1] - x[1]) ** 2
                r2 = np.where(r2 > 0, r2, 1e-300)
                acc += np.sum(w * s * (-np.log(r2) / (4.0 * np.pi)))
            else:
                m = 0.5 * (a + b)
                stack.append((a, m))
                stack.append((m, b))
        out[i] = acc
    return out


def circle(R=1.0):
    """unit-speed-scaled parametrisation of the circle of radius R (counter-clockwise)"""
    return (lambda t: (R * np.cos(t), R * np.sin(t))), (lambda t: (-R * np.sin(t), R * np.cos(t)))


def star(a=0.3, k=5):
    """r(theta) = 1 + a cos(k theta) (config 3's domain), counter-clockwise"""
    def curve(t):
        r = 1.0 + a * np.cos(k * t)
        return r * np.cos(t), r * np.sin(t)

    def dcurve(t):
        r = 1.0 + a * np.cos(k * t)
        dr = -a * k * np.sin(k * t)
        return dr * np.cos(t) - r * np.sin(t), dr * np.sin(t) + r * np.cos(t)
    return curve, dcurve


def _normal_out(dp):
    """outward unit normal of a counter-clockwise curve from gamma'(theta): (y', -x') / |gamma'|"""
    ds = np.hypot(dp[0], dp[1])
    return dp[1] / ds, -dp[0] / ds


def _closest_param(curve, x, n=4096):
    """parameter of the point of the curve closest to x: dense sample, then a bounded scalar minimisation"""
    from scipy.optimize import minimize_scalar
    t = np.linspace(0.0, 2.0 * np.pi, n, endpoint=False)
    p = curve(t)
    k = int(np.argmin((p[0] - x[0]) ** 2 + (p[1] - x[1]) ** 2))
    h = 2.0 * np.pi / n
    f = lambda u: float((curve(u)[0] - x[0]) ** 2 + (curve(u)[1] - x[1]) ** 2)  # noqa: E731
    return minimize_scalar(f, bounds=(t[k] - 2 * h, t[k] + 2 * h), method="bounded",
                           options={"xatol": 1e-14}).x


def double_layer(curve, dcurve, mu, targets, on_curve=None, n0=64, n_on=256):
    """D[mu] at targets [T, 2] (outward normal).  on_curve: optional bool mask of targets lying ON the curve
    (direct value, composite rule of n_on panels)."""
    targets = np.asarray(targets, dtype=np.float64)
    on = np.zeros(len(targets), bool) if on_curve is None else np.asarray(on_curve, bool)
    out = np.zeros(len(targets))
    edges = np.linspace(0.0, 2.0 * np.pi, n0 + 1)
    e_on = np.linspace(0.0, 2.0 * np.pi, n_on + 1)
    for i, x in enumerate(targets):
        acc = 0.0
        if on[i]:  # panels with a breakpoint at the target's parameter: no node closer than ~1e-3 panel lengths
            t0 = _closest_param(curve, x)
            stack, accept_all = [(t0 + e_on[k], t0 + e_on[k + 1]) for k in range(n_on)], True
        else:
            stack, accept_all = [(edges[k], edges[k + 1]) for k in range(n0)], False
        while stack:
            a, b = stack.pop()
            p, w, s = _panel(curve, dcurve, mu, a, b)
            length = np.sum(w)
            dist = np.min(np.hypot(p[0] - x[0], p[1] - x[1]))
            if accept_all or dist > ETA * length or (b - a) < MIN_LEN:
                t = 0.5 * (a + b) + 0.5 * (b - a) * _XG
                nx, ny = _normal_out(dcurve(t))
                dx, dy = x[0] - p[0], x[1] - p[1]
                r2 = dx * dx + dy * dy
                k = np.where(r2 > 0, (dx * nx + dy * ny) / np.where(r2 > 0, r2, 1.0), 0.0) / (2.0 * np.pi)
                acc += np.sum(w * s * k)
            else:
                m = 0.5 * (a + b)
                stack.append((a, m))
                stack.append((m, b))
        out[i] = acc
    return out
