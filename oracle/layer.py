"""CPU fp64 oracle for the single-layer potential -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    S[sigma](x) = int_Gamma G(x - y) sigma(y) ds_y,   G(z) = -(1/2 pi) log |z|        (PAPER.md lines 493-510,
                                                                                     eq. sheatdecomp)

on a closed curve given by an analytic parametrisation gamma(theta), theta in [0, 2 pi), and an analytic density
sigma(theta).  The integral is the plain definition evaluated by adaptive Gauss-Legendre quadrature in theta: a
panel is accepted when its distance to the target exceeds ETA times its length (the log kernel is then smooth on
it to ~1e-15 with 20 nodes), otherwise it is bisected; a target on the curve makes the recursion refine
geometrically towards the (integrable) logarithmic singularity, down to panels of length 1e-14.  Shares no code
with the CUDA path.  Pinned in tests/test_oracle.py (closed forms on the unit circle: S[1] = -log max(r, 1),
S[cos m theta] = r^{+-m} cos(m theta) / (2m); additivity over densities; a brute-force comparison with
scipy.integrate.quad for one off-curve target).
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
