"""C-ABI library: loads, exports every symbol include/vp.h declares, argument errors without a GPU,
and the host-callable scalar math of the method (local-part coefficients, multipliers) against
independent brute-force references (CPU)."""
import ctypes
import os
import re

import numpy as np
import pytest
import scipy.integrate as si
import scipy.special as sp

import paper_2409_11998_b200 as vp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "vp.h")).read()
    return sorted(set(re.findall(r"^\s*(?:vp_status|const char \*)\s*(vp_\w+)\s*\(", src, re.M)))


def test_library_exports_header_symbols():
    L = vp.lib()
    names = header_functions()
    assert "vp_plan" in names and "vp_eval" in names and "vp_destroy" in names and "vp_strerror" in names
    for n in names:
        assert hasattr(L, n), n


def test_struct_sizes_match_binding():
    """The ctypes mirrors of vp_opts / vp_info / vp_boundary have the library's sizes (vp_struct_sizes; the
    binding refuses to load a library with another layout)."""
    L = vp.lib()
    sz = (ctypes.c_int64 * 3)()
    assert L.vp_struct_sizes(sz) == vp.VP_OK
    assert tuple(sz) == (ctypes.sizeof(vp.VpOpts), ctypes.sizeof(vp.VpInfo), ctypes.sizeof(vp.VpBoundary))
    assert L.vp_struct_sizes(None) == vp.VP_ERR_ARG


def test_strerror_and_version():
    L = vp.lib()
    for s in range(-8, 1):
        assert len(L.vp_strerror(s)) > 0
    assert b"sm_100a" in L.vp_version()


def test_argument_errors_without_gpu():
    L = vp.lib()
    h = ctypes.c_void_p()
    o = vp.VpOpts()
    # null pointers / sizes / tol are rejected before any CUDA call
    assert L.vp_plan(None, None, 10, 12, None, 10, 1e-8, ctypes.byref(o), ctypes.byref(h)) == vp.VP_ERR_ARG
    assert L.vp_plan(1, 1, 0, 12, 1, 10, 1e-8, ctypes.byref(o), ctypes.byref(h)) == vp.VP_ERR_ARG
    assert L.vp_plan(1, 1, 10, 12, 1, 10, 1e-20, ctypes.byref(o), ctypes.byref(h)) == vp.VP_ERR_TOL
    assert L.vp_plan(1, 1, 10, 12, 1, 10, 0.5, ctypes.byref(o), ctypes.byref(h)) == vp.VP_ERR_TOL
    assert L.vp_eval(None, None, None) == vp.VP_ERR_ARG
    assert L.vp_eval_batch(None, 4, None, None) == vp.VP_ERR_ARG
    assert L.vp_eval_batch(1, 0, 1, 1) == vp.VP_ERR_ARG  # K < 1 is rejected before the handle is used
    # layer potentials, BIE solves, pipelined host evals: arguments checked before any CUDA call
    assert L.vp_slp_prepare(None) == vp.VP_ERR_ARG and L.vp_dlp_prepare(None) == vp.VP_ERR_ARG
    assert L.vp_eval_slp(None, None, None) == vp.VP_ERR_ARG and L.vp_eval_dlp(None, None, None) == vp.VP_ERR_ARG
    assert L.vp_layer_set_levels(None, 3) == vp.VP_ERR_ARG
    it, res = ctypes.c_int32(), ctypes.c_double()
    assert L.vp_bie_solve(None, 0, 1, 1, 1e-10, 10, 10, ctypes.byref(it), ctypes.byref(res)) == vp.VP_ERR_ARG
    assert L.vp_bie_solve(1, 7, 1, 1, 1e-10, 10, 10, ctypes.byref(it), ctypes.byref(res)) == vp.VP_ERR_ARG  # kind
    assert L.vp_bie_solve(1, 0, 1, 1, 0.0, 10, 10, ctypes.byref(it), ctypes.byref(res)) == vp.VP_ERR_ARG  # tol
    assert L.vp_bie_solve(1, 0, 1, 1, 1e-10, 10, 500, ctypes.byref(it), ctypes.byref(res)) == vp.VP_ERR_ARG
    assert L.vp_eval_host_many(None, 1, None, None) == vp.VP_ERR_ARG
    assert L.vp_eval_host_many(1, 0, None, None) == vp.VP_ERR_ARG
    nul = (ctypes.c_void_p * 2)(None, None)
    assert L.vp_eval_host_many(1, 2, nul, nul) == vp.VP_ERR_ARG
    assert L.vp_destroy(None) == vp.VP_OK


def test_multipliers_vs_definitions():
    # near history: int_{d1}^{d2} e^{-k^2 t} dt ; far history: e^{-k^2 d2} * (-int_0^R r log r J0(kr) dr)
    d1, d2, R = 1e-3, 3.2e-2, 2.1
    for k in [0.0, 1e-4, 0.7, 13.0, 60.0]:
        ref = d2 - d1 if k == 0 else si.quad(lambda t: np.exp(-k * k * t), d1, d2, epsabs=0, epsrel=1e-13)[0]
        assert abs(vp.debug_mult(0, k * k, d1, d2) - ref) < 1e-12 * max(abs(ref), 1e-300) + 1e-300
        W = -si.quad(lambda r: r * np.log(r) * sp.j0(k * r), 0, R, limit=400, epsabs=1e-15, epsrel=1e-13)[0]
        ref = np.exp(-k * k * d2) * W
        assert abs(vp.debug_mult(1, k * k, d2, R) - ref) < 1e-11 * max(1.0, abs(W))


def _taylor_value(coef, jet):
    return float(np.dot(coef, jet))


def _mono_index(a, b):
    d = a + b
    return d * (d + 1) // 2 + (d - a)


def test_interior_series_coefficients():
    b, c = vp.debug_local_coef("none", [0, 0, 0, 0], 0.3, 0.4, 1e-3, 3, 6)
    assert not b
    d = 1e-3
    assert c[_mono_index(0, 0)] == d
    assert abs(c[_mono_index(2, 0)] - d * d) < 1e-20 and abs(c[_mono_index(0, 2)] - d * d) < 1e-20
    assert abs(c[_mono_index(4, 0)] - 4 * d ** 3) < 1e-24 and abs(c[_mono_index(2, 2)] - 4 * d ** 3 / 3) < 1e-24


def test_circle_on_boundary_matches_corollary():
    """At c = 0 the V_L coefficients reduce to the paper's on-boundary corollary
    V_L = (d/2) f + d^{3/2} (2 f_eta - kappa f)/(3 sqrt pi) + (d^2/4) Lap f."""
    d, rho = 1e-4, 1.0
    b, c = vp.debug_local_coef("circle", [0, 0, rho, 0], 1.0, 0.0, d, 2, 6)   # point on the circle, normal -x
    assert b
    kap = 1 / rho
    assert abs(c[_mono_index(0, 0)] - (d / 2 - d ** 1.5 * kap / (3 * np.sqrt(np.pi)))) < 1e-15
    # f_eta = grad f . n, n = (-1, 0): coefficient of a10 = -2 d^{3/2}/(3 sqrt pi)
    assert abs(c[_mono_index(1, 0)] - (-2 * d ** 1.5 / (3 * np.sqrt(np.pi)))) < 1e-15
    # Lap f = 2 a20 + 2 a02 with weight d^2/4
    assert abs(c[_mono_index(2, 0)] - d * d / 2) < 1e-18 and abs(c[_mono_index(0, 2)] - d * d / 2) < 1e-18


def _brute_vl_halfplane(x2, delta, f):
    """int_0^delta int_{y2 > 0} K_t(x - y) f(y) dy dt for the half plane y2 > 0 (brute force)."""
    def inner(t):
        g = lambda y1, y2: np.exp(-((y1) ** 2 + (y2 - x2) ** 2) / (4 * t)) / (4 * np.pi * t) * f(y1, y2)
        s = 12 * np.sqrt(t)
        return si.dblquad(lambda y2, y1: g(y1, y2), -s, s, max(0, x2 - s), x2 + s, epsabs=1e-16, epsrel=1e-11)[0]
    return si.quad(inner, 0, delta, epsabs=1e-18, epsrel=1e-10, limit=100)[0]


@pytest.mark.parametrize("dist_over_sd", [0.0, 0.7, 3.0])
def test_rect_product_form_vs_brute_force(dist_over_sd):
    # near the bottom edge of a big rectangle (other edges far): quadratic f
    d = 1e-3
    sd = np.sqrt(d)
    x, y = 0.5, dist_over_sd * sd
    b, c = vp.debug_local_coef("rect", [0, 0, 1, 1], x, y, d, 3, 6)
    assert b
    a = {(0, 0): 0.7, (1, 0): -0.3, (0, 1): 1.1, (2, 0): 0.4, (1, 1): -0.8, (0, 2): 0.25}
    jet = np.zeros(15)
    for (p, q), v in a.items():
        jet[_mono_index(p, q)] = v
    f = lambda y1, y2: sum(v * (y1 - x) ** p * (y2 - y) ** q for (p, q), v in a.items())
    ref = _brute_vl_halfplane(y, d, lambda y1, y2: f(y1 + x, y2))
    got = _taylor_value(c, jet)
    assert abs(got - ref) < 1e-9 * abs(ref), (got, ref)


def test_rect_reduces_to_interior_far_from_edges():
    d = 1e-4
    b, c = vp.debug_local_coef("rect", [0, 0, 1, 1], 0.5, 0.5, d, 3, 6)
    assert not b       # beyond 12 sqrt(delta): interior series
    b, c = vp.debug_local_coef("rect", [0, 0, 1, 1], 0.5, 11.0 * np.sqrt(d), d, 3, 6)
    assert b
    _, ci = vp.debug_local_coef("none", [0, 0, 0, 0], 0.5, 0.5, d, 3, 6)
    assert np.max(np.abs(c - ci)) < 1e-12 * d   # exponentially close to the interior series


def test_circle_vs_rect_flat_limit():
    """A huge circle is locally a half plane: the (vplocO5) coefficients (kappa -> 0) agree with the
    exact product form up to O(delta^{5/2}) terms."""
    d = 1e-4
    rho = 1e4
    for cdist in [0.0, 1.0, 4.0]:
        yv = cdist * np.sqrt(d)
        b1, c1 = vp.debug_local_coef("circle", [0, rho, rho, 0], 0.0, yv, d, 2, 6)   # bottom point of circle at origin
        b2, c2 = vp.debug_local_coef("rect", [-1, 0, 1, 2], 0.0, yv, d, 2, 6)
        assert b1 and b2
        for idx in [_mono_index(0, 0), _mono_index(0, 1), _mono_index(2, 0), _mono_index(0, 2)]:
            # curvature terms kappa delta^{3/2} (kappa = 1/rho) and O(delta^{5/2}) remain
            assert abs(c1[idx] - c2[idx]) < 1e-3 * d ** 2 + 3 * d ** 1.5 / rho + 1e-9 * abs(c2[idx]), (cdist, idx)


def _brute_vl_quadrant(x1, x2, delta, f):
    """int_0^delta int_{y1 > 0, y2 > 0} K_t(x - y) f(y) dy dt for the quadrant (brute force, scipy)."""
    def inner(t):
        g = lambda y1, y2: np.exp(-((y1 - x1) ** 2 + (y2 - x2) ** 2) / (4 * t)) / (4 * np.pi * t) * f(y1, y2)
        s = 12 * np.sqrt(t)
        return si.dblquad(lambda y2, y1: g(y1, y2), max(0, x1 - s), x1 + s, max(0, x2 - s), x2 + s,
                          epsabs=1e-16, epsrel=1e-11)[0]
    return si.quad(inner, 0, delta, epsabs=1e-18, epsrel=1e-10, limit=100)[0]


@pytest.mark.parametrize("pos", [(0.0, 0.0), (0.4, 1.3), (2.0, 0.2), (5.0, 4.0)])
def test_rect_product_form_corner_vs_brute_force(pos):
    """Quarter-plane corner of the unit square (R8; the paper is silent on corners): the product-form
    coefficients of vp_coef_rect against a brute-force space-time integral over the quadrant, quadratic f with a
    mixed term; positions in units of sqrt(delta) from the corner (0, 0)."""
    d = 1e-3
    sd = np.sqrt(d)
    x, y = pos[0] * sd, pos[1] * sd
    b, c = vp.debug_local_coef("rect", [0, 0, 1, 1], x, y, d, 3, 6)
    assert b
    a = {(0, 0): 0.7, (1, 0): -0.3, (0, 1): 1.1, (2, 0): 0.4, (1, 1): -0.8, (0, 2): 0.25}
    jet = np.zeros(15)
    for (p, q), v in a.items():
        jet[_mono_index(p, q)] = v
    f = lambda y1, y2: sum(v * (y1 - x) ** p * (y2 - y) ** q for (p, q), v in a.items())
    ref = _brute_vl_quadrant(x, y, d, f)
    got = _taylor_value(c, jet)
    assert abs(got - ref) < 1e-9 * abs(ref), (got, ref)
