"""CPU fp64 oracle for the 2D Poisson volume potential -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  It shares no code with the CUDA product path
(paper_2409_11998_b200/), which never imports it.

Functions (see oracle/vp_oracle.c for the citations and the quadrature tiers):
  volume_potential(workload_or_geometry, targets) -> V*(x_t) = sum_T int_T G(x_t-y) f(y) dy
  smooth_direct(src, c, targets, delta)            -> sum_j c_j G_H[delta](x_t - x_j)
  smooth_dft(src, c, targets, d1, d2, ...)         -> same split through a direct Fourier sum
  e1(x), GH(r2, delta), WR(k, R)
  layer.single_layer(curve, dcurve, sigma, targets) -> S[sigma](x_t) on an analytic closed curve (oracle/layer.py)
  layer.double_layer(curve, dcurve, mu, targets, on_curve) -> D[mu](x_t), outward normal (oracle/layer.py)
Parity status of each function is listed in DESIGN.md §Oracle (all pinned).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=gnu11", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


class _Field(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n", ctypes.c_int32), ("a0", ctypes.c_double),
                ("a", ctypes.c_void_p), ("cx", ctypes.c_void_p), ("cy", ctypes.c_void_p), ("s", ctypes.c_void_p),
                ("k1", ctypes.c_void_p), ("k2", ctypes.c_void_p), ("fa", ctypes.c_void_p), ("fb", ctypes.c_void_p)]


class _Opts(ctypes.Structure):
    _fields_ = [("eta_far", ctypes.c_double), ("eta_polar", ctypes.c_double), ("nthreads", ctypes.c_int32),
                ("assume_resolved", ctypes.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d, i64, p = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p
        _lib.orc_volume_potential.argtypes = [i64, p, p, p, ctypes.POINTER(_Field), i64, p, p, ctypes.POINTER(_Opts)]
        _lib.orc_volume_potential.restype = ctypes.c_int
        _lib.orc_triangle_integral.argtypes = [p, ctypes.c_int8, p, ctypes.POINTER(_Field), d, d, ctypes.POINTER(_Opts)]
        _lib.orc_triangle_integral.restype = d
        _lib.orc_rule12_nodes.argtypes = [i64, p, p, p, p, p]
        _lib.orc_e1.argtypes = [d]
        _lib.orc_e1.restype = d
        _lib.orc_GH.argtypes = [d, d]
        _lib.orc_GH.restype = d
        _lib.orc_WR.argtypes = [d, d]
        _lib.orc_WR.restype = d
        _lib.orc_smooth_direct.argtypes = [i64, p, p, i64, p, d, p]
        _lib.orc_smooth_dft.argtypes = [i64, p, p, i64, p, d, d, d, i64, d, i64, d, d, d, p]
        _lib.orc_num_threads.restype = ctypes.c_int
        _lib.orc_prepare.argtypes = [i64, p, p, p, ctypes.POINTER(_Field), ctypes.POINTER(_Opts)]
        _lib.orc_prepare.restype = p
        _lib.orc_eval_prepared.argtypes = [p, i64, p, p]
        _lib.orc_eval_prepared.restype = ctypes.c_int
        _lib.orc_free.argtypes = [p]
        _lib.orc_field_values.argtypes = [ctypes.POINTER(_Field), i64, p, p]
        _lib.orc_set_gauss_legendre.argtypes = [ctypes.c_int, p, p]
        _lib.orc_set_gauss_legendre.restype = ctypes.c_int
        # Gauss-Legendre rules n = 1..40 from numpy (companion-matrix eigenvalues), handed to the C oracle
        xs, ws = zip(*(np.polynomial.legendre.leggauss(n) for n in range(1, 41)))
        _gl_keep = (np.ascontiguousarray(np.concatenate(xs)), np.ascontiguousarray(np.concatenate(ws)))
        if _lib.orc_set_gauss_legendre(40, _ptr(_gl_keep[0]), _ptr(_gl_keep[1])) != 0:
            raise RuntimeError("orc_set_gauss_legendre failed")
        _lib.orc_resolve_rules.argtypes = [i64, p, p, p, ctypes.POINTER(_Field), p]
        _lib.orc_resolve_rules.restype = ctypes.c_int
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _field_struct(field):
    keep = []
    F = _Field()
    kind = field["kind"]
    if kind == "const":
        F.kind, F.n, F.a0 = 0, 0, field["a"]
    elif kind == "gauss":
        arrs = [np.ascontiguousarray(field[k], np.float64) for k in ("a", "cx", "cy", "s")]
        keep += arrs
        F.kind, F.n = 1, arrs[0].size
        F.a, F.cx, F.cy, F.s = [a.ctypes.data for a in arrs]
    elif kind == "fourier":
        k1 = np.ascontiguousarray(field["k1"], np.int32)
        k2 = np.ascontiguousarray(field["k2"], np.int32)
        fa = np.ascontiguousarray(field["a"], np.float64)
        fb = np.ascontiguousarray(field["b"], np.float64)
        if k2.size and (k2.max() - k2.min() + 1) > 256:
            raise ValueError("fourier field too wide for the oracle's table")
        keep += [k1, k2, fa, fb]
        F.kind, F.n = 2, k1.size
        F.k1, F.k2, F.fa, F.fb = k1.ctypes.data, k2.ctypes.data, fa.ctypes.data, fb.ctypes.data
    else:
        raise ValueError(kind)
    return F, keep


def _opts(eta_far=0.0, eta_polar=0.0, nthreads=0, assume_resolved=False):
    return _Opts(eta_far, eta_polar, nthreads, 1 if assume_resolved else 0)


def volume_potential(tri, curved, circle, field, targets, eta_far=0.0, eta_polar=0.0, nthreads=0,
                     assume_resolved=False):
    """V*(targets) = sum over triangles of int_T G(x - y) f(y) dy (exact up to quadrature ~1e-13).
    assume_resolved: far field by the own 12-point rule on every triangle (skip the resolution ladder); valid
    only when resolve_rules() returns 0 for every triangle (checked on samples by the callers' tests)."""
    tri = np.ascontiguousarray(tri, np.float64)
    M = tri.shape[0]
    cur = np.ascontiguousarray(curved, np.int8) if curved is not None else None
    circ = np.ascontiguousarray(circle, np.float64) if circle is not None else None
    tg = np.ascontiguousarray(np.asarray(targets, np.float64).reshape(-1, 2))
    out = np.empty(tg.shape[0])
    F, keep = _field_struct(field)
    rc = lib().orc_volume_potential(M, _ptr(tri), _ptr(cur), _ptr(circ), ctypes.byref(F), tg.shape[0], _ptr(tg),
                                    _ptr(out), ctypes.byref(_opts(eta_far, eta_polar, nthreads, assume_resolved)))
    if rc != 0:
        raise RuntimeError(f"oracle failed rc={rc}")
    return out


class Prepared:
    """A triangulation prepared once (per-triangle far-field rules, CSR of weighted points); eval(targets) then
    costs only the per-target sums.  Same code path as volume_potential (which is prepare + eval + free)."""

    def __init__(self, w, **kw):
        if w.field["kind"] == "fourier":
            kw.setdefault("assume_resolved", True)
        self._keep = [np.ascontiguousarray(w.tri, np.float64),
                      np.ascontiguousarray(w.curved, np.int8) if w.curved is not None else None,
                      np.ascontiguousarray(w.circle, np.float64) if w.circle is not None else None]
        self._F, self._fk = _field_struct(w.field)
        self.h = lib().orc_prepare(self._keep[0].shape[0], _ptr(self._keep[0]), _ptr(self._keep[1]),
                                   _ptr(self._keep[2]), ctypes.byref(self._F), ctypes.byref(_opts(**kw)))
        if not self.h:
            raise RuntimeError("oracle prepare failed (out of host memory)")

    def eval(self, targets):
        tg = np.ascontiguousarray(np.asarray(targets, np.float64).reshape(-1, 2))
        out = np.empty(tg.shape[0])
        lib().orc_eval_prepared(self.h, tg.shape[0], _ptr(tg), _ptr(out))
        return out

    def close(self):
        if self.h:
            lib().orc_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


def field_values(field, xy):
    """The oracle's own evaluation of an analytic field spec at points xy [n, 2] (for pins)."""
    xy = np.ascontiguousarray(np.asarray(xy, np.float64).reshape(-1, 2))
    out = np.empty(xy.shape[0])
    F, keep = _field_struct(field)
    lib().orc_field_values(ctypes.byref(F), xy.shape[0], _ptr(xy), _ptr(out))
    return out


def workload_potential(w, target_idx=None, **kw):
    """Oracle V* for a workloads.configs.Workload at targets[target_idx] (all if None).
    Fourier fields (config 4) use assume_resolved (pinned by tests/test_oracle.py::test_fourier_field_resolved)."""
    tg = w.targets if target_idx is None else w.targets[target_idx]
    if w.field["kind"] == "fourier":
        kw.setdefault("assume_resolved", True)
    return volume_potential(w.tri, w.curved, w.circle, w.field, tg, **kw)


def resolve_rules(tri, field, curved=None, circle=None):
    """Per-triangle far-field rule the oracle's resolution ladder picks (0 = own 12-point rule)."""
    tri = np.ascontiguousarray(tri, np.float64)
    M = tri.shape[0]
    cur = np.ascontiguousarray(curved, np.int8) if curved is not None else None
    circ = np.ascontiguousarray(circle, np.float64) if circle is not None else None
    out = np.empty(M, np.int32)
    F, keep = _field_struct(field)
    lib().orc_resolve_rules(M, _ptr(tri), _ptr(cur), _ptr(circ), ctypes.byref(F), _ptr(out))
    return out


def triangle_integral(tri3, field, target, curved=0, circle=None, eta_far=0.0, eta_polar=0.0):
    t = np.ascontiguousarray(tri3, np.float64).reshape(3, 2)
    circ = np.ascontiguousarray(circle, np.float64) if circle is not None else None
    F, keep = _field_struct(field)
    return lib().orc_triangle_integral(_ptr(t), int(curved), _ptr(circ), ctypes.byref(F), float(target[0]),
                                       float(target[1]), ctypes.byref(_opts(eta_far, eta_polar, 0)))


def rule12_nodes(tri, curved=None, circle=None):
    tri = np.ascontiguousarray(tri, np.float64)
    M = tri.shape[0]
    cur = np.ascontiguousarray(curved, np.int8) if curved is not None else None
    circ = np.ascontiguousarray(circle, np.float64) if circle is not None else None
    nodes = np.empty((M, 12, 2))
    w = np.empty((M, 12))
    lib().orc_rule12_nodes(M, _ptr(tri), _ptr(cur), _ptr(circ), _ptr(nodes), _ptr(w))
    return nodes, w


def e1(x):
    return np.vectorize(lib().orc_e1)(np.asarray(x, float))


def GH(r2, delta):
    return np.vectorize(lambda r: lib().orc_GH(r, delta))(np.asarray(r2, float))


def WR(k, R):
    return np.vectorize(lambda kk: lib().orc_WR(kk, R))(np.asarray(k, float))


def smooth_direct(src, c, targets, delta):
    src = np.ascontiguousarray(np.asarray(src, np.float64).reshape(-1, 2))
    c = np.ascontiguousarray(np.asarray(c, np.float64).ravel())
    tg = np.ascontiguousarray(np.asarray(targets, np.float64).reshape(-1, 2))
    out = np.empty(tg.shape[0])
    lib().orc_smooth_direct(src.shape[0], _ptr(src), _ptr(c), tg.shape[0], _ptr(tg), float(delta), _ptr(out))
    return out


def smooth_dft(src, c, targets, d1, d2, L_nh, n_nh, L_fh, n_fh, R, x0=0.0, y0=0.0):
    src = np.ascontiguousarray(np.asarray(src, np.float64).reshape(-1, 2))
    c = np.ascontiguousarray(np.asarray(c, np.float64).ravel())
    tg = np.ascontiguousarray(np.asarray(targets, np.float64).reshape(-1, 2))
    out = np.empty(tg.shape[0])
    lib().orc_smooth_dft(src.shape[0], _ptr(src), _ptr(c), tg.shape[0], _ptr(tg), float(d1), float(d2),
                         float(L_nh), int(n_nh), float(L_fh), int(n_fh), float(R), float(x0), float(y0), _ptr(out))
    return out


def dft_params(src, targets, d1, d2, eps):
    """The oracle's own period/cutoff choice for smooth_dft (readings R2-R3):
    k_max = sqrt(ln(1/eps)/delta); L_NH = S + sqrt(4 d2 z) with E1(z) = eps;
    R = sqrt(2) S + sqrt(4 d2 ln(1/eps)); L_FH = S + R + sqrt(4 d2 ln(1/eps)); n = ceil(L k_max / pi) (even)."""
    pts = np.concatenate([np.reshape(src, (-1, 2)), np.reshape(targets, (-1, 2))])
    lo, hi = pts.min(0), pts.max(0)
    S = float((hi - lo).max())
    x0, y0 = (lo + hi) / 2
    lne = np.log(1.0 / eps)
    z = lne
    for _ in range(100):   # solve E1(z) = eps by Newton (E1'(z) = -e^{-z}/z)
        z = z + (lib().orc_e1(z) - eps) / (np.exp(-z) / z)
    L_nh = S + np.sqrt(4 * d2 * z)
    R = np.sqrt(2) * S + np.sqrt(4 * d2 * lne)
    L_fh = S + R + np.sqrt(4 * d2 * lne)
    n_nh = int(np.ceil(L_nh * np.sqrt(lne / d1) / np.pi))
    n_fh = int(np.ceil(L_fh * np.sqrt(lne / d2) / np.pi))
    n_nh += n_nh & 1
    n_fh += n_fh & 1
    return dict(L_nh=L_nh, n_nh=n_nh, L_fh=L_fh, n_fh=n_fh, R=R, x0=x0, y0=y0)


def num_threads():
    return lib().orc_num_threads()
