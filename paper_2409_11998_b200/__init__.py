"""B200-native evaluator of the 2D Poisson volume potential (arXiv 2409.11998 hot path).

Thin ctypes binding over the C ABI of libvp.so (include/vp.h): argument marshalling only; every
step of the method runs in the library's sm_100a kernels (+ cuFFT).  torch is used for device
memory and streams.  There is no CPU fallback: if libvp.so is missing or CUDA is unavailable,
constructing a Plan raises.

    plan = Plan(nodes, weights, targets, tol, boundary=("rect", 0, 0, 1, 1), targets_are_nodes=True)
    V = plan.eval(f)          # torch cuda tensor [T]
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VP_LIB") or os.path.join(_HERE, "libvp.so")  # VP_LIB: A/B builds (scripts/r2)

VP_OK, VP_ERR_ARG, VP_ERR_TOL, VP_ERR_NONFINITE, VP_ERR_GEOMETRY, VP_ERR_UNSUPPORTED, VP_ERR_OOM, VP_ERR_CUDA, \
    VP_ERR_CUFFT = 0, -1, -2, -3, -4, -5, -6, -7, -8
BDRY = {None: 0, "none": 0, "circle": 1, "rect": 2, "polygon": 3, "chunks": 4}
DERIV = {"auto": 0, "knn": 1, "triangle": 2}
PART_HISTORY, PART_LOCAL, PART_ALL = 1, 2, 3
BIE_DIRICHLET_INT, BIE_DIRICHLET_EXT, BIE_NEUMANN_INT = 0, 1, 2  # vp.h VP_BIE_*

EXPORTED = ["vp_plan", "vp_eval", "vp_eval_host", "vp_eval_batch", "vp_destroy", "vp_strerror", "vp_get_info", "vp_set_profiling",
            "vp_get_phase_times", "vp_eval_launch_count", "vp_check_finite", "vp_last_error_detail", "vp_version",
            "vp_slp_prepare", "vp_eval_slp", "vp_dlp_prepare", "vp_eval_dlp",
            "vp_layer_set_levels", "vp_bie_solve", "vp_eval_host_many", "vp_struct_sizes"]


class VpBoundary(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("q", ctypes.c_int32), ("n", ctypes.c_int64), ("pts", ctypes.c_void_p),
                ("p", ctypes.c_double * 4)]


class VpOpts(ctypes.Structure):
    _fields_ = [("C", ctypes.c_double), ("delta2_over_delta1", ctypes.c_double),
                ("delta1_override", ctypes.c_double), ("eps_nufft", ctypes.c_double),
                ("series_order", ctypes.c_int32), ("deriv_mode", ctypes.c_int32),
                ("deriv_degree", ctypes.c_int32), ("deriv_k", ctypes.c_int32), ("parts", ctypes.c_int32),
                ("targets_are_nodes", ctypes.c_int32), ("boundary", VpBoundary), ("cuda_stream", ctypes.c_void_p),
                ("ref_nodes", ctypes.c_void_p), ("tri_max_aspect", ctypes.c_double), ("levels", ctypes.c_int32),
                ("level_cmin", ctypes.c_double), ("level_rho", ctypes.c_double), ("deterministic", ctypes.c_int32),
                ("spread_tile", ctypes.c_int32), ("interp_tile", ctypes.c_int32), ("fft_mode", ctypes.c_int32),
                ("spread_pack", ctypes.c_int32), ("fft_rows", ctypes.c_int32),
                ("batch_pair", ctypes.c_int32)]


class VpInfo(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int64), ("N", ctypes.c_int64), ("T", ctypes.c_int64),
                ("p", ctypes.c_int32), ("w_es", ctypes.c_int32), ("beta_es", ctypes.c_double),
                ("dx2", ctypes.c_double), ("delta1", ctypes.c_double), ("delta2", ctypes.c_double),
                ("kmax_nh", ctypes.c_double), ("kmax_fh", ctypes.c_double), ("L_nh", ctypes.c_double),
                ("L_fh", ctypes.c_double), ("R_trunc", ctypes.c_double), ("nf_nh", ctypes.c_int64),
                ("nf_fh", ctypes.c_int64), ("nmode_nh", ctypes.c_int64), ("nmode_fh", ctypes.c_int64),
                ("x0", ctypes.c_double), ("y0", ctypes.c_double), ("S", ctypes.c_double),
                ("deriv_mode", ctypes.c_int32), ("deriv_degree", ctypes.c_int32), ("deriv_k", ctypes.c_int32),
                ("n_boundary_targets", ctypes.c_int64), ("plan_ms", ctypes.c_double),
                ("device_bytes", ctypes.c_int64), ("n_stencil_targets", ctypes.c_int64),
                ("n_batches", ctypes.c_int64), ("horner_err", ctypes.c_double), ("n_levels", ctypes.c_int32),
                ("n_boxes", ctypes.c_int64), ("n_level_targets", ctypes.c_int64), ("n_band_pairs", ctypes.c_int64),
                ("nf_band", ctypes.c_int64), ("level_targets", ctypes.c_int64 * 16),
                ("fft_path_nh", ctypes.c_int32), ("fft_path_fh", ctypes.c_int32)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["level_targets"] = list(self.level_targets)
        return d


_lib = None


def lib():
    """Load libvp.so (raises if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2409_11998_b200.build` (or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.vp_plan.argtypes = [vp, vp, i64, i32, vp, i64, d, ctypes.POINTER(VpOpts), ctypes.POINTER(vp)]
        L.vp_eval.argtypes = [vp, vp, vp]
        L.vp_eval_host.argtypes = [vp, vp, vp]
        L.vp_eval_host_many.argtypes = [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(vp)]
        L.vp_eval_batch.argtypes = [vp, i32, vp, vp]
        L.vp_slp_prepare.argtypes = [vp]
        L.vp_eval_slp.argtypes = [vp, vp, vp]
        L.vp_dlp_prepare.argtypes = [vp]
        L.vp_layer_set_levels.argtypes = [vp, i32]
        L.vp_bie_solve.argtypes = [vp, i32, vp, vp, d, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(d)]
        L.vp_eval_dlp.argtypes = [vp, vp, vp]
        L.vp_destroy.argtypes = [vp]
        L.vp_strerror.argtypes = [ctypes.c_int]
        L.vp_strerror.restype = ctypes.c_char_p
        L.vp_get_info.argtypes = [vp, ctypes.POINTER(VpInfo)]
        L.vp_set_profiling.argtypes = [vp, i32]
        L.vp_get_phase_times.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32),
                                         ctypes.POINTER(ctypes.c_char_p)]
        L.vp_eval_launch_count.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]
        L.vp_check_finite.argtypes = [vp, vp]
        L.vp_last_error_detail.restype = ctypes.c_char_p
        L.vp_version.restype = ctypes.c_char_p
        for name in EXPORTED:
            L[name].restype = L[name].restype if name in ("vp_strerror", "vp_last_error_detail", "vp_version") else ctypes.c_int
        L.vp_debug_local_coef.argtypes = [ctypes.c_int, vp, d, d, d, ctypes.c_int, ctypes.c_int, vp]
        L.vp_debug_local_coef.restype = ctypes.c_int
        L.vp_debug_mult.argtypes = [ctypes.c_int, d, d, d]
        L.vp_debug_mult.restype = d
        L.vp_debug_e1.argtypes = [d]
        L.vp_debug_e1.restype = d
        L.vp_struct_sizes.argtypes = [ctypes.POINTER(ctypes.c_int64)]
        L.vp_struct_sizes.restype = ctypes.c_int
        sz = (ctypes.c_int64 * 3)()
        mine = (ctypes.sizeof(VpOpts), ctypes.sizeof(VpInfo), ctypes.sizeof(VpBoundary))
        if L.vp_struct_sizes(sz) != VP_OK or tuple(sz) != mine:
            raise RuntimeError(f"{LIB_PATH}: struct layout mismatch (library {tuple(sz)}, binding {mine}): "
                               "rebuild with `python -m paper_2409_11998_b200.build --force`")
        _lib = L
    return _lib


class VpError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        detail = lib().vp_last_error_detail().decode()
        super().__init__(f"{where}: {lib().vp_strerror(status).decode()} ({status}) {detail}")


def _check(status, where):
    if status != VP_OK:
        raise VpError(status, where)


def _dev_f64(t, shape_last=None):
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch tensor")
    if t.device.type != "cuda" or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError("expected a contiguous float64 CUDA tensor")
    return t


class Plan:
    """vp_plan / vp_eval / vp_destroy as a Python object (argument marshalling only)."""

    def __init__(self, tri_nodes, weights, targets, tol, *, C=0.0, delta2_over_delta1=0.0, delta1_override=0.0,
                 eps_nufft=0.0, series_order=0, deriv="auto", deriv_degree=0, deriv_k=0, parts=PART_ALL,
                 targets_are_nodes=False, boundary=None, stream=None, ref_nodes=None, tri_max_aspect=0.0, levels=0,
                 level_cmin=0.0, level_rho=0.0, deterministic=False, spread_tile=0, interp_tile=0, fft_mode=0,
                 spread_pack=0, fft_rows=0, batch_pair=0):
        import torch
        L = lib()
        tri_nodes = _dev_f64(tri_nodes)
        weights = _dev_f64(weights)
        targets = _dev_f64(targets)
        M, p = int(weights.shape[0]), int(weights.shape[1])
        if tri_nodes.numel() != 2 * M * p or targets.dim() != 2 or targets.shape[1] != 2:
            raise ValueError("shapes: tri_nodes [M,p,2], weights [M,p], targets [T,2]")
        T = int(targets.shape[0])
        o = VpOpts()
        o.C, o.delta2_over_delta1, o.delta1_override, o.eps_nufft = C, delta2_over_delta1, delta1_override, eps_nufft
        o.series_order, o.deriv_mode, o.deriv_degree, o.deriv_k = series_order, DERIV[deriv], deriv_degree, deriv_k
        o.parts, o.targets_are_nodes = parts, 1 if targets_are_nodes else 0
        if boundary is not None and boundary[0] not in (None, "none"):
            o.boundary.kind = BDRY[boundary[0]]
            if boundary[0] == "polygon":      # ("polygon", pts [n, 2])
                self._bpts = np.ascontiguousarray(boundary[1], np.float64).reshape(-1, 2)
                o.boundary.n, o.boundary.pts = self._bpts.shape[0], self._bpts.ctypes.data
            elif boundary[0] == "chunks":     # ("chunks", pts [n, q+1, 2])
                self._bpts = np.ascontiguousarray(boundary[1], np.float64)
                if self._bpts.ndim != 3 or self._bpts.shape[2] != 2:
                    raise ValueError("chunks boundary: pts must be [n, q+1, 2]")
                o.boundary.n, o.boundary.q = self._bpts.shape[0], self._bpts.shape[1] - 1
                o.boundary.pts = self._bpts.ctypes.data
            else:
                for i, v in enumerate(boundary[1:5]):
                    o.boundary.p[i] = float(v)
        if stream is None:
            stream = torch.cuda.current_stream()
        self.stream = stream
        o.cuda_stream = ctypes.c_void_p(stream.cuda_stream)
        if ref_nodes is not None:
            self._ref = np.ascontiguousarray(ref_nodes, dtype=np.float64).reshape(-1, 2)
            if self._ref.shape[0] != p:
                raise ValueError("ref_nodes must be [p, 2]")
            o.ref_nodes = self._ref.ctypes.data
        o.tri_max_aspect = tri_max_aspect
        o.levels, o.level_cmin, o.level_rho = levels, level_cmin, level_rho
        o.deterministic = 1 if deterministic else 0
        o.spread_tile, o.interp_tile, o.fft_mode = spread_tile, interp_tile, fft_mode
        o.spread_pack, o.fft_rows = spread_pack, fft_rows
        o.batch_pair = batch_pair
        h = ctypes.c_void_p()
        _check(L.vp_plan(tri_nodes.data_ptr(), weights.data_ptr(), M, p, targets.data_ptr(), T, float(tol),
                         ctypes.byref(o), ctypes.byref(h)), "vp_plan")
        self.h = h
        self.M, self.p, self.T, self.N = M, p, T, M * p
        # boundary chunk nodes (single-layer densities live there)
        self._bq = (int(self._bpts.shape[0]) * int(self._bpts.shape[1])
                    if boundary is not None and boundary[0] == "chunks" else None)

    def _out(self, out, n, dev, shape=None):
        import torch
        if out is None:
            return torch.empty(shape or (n,), dtype=torch.float64, device=dev)
        out = _dev_f64(out)
        if out.numel() != n or out.device != dev:
            raise ValueError(f"out must be a contiguous float64 tensor of {n} entries on {dev}")
        return out

    def eval(self, f, out=None):
        f = _dev_f64(f)
        if f.numel() != self.N:
            raise ValueError("f must have M*p entries")
        out = self._out(out, self.T, f.device)
        _check(lib().vp_eval(self.h, f.data_ptr(), out.data_ptr()), "vp_eval")
        return out

    def eval_batch(self, F, out=None):
        """K fields at once (C ABI vp_eval_batch): F [K, M, p] or [K, M*p] device fp64 -> [K, T]
        (a caller-supplied out must hold K*T contiguous float64 entries on F's device)."""
        F = _dev_f64(F)
        if F.numel() % self.N:
            raise ValueError("F must hold K x M*p entries")
        K = F.numel() // self.N
        if K < 1:
            raise ValueError("F must hold at least one field")
        out = self._out(out, K * self.T, F.device, (K, self.T))
        _check(lib().vp_eval_batch(self.h, K, F.data_ptr(), out.data_ptr()), "vp_eval_batch")
        return out

    def set_layer_levels(self, J):
        """Dyadic telescoping levels of the layer local parts (C ABI vp_layer_set_levels; before prepare_*)."""
        _check(lib().vp_layer_set_levels(self.h, int(J)), "vp_layer_set_levels")

    def prepare_slp(self):
        """Boundary sources and local stencils of the single-layer potential (C ABI vp_slp_prepare; the plan's
        boundary must be "chunks")."""
        _check(lib().vp_slp_prepare(self.h), "vp_slp_prepare")

    def eval_slp(self, sigma, out=None):
        """S[sigma] at the targets (C ABI vp_eval_slp): sigma [n_chunks, q+1] device fp64 at the chunk nodes."""
        sigma = _dev_f64(sigma)
        if self._bq is None or sigma.numel() != self._bq:
            raise ValueError("sigma must hold one value per boundary chunk node ([n, q+1]; plan with chunks)")
        out = self._out(out, self.T, sigma.device)
        _check(lib().vp_eval_slp(self.h, sigma.data_ptr(), out.data_ptr()), "vp_eval_slp")
        return out

    def prepare_dlp(self):
        """Dipole sources, local stencils and spectral-derivative buffers of the double-layer potential (C ABI
        vp_dlp_prepare; the plan's boundary must be "chunks")."""
        _check(lib().vp_dlp_prepare(self.h), "vp_dlp_prepare")

    def eval_dlp(self, mu, out=None):
        """D[mu] at the targets (C ABI vp_eval_dlp; outward normal): mu [n_chunks, q+1] device fp64 at the chunk
        nodes."""
        mu = _dev_f64(mu)
        if self._bq is None or mu.numel() != self._bq:
            raise ValueError("mu must hold one value per boundary chunk node ([n, q+1]; plan with chunks)")
        out = self._out(out, self.T, mu.device)
        _check(lib().vp_eval_dlp(self.h, mu.data_ptr(), out.data_ptr()), "vp_eval_dlp")
        return out

    def bie_solve(self, kind, rhs, tol=1e-12, maxit=200, restart=50, out=None):
        """GMRES solve of a boundary integral equation with the GPU double-layer operator (C ABI vp_bie_solve; the
        plan's targets are the chunk nodes, prepare_dlp() done).  kind: BIE_DIRICHLET_INT / BIE_DIRICHLET_EXT /
        BIE_NEUMANN_INT.  Returns (x [T] device, iterations, relative residual)."""
        rhs = _dev_f64(rhs)
        if rhs.numel() != self.T:
            raise ValueError("rhs must hold one value per target (= chunk node)")
        out = self._out(out, self.T, rhs.device)
        it, res = ctypes.c_int32(0), ctypes.c_double(0.0)
        _check(lib().vp_bie_solve(self.h, int(kind), rhs.data_ptr(), out.data_ptr(), float(tol), int(maxit),
                                  int(restart), ctypes.byref(it), ctypes.byref(res)), "vp_bie_solve")
        return out, it.value, res.value

    def eval_host(self, f_host, out_host=None):
        """f_host: numpy float64 (ideally pinned, e.g. torch pinned tensor .numpy()); returns numpy [T]."""
        f_host = np.ascontiguousarray(f_host, dtype=np.float64).reshape(-1)
        if f_host.size != self.N:
            raise ValueError("f_host must have M*p entries")
        if out_host is None:
            out_host = np.empty(self.T)
        if (not isinstance(out_host, np.ndarray) or out_host.dtype != np.float64 or out_host.size != self.T
                or not out_host.flags.c_contiguous or not out_host.flags.writeable):
            raise ValueError(f"out_host must be a writeable C-contiguous float64 array of {self.T} entries")
        _check(lib().vp_eval_host(self.h, f_host.ctypes.data, out_host.ctypes.data), "vp_eval_host")
        return out_host

    def eval_host_many(self, f_hosts, out_hosts):
        """K fields from host memory with overlapped transfers (C ABI vp_eval_host_many): f_hosts / out_hosts are
        lists of K float64 C-contiguous numpy arrays (pinned for the overlap) of N / T entries."""
        K = len(f_hosts)
        if K < 1 or len(out_hosts) != K:
            raise ValueError("need K >= 1 input and output arrays")
        for a, n, ro in [(a, self.N, True) for a in f_hosts] + [(a, self.T, False) for a in out_hosts]:
            if (not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.size != n or not a.flags.c_contiguous
                    or (not ro and not a.flags.writeable)):
                raise ValueError(f"host arrays must be C-contiguous float64 numpy arrays of {n} entries")
        fp = (ctypes.c_void_p * K)(*[a.ctypes.data for a in f_hosts])
        op = (ctypes.c_void_p * K)(*[a.ctypes.data for a in out_hosts])
        _check(lib().vp_eval_host_many(self.h, K, fp, op), "vp_eval_host_many")
        return out_hosts

    def check_finite(self, f):
        f = _dev_f64(f)
        return lib().vp_check_finite(self.h, f.data_ptr()) == VP_OK

    def info(self):
        I = VpInfo()
        _check(lib().vp_get_info(self.h, ctypes.byref(I)), "vp_get_info")
        return I.as_dict()

    def set_profiling(self, on=True):
        _check(lib().vp_set_profiling(self.h, 1 if on else 0), "vp_set_profiling")

    def phase_times(self):
        ms = (ctypes.c_double * 16)()
        names = (ctypes.c_char_p * 16)()
        n = ctypes.c_int32()
        _check(lib().vp_get_phase_times(self.h, ms, ctypes.byref(n), names), "vp_get_phase_times")
        return {names[i].decode(): ms[i] for i in range(n.value)}

    def launch_count(self):
        k, f = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().vp_eval_launch_count(self.h, ctypes.byref(k), ctypes.byref(f)), "vp_eval_launch_count")
        return k.value, f.value

    def destroy(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().vp_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def debug_local_coef(kind, bp, x, y, delta, nterms=3, deg=6):
    """Host evaluation of the local-part Taylor-coefficient weights (vp_math.cuh) for tests."""
    c = np.zeros(15)
    bpa = np.ascontiguousarray(bp, np.float64)
    b = lib().vp_debug_local_coef(BDRY[kind] if isinstance(kind, str) else kind, bpa.ctypes.data, x, y, delta,
                                  nterms, deg, c.ctypes.data)
    return bool(b), c


def debug_mult(kind, k2, a, b):
    return lib().vp_debug_mult(kind, k2, a, b)
