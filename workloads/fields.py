"""Analytic source densities f for the synthetic workloads (input data).

Each field is a plain dict so it can be handed unchanged to the CPU oracle
(which evaluates f itself, in C, for its near-field refinement) and evaluated
here at the quadrature nodes for the GPU path.

kinds
  const   : f = a
  gauss   : f = sum_i a_i exp(-|x - c_i|^2 / s_i)          (s_i = width_i^2, SURVEY §8(c) reading 16)
  fourier : f = sum_k a_k cos(2 pi k.x) + b_k sin(2 pi k.x)  (k in Z^2, half plane)
"""
import numpy as np


def const(a=1.0):
    return {"kind": "const", "a": float(a)}


def gauss(a, cx, cy, s):
    return {"kind": "gauss", "a": np.asarray(a, float), "cx": np.asarray(cx, float),
            "cy": np.asarray(cy, float), "s": np.asarray(s, float)}


def fourier(k1, k2, a, b):
    return {"kind": "fourier", "k1": np.asarray(k1, np.int32), "k2": np.asarray(k2, np.int32),
            "a": np.asarray(a, float), "b": np.asarray(b, float)}


def random_fourier(rng, kmax=64):
    """Modes 0 < |k| <= kmax on the half plane, coefficients N(0,1)/(1+|k|^2)."""
    k1, k2 = np.meshgrid(np.arange(-kmax, kmax + 1), np.arange(-kmax, kmax + 1), indexing="ij")
    k1, k2 = k1.ravel(), k2.ravel()
    r2 = k1 * k1 + k2 * k2
    half = (k1 > 0) | ((k1 == 0) & (k2 > 0))
    keep = half & (r2 > 0) & (r2 <= kmax * kmax)
    k1, k2, r2 = k1[keep], k2[keep], r2[keep]
    a = rng.standard_normal(k1.size) / (1.0 + r2)
    b = rng.standard_normal(k1.size) / (1.0 + r2)
    return fourier(k1, k2, a, b)


def evaluate(field, x, y, device=None):
    """f at points (x, y) (numpy arrays of equal shape). Fourier fields use torch in chunks."""
    x = np.asarray(x, float)
    y = np.asarray(y, float)
    kind = field["kind"]
    if kind == "const":
        return np.full(x.shape, field["a"])
    if kind == "gauss" and x.size > 4_000_000:
        return _eval_gauss_torch(field, x, y, device)
    if kind == "gauss":
        out = np.zeros(x.shape)
        for a, cx, cy, s in zip(field["a"], field["cx"], field["cy"], field["s"]):
            out += a * np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / s)
        return out
    if kind == "fourier":
        return _eval_fourier(field, x, y, device)
    raise ValueError(kind)


def _eval_gauss_torch(field, x, y, device=None):
    import torch
    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    xs, ys = x.ravel(), y.ravel()
    out = np.empty(xs.size)
    step = 1 << 24
    for s0 in range(0, xs.size, step):
        xx = torch.from_numpy(xs[s0:s0 + step]).to(device)
        yy = torch.from_numpy(ys[s0:s0 + step]).to(device)
        acc = torch.zeros_like(xx)
        for a, cx, cy, s in zip(field["a"], field["cx"], field["cy"], field["s"]):
            acc += float(a) * torch.exp(-((xx - float(cx)) ** 2 + (yy - float(cy)) ** 2) / float(s))
        out[s0:s0 + step] = acc.cpu().numpy()
    return out.reshape(x.shape)


def _eval_fourier(field, x, y, device=None):
    import torch
    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    k1 = field["k1"].astype(np.int64)
    k2 = field["k2"].astype(np.int64)
    K1 = int(k1.max()) if k1.size else 0
    lo2, hi2 = int(k2.min()), int(k2.max())
    n2 = hi2 - lo2 + 1
    C = np.zeros((K1 + 1, n2), np.complex128)
    # f = Re sum (a - i b) e^{2 pi i k.x}
    np.add.at(C, (k1, k2 - lo2), field["a"] - 1j * field["b"])
    Ct = torch.from_numpy(C).to(device)
    xs, ys = x.ravel(), y.ravel()
    out = np.empty(xs.size)
    m1 = torch.arange(0, K1 + 1, device=device, dtype=torch.float64)
    m2 = torch.arange(lo2, hi2 + 1, device=device, dtype=torch.float64)
    step = 1 << 18
    for s0 in range(0, xs.size, step):
        xx = torch.from_numpy(xs[s0:s0 + step]).to(device)
        yy = torch.from_numpy(ys[s0:s0 + step]).to(device)
        E1 = torch.polar(torch.ones(1, device=device, dtype=torch.float64),
                         2 * np.pi * xx[:, None] * m1[None, :])          # (n, K1+1)
        E2 = torch.polar(torch.ones(1, device=device, dtype=torch.float64),
                         2 * np.pi * yy[:, None] * m2[None, :])          # (n, n2)
        inner = E2 @ Ct.T                                                # (n, K1+1)
        out[s0:s0 + step] = (E1 * inner).sum(dim=1).real.cpu().numpy()
    return out.reshape(x.shape)
