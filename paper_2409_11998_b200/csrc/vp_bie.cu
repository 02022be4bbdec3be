// vp_bie.cu -- boundary integral equations of the Poisson solve (§5 "s:bie", lines 1271-1330; SURVEY
// §8(f) f2) by restarted GMRES whose matrix-vector product is the GPU double-layer operator of vp_layer.cu.
//
//   interior Dirichlet (eq. dir_inteq):   -mu/2 + D[mu] = g - V[f]          on Gamma
//   exterior Dirichlet (eq. dir_repext):  +mu/2 + D_E[mu] = g - V[f] - A log|x - x0|,
//                                                          D_E[mu] = D[mu] + int_Gamma mu ds
//   interior Neumann (lines 1310-1318):                    u/2 + D[u] = V[f] + S[g]          (consistent, singular:
//                                                          constants span the null space)
// The paper solves these with GMRES + an FMM (lines 1319-1324); here the product D[mu] at the boundary nodes is
// vp_eval_dlp on a plan whose targets ARE the chunk nodes (the direct value at an on-curve target, reading R21),
// so every step of the product runs in this library's kernels.  GMRES(m) with classical Gram-Schmidt applied twice
// (CGS2): the k projections of one Arnoldi step are one multi-dot kernel + one multi-axpy kernel, partial sums per
// block reduced on the host in a fixed order (deterministic); the small Hessenberg least-squares problem (Givens
// rotations) is solved on the host.
#include <cmath>
#include <vector>

#include "vp_common.cuh"

// part[i * nb + b] = sum over block b's strided range of V[i][t] w[t], i < k
__global__ void k_bie_mdot(const double *__restrict__ V, int64_t ld, int k, const double *__restrict__ w, int64_t T,
                           double *__restrict__ part) {
  __shared__ double red[8][32];
  const int nb = gridDim.x;
  for (int i = 0; i < k; i++) {
    double acc = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)nb * blockDim.x)
      acc = fma(V[i * ld + t], w[t], acc);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][0] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); q++) s += red[q][0];
      part[i * nb + blockIdx.x] = s;
    }
    __syncthreads();
  }
}

// w[t] = a w[t] - sum_{i < k} h[i] V[i][t]   (h in device memory)
__global__ void k_bie_maxpy(double *__restrict__ w, double a, const double *__restrict__ V, int64_t ld, int k,
                            const double *__restrict__ h, int64_t T) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    double v = a * w[t];
    for (int i = 0; i < k; i++) v = fma(-h[i], V[i * ld + t], v);
    w[t] = v;
  }
}

// y += c x (+ s, a device scalar, when s != nullptr)
__global__ void k_bie_diag(double *__restrict__ y, const double *__restrict__ x, double c, const double *__restrict__ s,
                           int64_t T) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  y[t] = fma(c, x[t], y[t]) + (s ? s[0] : 0.0);
}

// max over user-order targets of the distance to the chunk node of the same index
__global__ void k_bie_check(const double *__restrict__ tx, const double *__restrict__ ty,
                            const int32_t *__restrict__ tperm, const double *__restrict__ pts, int64_t T,
                            unsigned long long *__restrict__ bad) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int64_t u = tperm[t];
  const double d = hypot(tx[t] - pts[2 * u], ty[t] - pts[2 * u + 1]);
  if (!(d <= 1e-12 * (1.0 + fabs(pts[2 * u]) + fabs(pts[2 * u + 1])))) atomicAdd(bad, 1ull);
}

namespace {
struct Bie {
  vp_plan_s *P;
  int kind;
  int64_t T;
  int nb;
  double *part, *hd, *sdev;
  std::vector<double> parth;
  cudaStream_t s;

  // A x -> y
  void apply(const double *x, double *y) {
    vp_status st = vp_eval_dlp(P, x, y);
    if (st != VP_OK) throw VpError{st};
    const unsigned g = (unsigned)((T + 255) / 256);
    if (kind == VP_BIE_DIRICHLET_EXT) {
      dots(P->lay_W, 0, 1, x);  // int mu ds = sum_j W_j mu_j
      VP_CUDA(cudaMemcpyAsync(sdev, parth.data(), sizeof(double), cudaMemcpyHostToDevice, s));
    }
    k_bie_diag<<<g, 256, 0, s>>>(y, x, kind == VP_BIE_DIRICHLET_INT ? -0.5 : 0.5,
                                 kind == VP_BIE_DIRICHLET_EXT ? sdev : nullptr, T);
    VP_CHECK_LAUNCH();
  }
  // parth[i] = <V_i, w>, i < k (V rows ld apart); synchronises
  void dots(const double *V, int64_t ld, int k, const double *w) {
    k_bie_mdot<<<nb, 256, 0, s>>>(V, ld, k, w, T, part);
    VP_CHECK_LAUNCH();
    std::vector<double> ph((size_t)k * nb);
    VP_CUDA(cudaMemcpyAsync(ph.data(), part, sizeof(double) * k * nb, cudaMemcpyDeviceToHost, s));
    VP_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < k; i++) {
      double a = 0.0;
      for (int b = 0; b < nb; b++) a += ph[(size_t)i * nb + b];
      parth[i] = a;
    }
  }
  double norm(const double *w) {
    dots(w, 0, 1, w);
    return std::sqrt(parth[0]);
  }
  // w <- a w - sum h_i V_i
  void maxpy(double *w, double a, const double *V, int64_t ld, int k, const double *h) {
    VP_CUDA(cudaMemcpyAsync(hd, h, sizeof(double) * k, cudaMemcpyHostToDevice, s));
    k_bie_maxpy<<<nb, 256, 0, s>>>(w, a, V, ld, k, hd, T);
    VP_CHECK_LAUNCH();
  }
};
}  // namespace

extern "C" vp_status vp_bie_solve(vp_handle P, int32_t kind, const double *rhs, double *x, double tol, int32_t maxit,
                                  int32_t restart, int32_t *iters, double *resid) {
  if (!P || !rhs || !x || !(tol > 0) || maxit < 1 || restart < 1 || restart > 200) return VP_ERR_ARG;
  if (kind != VP_BIE_DIRICHLET_INT && kind != VP_BIE_DIRICHLET_EXT && kind != VP_BIE_NEUMANN_INT) return VP_ERR_ARG;
  std::vector<void *> tmp;
  cudaStream_t s = P->stream;
  try {
    if (!P->dlp_ready) throw VpError{VP_ERR_ARG};
    const int64_t T = P->T, qp = P->bdev.q + 1;
    if (T != P->bdev.n * qp) throw VpError{VP_ERR_ARG};
    auto dalloc = [&](size_t n) {
      void *p = nullptr;
      VP_CUDA(cudaMallocAsync(&p, n * sizeof(double), s));
      tmp.push_back(p);
      return (double *)p;
    };
    {  // the targets must be the chunk nodes, in the descriptor's order
      unsigned long long *bad = (unsigned long long *)dalloc(1), hbad = 0;
      VP_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), s));
      k_bie_check<<<(unsigned)((T + 255) / 256), 256, 0, s>>>(P->tx, P->ty, P->tperm, P->bdev.pts, T, bad);
      VP_CHECK_LAUNCH();
      VP_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, s));
      VP_CUDA(cudaStreamSynchronize(s));
      if (hbad) throw VpError{VP_ERR_ARG};
    }
    const int m = restart;
    Bie B{P, kind, T, (int)std::min<int64_t>(296, (T + 255) / 256), nullptr, nullptr, nullptr, {}, s};
    B.part = dalloc((size_t)(m + 1) * B.nb);
    B.hd = dalloc(m + 1);
    B.sdev = dalloc(1);
    B.parth.assign(m + 1, 0.0);
    double *V = dalloc((size_t)(m + 1) * T), *w = dalloc(T);
    const double bnorm = B.norm(rhs);
    int it = 0;
    double res = 0.0;
    VP_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * T, s));
    if (bnorm == 0.0) {
      if (iters) *iters = 0;
      if (resid) *resid = 0.0;
      for (void *p : tmp) cudaFreeAsync(p, s);
      VP_CUDA(cudaStreamSynchronize(s));
      return VP_OK;
    }
    std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m), h(m + 1);
    while (true) {
      // r = b - A x  into V_0
      B.apply(x, w);
      VP_CUDA(cudaMemcpyAsync(V, rhs, sizeof(double) * T, cudaMemcpyDeviceToDevice, s));
      const double one = 1.0;
      B.maxpy(V, 1.0, w, 0, 1, &one);
      const double beta = B.norm(V);
      res = beta / bnorm;
      if (res <= tol || it >= maxit) break;
      h[0] = 1.0 / beta;
      {
        const double zero = 0.0;  // V_0 /= beta: a w - 0 with a = 1/beta
        B.maxpy(V, h[0], V, 0, 0, &zero);
      }
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      int j = 0;
      for (; j < m && it < maxit; j++, it++) {
        double *vj1 = V + (size_t)(j + 1) * T;
        B.apply(V + (size_t)j * T, vj1);
        // CGS2: two passes of classical Gram-Schmidt against V_0..V_j
        for (int i = 0; i <= j; i++) H[(size_t)i * m + j] = 0.0;
        for (int pass = 0; pass < 2; pass++) {
          B.dots(V, T, j + 1, vj1);
          for (int i = 0; i <= j; i++) h[i] = B.parth[i];
          B.maxpy(vj1, 1.0, V, T, j + 1, h.data());
          for (int i = 0; i <= j; i++) H[(size_t)i * m + j] += h[i];
        }
        const double hn = B.norm(vj1);
        H[(size_t)(j + 1) * m + j] = hn;
        if (hn > 0) {
          const double zero = 0.0;
          B.maxpy(vj1, 1.0 / hn, V, 0, 0, &zero);
        }
        // Givens rotations on column j
        for (int i = 0; i < j; i++) {
          const double a = H[(size_t)i * m + j], b = H[(size_t)(i + 1) * m + j];
          H[(size_t)i * m + j] = cs[i] * a + sn[i] * b;
          H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * b;
        }
        const double a = H[(size_t)j * m + j], b = H[(size_t)(j + 1) * m + j], r = std::hypot(a, b);
        cs[j] = r > 0 ? a / r : 1.0;
        sn[j] = r > 0 ? b / r : 0.0;
        H[(size_t)j * m + j] = r;
        H[(size_t)(j + 1) * m + j] = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        res = std::fabs(g[j + 1]) / bnorm;
        if (res <= tol || hn == 0.0) {
          j++;
          it++;
          break;
        }
      }
      // y = R^{-1} g, x += V y
      for (int i = j - 1; i >= 0; i--) {
        double v = g[i];
        for (int k = i + 1; k < j; k++) v -= H[(size_t)i * m + k] * y[k];
        y[i] = H[(size_t)i * m + i] != 0.0 ? v / H[(size_t)i * m + i] : 0.0;
      }
      for (int i = 0; i < j; i++) h[i] = -y[i];
      B.maxpy(x, 1.0, V, T, j, h.data());
    }
    if (iters) *iters = it;
    if (resid) *resid = res;
    for (void *p : tmp) VP_CUDA(cudaFreeAsync(p, s));
    tmp.clear();
    VP_CUDA(cudaStreamSynchronize(s));
  } catch (VpError &e) {
    for (void *p : tmp) cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
    return e.s;
  }
  return VP_OK;
}
