// vp_layer.cu -- the single-layer potential S[sigma] on the volume plan's grids (first part).
//
//   S[sigma](x) = int_Gamma G(x - y) sigma(y) ds_y = S_L + S_NH + S_FH              (PAPER.md lines 493-510,
//                                                                                     eq. sheatdecomp)
// History part (lemmas snearkspace / sfarkspace, lines 511-553): the same kernels as the volume history with
// point sources at the boundary's quadrature nodes y_j (the chunks' Gauss-Legendre nodes, PAPER.md lines
// 633-653) and strengths sigma_j W_j, W_j = w_k |gamma'(s_k)| -- spread onto the NH grid, restriction to FH,
// transforms with the same multipliers, prolongation, interpolation at the targets (history only).
// Local part (Lemma slp, eq. slplocO5): for targets within 12 sqrt(delta_1) of Gamma,
//   S_L(x) = -[ A0 sigma_b + A1 sigma'_b + A2 sigma''_b ]
//   A0 = sqrt(d)/2 F1 + sgn d c kappa/4 F1 + d^{3/2} kappa^2/12 F2 + d^2 sgn (c kappa^3/16 F3 + c gamma4/48 F4)
//   A1 = d^2 sgn c gamma3/12 F4,   A2 = d^{3/2}/12 F4 + d^2 sgn c kappa/8 F4
//   F1 = c erfc(c/2) - 2 e^{-c^2/4}/sqrt(pi), F2 = 2c^3 erfc - (4c^2+1) e/sqrt(pi), F3 = 3c^3 erfc - (6c^2-2) e/sqrt(pi),
//   F4 = 2(c^2-2) e/sqrt(pi) - c^3 erfc,
// with c = r / sqrt(delta_1), the curve written over its tangent line at the closest point b as eta(xi) along the
// INWARD normal (kappa = eta'', gamma3 = eta''', gamma4 = eta''''), sgn = +1 on the interior side, and the
// density derivatives along xi.  The overall minus sign is DESIGN.md reading R19: the printed formula's leading
// term at c = 0 is -sqrt(delta) sigma_b / sqrt(pi), but S_L = int_0^delta int K_t sigma ds dt is positive for
// sigma > 0 (checked against the oracle: tests/test_layer.py).  S_L is linear in the chunk's nodal densities, so
// plan time stores it as a (q+1)-entry stencil per near target (chunk index + weights); eval applies it.
#include <cub/cub.cuh>

#include <cmath>
#include <vector>

#include "vp_boundary.cuh"
#include "vp_common.cuh"

void vp_gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w);  // vp_api.cu, on [-1, 1]

// nearest chunk node of (x, y) in the boundary bins; -1 if none within reach + gap
__device__ static int64_t slp_nearest_node(const VpBdryDev &B, double x, double y, double reach) {
  const int64_t bx = (int64_t)floor((x - B.bx0) / B.bcell), by = (int64_t)floor((y - B.by0) / B.bcell);
  double dn = 1e300;
  int64_t nid = -1;
  for (int64_t yy = by - 1; yy <= by + 1; yy++) {
    if (yy < 0 || yy >= B.nby) continue;
    for (int64_t xx = bx - 1; xx <= bx + 1; xx++) {
      if (xx < 0 || xx >= B.nbx) continue;
      const int64_t b = yy * B.nbx + xx;
      for (int32_t k = B.bstart[b]; k < B.bstart[b + 1]; k++) {
        const int64_t id = B.bidx[k];
        const double px = B.pts[2 * id] - x, py = B.pts[2 * id + 1] - y;
        const double d = px * px + py * py;
        if (d < dn) {
          dn = d;
          nid = id;
        }
      }
    }
  }
  return (nid >= 0 && sqrt(dn) < reach + B.gap) ? nid : -1;
}

// pass 1: flag the targets (sorted order) within reach of Gamma
__global__ void k_slp_near(const double *__restrict__ tx, const double *__restrict__ ty, int64_t T, VpBdryDev B,
                           double reach, int32_t *__restrict__ flag) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  flag[t] = slp_nearest_node(B, tx[t], ty[t], reach) >= 0 ? 1 : 0;
}

// pass 2: closest point (nearest node + Newton), tangent-line jets and the stencil
// weights over the closest chunk's q + 1 nodal densities
__global__ void k_slp_stencil(const int32_t *__restrict__ list, int64_t n, const double *__restrict__ tx,
                              const double *__restrict__ ty, VpBdryDev B, const double *__restrict__ swt,
                              double delta, double reach, int32_t *__restrict__ schunk, double *__restrict__ sw) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t t = list[i];
  const double x = tx[t], y = ty[t];
  const int qp = B.q + 1;
  double *w = sw + i * qp;
  for (int k = 0; k < qp; k++) w[k] = 0.0;
  schunk[i] = -1;
  const int64_t nid = slp_nearest_node(B, x, y, reach);
  if (nid < 0) return;
  int64_t c;
  double sb, nx, ny, kap0;
  const double r = vp_chunk_closest(B, x, y, nid / qp, B.snode[nid % qp], &c, &sb, &nx, &ny, &kap0);
  if (r >= reach) return;
  // curve derivatives d^k gamma / ds^k (k = 0..4) at sb from the Legendre coefficients; Legendre derivatives by
  // (m+1) P_{m+1}^{(k)} = (2m+1)(s P_m^{(k)} + k P_m^{(k-1)}) - m P_{m-1}^{(k)}
  const double *cf = B.coef + c * (int64_t)qp * 2;
  double g[5][2] = {{cf[0], cf[1]}, {0, 0}, {0, 0}, {0, 0}, {0, 0}};
  double Pm[5] = {1, 0, 0, 0, 0}, Pp[5] = {0, 0, 0, 0, 0};  // P_m^{(k)}, P_{m-1}^{(k)} at sb
  double Lk[3][VP_CHUNK_MAXQ + 1];                          // Lagrange basis L_j^{(k)}(sb), k = 0..2
  for (int j = 0; j < qp; j++) Lk[0][j] = Lk[1][j] = Lk[2][j] = 0.0;
  // L_j(s) = sum_m (2m+1)/2 w_j P_m(s_j) P_m(s) (exact for the degree-q interpolant at the Gauss-Legendre nodes)
  double Pj0[VP_CHUNK_MAXQ + 1], Pj1[VP_CHUNK_MAXQ + 1];  // P_{m-1}(s_j), P_m(s_j)
  for (int j = 0; j < qp; j++) {
    Pj0[j] = 0.0;
    Pj1[j] = 1.0;
  }
  for (int m = 0; m <= B.q; m++) {
    if (m > 0) {
      for (int k = 1; k <= 4; k++) {
        g[k][0] = fma(cf[2 * m], Pm[k], g[k][0]);
        g[k][1] = fma(cf[2 * m + 1], Pm[k], g[k][1]);
      }
      g[0][0] = fma(cf[2 * m], Pm[0], g[0][0]);
      g[0][1] = fma(cf[2 * m + 1], Pm[0], g[0][1]);
    }
    for (int j = 0; j < qp; j++) {
      const double f = 0.5 * (2 * m + 1) * swt[j] * Pj1[j];
      Lk[0][j] = fma(f, Pm[0], Lk[0][j]);
      Lk[1][j] = fma(f, Pm[1], Lk[1][j]);
      Lk[2][j] = fma(f, Pm[2], Lk[2][j]);
    }
    // advance m -> m + 1
    double Pn[5];
    for (int k = 4; k >= 0; k--)
      Pn[k] = ((2 * m + 1) * (sb * Pm[k] + (k > 0 ? k * Pm[k - 1] : 0.0)) - m * Pp[k]) / (m + 1);
    for (int k = 0; k <= 4; k++) {
      Pp[k] = Pm[k];
      Pm[k] = Pn[k];
    }
    for (int j = 0; j < qp; j++) {
      const double pn = ((2 * m + 1) * B.snode[j] * Pj1[j] - m * Pj0[j]) / (m + 1);
      Pj0[j] = Pj1[j];
      Pj1[j] = pn;
    }
  }
  // frame at b: T along gamma' (counter-clockwise), N = inward normal; jets over the tangent line
  const double sp = hypot(g[1][0], g[1][1]);
  const double Tx = g[1][0] / sp, Ty = g[1][1] / sp, Nx = -Ty, Ny = Tx;
  const double a1 = sp, a2 = (g[2][0] * Tx + g[2][1] * Ty) / 2, a3 = (g[3][0] * Tx + g[3][1] * Ty) / 6;
  const double e2 = (g[2][0] * Nx + g[2][1] * Ny) / 2, e3 = (g[3][0] * Nx + g[3][1] * Ny) / 6,
               e4 = (g[4][0] * Nx + g[4][1] * Ny) / 24;
  // u(xi) = b1 xi + b2 xi^2 + b3 xi^3 (series reversion of xi(u) = a1 u + a2 u^2 + a3 u^3 + ...)
  const double b1 = 1.0 / a1, b2 = -a2 / (a1 * a1 * a1), b3 = (2 * a2 * a2 - a1 * a3) / (a1 * a1 * a1 * a1 * a1);
  const double kap = 2 * e2 * b1 * b1;
  const double gam3 = 6 * (2 * e2 * b1 * b2 + e3 * b1 * b1 * b1);
  const double gam4 = 24 * (e2 * (b2 * b2 + 2 * b1 * b3) + 3 * e3 * b1 * b1 * b2 + e4 * b1 * b1 * b1 * b1);
  const double side = (x - g[0][0]) * Nx + (y - g[0][1]) * Ny;
  const double sg = side > 0 ? 1.0 : (side < 0 ? -1.0 : 0.0);
  const double sd = sqrt(delta), cc = r / sd;
  const double ex = exp(-0.25 * cc * cc) / sqrt(VP_PI), er = erfc(0.5 * cc);
  const double F1 = cc * er - 2 * ex, F2 = 2 * cc * cc * cc * er - (4 * cc * cc + 1) * ex,
               F3 = 3 * cc * cc * cc * er - (6 * cc * cc - 2) * ex, F4 = 2 * (cc * cc - 2) * ex - cc * cc * cc * er;
  const double d32 = delta * sd, d2 = delta * delta;
  const double A0 = 0.5 * sd * F1 + sg * delta * cc * kap / 4 * F1 + d32 * kap * kap / 12 * F2 +
                    d2 * sg * (cc * kap * kap * kap / 16 * F3 + cc * gam4 / 48 * F4);
  const double A1 = d2 * sg * cc * gam3 / 12 * F4;
  const double A2 = d32 / 12 * F4 + d2 * sg * cc * kap / 8 * F4;
  // sigma(xi) = sigma(s_b + u(xi)):  sigma' = b1 sigma_s, sigma'' = 2 b2 sigma_s + b1^2 sigma_ss
  for (int j = 0; j < qp; j++)
    w[j] = -(A0 * Lk[0][j] + A1 * b1 * Lk[1][j] + A2 * (2 * b2 * Lk[1][j] + b1 * b1 * Lk[2][j]));
  schunk[i] = (int32_t)c;
}

// eval: out[user index of target] += sum_k w[k] sigma[chunk][k]
__global__ void k_slp_local(const int32_t *__restrict__ list, const int32_t *__restrict__ schunk,
                            const double *__restrict__ sw, int64_t n, int qp, const int32_t *__restrict__ tperm,
                            const double *__restrict__ sigma, double *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t c = schunk[i];
  if (c < 0) return;
  const double *w = sw + i * qp, *s = sigma + (int64_t)c * qp;
  double acc = 0.0;
  for (int k = 0; k < qp; k++) acc = fma(w[k], s[k], acc);
  out[tperm[list[i]]] += acc;
}

// boundary source nodes and weights W = w_k |gamma'(s_k)| (host, from the chunk Legendre coefficients)
__global__ void k_slp_sources(const double *__restrict__ coef, const double *__restrict__ pts,
                              const double *__restrict__ snode, const double *__restrict__ swt, int64_t n, int q,
                              double *__restrict__ W) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int qp = q + 1;
  if (id >= n * qp) return;
  const int64_t c = id / qp;
  const int k = (int)(id % qp);
  const double s = snode[k];
  const double *cf = coef + c * (int64_t)qp * 2;
  double P0 = 1.0, P1 = s, D0 = 0.0, D1 = 1.0, gx = 0.0, gy = 0.0;
  for (int m = 1; m <= q; m++) {
    gx = fma(cf[2 * m], D1, gx);
    gy = fma(cf[2 * m + 1], D1, gy);
    const double Pn = ((2 * m + 1) * s * P1 - m * P0) / (m + 1), Dn = D0 + (2 * m + 1) * P1;
    P0 = P1;
    P1 = Pn;
    D0 = D1;
    D1 = Dn;
  }
  (void)pts;
  W[id] = swt[k] * hypot(gx, gy);
}

void vp_build_strip_order(vp_plan_s *P, VpSpreadSet &S, const double *xy, const double *weights,
                          const int32_t *node_of, int64_t n, const GridArgs &g);

void vp_slp_build(vp_plan_s *P) {
  if (P->slp_ready) return;
  const VpBdryDev &B = P->bdev;
  if (B.kind != VP_BDRY_CHUNKS) throw VpError{VP_ERR_UNSUPPORTED};
  cudaStream_t s = P->stream;
  const int qp = B.q + 1;
  const int64_t nb = B.n * qp;
  std::vector<double> sn, swh;
  vp_gauss_legendre(qp, sn, swh);
  P->slp_swt = vp_alloc<double>(P, qp);
  VP_CUDA(cudaMemcpy(P->slp_swt, swh.data(), sizeof(double) * qp, cudaMemcpyHostToDevice));
  // boundary sources on the NH grid (strip order, like the volume nodes)
  double *W = nullptr;
  VP_CUDA(cudaMallocAsync(&W, sizeof(double) * nb, s));
  k_slp_sources<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(B.coef, B.pts, B.snode, P->slp_swt, B.n, B.q, W);
  VP_CHECK_LAUNCH();
  vp_build_strip_order(P, P->bsp, B.pts, W, nullptr, nb, grid_args(P->nh));
  VP_CUDA(cudaFreeAsync(W, s));
  // local stencils of the targets within reach
  const double reach = 12.0 * sqrt(P->delta1);
  int32_t *flag = nullptr, *d_n = nullptr, *list = nullptr;
  VP_CUDA(cudaMallocAsync(&flag, sizeof(int32_t) * (P->T + 1), s));
  VP_CUDA(cudaMallocAsync(&d_n, sizeof(int32_t), s));
  const unsigned nbT = (unsigned)((P->T + 255) / 256);
  k_slp_near<<<nbT, 256, 0, s>>>(P->tx, P->ty, P->T, B, reach, flag);
  VP_CHECK_LAUNCH();
  list = vp_alloc<int32_t>(P, P->T + 1);
  cub::CountingInputIterator<int32_t> cnt(0);
  size_t tb = 0;
  cub::DeviceSelect::Flagged(nullptr, tb, cnt, flag, list, d_n, (int)P->T, s);
  void *tmp = nullptr;
  VP_CUDA(cudaMallocAsync(&tmp, tb + 16, s));
  VP_CUDA(cub::DeviceSelect::Flagged(tmp, tb, cnt, flag, list, d_n, (int)P->T, s));
  int32_t nn = 0;
  VP_CUDA(cudaMemcpyAsync(&nn, d_n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  VP_CUDA(cudaStreamSynchronize(s));
  P->slp_n = nn;
  P->slp_list = list;
  P->slp_chunk = vp_alloc<int32_t>(P, std::max<int64_t>(nn, 1));
  P->slp_w = vp_alloc<double>(P, (size_t)std::max<int64_t>(nn, 1) * qp);
  if (nn > 0) {
    k_slp_stencil<<<(unsigned)((nn + 127) / 128), 128, 0, s>>>(list, nn, P->tx, P->ty, B, P->slp_swt, P->delta1,
                                                                reach, P->slp_chunk, P->slp_w);
    VP_CHECK_LAUNCH();
  }
  for (void *p : {(void *)flag, (void *)d_n, tmp}) VP_CUDA(cudaFreeAsync(p, s));
  VP_CUDA(cudaStreamSynchronize(s));
  P->slp_ready = true;
}

void vp_launch_slp_local(vp_plan_s *P, const double *sigma, double *out) {
  if (P->slp_n == 0) return;
  k_slp_local<<<(unsigned)((P->slp_n + 255) / 256), 256, 0, P->stream>>>(
      P->slp_list, P->slp_chunk, P->slp_w, P->slp_n, P->bdev.q + 1, P->tperm, sigma, out);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}
