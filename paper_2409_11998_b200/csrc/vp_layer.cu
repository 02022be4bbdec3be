// vp_layer.cu -- the layer potentials S[sigma] and D[mu] on the volume plan's grids.
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
//
//   D[mu](x) = int_Gamma dG(x - y)/dnu_y mu(y) ds_y = D_L + D_NH + D_FH, nu the OUTWARD normal  (lines 511-521,
//                                                                                     eq. dheatdecomp; line 86)
// History (lemmas dnearkspace / dfarkspace, lines 522-553): the multiplier of S times i k . nu-hat, i.e. the
// history of the point sources mu_j nu_j W_j differentiated once.  Reading R20: with the transform convention of
// the lemma (sigma-hat(k) = int sigma e^{-i k.x} ds) d/dnu_{x'} of e^{i k.(x - x')} is -i k.nu, not the printed
// +i k.nu (the printed sign fails the unit-circle closed forms).  Built as: spread mu nu_1 W and mu nu_2 W onto
// the NH grid (two passes of the volume spreader) and restrict each to the FH grid, take the spectral derivative
// -(d_1 g_1 + d_2 g_2) on each grid's own DFT (cuFFT D2Z, k_dlp_combine, Z2D), then the volume path's transforms,
// multipliers, prolongation and interpolation unchanged (the multipliers are diagonal in the same DFT bases, so
// this IS the -i k multiplier).
// Local part (Lemma dlp, eq. dlplocO5) as printed, in the frame whose eta axis is the OUTWARD
// normal and sgn = +1 on the exterior side (reading R21; checked against the oracle minus the direct history sum in
// tests/test_layer.py), with the density's xi-derivatives (orders 1, 2, 4) by Faa di Bruno from the chunk parameter.
#include <cub/cub.cuh>
#include <cufft.h>

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

// closest point and tangent-line jets of a near target (the curve over its tangent line at
// b, eta(xi) along the INWARD normal N; density derivatives along xi through u(xi) = s - s_b)
struct LayerFrame {
  int64_t c;               // closest chunk (-1: none within reach)
  double r, side;          // distance to b, (x - b).N
  double b1, b2, b3, b4;   // u(xi) = b1 xi + b2 xi^2 + b3 xi^3 + b4 xi^4 (series reversion of xi(u))
  double kap, gam3, gam4;  // eta'', eta''', eta'''' at b (inward frame)
  double Lk[5][VP_CHUNK_MAXQ + 1];  // d^k/ds^k of the chunk's Lagrange basis at s_b, k = 0..4
};

__device__ static void layer_frame(const VpBdryDev &B, const double *__restrict__ swt, double x, double y, double reach,
                                   LayerFrame &F) {
  const int qp = B.q + 1;
  F.c = -1;
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
  for (int k = 0; k < 5; k++)
    for (int j = 0; j < qp; j++) F.Lk[k][j] = 0.0;
  // L_j(s) = sum_m (2m+1)/2 w_j P_m(s_j) P_m(s) (exact for the degree-q interpolant at the Gauss-Legendre nodes)
  double Pj0[VP_CHUNK_MAXQ + 1], Pj1[VP_CHUNK_MAXQ + 1];  // P_{m-1}(s_j), P_m(s_j)
  for (int j = 0; j < qp; j++) {
    Pj0[j] = 0.0;
    Pj1[j] = 1.0;
  }
  for (int m = 0; m <= B.q; m++) {
    if (m > 0) {
      for (int k = 0; k <= 4; k++) {
        g[k][0] = fma(cf[2 * m], Pm[k], g[k][0]);
        g[k][1] = fma(cf[2 * m + 1], Pm[k], g[k][1]);
      }
    }
    for (int j = 0; j < qp; j++) {
      const double f = 0.5 * (2 * m + 1) * swt[j] * Pj1[j];
      for (int k = 0; k <= 4; k++) F.Lk[k][j] = fma(f, Pm[k], F.Lk[k][j]);
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
  const double a1 = sp, a2 = (g[2][0] * Tx + g[2][1] * Ty) / 2, a3 = (g[3][0] * Tx + g[3][1] * Ty) / 6,
               a4 = (g[4][0] * Tx + g[4][1] * Ty) / 24;
  const double e2 = (g[2][0] * Nx + g[2][1] * Ny) / 2, e3 = (g[3][0] * Nx + g[3][1] * Ny) / 6,
               e4 = (g[4][0] * Nx + g[4][1] * Ny) / 24;
  // series reversion of xi(u) = a1 u + a2 u^2 + a3 u^3 + a4 u^4
  const double ia = 1.0 / a1, ia3 = ia * ia * ia;
  F.b1 = ia;
  F.b2 = -a2 * ia3;
  F.b3 = (2 * a2 * a2 - a1 * a3) * ia3 * ia * ia;
  F.b4 = (5 * a1 * a2 * a3 - a1 * a1 * a4 - 5 * a2 * a2 * a2) * ia3 * ia3 * ia;
  const double b1 = F.b1, b2 = F.b2, b3 = F.b3;
  F.kap = 2 * e2 * b1 * b1;
  F.gam3 = 6 * (2 * e2 * b1 * b2 + e3 * b1 * b1 * b1);
  F.gam4 = 24 * (e2 * (b2 * b2 + 2 * b1 * b3) + 3 * e3 * b1 * b1 * b2 + e4 * b1 * b1 * b1 * b1);
  F.side = (x - g[0][0]) * Nx + (y - g[0][1]) * Ny;
  F.r = r;
  F.c = c;
}

// asymptotic local-part weights over the closest chunk's q + 1 nodal densities at short-time cutoff delta
// S (eq. slplocO5, reading R19):  S_L = -[A0 sigma + A1 sigma_1 + A2 sigma_2]  (sigma_k: k-th derivative along xi)
__device__ static void slp_asym_weights(const LayerFrame &F, double delta, int qp, double *__restrict__ w) {
  const double kap = F.kap, gam3 = F.gam3, gam4 = F.gam4, b1 = F.b1, b2 = F.b2;
  const double sg = F.side > 0 ? 1.0 : (F.side < 0 ? -1.0 : 0.0);
  const double sd = sqrt(delta), cc = F.r / sd;
  const double ex = exp(-0.25 * cc * cc) / sqrt(VP_PI), er = erfc(0.5 * cc);
  const double F1 = cc * er - 2 * ex, F2 = 2 * cc * cc * cc * er - (4 * cc * cc + 1) * ex,
               F3 = 3 * cc * cc * cc * er - (6 * cc * cc - 2) * ex, F4 = 2 * (cc * cc - 2) * ex - cc * cc * cc * er;
  const double d32 = delta * sd, d2 = delta * delta;
  const double A0 = 0.5 * sd * F1 + sg * delta * cc * kap / 4 * F1 + d32 * kap * kap / 12 * F2 +
                    d2 * sg * (cc * kap * kap * kap / 16 * F3 + cc * gam4 / 48 * F4);
  const double A1 = d2 * sg * cc * gam3 / 12 * F4;
  const double A2 = d32 / 12 * F4 + d2 * sg * cc * kap / 8 * F4;
  // sigma(xi) = sigma(s_b + u(xi)):  sigma_1 = b1 sigma_s, sigma_2 = 2 b2 sigma_s + b1^2 sigma_ss
  for (int j = 0; j < qp; j++)
    w[j] -= A0 * F.Lk[0][j] + A1 * b1 * F.Lk[1][j] + A2 * (2 * b2 * F.Lk[1][j] + b1 * b1 * F.Lk[2][j]);
}

// D (eq. dlplocO5 in the outward frame, reading R21: eta along nu = -N, so kappa, gamma3, gamma4 and the side
// change sign): D_L = B0 mu + B1 mu_1 + B2 mu_2 + B4 mu_4 with the xi-derivatives by Faa di Bruno
//   mu_1 = b1 mu_s, mu_2 = 2 b2 mu_s + b1^2 mu_ss,
//   mu_4 = 24 b4 mu_s + (24 b1 b3 + 12 b2^2) mu_ss + 12 b1^2 b2 mu_sss + b1^4 mu_ssss
__device__ static void dlp_asym_weights(const LayerFrame &F, double delta, int qp, double *__restrict__ w) {
  const double kap = -F.kap, g3 = -F.gam3, g4 = -F.gam4, b1 = F.b1, b2 = F.b2, b3 = F.b3, b4 = F.b4;
  const double sd = sqrt(delta), c = F.r / sd;
  // +1 outside; a target within 1e-10 sqrt(delta) of Gamma counts as ON it (sgn = 0: the direct value D(b), the
  // corollary's eq. dlplocO5onsurf) -- the leading term sgn mu/2 erfc(c/2) jumps there (reading R21)
  const double sg = c < 1e-10 ? 0.0 : (F.side < 0 ? 1.0 : -1.0);
  const double E = exp(-0.25 * c * c) / sqrt(VP_PI), er = erfc(0.5 * c);
  const double c2 = c * c, c3 = c2 * c, d32 = delta * sd, d2 = delta * delta;
  const double G1 = 2 * (c2 + 1) * E - c3 * er, G4 = 2 * (c2 + 4) * E - c3 * er;
  const double k2 = kap * kap;
  const double B0 = sg * 0.5 * er + sd * kap * 0.5 * E + delta * sg * 3 * c * k2 / 8 * E +
                    d32 * (5 * (c2 - 2) * k2 * kap / 16 * E + g4 / 4 * E) +
                    d2 * sg * (35 * c * k2 * k2 * (c2 - 6) / 128 * E + 5 * c * g3 * g3 / 12 * E + 5 * c * kap * g4 / 8 * E);
  const double B1 = d32 * g3 / 12 * G4 + d2 * sg * 5 * c * kap * g3 / 24 * G4;
  const double B2 = delta * sg * c / 4 * (2 * E - c * er) + d32 * kap / 4 * G1 + d2 * sg * 5 * c * k2 / 16 * G1;
  const double B4 = d2 * sg * c / 48 * (c3 * er - 2 * (c2 - 2) * E);
  const double b12 = b1 * b1;
  const double Ws = B1 * b1 + B2 * 2 * b2 + B4 * 24 * b4, Wss = B2 * b12 + B4 * (24 * b1 * b3 + 12 * b2 * b2),
               Wsss = B4 * 12 * b12 * b2, Wssss = B4 * b12 * b12;
  for (int j = 0; j < qp; j++)
    w[j] += B0 * F.Lk[0][j] + Ws * F.Lk[1][j] + Wss * F.Lk[2][j] + Wsss * F.Lk[3][j] + Wssss * F.Lk[4][j];
}

// chunks with a node within reach + gap of (x, y), unique, in bin order; returns the count (may exceed cap)
__device__ static int layer_near_chunks(const VpBdryDev &B, double x, double y, double reach, int cap,
                                        int32_t *__restrict__ ch) {
  const int qp = B.q + 1;
  const int64_t bx = (int64_t)floor((x - B.bx0) / B.bcell), by = (int64_t)floor((y - B.by0) / B.bcell);
  int n = 0;
  for (int64_t yy = by - 1; yy <= by + 1; yy++) {
    if (yy < 0 || yy >= B.nby) continue;
    for (int64_t xx = bx - 1; xx <= bx + 1; xx++) {
      if (xx < 0 || xx >= B.nbx) continue;
      const int64_t b = yy * B.nbx + xx;
      for (int32_t k = B.bstart[b]; k < B.bstart[b + 1]; k++) {
        const int64_t id = B.bidx[k];
        const double px = B.pts[2 * id] - x, py = B.pts[2 * id + 1] - y;
        if (sqrt(px * px + py * py) >= reach + B.gap) continue;
        const int32_t c = (int32_t)(id / qp);
        bool seen = false;
        for (int i = 0; i < min(n, cap); i++) seen |= ch[i] == c;
        if (seen) continue;
        if (n < cap) ch[n] = c;
        n++;
      }
    }
  }
  return n;
}

#define LAYER_NC_SCAN 64  // chunks per target the counting pass can tell apart

__global__ void k_layer_count(const int32_t *__restrict__ list, int64_t n, const double *__restrict__ tx,
                              const double *__restrict__ ty, VpBdryDev B, double reach, int32_t *__restrict__ maxnc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t ch[LAYER_NC_SCAN];
  const int64_t t = list[i];
  atomicMax(maxnc, layer_near_chunks(B, tx[t], ty[t], reach, LAYER_NC_SCAN, ch));
}

// Local-part stencil of one near target (§4.1 "s:dyadicref", lines 1181-1269): the asymptotic expansion at
// delta* = delta_1 / 4^J on the closest chunk plus the telescoped levels
//   sum_{j=1..J} int_Gamma K_j(x, y) dens(y) ds_y,   K_j = int_{delta_1/4^j}^{delta_1/4^{j-1}} (heat kernel) dt
// by direct smooth quadrature over every chunk within reach: the chunk parameter is cut into NP panels of 16
// Gauss-Legendre points (panel length <= 2.5 sqrt(delta*) / 1.5, tables Tq / Tq1 of the Lagrange basis and its
// derivative), so the sharpest level is resolved.  S: K_j = (1/4 pi) int over the level of e^{-rho^2/4t}/t dt by
// 12-point Gauss-Legendre in log t per level (the difference kernel (1/4 pi)[E1(4^{j-2} r) - E1(4^{j-1} r)] of the
// paper, r = rho^2 / delta_1, to 1e-14).  D: d/dnu_y of the same, summed over the levels in closed form,
//   (1/2 pi) (x - y).nu / rho^2 [e^{-rho^2/4 delta_1} - e^{-rho^2/4 delta*}].
template <int KIND>  // 0: S, 1: D
__global__ void k_layer_stencil(const int32_t *__restrict__ list, int64_t n, const double *__restrict__ tx,
                                const double *__restrict__ ty, VpBdryDev B, const double *__restrict__ swt,
                                double delta1, int J, double reach, int NC, int NP, const double *__restrict__ Tq,
                                const double *__restrict__ Tq1, const double *__restrict__ gw,
                                const double *__restrict__ lgx, const double *__restrict__ lgw,
                                int32_t *__restrict__ schunk, double *__restrict__ sw) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int qp = B.q + 1;
  const int64_t t = list[i];
  const double x = tx[t], y = ty[t];
  int32_t *ch = schunk + i * NC;
  double *w = sw + i * (int64_t)NC * qp;
  for (int k = 0; k < NC; k++) ch[k] = -1;
  for (int k = 0; k < NC * qp; k++) w[k] = 0.0;
  const int nc = min(layer_near_chunks(B, x, y, reach, NC, ch), NC);
  // asymptotic part at delta*
  const double dstar = ldexp(delta1, -2 * J);
  LayerFrame F;
  layer_frame(B, swt, x, y, reach, F);
  if (F.c >= 0) {
    int slot = -1;
    for (int k = 0; k < nc; k++)
      if (ch[k] == (int32_t)F.c) slot = k;
    if (slot >= 0) {
      if (KIND == 0)
        slp_asym_weights(F, dstar, qp, w + slot * qp);
      else
        dlp_asym_weights(F, dstar, qp, w + slot * qp);
    }
  }
  if (J == 0) return;
  // telescoped levels by direct quadrature
  const double a1 = 0.25 / delta1, as = 0.25 / dstar, reach2 = reach * reach;
  for (int k = 0; k < nc; k++) {
    const double *X = B.pts + (int64_t)ch[k] * qp * 2;
    double *wk = w + k * qp;
    for (int p = 0; p < NP; p++) {
      // panel test at its middle point: skip panels farther than reach + the panel's length
      {
        const double *T0 = Tq + (int64_t)(p * 16 + 8) * qp, *T1 = Tq1 + (int64_t)(p * 16 + 8) * qp;
        double gx = 0, gy = 0, dx = 0, dy = 0;
        for (int j = 0; j < qp; j++) {
          gx = fma(T0[j], X[2 * j], gx);
          gy = fma(T0[j], X[2 * j + 1], gy);
          dx = fma(T1[j], X[2 * j], dx);
          dy = fma(T1[j], X[2 * j + 1], dy);
        }
        const double half = 1.5 * hypot(dx, dy) / NP;  // |gamma'| x panel half-width (2 / NP / 2) x 1.5
        const double dd = hypot(gx - x, gy - y);
        if (dd > reach + half) continue;
      }
      for (int g = 0; g < 16; g++) {
        const int64_t pp = p * 16 + g;
        const double *T0 = Tq + pp * qp, *T1 = Tq1 + pp * qp;
        double gx = 0, gy = 0, dx = 0, dy = 0;
        for (int j = 0; j < qp; j++) {
          gx = fma(T0[j], X[2 * j], gx);
          gy = fma(T0[j], X[2 * j + 1], gy);
          dx = fma(T1[j], X[2 * j], dx);
          dy = fma(T1[j], X[2 * j + 1], dy);
        }
        const double rx = x - gx, ry = y - gy, r2 = rx * rx + ry * ry;
        if (r2 > reach2) continue;
        double kv;
        if (KIND == 0) {
          double s = 0.0;  // sum over levels of int e^{-r2/4t}/t dt = int e^{-(r2/4) e^{-u}} du, u = log t
          for (int l = 1; l <= J; l++) {
            const double ua = log(ldexp(delta1, -2 * l)), ub = log(ldexp(delta1, -2 * (l - 1)));
            const double hm = 0.5 * (ub - ua), um = 0.5 * (ub + ua);
            for (int m = 0; m < 12; m++) s = fma(hm * lgw[m], exp(-0.25 * r2 * exp(-(um + hm * lgx[m]))), s);
          }
          kv = s / (4.0 * VP_PI) * hypot(dx, dy);
        } else {
          // (x - y).nu |gamma'| = rx dy - ry dx;  e^{-a1 r2} - e^{-as r2} = -e^{-a1 r2} expm1(-(as - a1) r2)
          kv = r2 > 0.0 ? -(rx * dy - ry * dx) / r2 * exp(-a1 * r2) * expm1(-(as - a1) * r2) / (2.0 * VP_PI) : 0.0;
        }
        const double wq = kv * gw[pp];
        for (int j = 0; j < qp; j++) wk[j] = fma(wq, T0[j], wk[j]);
      }
    }
  }
}

// eval: out[user index of target] += sum over the target's NC chunk slots of sum_k w[k] dens[chunk][k]
__global__ void k_layer_local(const int32_t *__restrict__ list, const int32_t *__restrict__ schunk,
                              const double *__restrict__ sw, int64_t n, int NC, int qp, const int32_t *__restrict__ tperm,
                              const double *__restrict__ dens, double *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int k = 0; k < NC; k++) {
    const int32_t c = schunk[i * NC + k];
    if (c < 0) continue;
    const double *w = sw + (i * NC + k) * qp, *s = dens + (int64_t)c * qp;
    for (int j = 0; j < qp; j++) acc = fma(w[j], s[j], acc);
  }
  out[tperm[list[i]]] += acc;
}

// boundary source nodes, weights W = w_k |gamma'(s_k)| and (dipole sets) W nu_1, W nu_2 with the OUTWARD normal
// nu = (y', -x') / |gamma'| of the counter-clockwise chunk (from the chunk Legendre coefficients)
__global__ void k_slp_sources(const double *__restrict__ coef, const double *__restrict__ snode,
                              const double *__restrict__ swt, int64_t n, int q, double *__restrict__ W,
                              double *__restrict__ Wx, double *__restrict__ Wy) {
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
  const double sp = hypot(gx, gy);
  if (W) W[id] = swt[k] * sp;
  if (Wx) Wx[id] = swt[k] * gy;   // W nu_1 = w |gamma'| y' / |gamma'|
  if (Wy) Wy[id] = -swt[k] * gx;  // W nu_2
}

void vp_build_strip_order(vp_plan_s *P, VpSpreadSet &S, const double *xy, const double *weights,
                          const int32_t *node_of, int64_t n, const GridArgs &g);

// shared by S and D: Gauss-Legendre weights of the chunk rule and the list of targets (sorted order) within
// 12 sqrt(delta_1) of the boundary
static void layer_common(vp_plan_s *P) {
  if (P->lay_common) return;
  const VpBdryDev &B = P->bdev;
  if (B.kind != VP_BDRY_CHUNKS) throw VpError{VP_ERR_UNSUPPORTED};
  cudaStream_t s = P->stream;
  const int qp = B.q + 1;
  std::vector<double> sn, swh;
  vp_gauss_legendre(qp, sn, swh);
  P->slp_swt = vp_alloc<double>(P, qp);
  VP_CUDA(cudaMemcpy(P->slp_swt, swh.data(), sizeof(double) * qp, cudaMemcpyHostToDevice));
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
  for (void *p : {(void *)flag, (void *)d_n, tmp}) VP_CUDA(cudaFreeAsync(p, s));
  P->slp_n = nn;
  P->slp_list = list;
  // chunk slots per near target (counting pass)
  int32_t *d_max = nullptr;
  VP_CUDA(cudaMallocAsync(&d_max, sizeof(int32_t), s));
  VP_CUDA(cudaMemsetAsync(d_max, 0, sizeof(int32_t), s));
  if (nn > 0) {
    k_layer_count<<<(unsigned)((nn + 127) / 128), 128, 0, s>>>(list, nn, P->tx, P->ty, B, reach, d_max);
    VP_CHECK_LAUNCH();
  }
  int32_t mx = 0;
  VP_CUDA(cudaMemcpyAsync(&mx, d_max, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  VP_CUDA(cudaStreamSynchronize(s));
  VP_CUDA(cudaFreeAsync(d_max, s));
  if (mx > LAYER_NC_SCAN) throw VpError{VP_ERR_UNSUPPORTED};  // chunks far shorter than sqrt(delta_1)
  P->lay_nc = std::max(mx, 1);
  // panels of the telescoped quadrature: 16-point Gauss-Legendre per panel, panel length <= 2.5 sqrt(delta*)/1.5
  const int J = P->lay_J;
  const double dstar = std::ldexp(P->delta1, -2 * J);
  const int NP = J == 0 ? 1 : (int)std::min<double>(4096.0, std::ceil(1.5 * B.len_max / (2.5 * std::sqrt(dstar))));
  P->lay_np = NP;
  std::vector<double> g16, w16, g12, w12;
  vp_gauss_legendre(16, g16, w16);
  vp_gauss_legendre(12, g12, w12);
  std::vector<double> tq((size_t)NP * 16 * qp), tq1((size_t)NP * 16 * qp), gw((size_t)NP * 16);
  for (int p = 0; p < NP; p++)
    for (int g = 0; g < 16; g++) {
      const size_t pp = (size_t)p * 16 + g;
      const double x = -1.0 + (p + 0.5 * (g16[g] + 1.0)) * 2.0 / NP;
      gw[pp] = w16[g] / NP;
      for (int j = 0; j < qp; j++) {  // Lagrange basis on the chunk nodes and its derivative (product rule)
        double L = 1.0, dL = 0.0;
        for (int m = 0; m < qp; m++) {
          if (m == j) continue;
          const double f = 1.0 / (sn[j] - sn[m]);
          dL = dL * (x - sn[m]) * f + L * f;
          L *= (x - sn[m]) * f;
        }
        tq[pp * qp + j] = L;
        tq1[pp * qp + j] = dL;
      }
    }
  P->lay_tq = vp_alloc<double>(P, tq.size());
  P->lay_tq1 = vp_alloc<double>(P, tq1.size());
  P->lay_gw = vp_alloc<double>(P, gw.size());
  P->lay_lg = vp_alloc<double>(P, 24);
  VP_CUDA(cudaMemcpy(P->lay_tq, tq.data(), sizeof(double) * tq.size(), cudaMemcpyHostToDevice));
  VP_CUDA(cudaMemcpy(P->lay_tq1, tq1.data(), sizeof(double) * tq1.size(), cudaMemcpyHostToDevice));
  VP_CUDA(cudaMemcpy(P->lay_gw, gw.data(), sizeof(double) * gw.size(), cudaMemcpyHostToDevice));
  VP_CUDA(cudaMemcpy(P->lay_lg, g12.data(), sizeof(double) * 12, cudaMemcpyHostToDevice));
  VP_CUDA(cudaMemcpy(P->lay_lg + 12, w12.data(), sizeof(double) * 12, cudaMemcpyHostToDevice));
  P->lay_common = true;
}

template <int KIND>
static void launch_layer_stencil(vp_plan_s *P, int32_t **chunk, double **w) {
  const int64_t nn = P->slp_n;
  const int qp = P->bdev.q + 1, NC = P->lay_nc;
  *chunk = vp_alloc<int32_t>(P, (size_t)std::max<int64_t>(nn, 1) * NC);
  *w = vp_alloc<double>(P, (size_t)std::max<int64_t>(nn, 1) * NC * qp);
  if (nn > 0) {
    k_layer_stencil<KIND><<<(unsigned)((nn + 63) / 64), 64, 0, P->stream>>>(
        P->slp_list, nn, P->tx, P->ty, P->bdev, P->slp_swt, P->delta1, P->lay_J, 12.0 * sqrt(P->delta1), NC,
        P->lay_np, P->lay_tq, P->lay_tq1, P->lay_gw, P->lay_lg, P->lay_lg + 12, *chunk, *w);
    VP_CHECK_LAUNCH();
  }
  VP_CUDA(cudaStreamSynchronize(P->stream));
}

void vp_slp_build(vp_plan_s *P) {
  if (P->slp_ready) return;
  layer_common(P);
  const VpBdryDev &B = P->bdev;
  cudaStream_t s = P->stream;
  const int qp = B.q + 1;
  const int64_t nb = B.n * qp;
  // boundary sources on the NH grid (strip order, like the volume nodes)
  double *W = nullptr;
  VP_CUDA(cudaMallocAsync(&W, sizeof(double) * nb, s));
  k_slp_sources<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(B.coef, B.snode, P->slp_swt, B.n, B.q, W, nullptr,
                                                             nullptr);
  VP_CHECK_LAUNCH();
  vp_build_strip_order(P, P->bsp, B.pts, W, nullptr, nb, grid_args(P->nh));
  VP_CUDA(cudaFreeAsync(W, s));
  launch_layer_stencil<0>(P, &P->slp_chunk, &P->slp_w);
  P->slp_ready = true;
}

void vp_dlp_build(vp_plan_s *P) {
  if (P->dlp_ready) return;
  layer_common(P);
  const VpBdryDev &B = P->bdev;
  cudaStream_t s = P->stream;
  const int qp = B.q + 1;
  const int64_t nb = B.n * qp;
  double *Wx = nullptr, *Wy = nullptr;
  VP_CUDA(cudaMallocAsync(&Wx, sizeof(double) * nb, s));
  VP_CUDA(cudaMallocAsync(&Wy, sizeof(double) * nb, s));
  P->lay_W = vp_alloc<double>(P, nb);  // W_j = w_k |gamma'(s_k)|: the boundary rule (D_E's int mu ds, BIE solves)
  k_slp_sources<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(B.coef, B.snode, P->slp_swt, B.n, B.q, P->lay_W, Wx,
                                                             Wy);
  VP_CHECK_LAUNCH();
  vp_build_strip_order(P, P->dsp1, B.pts, Wx, nullptr, nb, grid_args(P->nh));
  vp_build_strip_order(P, P->dsp2, B.pts, Wy, nullptr, nb, grid_args(P->nh));
  VP_CUDA(cudaFreeAsync(Wx, s));
  VP_CUDA(cudaFreeAsync(Wy, s));
  launch_layer_stencil<1>(P, &P->dlp_chunk, &P->dlp_w);
  // spectral derivatives on the NH and FH grids: two half spectra per grid, cuFFT D2Z / Z2D plans over the rows
  P->dlp_has_plans = true;  // free_plan destroys the handles that were created
  for (int gi = 0; gi < 2; gi++) {
    const VpGrid &G = gi == 0 ? P->nh : P->fh;
    const int64_t ncol = G.nf / 2 + 1;
    P->dlp_spec[gi] = (double2 *)vp_alloc<double>(P, (size_t)2 * 2 * G.nf * ncol);
    int n[2] = {(int)G.nf, (int)G.nf}, inem[2] = {(int)G.nf, (int)G.row}, onem[2] = {(int)G.nf, (int)ncol};
    VP_CUFFT(cufftPlanMany(&P->dlp_fwd[gi], 2, n, inem, 1, (int)(G.nf * G.row), onem, 1, (int)(G.nf * ncol),
                           CUFFT_D2Z, 1));
    VP_CUFFT(cufftPlanMany(&P->dlp_inv[gi], 2, n, onem, 1, (int)(G.nf * ncol), inem, 1, (int)(G.nf * G.row),
                           CUFFT_Z2D, 1));
  }
  VP_CUDA(cudaStreamSynchronize(s));
  P->dlp_ready = true;
}

// A <- -(i k_1 A + i k_2 B) / nf^2 on the half spectrum [nf][nf/2+1] (k = dk m, m the signed DFT index; the
// Nyquist row and column are zeroed -- the NH multiplier truncates at |m| <= nmode/2 < nf/2 anyway)
__global__ void k_dlp_combine(double2 *__restrict__ A, const double2 *__restrict__ Bs, int64_t nf, double dk,
                              double scale) {
  const int64_t ncol = nf / 2 + 1, total = nf * ncol;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = id / ncol, c = id - r * ncol;
    if (2 * r == nf || 2 * c == nf) {
      A[id] = make_double2(0.0, 0.0);
      continue;
    }
    const double k1 = dk * (double)c, k2 = dk * (double)(2 * r < nf ? r : r - nf);
    const double2 a = A[id], b = Bs[id];
    // -(i k1 a + i k2 b) = (k1 a.y + k2 b.y, -(k1 a.x + k2 b.x))
    A[id] = make_double2(scale * (k1 * a.y + k2 * b.y), -scale * (k1 * a.x + k2 * b.x));
  }
}



// the D history's source grids: NH <- -(d_1 g_1 + d_2 g_2), FH <- -(d_1 R g_1 + d_2 R g_2), g_i the NH spread of
// mu nu_i W, R the FH restriction, d_i the spectral derivative on the grid's own DFT.  Differentiating on each
// grid (rather than restricting the differentiated NH grid) keeps the restriction's aliased content from being
// amplified by |k'| / |k| at the low modes the far history is made of.
void vp_dlp_source_grids(vp_plan_s *P, const double *mu) {
  VpGrid *Gs[2] = {&P->nh, &P->fh};
  for (int gi = 0; gi < 2; gi++) {
    VP_CUFFT(cufftSetStream(P->dlp_fwd[gi], P->stream));
    VP_CUFFT(cufftSetStream(P->dlp_inv[gi], P->stream));
  }
  for (int i = 0; i < 2; i++) {
    VP_CUDA(cudaMemsetAsync(P->nh.data, 0, sizeof(double) * P->nh.nf * P->nh.row, P->stream));
    VP_CUDA(cudaMemsetAsync(P->fh.data, 0, sizeof(double) * P->fh.nf * P->fh.row, P->stream));
    VpSpreadSet S = i == 0 ? P->dsp1 : P->dsp2;
    S.fs_out = nullptr;
    vp_launch_spread(P, S, grid_args(P->nh), mu);
    vp_launch_restrict(P);
    for (int gi = 0; gi < 2; gi++) {
      const int64_t nc = Gs[gi]->nf * (Gs[gi]->nf / 2 + 1);
      VP_CUFFT(cufftExecD2Z(P->dlp_fwd[gi], Gs[gi]->data, (cufftDoubleComplex *)(P->dlp_spec[gi] + i * nc)));
    }
  }
  for (int gi = 0; gi < 2; gi++) {
    VpGrid &G = *Gs[gi];
    const int64_t total = G.nf * (G.nf / 2 + 1);
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    k_dlp_combine<<<blocks, 256, 0, P->stream>>>(P->dlp_spec[gi], P->dlp_spec[gi] + total, G.nf, 2.0 * VP_PI / G.L,
                                                 1.0 / ((double)G.nf * (double)G.nf));
    VP_CHECK_LAUNCH();
    VP_CUFFT(cufftExecZ2D(P->dlp_inv[gi], (cufftDoubleComplex *)P->dlp_spec[gi], G.data));
  }
  P->n_ffts += 6;
  P->n_kernels += 2;
}

static void launch_layer_local(vp_plan_s *P, const int32_t *chunk, const double *w, const double *dens,
                               double *out) {
  if (P->slp_n == 0) return;
  k_layer_local<<<(unsigned)((P->slp_n + 255) / 256), 256, 0, P->stream>>>(P->slp_list, chunk, w, P->slp_n,
                                                                           P->lay_nc, P->bdev.q + 1, P->tperm, dens,
                                                                           out);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

void vp_launch_slp_local(vp_plan_s *P, const double *sigma, double *out) {
  launch_layer_local(P, P->slp_chunk, P->slp_w, sigma, out);
}

void vp_launch_dlp_local(vp_plan_s *P, const double *mu, double *out) {
  launch_layer_local(P, P->dlp_chunk, P->dlp_w, mu, out);
}
