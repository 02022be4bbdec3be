// vp_math.cuh -- scalar math of the method, usable on host and device (product path).
//
//  * ES spreading kernel psi(z) = exp(beta (sqrt(1 - z^2) - 1)), |z| < 1 (the "exponential of
//    semicircle" kernel named by BASELINE.json's north_star).
//  * Kernel-split Fourier multipliers (§2: near history (vnearkspace) line 385, far history
//    (vfarkspace)/(Wdef) lines 416-435 with a general truncation radius R, R2).
//  * Local-part coefficients: the Taylor coefficient weights of V_L for
//      - interior targets: sum_n delta^n Lap^{n-1} f / n!   (extended)
//      - near a circle: eq. (vplocO5) with the delta^{3/2} sign reading
//        (2 f_eta - kappa f) (R7), which reproduces the on-boundary corollary (lines 1122-1127)
//      - near an axis-aligned rectangle: exact product form int_0^delta M_a(x1,t) M_b(x2,t) dt
//        (R8; paper silent on corners).
#pragma once
#include <math.h>

#ifdef __CUDACC__
#define VP_HD __host__ __device__ __forceinline__
#else
#define VP_HD inline
#endif

#define VP_MAXDEG 6
#define VP_NTAYLOR 15  // Taylor coefficients a_{ab}, a + b <= 4

// monomial (a, b) of total degree d ordered (d, d-a): index of x^a y^b
VP_HD int vp_mono_index(int a, int b) {
  int d = a + b;
  return d * (d + 1) / 2 + (d - a);
}
VP_HD int vp_ncoef(int deg) { return (deg + 1) * (deg + 2) / 2; }

VP_HD double vp_es(double z, double beta) {
  double s = 1.0 - z * z;
  return s > 0.0 ? exp(beta * (sqrt(s) - 1.0)) : 0.0;
}

// ---------------------------------------------------------------- Fourier multipliers
// near history: (e^{-k^2 d1} - e^{-k^2 d2}) / k^2, limit d2 - d1 at k = 0 (PAPER.md (vnearkspace))
VP_HD double vp_mult_nh(double k2, double d1, double d2) {
  if (k2 == 0.0) return d2 - d1;
  return (expm1(-k2 * d1) - expm1(-k2 * d2)) / k2;
}
// far history: e^{-k^2 d2} W_R(k), W_R = (1 - J0(Rk))/k^2 - R log R J1(Rk)/k (PAPER.md (Wdef), general R)
VP_HD double vp_mult_fh(double k2, double d2, double R) {
  double k = sqrt(k2), z = R * k, W;
  if (z < 1e-3) {
    double z2 = z * z;
    W = R * R * (0.25 - z2 / 64.0 + z2 * z2 / 2304.0) - R * log(R) * R * (0.5 - z2 / 16.0 + z2 * z2 / 384.0);
  } else {
    W = (1.0 - j0(z)) / k2 - R * log(R) * j1(z) / k;
  }
  return exp(-k2 * d2) * W;
}

// ---------------------------------------------------------------- local part coefficients
// coef[vp_mono_index(a,b)] multiplies the Taylor coefficient a_{ab} of f at the target
// (f(x + z) = sum a_ab z1^a z2^b).  deg = degree available from the jet (terms above dropped).
VP_HD void vp_coef_clear(double *coef) {
  for (int i = 0; i < VP_NTAYLOR; i++) coef[i] = 0.0;
}

VP_HD void vp_coef_interior(double delta, int nterms, int deg, double *coef) {
  vp_coef_clear(coef);
  coef[vp_mono_index(0, 0)] = delta;
  if (nterms >= 2 && deg >= 2) {  // delta^2/2 Lap f, Lap f = 2 a20 + 2 a02
    coef[vp_mono_index(2, 0)] = delta * delta;
    coef[vp_mono_index(0, 2)] = delta * delta;
  }
  if (nterms >= 3 && deg >= 4) {  // delta^3/6 Lap^2 f, Lap^2 f = 24 a40 + 8 a22 + 24 a04
    double d3 = delta * delta * delta;
    coef[vp_mono_index(4, 0)] = 4.0 * d3;
    coef[vp_mono_index(2, 2)] = 4.0 * d3 / 3.0;
    coef[vp_mono_index(0, 4)] = 4.0 * d3;
  }
}

// eq. (vplocO5) in the frame of the closest boundary point b: r = |x - b| >= 0,
// (nx, ny) the inward unit normal at b, kap the curvature at b (> 0 convex).  The caller has checked
// r < 12 sqrt(delta).  Sign of the delta^{3/2} line: DESIGN.md R7.
VP_HD void vp_coef_smooth(double r, double nx, double ny, double kap, double delta, int nterms, int deg,
                          double *coef) {
  double sd = sqrt(delta);
  double c = r / sd;
  vp_coef_clear(coef);
  double tx = -ny, ty = nx;
  const double sp = 1.7724538509055160273;  // sqrt(pi)
  double E = exp(-c * c / 4.0), ec = erfc(c / 2.0), ef = erf(c / 2.0);
  double c2 = c * c, c4 = c2 * c2;
  double A0 = delta / 4.0 * (2.0 * ef + 2.0 * E * c / sp - c2 * ec + 2.0);
  double A1 = delta * sd * ((4.0 - 2.0 * c2) * E + sp * c2 * c * ec) / (12.0 * sp);
  double E2 = 2.0 * c * (c2 - 2.0) * E / sp;
  double q = delta * delta / 48.0;
  double cf = A0 - kap * A1 + q * (-3.0 * c4 * kap * kap * ec + 3.0 * kap * kap * E2);
  double cfe = 2.0 * A1 + q * (4.0 * c4 * kap * ec - 4.0 * kap * E2);
  double cfee = q * (-3.0 * (c4 + 4.0) * ec + 3.0 * E2 + 24.0);
  double cfxx = q * ((c4 - 12.0) * ec - E2 + 24.0);
  if (deg < 2) { cfee = 0.0; cfxx = 0.0; }
  coef[vp_mono_index(0, 0)] = cf;
  coef[vp_mono_index(1, 0)] = cfe * nx;
  coef[vp_mono_index(0, 1)] = cfe * ny;
  // f_ss along unit u: 2 a20 u1^2 + 2 a11' ... with a11 the xy coefficient: u^T H u, H = [[2a20, a11],[a11, 2a02]]
  coef[vp_mono_index(2, 0)] = 2.0 * (cfee * nx * nx + cfxx * tx * tx);
  coef[vp_mono_index(1, 1)] = 2.0 * (cfee * nx * ny + cfxx * tx * ty);
  coef[vp_mono_index(0, 2)] = 2.0 * (cfee * ny * ny + cfxx * ty * ty);
  if (nterms >= 3 && deg >= 4) {  // delta^3/6 Lap^2 f weighted by the boundary factor A0/delta
    double d3 = delta * delta * delta * (A0 / delta);
    coef[vp_mono_index(4, 0)] = 4.0 * d3;
    coef[vp_mono_index(2, 2)] = 4.0 * d3 / 3.0;
    coef[vp_mono_index(0, 4)] = 4.0 * d3;
  }
}

// near a circle of radius rho centred at (ccx, ccy); target inside at (x, y).
// Returns false if the target is farther than 12 sqrt(delta) (caller uses the interior form).
VP_HD bool vp_coef_circle(double x, double y, double ccx, double ccy, double rho, double delta, int nterms,
                          int deg, double *coef) {
  double dx = x - ccx, dy = y - ccy;
  double rr = sqrt(dx * dx + dy * dy);
  double r = rho - rr;
  if (r < 0.0) r = 0.0;
  if (r >= 12.0 * sqrt(delta)) return false;
  // inward normal n (towards the centre)
  double nx = rr > 0 ? -dx / rr : 1.0, ny = rr > 0 ? -dy / rr : 0.0;
  vp_coef_smooth(r, nx, ny, 1.0 / rho, delta, nterms, deg, coef);
  return true;
}

// 1D moments M_a(t) = int_lo^hi g_t(z) z^a dz, g_t = e^{-z^2/4t}/sqrt(4 pi t), a = 0..4
VP_HD void vp_moments(double lo, double hi, double t, double *Mo) {
  double st = sqrt(t);
  double inv = 1.0 / sqrt(4.0 * VP_PI * t);
  double glo = exp(-lo * lo / (4.0 * t)) * inv, ghi = exp(-hi * hi / (4.0 * t)) * inv;
  Mo[0] = 0.5 * (erf(hi / (2.0 * st)) - erf(lo / (2.0 * st)));
  Mo[1] = -2.0 * t * (ghi - glo);
  double plo = lo, phi = hi;  // z^{a-1} at the ends
  for (int a = 2; a <= 4; a++) {
    Mo[a] = -2.0 * t * (phi * ghi - plo * glo) + 2.0 * t * (a - 1) * Mo[a - 2];
    plo *= lo;
    phi *= hi;
  }
}

// Gauss-Legendre 12 nodes / weights on [0, 1]
VP_HD double vp_gl12_x(int i) {
  const double x[12] = {0.0092196828766403782, 0.047941371814762601, 0.11504866290284765, 0.20634102285669126, 0.31608425050090994, 0.43738329574426554, 0.5626167042557344, 0.68391574949909006, 0.79365897714330869, 0.88495133709715235, 0.95205862818523745, 0.99078031712335957};
  return x[i];
}
VP_HD double vp_gl12_w(int i) {
  const double w[12] = {0.023587668193255706, 0.053469662997659533, 0.080039164271673208, 0.10158371336153287, 0.11674626826917731, 0.12457352290670134, 0.12457352290670134, 0.11674626826917731, 0.10158371336153287, 0.080039164271673208, 0.053469662997659533, 0.023587668193255706};
  return w[i];
}

// local box integral: coef_ab = int_0^delta M_a([lo1, hi1], t) M_b([lo2, hi2], t) dt, bounds relative to the target
// (infinite bounds allowed), by Gauss-Legendre in tau = sqrt(t) on panels split at the finite edge distances
// (R8).  The exact local integral of the Taylor polynomial over the box (Taylor basis of the box frame).
VP_HD void vp_coef_box(double lo1, double hi1, double lo2, double hi2, double delta, int deg, double *coef) {
  double sd = sqrt(delta);
  const double big = 60.0 * sd;  // exp(-big^2 / 4 delta) = e^{-900}: an infinite bound
  lo1 = fmax(lo1, -big); lo2 = fmax(lo2, -big);
  hi1 = fmin(hi1, big); hi2 = fmin(hi2, big);
  double dist[4] = {-lo1, hi1, -lo2, hi2};
  vp_coef_clear(coef);
  double brk[20];
  int nb = 0;
  brk[nb++] = 0.0;
  const double fr[4] = {1.0 / 12.0, 1.0 / 6.0, 1.0 / 3.0, 1.0 / 1.5};
  for (int e = 0; e < 4; e++) {
    double d = dist[e] > 0 ? dist[e] : 0.0;
    for (int k = 0; k < 4; k++) {
      double b = d * fr[k];
      if (b > 0.0 && b < sd) brk[nb++] = b;
    }
  }
  brk[nb++] = sd;
  // insertion sort
  for (int i = 1; i < nb; i++) {
    double v = brk[i];
    int j = i - 1;
    while (j >= 0 && brk[j] > v) { brk[j + 1] = brk[j]; j--; }
    brk[j + 1] = v;
  }
  int dmax = deg < 4 ? deg : 4;
  for (int pnl = 0; pnl + 1 < nb; pnl++) {
    double a0 = brk[pnl], a1 = brk[pnl + 1], h = a1 - a0;
    if (h <= 0.0) continue;
    for (int i = 0; i < 12; i++) {
      double tau = a0 + h * vp_gl12_x(i);
      double wt = h * vp_gl12_w(i) * 2.0 * tau;
      double t = tau * tau;
      double Mx[5], My[5];
      vp_moments(lo1, hi1, t, Mx);
      vp_moments(lo2, hi2, t, My);
      for (int d = 0; d <= dmax; d++)
        for (int a = d; a >= 0; a--) coef[vp_mono_index(a, d - a)] += wt * Mx[a] * My[d - a];
    }
  }
}

// Taylor-coefficient weights of a rotated frame -> the global frame: the local frame has orthonormal axes
// (ax, ay), (bx, by); f(x + s1 a + s2 b) = sum a'_ij s1^i s2^j with a'_ij = sum_ab T[ab][ij] a_ab, T the
// coefficients of (s1 ax + s2 bx)^a (s1 ay + s2 by)^b.  Returns coef_ab = sum_ij T[ab][ij] cloc_ij (degree <= 4).
VP_HD void vp_coef_rotate(const double *cloc, double ax, double ay, double bx, double by, int deg, double *coef) {
  vp_coef_clear(coef);
  const int dmax = deg < 4 ? deg : 4;
  for (int d = 0; d <= dmax; d++)
    for (int a = d; a >= 0; a--) {
      const int b = d - a;
      double P[5] = {1.0, 0.0, 0.0, 0.0, 0.0};  // P[i]: coefficient of s1^i s2^(deg_so_far - i)
      int n = 0;
      for (int m = 0; m < d; m++) {
        const double u = m < a ? ax : ay, v = m < a ? bx : by;  // factor (u s1 + v s2)
        double Q[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i <= n; i++) {
          Q[i + 1] += P[i] * u;
          Q[i] += P[i] * v;
        }
        n++;
        for (int i = 0; i <= n; i++) P[i] = Q[i];
      }
      double acc = 0.0;
      for (int i = 0; i <= d; i++) acc += P[i] * cloc[vp_mono_index(i, d - i)];
      coef[vp_mono_index(a, b)] = acc;
    }
}

// near an axis-aligned rectangle [x0,x1]x[y0,y1]: coef_ab = int_0^delta M_a(x-range, t) M_b(y-range, t) dt.
// Returns false when all edges are farther than 12 sqrt(delta).
VP_HD bool vp_coef_rect(double x, double y, double x0, double y0, double x1, double y1, double delta, int deg,
                        double *coef) {
  double sd = sqrt(delta);
  double dmin = fmin(fmin(x - x0, x1 - x), fmin(y - y0, y1 - y));
  if (dmin >= 12.0 * sd) return false;
  vp_coef_box(x0 - x, x1 - x, y0 - y, y1 - y, delta, deg, coef);
  return true;
}
