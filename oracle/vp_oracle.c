/*
 * vp_oracle.c -- CPU fp64 ORACLE for the 2D Poisson volume potential.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * product path (paper_2409_11998_b200/); neither includes the other.
 *
 * What it computes (§1 eq. (volpotposgreen)/(GreenPoisson), lines 55-68):
 *
 *     V*(x) = sum_T  \int_T  G(x - y) f(y) dy,     G(x) = -(1/2pi) log|x|
 *
 * over the given triangles (straight, or with circular-arc edges mapped by the
 * smooth blending map of workloads/geometry.py -- the same *geometric definition*,
 * implemented here independently), with f evaluated analytically.  This is the plain
 * definition the method approximates (the error
 * split of eq. (volint_error)).  Quadrature, per (target, triangle), by the relative
 * distance eta = dist / diam:
 *     eta >= 6        : own 12-point degree-6 rule (Dunavant), f analytic
 *     0.5 <= eta < 6  : Duffy-collapsed tensor Gauss-Legendre, n = 6..20 by eta
 *     eta < 0.5       : polar (Duffy) rule centred at the target's reference-space
 *                       pre-image; radial variable u = exp(-tau) removes the u log u
 *                       singularity; angular panels graded toward the near-singular
 *                       direction.  Works for targets inside, on, or just outside T.
 *
 * Also:
 *   orc_smooth_direct : sum_j c_j G_H[delta](x_t - x_j), the smooth part of the Ewald/heat
 *                       split, G_H = -(1/2pi)log r - (1/4pi)E1(r^2/4delta)  (PAPER.md eq.
 *                       (splitting2), lines 329-341; identity (eiformula), lines 351-356).
 *   orc_smooth_dft    : the same quantity through a direct (non-fast) Fourier sum of the
 *                       near/far history split (§3 Steps 2-4, lines 826-893; lemmas
 *                       (vnearkspace) line 385 and (vfarkspace)/(Wdef) lines 416-435), with the
 *                       normalisation and period readings of DESIGN.md §Readings R1-R3.
 *   orc_e1            : exponential integral E1 (series / continued fraction).
 *
 * Parity pins: tests/test_oracle.py (closed forms for the disk, Gaussian and rectangle,
 * 4th-order finite-difference -Laplace V = f, brute-force scipy quadrature on tiny cases,
 * additivity and translation invariance, E1 vs scipy).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_PI 3.14159265358979323846

/* Neumaier (compensated) summation: the target sums run over up to ~2e8 terms (config 5), whose naive rounding
 * error (~sqrt(N) eps sum|t|, measured 1e-12..3e-11 relative at config 5) would exceed the 1e-12 smooth-part gate
 * of the north star; compensated, the error is ~eps sum|t| */
typedef struct { double s, c; } orc_ksum;
static inline void ksum_add(orc_ksum *k, double v) {
  double t = k->s + v;
  if (fabs(k->s) >= fabs(v)) k->c += (k->s - t) + v;
  else k->c += (v - t) + k->s;
  k->s = t;
}
#define ORC_EULER 0.57721566490153286061

/* ------------------------------------------------------------------ fields */
typedef struct {
  int32_t kind; /* 0 const, 1 gauss, 2 fourier */
  int32_t n;
  double a0;                               /* const */
  const double *a, *cx, *cy, *s;           /* gauss: f = sum a exp(-|x-c|^2/s) */
  const int32_t *k1, *k2;                  /* fourier */
  const double *fa, *fb;                   /* f = sum fa cos(2pi k.x) + fb sin(2pi k.x) */
} orc_field;

typedef struct {
  /* fourier evaluation helper (dense coefficient table, built once) */
  int K1, lo2, n2;
  double complex *C; /* (K1+1) x n2 : fa - i fb */
} orc_fourier_tab;

static orc_fourier_tab g_ftab;

static void build_fourier_tab(const orc_field *F) {
  free(g_ftab.C);
  memset(&g_ftab, 0, sizeof g_ftab);
  if (F->kind != 2) return;
  int K1 = 0, lo2 = 0, hi2 = 0;
  for (int i = 0; i < F->n; i++) {
    if (F->k1[i] > K1) K1 = F->k1[i];
    if (F->k2[i] < lo2) lo2 = F->k2[i];
    if (F->k2[i] > hi2) hi2 = F->k2[i];
  }
  g_ftab.K1 = K1; g_ftab.lo2 = lo2; g_ftab.n2 = hi2 - lo2 + 1;
  g_ftab.C = calloc((size_t)(K1 + 1) * g_ftab.n2, sizeof(double complex));
  for (int i = 0; i < F->n; i++)
    g_ftab.C[(size_t)F->k1[i] * g_ftab.n2 + (F->k2[i] - lo2)] += F->fa[i] - I * F->fb[i];
}

static double field_eval(const orc_field *F, double x, double y) {
  if (F->kind == 0) return F->a0;
  if (F->kind == 1) {
    double v = 0.0;
    for (int i = 0; i < F->n; i++) {
      double dx = x - F->cx[i], dy = y - F->cy[i];
      v += F->a[i] * exp(-(dx * dx + dy * dy) / F->s[i]);
    }
    return v;
  }
  /* fourier: Re sum_{k1} e^{2pi i k1 x} sum_{k2} C[k1,k2] e^{2pi i k2 y} */
  int K1 = g_ftab.K1, n2 = g_ftab.n2, lo2 = g_ftab.lo2;
  double complex ey[256];
  double complex sy = cexp(2.0 * ORC_PI * I * y);
  ey[0] = cexp(2.0 * ORC_PI * I * y * lo2);
  for (int j = 1; j < n2; j++) ey[j] = (j % 16 == 0) ? cexp(2.0 * ORC_PI * I * y * (lo2 + j)) : ey[j - 1] * sy;
  double complex sx = cexp(2.0 * ORC_PI * I * x), ex = 1.0;
  double v = 0.0;
  for (int k = 0; k <= K1; k++) {
    if (k % 16 == 0) ex = cexp(2.0 * ORC_PI * I * x * k);
    const double complex *row = g_ftab.C + (size_t)k * n2;
    double complex acc = 0.0;
    for (int j = 0; j < n2; j++) acc += row[j] * ey[j];
    v += creal(ex * acc);
    ex *= sx;
  }
  return v;
}

/* ------------------------------------------------------------------ Gauss-Legendre */
/* Nodes/weights on [0,1] for n = 1..GL_MAX are NOT generated here: the Python layer (oracle/__init__.py) passes
 * numpy.polynomial.legendre.leggauss (companion-matrix eigenvalues + Newton polish, a library routine) through
 * orc_set_gauss_legendre before any quadrature runs.  The oracle thereby shares no Gauss-Legendre generator
 * with the product path (which builds its own by Newton iteration on P_n). */
#define GL_MAX 40
static double g_glx[GL_MAX + 1][GL_MAX], g_glw[GL_MAX + 1][GL_MAX];
static int g_gl_init = 0;

/* x, w: concatenated rules n = 1..nmax on [-1, 1] (n entries each) */
int orc_set_gauss_legendre(int nmax, const double *x, const double *w) {
  if (nmax < GL_MAX) return -1;
  int64_t o = 0;
  for (int n = 1; n <= nmax; n++) {
    for (int i = 0; i < n; i++)
      if (n <= GL_MAX) {
        g_glx[n][i] = 0.5 * (x[o + i] + 1.0);
        g_glw[n][i] = 0.5 * w[o + i];
      }
    o += n;
  }
  g_gl_init = 1;
  return 0;
}

static void gl_init(void) {
  if (!g_gl_init) abort(); /* orc_set_gauss_legendre must run first (oracle/__init__.py does) */
}

/* ------------------------------------------------------------------ 12-point rule (own copy) */
/* Dunavant (1985) degree-6 rule: two S21 orbits, one S111 orbit; barycentric, weights sum to 1. */
static double g_r12[12][3], g_w12[12];
static void rule12_init(void) {
  const double a1 = 0.249286745170910, w1 = 0.116786275726379;
  const double a2 = 0.063089014491502, w2 = 0.050844906370207;
  const double p = 0.053145049844817, q = 0.310352451033784, r = 0.636502499121399, w3 = 0.082851075618374;
  int k = 0;
  double s21[2][2] = {{a1, w1}, {a2, w2}};
  for (int o = 0; o < 2; o++) {
    double a = s21[o][0], b = 1.0 - 2.0 * a;
    double pts[3][3] = {{a, a, b}, {a, b, a}, {b, a, a}};
    for (int m = 0; m < 3; m++, k++) {
      g_r12[k][1] = pts[m][1]; g_r12[k][2] = pts[m][2]; g_r12[k][0] = 1.0 - pts[m][1] - pts[m][2];
      g_w12[k] = s21[o][1];
    }
  }
  double perm[6][3] = {{p, q, r}, {p, r, q}, {q, p, r}, {q, r, p}, {r, p, q}, {r, q, p}};
  for (int m = 0; m < 6; m++, k++) {
    g_r12[k][1] = perm[m][1]; g_r12[k][2] = perm[m][2]; g_r12[k][0] = 1.0 - perm[m][1] - perm[m][2];
    g_w12[k] = w3;
  }
}

/* ------------------------------------------------------------------ triangle maps */
typedef struct {
  double v[3][2];
  int curved;          /* bitmask of arc edges */
  double cx, cy, rho;  /* circle */
  double diam, sag;
} orc_tri;

static double complex csinc(double complex z) {
  if (cabs(z) < 1e-4) return 1.0 - z * z / 6.0 + z * z * z * z / 120.0;
  return csin(z) / z;
}

/* q(lam) = (arc(lam) - chord(lam)) / (lam (1-lam)) for arc va->vb (complex-step safe) */
static void arc_q(const orc_tri *t, int i, int j, double complex lam, double complex *qx, double complex *qy) {
  const double *va = t->v[i], *vb = t->v[j];
  double ta = atan2(va[1] - t->cy, va[0] - t->cx), tb = atan2(vb[1] - t->cy, vb[0] - t->cx);
  double dt = remainder(tb - ta, 2.0 * ORC_PI);
  double dvx = vb[0] - va[0], dvy = vb[1] - va[1];
  if (creal(lam) <= 0.5) {
    double complex ph = ta + lam * dt / 2.0;
    double complex s = t->rho * dt * csinc(lam * dt / 2.0);
    *qx = (s * (-csin(ph)) - dvx) / (1.0 - lam);
    *qy = (s * ccos(ph) - dvy) / (1.0 - lam);
  } else {
    double complex mu = 1.0 - lam;
    double complex ph = tb - mu * dt / 2.0;
    double complex s = -t->rho * dt * csinc(mu * dt / 2.0);
    *qx = (s * (-csin(ph)) + dvx) / lam;
    *qy = (s * ccos(ph) + dvy) / lam;
  }
}

/* X(xi) (complex-step capable) */
static void tri_map_c(const orc_tri *t, double complex x1, double complex x2, double complex *X, double complex *Y) {
  double complex l[3] = {1.0 - x1 - x2, x1, x2};
  double complex x = 0, y = 0;
  for (int k = 0; k < 3; k++) { x += l[k] * t->v[k][0]; y += l[k] * t->v[k][1]; }
  if (t->curved) {
    for (int e = 0; e < 3; e++) {
      if (!(t->curved & (1 << e))) continue;
      int i = e, j = (e + 1) % 3;
      double complex lam = (1.0 + l[j] - l[i]) / 2.0, qx, qy;
      arc_q(t, i, j, lam, &qx, &qy);
      x += l[i] * l[j] * qx;
      y += l[i] * l[j] * qy;
    }
  }
  *X = x; *Y = y;
}

/* X, Jacobian J (row-major: J[0]=dX/dxi1, J[1]=dX/dxi2, J[2]=dY/dxi1, J[3]=dY/dxi2) */
static void tri_map(const orc_tri *t, double x1, double x2, double *X, double *Y, double *J) {
  if (!t->curved) {
    *X = (1 - x1 - x2) * t->v[0][0] + x1 * t->v[1][0] + x2 * t->v[2][0];
    *Y = (1 - x1 - x2) * t->v[0][1] + x1 * t->v[1][1] + x2 * t->v[2][1];
    if (J) {
      J[0] = t->v[1][0] - t->v[0][0]; J[1] = t->v[2][0] - t->v[0][0];
      J[2] = t->v[1][1] - t->v[0][1]; J[3] = t->v[2][1] - t->v[0][1];
    }
    return;
  }
  double complex cx, cy;
  tri_map_c(t, x1, x2, &cx, &cy);
  *X = creal(cx); *Y = creal(cy);
  if (J) {
    const double h = 1e-30;
    tri_map_c(t, x1 + I * h, x2, &cx, &cy);
    J[0] = cimag(cx) / h; J[2] = cimag(cy) / h;
    tri_map_c(t, x1, x2 + I * h, &cx, &cy);
    J[1] = cimag(cx) / h; J[3] = cimag(cy) / h;
  }
}

static void load_tri(orc_tri *t, const double *tri, const int8_t *curved, const double *circle, int64_t m) {
  for (int k = 0; k < 3; k++) { t->v[k][0] = tri[6 * m + 2 * k]; t->v[k][1] = tri[6 * m + 2 * k + 1]; }
  t->curved = (curved && circle) ? curved[m] : 0;
  if (circle) { t->cx = circle[0]; t->cy = circle[1]; t->rho = circle[2]; } else { t->cx = t->cy = 0; t->rho = 1; }
  double d = 0.0;
  for (int k = 0; k < 3; k++) {
    int j = (k + 1) % 3;
    double e = hypot(t->v[j][0] - t->v[k][0], t->v[j][1] - t->v[k][1]);
    if (e > d) d = e;
  }
  t->sag = 0.0;
  if (t->curved) {
    for (int e = 0; e < 3; e++) if (t->curved & (1 << e)) {
      int j = (e + 1) % 3;
      double c = hypot(t->v[j][0] - t->v[e][0], t->v[j][1] - t->v[e][1]);
      double half = asin(fmin(1.0, c / (2 * t->rho)));
      double s = t->rho * (1 - cos(half));
      if (s > t->sag) t->sag = s;
    }
  }
  t->diam = d + 2.0 * t->sag;
}

/* distance from p to the straight triangle (0 if inside) */
static double seg_dist2(double px, double py, const double *a, const double *b) {
  double dx = b[0] - a[0], dy = b[1] - a[1];
  double L2 = dx * dx + dy * dy;
  double u = L2 > 0 ? ((px - a[0]) * dx + (py - a[1]) * dy) / L2 : 0.0;
  if (u < 0) u = 0; else if (u > 1) u = 1;
  double ex = a[0] + u * dx - px, ey = a[1] + u * dy - py;
  return ex * ex + ey * ey;
}
static double tri_dist(const orc_tri *t, double px, double py) {
  double c[3];
  for (int k = 0; k < 3; k++) {
    int j = (k + 1) % 3;
    c[k] = (t->v[j][0] - t->v[k][0]) * (py - t->v[k][1]) - (t->v[j][1] - t->v[k][1]) * (px - t->v[k][0]);
  }
  if ((c[0] >= 0 && c[1] >= 0 && c[2] >= 0) || (c[0] <= 0 && c[1] <= 0 && c[2] <= 0)) return 0.0;
  double d = seg_dist2(px, py, t->v[0], t->v[1]);
  double d2 = seg_dist2(px, py, t->v[1], t->v[2]); if (d2 < d) d = d2;
  d2 = seg_dist2(px, py, t->v[2], t->v[0]); if (d2 < d) d = d2;
  return sqrt(d);
}

/* ------------------------------------------------------------------ quadrature tiers */
static inline double Gk(double dx, double dy) { return -log(dx * dx + dy * dy) / (4.0 * ORC_PI); }

/* Duffy-collapsed n x n Gauss rule on the reference triangle: xi = (u, (1-u) v), J = 1-u */
static double tri_duffy(const orc_tri *t, const orc_field *F, double px, double py, int n) {
  const double *x = g_glx[n], *w = g_glw[n];
  double acc = 0.0, Jm[4];
  for (int a = 0; a < n; a++) {
    double u = x[a];
    for (int b = 0; b < n; b++) {
      double v = x[b];
      double X, Y;
      tri_map(t, u, (1.0 - u) * v, &X, &Y, Jm);
      double det = fabs(Jm[0] * Jm[3] - Jm[1] * Jm[2]);
      acc += w[a] * w[b] * (1.0 - u) * det * Gk(X - px, Y - py) * field_eval(F, X, Y);
    }
  }
  return acc;
}

/* Newton inversion X(xi) = p, starting from the affine pre-image */
static void tri_inverse(const orc_tri *t, double px, double py, double *x1, double *x2) {
  double J[4];
  double e1x = t->v[1][0] - t->v[0][0], e1y = t->v[1][1] - t->v[0][1];
  double e2x = t->v[2][0] - t->v[0][0], e2y = t->v[2][1] - t->v[0][1];
  double det = e1x * e2y - e2x * e1y;
  double rx = px - t->v[0][0], ry = py - t->v[0][1];
  *x1 = (rx * e2y - e2x * ry) / det;
  *x2 = (e1x * ry - rx * e1y) / det;
  if (!t->curved) return;
  for (int it = 0; it < 30; it++) {
    double X, Y;
    tri_map(t, *x1, *x2, &X, &Y, J);
    double fx = X - px, fy = Y - py;
    double d = J[0] * J[3] - J[1] * J[2];
    double s1 = (fx * J[3] - J[1] * fy) / d, s2 = (J[0] * fy - fx * J[2]) / d;
    *x1 -= s1; *x2 -= s2;
    if (fabs(s1) + fabs(s2) < 1e-16) break;
  }
}

/* radial tau-panels for u = exp(-tau) */
static const double TAU_BRK[] = {0.0, 1.0, 3.0, 7.0, 15.0, 37.0};
#define N_TAU_PAN 5
#ifndef N_TAU_GL
#define N_TAU_GL 14
#endif

/* integral over the signed sub-triangle (xi_t, A, B) in reference space, apex singular */
static double polar_sub(const orc_tri *t, const orc_field *F, double px, double py,
                        double t1, double t2, const double *A, const double *B, int NV) {
  double ax = A[0] - t1, ay = A[1] - t2, bx = B[0] - t1, by = B[1] - t2;
  double cr = ax * by - ay * bx;
  if (fabs(cr) < 1e-15) return 0.0;
  double sgn = cr > 0 ? 1.0 : -1.0, acr = fabs(cr);
  double J0[4], X0, Y0;
  tri_map(t, t1, t2, &X0, &Y0, J0);
  /* angular near-singularity: minimise |J0 e(v)|^2 over v */
  double pax = J0[0] * ax + J0[1] * ay, pay = J0[2] * ax + J0[3] * ay;
  double pbx = J0[0] * bx + J0[1] * by, pby = J0[2] * bx + J0[3] * by;
  double dx = pbx - pax, dy = pby - pay;
  double A2 = dx * dx + dy * dy;
  double vstar = A2 > 0 ? -(pax * dx + pay * dy) / A2 : 0.5;
  /* near-singular direction: the closest point of the (linearised) base to the apex, clamped to
   * the panel [0,1]; grade geometrically toward it when it is close relative to the base length */
  if (vstar < 0.0) vstar = 0.0;
  if (vstar > 1.0) vstar = 1.0;
  double brk[100];
  int nb = 0;
  brk[nb++] = 0.0;
  {
    double mx = pax + vstar * dx, my = pay + vstar * dy;
    double dmin = hypot(mx, my) / sqrt(A2); /* relative distance scale in v */
    if (dmin < 0.5) {
      if (dmin < 1e-15) dmin = 1e-15;
      double lo[45], hi[45];
      int nl = 0, nh = 0;
      for (double s = dmin; s < vstar && nl < 45; s *= 3.0) lo[nl++] = vstar - s;
      for (double s = dmin; s < 1.0 - vstar && nh < 45; s *= 3.0) hi[nh++] = vstar + s;
      for (int k = nl - 1; k >= 0; k--) brk[nb++] = lo[k];
      if (vstar > 0.0 && vstar < 1.0) brk[nb++] = vstar;
      for (int k = 0; k < nh; k++) brk[nb++] = hi[k];
    }
  }
  brk[nb++] = 1.0;
  const double *gvx = g_glx[NV], *gvw = g_glw[NV];
  const double *grx = g_glx[N_TAU_GL], *grw = g_glw[N_TAU_GL];
  double acc = 0.0;
  for (int p = 0; p + 1 < nb; p++) {
    double v0 = brk[p], v1 = brk[p + 1], hv = v1 - v0;
    if (hv <= 0) continue;
    for (int b = 0; b < NV; b++) {
      double v = v0 + hv * gvx[b];
      double ex = ax + v * (bx - ax), ey = ay + v * (by - ay);
      double rad = 0.0;
      for (int q = 0; q < N_TAU_PAN; q++) {
        double ta = TAU_BRK[q], tb = TAU_BRK[q + 1], ht = tb - ta;
        for (int a = 0; a < N_TAU_GL; a++) {
          double tau = ta + ht * grx[a];
          double u = exp(-tau);
          double Jm[4], X, Y, Rx, Ry;
          tri_map(t, t1 + u * ex, t2 + u * ey, &X, &Y, Jm);
          if (!t->curved) {
            Rx = J0[0] * ex + J0[1] * ey; Ry = J0[2] * ex + J0[3] * ey;
          } else if (u > 1e-7) {
            Rx = (X - X0) / u; Ry = (Y - Y0) / u;
          } else {
            double Jh[4], Xh, Yh;
            tri_map(t, t1 + 0.5 * u * ex, t2 + 0.5 * u * ey, &Xh, &Yh, Jh);
            Rx = Jh[0] * ex + Jh[1] * ey; Ry = Jh[2] * ex + Jh[3] * ey;
          }
          double det = fabs(Jm[0] * Jm[3] - Jm[1] * Jm[2]);
          /* G = -(1/2pi)(log u + log|R|),  log u = -tau;  du = -u dtau;  integrand u*g(u) */
          double G = -(-tau + 0.5 * log(Rx * Rx + Ry * Ry)) / (2.0 * ORC_PI);
          rad += grw[a] * ht * u * u * G * field_eval(F, X, Y) * det;
        }
      }
      acc += gvw[b] * hv * rad;
    }
  }
  return sgn * acc * acr;
}

static double tri_polar(const orc_tri *t, const orc_field *F, double px, double py, int NV) {
  double t1, t2;
  tri_inverse(t, px, py, &t1, &t2);
  static const double R[3][2] = {{0, 0}, {1, 0}, {0, 1}};
  double acc = 0.0;
  for (int e = 0; e < 3; e++) acc += polar_sub(t, F, px, py, t1, t2, R[e], R[(e + 1) % 3], NV);
  return acc;
}

/* ------------------------------------------------------------------ public entry points */
typedef struct {
  double eta_far;    /* >= : own 12-point rule (default 6) */
  double eta_polar;  /* <  : polar rule (default 0.25) */
  int32_t nthreads;  /* 0 = OpenMP default */
  int32_t assume_resolved; /* 1: skip the per-triangle resolution ladder (far field = own 12-point rule on every
                              triangle).  Only for fields the 12-point rule resolves everywhere; the caller
                              checks that claim with orc_resolve_rules on a sample (tests/test_oracle.py). */
} orc_opts;

static int duffy_n(double eta) {
  if (eta >= 3.0) return 6;
  if (eta >= 1.5) return 9;
  if (eta >= 0.75) return 12;
  return 20;
}

/* ---- resolution of f on a triangle: which rule integrates f (times low-order moments) to
 * ~1e-15 relative?  0 -> own 12-point rule, else the Duffy n x n order (8, 14, 20, 30).
 * The kernel G is smooth on T when eta >= eta_far; the product G f is then resolved when f and
 * its first moments are (checked against the next finer rule). */
static void moments_12(const orc_tri *t, const orc_field *F, double gx, double gy, double D, double *mom, double *absw) {
  for (int k = 0; k < 6; k++) mom[k] = 0.0;
  *absw = 0.0;
  for (int k = 0; k < 12; k++) {
    double X, Y, Jm[4];
    tri_map(t, g_r12[k][1], g_r12[k][2], &X, &Y, Jm);
    double w = g_w12[k] * 0.5 * fabs(Jm[0] * Jm[3] - Jm[1] * Jm[2]) * field_eval(F, X, Y);
    /* moment coordinates in the reference triangle (exact; physical X - gx loses digits on tiny triangles) */
    double a = g_r12[k][1] - 1.0 / 3.0, b = g_r12[k][2] - 1.0 / 3.0;
    (void)gx; (void)gy; (void)D;
    mom[0] += w; mom[1] += w * a; mom[2] += w * b; mom[3] += w * a * a; mom[4] += w * a * b; mom[5] += w * b * b;
    *absw += fabs(w);
  }
}
static void moments_duffy(const orc_tri *t, const orc_field *F, double gx, double gy, double D, int n, double *mom, double *absw) {
  for (int k = 0; k < 6; k++) mom[k] = 0.0;
  *absw = 0.0;
  for (int i = 0; i < n; i++)
    for (int j = 0; j < n; j++) {
      double u = g_glx[n][i], v = g_glx[n][j], X, Y, Jm[4];
      tri_map(t, u, (1.0 - u) * v, &X, &Y, Jm);
      double w = g_glw[n][i] * g_glw[n][j] * (1.0 - u) * fabs(Jm[0] * Jm[3] - Jm[1] * Jm[2]) * field_eval(F, X, Y);
      double a = u - 1.0 / 3.0, b = (1.0 - u) * v - 1.0 / 3.0;
      (void)gx; (void)gy; (void)D;
      mom[0] += w; mom[1] += w * a; mom[2] += w * b; mom[3] += w * a * a; mom[4] += w * a * b; mom[5] += w * b * b;
      *absw += fabs(w);
    }
}
static double mom_diff(const double *a, const double *b) {
  double d = 0.0;
  for (int k = 0; k < 6; k++) d = fmax(d, fabs(a[k] - b[k]));
  return d;
}
/* fscale = max |f| over the domain's nodes: a triangle whose integrand is below 1e-6 fscale everywhere is
 * resolved to an absolute 1e-19 fscale |T| (its contribution to V is negligible at any tolerance) instead of
 * to its own (possibly 1e-200) size -- otherwise Gaussian tails demand 30 x 30 rules for nothing. */
static double g_fscale = 0.0;
static int resolve_rule(const orc_tri *t, const orc_field *F, double gx, double gy) {
  if (F->kind == 0 && !t->curved) return 0;
  static const int ladder[4] = {8, 14, 20, 30};
  double m12[6], mA[6], mB[6], s12, sA, sB;
  const double tolr = 1e-13;  /* per-triangle relative accuracy; the rounding floor of the sums is ~1e-15 */
  moments_12(t, F, gx, gy, t->diam, m12, &s12);
  moments_duffy(t, F, gx, gy, t->diam, ladder[0], mA, &sA);
  double area = 0.5 * fabs((t->v[1][0] - t->v[0][0]) * (t->v[2][1] - t->v[0][1]) -
                           (t->v[1][1] - t->v[0][1]) * (t->v[2][0] - t->v[0][0]));
  double scale = fmax(fmax(sA, 1e-6 * g_fscale * area), 1e-300);
  if (mom_diff(m12, mA) <= tolr * scale) return 0;
  for (int r = 0; r + 1 < 4; r++) {
    moments_duffy(t, F, gx, gy, t->diam, ladder[r + 1], mB, &sB);
    if (mom_diff(mA, mB) <= tolr * scale) return ladder[r];
    memcpy(mA, mB, sizeof mA);
  }
  return ladder[3];
}

/* near/singular contribution of one triangle to one target (eta < eta_far) */
static double tri_near(const orc_tri *t, const orc_field *F, double px, double py, int nres, const orc_opts *o) {
  double d = tri_dist(t, px, py) - t->sag;
  if (d < 0) d = 0;
  double eta = d / t->diam;
  if (eta >= o->eta_polar) {
    int n = duffy_n(eta);
    if (nres > n) n = nres;
    return tri_duffy(t, F, px, py, n);
  }
  return tri_polar(t, F, px, py, t->curved ? 40 : (nres >= 14 ? 30 : 20));
}

/* far contribution with the triangle's resolved rule computed on the fly (single-triangle API) */
static double tri_far_onfly(const orc_tri *t, const orc_field *F, double px, double py, int nres) {
  if (nres > 0) {
    /* Duffy n x n, kernel smooth at eta >= eta_far */
    return tri_duffy(t, F, px, py, nres);
  }
  double acc = 0.0;
  for (int k = 0; k < 12; k++) {
    double X, Y, Jm[4];
    tri_map(t, g_r12[k][1], g_r12[k][2], &X, &Y, Jm);
    double w = g_w12[k] * 0.5 * fabs(Jm[0] * Jm[3] - Jm[1] * Jm[2]);
    acc += w * field_eval(F, X, Y) * Gk(X - px, Y - py);
  }
  return acc;
}

static void init_all(const orc_field *F) {
  gl_init();
  rule12_init();
  build_fourier_tab(F);
}

static void opts_default(orc_opts *o, const orc_opts *in) {
  o->eta_far = 6.0; o->eta_polar = 0.5; o->nthreads = 0; o->assume_resolved = 0;
  if (in) {
    if (in->eta_far > 0) o->eta_far = in->eta_far;
    if (in->eta_polar > 0) o->eta_polar = in->eta_polar;
    o->nthreads = in->nthreads;
    o->assume_resolved = in->assume_resolved;
  }
}

static void set_fscale(int64_t M, const double *tri, const int8_t *curved, const double *circle, const orc_field *F) {
  double mx = 0.0;
#pragma omp parallel for schedule(static) reduction(max : mx)
  for (int64_t m = 0; m < M; m++) {
    orc_tri t;
    load_tri(&t, tri, curved, circle, m);
    for (int k = 0; k < 12; k++) {
      double X, Y;
      tri_map(&t, g_r12[k][1], g_r12[k][2], &X, &Y, NULL);
      double v = fabs(field_eval(F, X, Y));
      if (v > mx) mx = v;
    }
  }
  g_fscale = mx;
}

/* A prepared triangulation: per triangle its bounding circle and the far-field rule resolving f, expanded
 * into a CSR of (x, y, w f) points.  orc_volume_potential = prepare + eval + free; the split lets a caller
 * (bench.py's reference arm) pay the per-triangle setup once and time target batches separately. */
typedef struct {
  int64_t M;
  const double *tri;
  const int8_t *curved;
  const double *circle;
  orc_field F;
  orc_opts o;
  double *cen;
  int32_t *nres;
  int64_t *off;
  double *pts;
} orc_prepared;

void orc_free(orc_prepared *h) {
  if (!h) return;
  free(h->pts); free(h->cen); free(h->nres); free(h->off);
  free(h);
}

/* tri: M x 3 x 2 CCW; curved: M edge bitmasks or NULL; circle: (cx, cy, rho) or NULL.  The arrays (and the
 * field's) must outlive the handle.  NULL on allocation failure. */
orc_prepared *orc_prepare(int64_t M, const double *tri, const int8_t *curved, const double *circle,
                          const orc_field *F, const orc_opts *oin) {
  orc_prepared *h = calloc(1, sizeof(orc_prepared));
  if (!h) return NULL;
  opts_default(&h->o, oin);
  init_all(F);
#ifdef _OPENMP
  if (h->o.nthreads > 0) omp_set_num_threads(h->o.nthreads);
#endif
  h->M = M; h->tri = tri; h->curved = curved; h->circle = circle; h->F = *F;
  h->cen = malloc(sizeof(double) * 4 * (size_t)M); /* gx, gy, rbound, diam */
  h->nres = malloc(sizeof(int32_t) * (size_t)M);
  h->off = malloc(sizeof(int64_t) * ((size_t)M + 1));
  if (!h->cen || !h->nres || !h->off) { orc_free(h); return NULL; }
  set_fscale(M, tri, curved, circle, F);
  double *cen = h->cen;
  int32_t *nres = h->nres;
  int64_t *off = h->off;
  const orc_opts o = h->o;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t m = 0; m < M; m++) {
    orc_tri t;
    load_tri(&t, tri, curved, circle, m);
    double gx = (t.v[0][0] + t.v[1][0] + t.v[2][0]) / 3.0, gy = (t.v[0][1] + t.v[1][1] + t.v[2][1]) / 3.0;
    double rb = 0.0;
    for (int k = 0; k < 3; k++) { double r = hypot(t.v[k][0] - gx, t.v[k][1] - gy); if (r > rb) rb = r; }
    cen[4 * m] = gx; cen[4 * m + 1] = gy; cen[4 * m + 2] = rb + t.sag; cen[4 * m + 3] = t.diam;
    nres[m] = o.assume_resolved ? 0 : resolve_rule(&t, F, gx, gy);
  }
  off[0] = 0;
  for (int64_t m = 0; m < M; m++) off[m + 1] = off[m] + (nres[m] ? (int64_t)nres[m] * nres[m] : 12);
  h->pts = malloc(sizeof(double) * 3 * (size_t)off[M]);
  if (!h->pts) { orc_free(h); return NULL; }
  double *pts = h->pts;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t m = 0; m < M; m++) {
    orc_tri t;
    load_tri(&t, tri, curved, circle, m);
    double *q = pts + 3 * off[m];
    int n = nres[m];
    if (!n) {
      for (int k = 0; k < 12; k++) {
        double X, Y, Jm[4];
        tri_map(&t, g_r12[k][1], g_r12[k][2], &X, &Y, Jm);
        double w = g_w12[k] * 0.5 * fabs(Jm[0] * Jm[3] - Jm[1] * Jm[2]);
        q[3 * k] = X; q[3 * k + 1] = Y; q[3 * k + 2] = w * field_eval(F, X, Y);
      }
    } else {
      int k = 0;
      for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++, k++) {
          double u = g_glx[n][i], v = g_glx[n][j], X, Y, Jm[4];
          tri_map(&t, u, (1.0 - u) * v, &X, &Y, Jm);
          double w = g_glw[n][i] * g_glw[n][j] * (1.0 - u) * fabs(Jm[0] * Jm[3] - Jm[1] * Jm[2]);
          q[3 * k] = X; q[3 * k + 1] = Y; q[3 * k + 2] = w * field_eval(F, X, Y);
        }
    }
  }
  return h;
}

/* V*(targets) on a prepared triangulation */
int orc_eval_prepared(const orc_prepared *h, int64_t T, const double *tg, double *out) {
  const int64_t M = h->M;
  const double *cen = h->cen, *pts = h->pts;
  const int64_t *off = h->off;
  const int32_t *nres = h->nres;
  const orc_field *F = &h->F;
  const orc_opts o = h->o;
  init_all(F);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < T; i++) {
    double px = tg[2 * i], py = tg[2 * i + 1];
    orc_ksum acc = {0.0, 0.0};
    for (int64_t m = 0; m < M; m++) {
      const double *c = cen + 4 * m;
      double lb = hypot(px - c[0], py - c[1]) - c[2];
      double tsum = 0.0;  /* one triangle's contribution (<= 900 terms), then compensated across triangles */
      if (lb >= o.eta_far * c[3]) {
        const double *q = pts + 3 * off[m];
        int64_t np = off[m + 1] - off[m];
        for (int64_t k = 0; k < np; k++) tsum += q[3 * k + 2] * Gk(q[3 * k] - px, q[3 * k + 1] - py);
      } else {
        orc_tri t;
        load_tri(&t, h->tri, h->curved, h->circle, m);
        double d = tri_dist(&t, px, py) - t.sag;
        if (d >= o.eta_far * t.diam) {
          const double *q = pts + 3 * off[m];
          int64_t np = off[m + 1] - off[m];
          for (int64_t k = 0; k < np; k++) tsum += q[3 * k + 2] * Gk(q[3 * k] - px, q[3 * k + 1] - py);
        } else {
          tsum = tri_near(&t, F, px, py, nres[m], &o);
        }
      }
      ksum_add(&acc, tsum);
    }
    out[i] = acc.s + acc.c;
  }
  return 0;
}

/* V*(targets) for a triangulation (tri: M x 3 x 2 CCW; curved: M edge bitmasks or NULL;
 * circle: (cx, cy, rho) or NULL).  Returns 0 on success, -6 on allocation failure. */
int orc_volume_potential(int64_t M, const double *tri, const int8_t *curved, const double *circle,
                         const orc_field *F, int64_t T, const double *tg, double *out, const orc_opts *oin) {
  orc_prepared *h = orc_prepare(M, tri, curved, circle, F, oin);
  if (!h) return -6;
  int rc = orc_eval_prepared(h, T, tg, out);
  orc_free(h);
  return rc;
}

/* per-triangle resolved far rule order (0 = 12-point) -- diagnostics */
int orc_resolve_rules(int64_t M, const double *tri, const int8_t *curved, const double *circle,
                      const orc_field *F, int32_t *nres) {
  init_all(F);
  set_fscale(M, tri, curved, circle, F);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t m = 0; m < M; m++) {
    orc_tri t;
    load_tri(&t, tri, curved, circle, m);
    double gx = (t.v[0][0] + t.v[1][0] + t.v[2][0]) / 3.0, gy = (t.v[0][1] + t.v[1][1] + t.v[2][1]) / 3.0;
    nres[m] = resolve_rule(&t, F, gx, gy);
  }
  return 0;
}

/* single-triangle integral (tests: brute-force pins, additivity) */
double orc_triangle_integral(const double *tri3, int8_t curved, const double *circle, const orc_field *F,
                             double px, double py, const orc_opts *oin) {
  orc_opts o;
  opts_default(&o, oin);
  init_all(F);
  orc_tri t;
  load_tri(&t, tri3, &curved, circle, 0);
  set_fscale(1, tri3, &curved, circle, F);
  double gx = (t.v[0][0] + t.v[1][0] + t.v[2][0]) / 3.0, gy = (t.v[0][1] + t.v[1][1] + t.v[2][1]) / 3.0;
  int n = resolve_rule(&t, F, gx, gy);
  double d = tri_dist(&t, px, py) - t.sag;
  if (d >= o.eta_far * t.diam) return tri_far_onfly(&t, F, px, py, n);
  return tri_near(&t, F, px, py, n, &o);
}

/* own quadrature nodes/weights (tests: independence check against the generator) */
void orc_rule12_nodes(int64_t M, const double *tri, const int8_t *curved, const double *circle,
                      double *nodes, double *weights) {
  gl_init(); rule12_init();
  for (int64_t m = 0; m < M; m++) {
    orc_tri t;
    load_tri(&t, tri, curved, circle, m);
    for (int k = 0; k < 12; k++) {
      double X, Y, Jm[4];
      tri_map(&t, g_r12[k][1], g_r12[k][2], &X, &Y, Jm);
      nodes[24 * m + 2 * k] = X; nodes[24 * m + 2 * k + 1] = Y;
      weights[12 * m + k] = g_w12[k] * 0.5 * fabs(Jm[0] * Jm[3] - Jm[1] * Jm[2]);
    }
  }
}

/* ------------------------------------------------------------------ E1 and the smooth part */
/* Ein(z) = E1(z) + log z + gamma = sum_{k>=1} (-1)^{k+1} z^k / (k k!)  (DLMF 6.6.4), summed in long double */
static double ein(double z) {
  long double sum = 0.0L, term = 1.0L;
  for (int k = 1; k < 90; k++) {
    term *= (long double)z / k;
    long double d = ((k & 1) ? 1.0L : -1.0L) * term / k;
    sum += d;
    if (fabsl(d) < 1e-21L * fabsl(sum)) break;
  }
  return (double)sum;
}

/* E1(x) = e^{-x} int_0^inf e^{-v} / (x + v) dv  (DLMF 6.2.2 with t = 1 + v/x), x > 2: composite Gauss-Legendre
 * on [0, 44] (e^{-44} < 1e-19), panels growing in length; the integrand is positive (no cancellation) and
 * analytic with its pole at v = -x <= -2, so 24 nodes per panel reach full precision.  x <= 2: the series
 * E1 = -gamma - log x + Ein(x).  (A different method from the product path's series / continued fraction.) */
double orc_e1(double x) {
  if (x <= 0) return INFINITY;
  if (x <= 2.0) return -ORC_EULER - log(x) + ein(x);
  if (x > 745.0) return 0.0;
  gl_init();
  static const double brk[] = {0.0, 0.5, 1.0, 2.0, 4.0, 8.0, 14.0, 22.0, 32.0, 44.0};
  const int npan = 9, ng = 24;
  double acc = 0.0;
  for (int p = 0; p < npan; p++) {
    double a = brk[p], h = brk[p + 1] - a;
    for (int i = 0; i < ng; i++) {
      double v = a + h * g_glx[ng][i];
      acc += h * g_glw[ng][i] * exp(-v) / (x + v);
    }
  }
  return exp(-x) * acc;
}

/* G_H[delta](r) = -(1/4pi)[log r^2 + E1(r^2/4delta)], G_H(0) = (gamma - log 4delta)/(4pi) */
double orc_GH(double r2, double delta) {
  double z = r2 / (4.0 * delta);
  if (z <= 1.0) return -(log(4.0 * delta) - ORC_EULER + ein(z)) / (4.0 * ORC_PI);
  return -(log(r2) + orc_e1(z)) / (4.0 * ORC_PI);
}

int orc_smooth_direct(int64_t N, const double *src, const double *c, int64_t T, const double *tg,
                      double delta, double *out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < T; i++) {
    double px = tg[2 * i], py = tg[2 * i + 1];
    orc_ksum acc = {0.0, 0.0};
    for (int64_t j = 0; j < N; j++) {
      double dx = px - src[2 * j], dy = py - src[2 * j + 1];
      ksum_add(&acc, c[j] * orc_GH(dx * dx + dy * dy, delta));
    }
    out[i] = acc.s + acc.c;
  }
  return 0;
}

/* Truncated-Green's-function transform (PAPER.md eq. (Wdef), with a general radius R):
 * W_R(k) = -int_0^R r log(r) J0(k r) dr  -- the 2D transform of -log|x| restricted to |x| < R, over 2 pi.
 * Evaluated here from that DEFINITION (not the closed form (1 - J0(Rk))/k^2 - R log R J1(Rk)/k the product
 * path uses): r = R u^2 makes the integrand -2 R^2 u^3 (log R + 2 log u) J0(k R u^2) smooth at u = 0; composite
 * Gauss-Legendre in u with panels graded toward 0, then panels uniform in r (about one per third of a period
 * of J0); J0 from libm. */
double orc_WR(double k, double R) {
  gl_init();
  const int ng = 24;
  int npan = (int)ceil(k * R / 1.0);
  if (npan < 4) npan = 4;
  if (npan > 20000) npan = 20000;
  double acc = 0.0, lr = log(R);
  double u1 = sqrt(1.0 / npan);
  double edges[6] = {0.0, 1e-6 * u1, 1e-4 * u1, 1e-2 * u1, 0.1 * u1, u1};
  for (int p = 0; p < 5; p++) {
    double a = edges[p], h = edges[p + 1] - a;
    for (int i = 0; i < ng; i++) {
      double u = a + h * g_glx[ng][i];
      acc += h * g_glw[ng][i] * (-2.0 * R * R * u * u * u * (lr + 2.0 * log(u)) * j0(k * R * u * u));
    }
  }
  for (int p = 1; p < npan; p++) {
    double ua = sqrt((double)p / npan), ub = sqrt((double)(p + 1) / npan), h = ub - ua;
    for (int i = 0; i < ng; i++) {
      double u = ua + h * g_glx[ng][i];
      acc += h * g_glw[ng][i] * (-2.0 * R * R * u * u * u * (lr + 2.0 * log(u)) * j0(k * R * u * u));
    }
  }
  return acc;
}

/* f at arbitrary points (pins of field_eval against a numpy evaluation of the same analytic field) */
void orc_field_values(const orc_field *F, int64_t n, const double *xy, double *out) {
  build_fourier_tab(F);
  for (int64_t i = 0; i < n; i++) out[i] = field_eval(F, xy[2 * i], xy[2 * i + 1]);
}

/* Direct (slow) Fourier evaluation of V_NH + V_FH with trapezoid rule on k = 2 pi m / L:
 *   V_H(x) = (1/L^2) sum_m M(k_m) chat(k_m) e^{i k_m . x},  chat(k) = sum_j c_j e^{-i k . x_j}
 * M_NH = (e^{-k^2 d1} - e^{-k^2 d2})/k^2 (k=0: d2-d1), M_FH = e^{-k^2 d2} W_R(k); modes |m_i| <= n/2.
 * Periods/cutoffs are arguments (chosen by the caller per DESIGN.md readings R1-R3). */
int orc_smooth_dft(int64_t N, const double *src, const double *c, int64_t T, const double *tg,
                   double d1, double d2, double L_nh, int64_t n_nh, double L_fh, int64_t n_fh, double R,
                   double x0, double y0, double *out) {
  for (int64_t i = 0; i < T; i++) out[i] = 0.0;
  for (int part = 0; part < 2; part++) {
    double L = part ? L_fh : L_nh;
    int64_t n = part ? n_fh : n_nh;
    int64_t h = n / 2, nm = 2 * h + 1;
    double dk = 2.0 * ORC_PI / L;
    double complex *ch = calloc((size_t)nm * nm, sizeof(double complex));
    /* chat over modes m in [-h, h]^2, parallel over m1 */
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < nm; a++) {
      double k1 = dk * (a - h);
      for (int64_t j = 0; j < N; j++) {
        double complex e1 = c[j] * cexp(-I * k1 * (src[2 * j] - x0));
        double complex s = cexp(-I * dk * (src[2 * j + 1] - y0)), e = e1 * cexp(I * dk * h * (src[2 * j + 1] - y0));
        for (int64_t b = 0; b < nm; b++) {
          if ((b & 63) == 0) e = e1 * cexp(-I * dk * (b - h) * (src[2 * j + 1] - y0));
          ch[a * nm + b] += e;
          e *= s;
        }
      }
    }
    /* multiply */
    for (int64_t a = 0; a < nm; a++)
      for (int64_t b = 0; b < nm; b++) {
        double k2 = dk * dk * ((double)(a - h) * (a - h) + (double)(b - h) * (b - h));
        double Mk;
        if (part == 0) Mk = (k2 == 0.0) ? (d2 - d1) : (exp(-k2 * d1) - exp(-k2 * d2)) / k2;
        else Mk = exp(-k2 * d2) * orc_WR(sqrt(k2), R);
        ch[a * nm + b] *= Mk / (L * L);
      }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < T; i++) {
      double complex acc = 0.0;
      double px = tg[2 * i] - x0, py = tg[2 * i + 1] - y0;
      for (int64_t a = 0; a < nm; a++) {
        double complex e1 = cexp(I * dk * (a - h) * px);
        double complex s = cexp(I * dk * py), e = e1 * cexp(-I * dk * h * py);
        for (int64_t b = 0; b < nm; b++) {
          if ((b & 63) == 0) e = e1 * cexp(I * dk * (b - h) * py);
          acc += ch[a * nm + b] * e;
          e *= s;
        }
      }
      out[i] += creal(acc);
    }
    free(ch);
  }
  return 0;
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
