// vp_api.cu -- the C ABI of libvp.so (include/vp.h): plan construction and evaluation.
//
// Plan (§3 "Input" and "Step 1", lines 782-821; readings R1-R5 of DESIGN.md):
//   Dx^2 = sum(w)/N, delta1 = C Dx^2 (C = 3), delta2 = 32 delta1; k_max = sqrt(ln(1/eps)/delta);
//   periods L_NH = S + sqrt(4 delta2 z_eps) (E1(z_eps) = eps), R = sqrt2 S + sqrt(4 delta2 ln(1/eps)),
//   L_FH = S + R + sqrt(4 delta2 ln(1/eps)); modes n = 2 ceil(L k_max / 2pi); fine grids nf = 2n
//   (next 2,3,5,7-smooth); ES kernel width w = ceil(log10(1/eps)) + 1, beta = 2.30 w.
//   Sources and targets are binned into 32x32 tiles of the NH fine grid and sorted (CUB radix sort);
//   the local-part stencils are built (vp_local.cu); cuFFT D2Z/Z2D plans share one work area.
// Eval (one stream, no host synchronisation): zero grids -> spread -> D2Z x2 -> multiply x2 ->
//   Z2D x2 -> interpolation + local part + scatter.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>

#include "vp_boundary.cuh"
#include "vp_common.cuh"
#include "vp_math.cuh"

static thread_local std::string g_last_error;
void vp_set_last_error(const std::string &s) { g_last_error = s; }

int vp_current_device() {
  int d = 0;
  VP_CUDA(cudaGetDevice(&d));
  return d;
}

void vp_smem_attr(const void *func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, size_t> done;
  if (bytes <= 48 * 1024) return;
  const int dev = vp_current_device();
  std::lock_guard<std::mutex> lk(mu);
  size_t &have = done[std::make_pair(dev, func)];
  if (bytes <= have) return;
  VP_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  have = bytes;
}

extern "C" vp_status vp_struct_sizes(int64_t *out) {
  if (!out) return VP_ERR_ARG;
  out[0] = (int64_t)sizeof(vp_opts);
  out[1] = (int64_t)sizeof(vp_info);
  out[2] = (int64_t)sizeof(vp_boundary);
  return VP_OK;
}

extern "C" const char *vp_strerror(vp_status s) {
  switch (s) {
    case VP_OK: return "ok";
    case VP_ERR_ARG: return "invalid argument";
    case VP_ERR_TOL: return "tolerance outside [1e-14, 1e-2]";
    case VP_ERR_NONFINITE: return "non-finite value in input";
    case VP_ERR_GEOMETRY: return "invalid geometry / boundary descriptor";
    case VP_ERR_UNSUPPORTED: return "unsupported option combination";
    case VP_ERR_OOM: return "out of device memory (or grid too large)";
    case VP_ERR_CUDA: return "CUDA runtime error";
    case VP_ERR_CUFFT: return "cuFFT error";
  }
  return "unknown status";
}

extern "C" const char *vp_version(void) { return "vp 0.1 (sm_100a, fp64)"; }
extern "C" const char *vp_last_error_detail(void) { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------------------------
// host helpers
static double host_e1(double x) {  // exponential integral E1, x > 0 (series / continued fraction)
  if (x <= 1.0) {
    double s = 0.0, t = 1.0;
    for (int k = 1; k < 80; k++) {
      t *= -x / k;
      s -= t / k;
      if (fabs(t / k) < 1e-17 * fabs(s)) break;
    }
    return -0.5772156649015329 - log(x) + s;
  }
  double b = x + 1.0, c = 1e300, d = 1.0 / b, h = d;
  for (int i = 1; i < 400; i++) {
    double an = -(double)i * i;
    b += 2.0;
    d = 1.0 / (an * d + b);
    c = b + an / c;
    double del = c * d;
    h *= del;
    if (fabs(del - 1.0) < 1e-16) break;
  }
  return h * exp(-x);
}

double vp_solve_e1(double eps) {  // z with E1(z) = eps
  double z = log(1.0 / eps);
  for (int it = 0; it < 100; it++) {
    double f = host_e1(z) - eps;
    double df = -exp(-z) / z;
    double dz = f / df;
    z -= dz;
    if (fabs(dz) < 1e-12 * z) break;
  }
  return z;
}

int64_t vp_next_smooth(int64_t n) {  // smallest even 2^a 3^b 5^c 7^d >= n
  if (n < 2) n = 2;
  for (int64_t m = n + (n & 1);; m += 2) {
    int64_t r = m;
    for (int p : {2, 3, 5, 7})
      while (r % p == 0) r /= p;
    if (r == 1) return m;
  }
}

static void gauss_legendre01(int n, std::vector<double> &x, std::vector<double> &w) {
  x.resize(n);
  w.resize(n);
  for (int i = 0; i < n; i++) {
    double z = cos(VP_PI * (i + 0.75) / (n + 0.5)), pp = 1.0;
    for (int it = 0; it < 100; it++) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; j++) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      double dz = p1 / pp;
      z -= dz;
      if (fabs(dz) < 1e-16) break;
    }
    x[i] = 0.5 * (1.0 - z);
    w[i] = 1.0 / ((1.0 - z * z) * pp * pp);
  }
}

// Gauss-Legendre nodes (increasing) and weights on [-1, 1]
void vp_gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w) {
  gauss_legendre01(n, x, w);
  for (int i = 0; i < n; i++) {
    x[i] = 2.0 * x[i] - 1.0;
    w[i] *= 2.0;
  }
}

// ---------------------------------------------------------------------------------------------
// validation / statistics of the inputs (one pass over nodes, weights and targets)
struct Stats {
  double sumw, xmin, xmax, ymin, ymax;
  int bad;
};

__global__ void k_stats(const double *__restrict__ nodes, const double *__restrict__ w, int64_t N,
                        const double *__restrict__ tg, int64_t T, double *out_sum, double *out_box, int *out_bad) {
  double s = 0.0, x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
  int bad = 0;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N + T; i += stride) {
    double x, y;
    if (i < N) {
      x = nodes[2 * i];
      y = nodes[2 * i + 1];
      double ww = w[i];
      if (!isfinite(ww) || ww < 0.0) bad = 1;
      s += ww;
    } else {
      x = tg[2 * (i - N)];
      y = tg[2 * (i - N) + 1];
    }
    if (!isfinite(x) || !isfinite(y)) bad = 1;
    x0 = fmin(x0, x); x1 = fmax(x1, x); y0 = fmin(y0, y); y1 = fmax(y1, y);
  }
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage ts;
  double bs = BR(ts).Sum(s);
  __syncthreads();
  double bx0 = BR(ts).Reduce(x0, cub::Min());
  __syncthreads();
  double bx1 = BR(ts).Reduce(x1, cub::Max());
  __syncthreads();
  double by0 = BR(ts).Reduce(y0, cub::Min());
  __syncthreads();
  double by1 = BR(ts).Reduce(y1, cub::Max());
  __syncthreads();
  int any = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    out_sum[blockIdx.x] = bs;
    out_box[4 * blockIdx.x] = bx0;
    out_box[4 * blockIdx.x + 1] = bx1;
    out_box[4 * blockIdx.x + 2] = by0;
    out_box[4 * blockIdx.x + 3] = by1;
    if (any) *out_bad = 1;
  }
}

__global__ void k_check_finite(const double *__restrict__ f, int64_t n, int *bad) {
  int b = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(f[i])) b = 1;
  if (__syncthreads_or(b) && threadIdx.x == 0) *bad = 1;
}

// ---------------------------------------------------------------------------------------------
static void setup_grid(vp_plan_s *P, VpGrid &G, int kind, double L, double kmax) {
  G.kind = kind;
  G.L = L;
  int64_t n = 2 * (int64_t)ceil(L * kmax / (2.0 * VP_PI));
  if (n < 4) n = 4;
  G.nmode = n;
  G.nf = vp_next_smooth(2 * n);
  if (G.nf < 2 * P->w) G.nf = vp_next_smooth(2 * P->w);
  G.h = L / (double)G.nf;
  G.ox = P->cx - 0.5 * L;
  G.oy = P->cy - 0.5 * L;
  G.row = G.nf;                 // real grid rows (unpadded); the half spectrum lives in G.cdata
  G.crow = 2 * (G.nf / 2 + 1);  // doubles per half-spectrum row
  if ((double)G.nf * (double)(G.row + G.crow) * 8.0 > 120e9) throw VpError{VP_ERR_OOM};
  G.data = vp_alloc<double>(P, (size_t)G.nf * G.row);
  G.cdata = vp_alloc<double>(P, (size_t)G.nf * G.crow);
}

// Far-history grid on the NH lattice: spacing h2 = m h1 (integer m), origin on an NH
// node, period L2 = nf2 h2 >= L_req.  Every FH node then coincides with an NH node, so the restriction
// weights psi_FH((X1(i) - X2(i')) / (w h2 / 2)) depend on i - m i' only: one tap vector for all outputs.
static void setup_grid_fh(vp_plan_s *P, VpGrid &G, double L_req, double kmax) {
  const VpGrid &N = P->nh;
  int64_t n_req = 2 * (int64_t)ceil(L_req * kmax / (2.0 * VP_PI));
  if (n_req < 4) n_req = 4;
  const double h_max = L_req / (double)(2 * n_req);  // sigma = 2
  int64_t m = (int64_t)floor(h_max / N.h * (1.0 + 1e-12));
  if (m < 1) m = 1;
  G.kind = 1;
  G.h = m * N.h;
  G.nf = vp_next_smooth((int64_t)ceil(L_req / G.h));
  if (G.nf < 2 * P->w) G.nf = vp_next_smooth(2 * P->w);
  G.L = G.nf * G.h;
  G.nmode = 2 * (int64_t)ceil(G.L * kmax / (2.0 * VP_PI));
  if (G.nmode > G.nf) G.nmode = G.nf - (G.nf & 1);
  const int64_t j = llround((N.ox - (P->cx - 0.5 * G.L)) / N.h);
  G.ox = N.ox - (double)j * N.h;
  G.oy = N.oy - (double)j * N.h;
  G.row = G.nf;
  G.crow = 2 * (G.nf / 2 + 1);
  P->fh_ratio = (int)m;
  P->fh_shift = j;
  if ((double)G.nf * (double)(G.row + G.crow) * 8.0 > 120e9) throw VpError{VP_ERR_OOM};
  G.data = vp_alloc<double>(P, (size_t)G.nf * G.row);
  G.cdata = vp_alloc<double>(P, (size_t)G.nf * G.crow);
}

// 1D transform of the ES kernel at spacing h: Phi(k) = 2 alpha int_0^1 psi(s) cos(k alpha s) ds, alpha = w h/2
static double es_transform(const vp_plan_s *P, double h, double k, const std::vector<double> &gx,
                           const std::vector<double> &gw) {
  double alpha = P->w * h / 2.0, s = 0.0;
  for (size_t q = 0; q < gx.size(); q++) s += gw[q] * vp_es(gx[q], P->beta) * cos(k * alpha * gx[q]);
  return 2.0 * alpha * s;
}

// 1 / Phi(2 pi m / L)^2, m = 0..nhalf, for the ES kernel at spacing h (deconvolution table)
void vp_es_deconv_table(const vp_plan_s *P, double h, double L, int64_t nhalf, std::vector<double> &out) {
  std::vector<double> gx, gw;
  gauss_legendre01(2 * P->w + 60, gx, gw);
  out.resize(nhalf + 1);
  for (int64_t m = 0; m <= nhalf; m++) {
    double Phi = es_transform(P, h, 2.0 * VP_PI * m / L, gx, gw);
    out[m] = 1.0 / (Phi * Phi);
  }
}

// deconvolution tables: NH kernel psi_1 (one stage); FH kernel psi_1 * psi_2 (NH spread, then restriction)
static void setup_deconv(vp_plan_s *P) {
  std::vector<double> gx, gw;
  gauss_legendre01(2 * P->w + 60, gx, gw);
  for (VpGrid *G : {&P->nh, &P->fh}) {
    int64_t nh = G->nmode / 2;
    std::vector<double> dec(nh + 1);
    for (int64_t m = 0; m <= nh; m++) {
      double k = 2.0 * VP_PI * m / G->L;
      double Phi = es_transform(P, P->nh.h, k, gx, gw);
      if (G->kind == 1) Phi *= es_transform(P, P->fh.h, k, gx, gw);
      dec[m] = 1.0 / (Phi * Phi);
    }
    G->deconv = vp_alloc<double>(P, nh + 1);
    VP_CUDA(cudaMemcpy(G->deconv, dec.data(), sizeof(double) * (nh + 1), cudaMemcpyHostToDevice));
  }
  double h1 = P->nh.h, h2 = P->fh.h;
  P->nh.mult_scale = h1 * h1 / ((double)P->nh.nf * (double)P->nh.nf);
  P->fh.mult_scale = h2 * h2 * (h1 * h1) * (h1 * h1) / ((double)P->fh.nf * (double)P->fh.nf);
}

// Horner coefficients of the W ES taps (Chebyshev interpolation at D+1 nodes, then monomial basis in t)
static void setup_horner(vp_plan_s *P) {
  const int W = P->w, D = VP_HORNER_DEG(W);
  memset(&P->horner, 0, sizeof(P->horner));
  double maxerr = 0.0;
  for (int k = 0; k < W; k++) {
    const int n = D + 1;
    std::vector<double> ch(n, 0.0), fv(n);
    for (int i = 0; i < n; i++) {
      double t = cos(VP_PI * (i + 0.5) / n);
      fv[i] = vp_es((k + 0.5 * (t + 1.0) - 0.5 * W) * 2.0 / W, P->beta);
    }
    for (int j = 0; j < n; j++) {
      double s = 0.0;
      for (int i = 0; i < n; i++) s += fv[i] * cos(VP_PI * j * (i + 0.5) / n);
      ch[j] = s * (j == 0 ? 1.0 : 2.0) / n;
    }
    // Chebyshev -> monomial: T_0 = 1, T_1 = t, T_{j+1} = 2 t T_j - T_{j-1}
    std::vector<double> Tm(n, 0.0), Tp(n, 0.0), Tc(n, 0.0), mono(n, 0.0);
    Tm[0] = 1.0;
    Tc[1 % n] = (n > 1) ? 1.0 : 0.0;
    for (int j = 0; j < n; j++) {
      const std::vector<double> &T = (j == 0) ? Tm : Tc;
      for (int q = 0; q < n; q++) mono[q] += ch[j] * T[q];
      if (j >= 1) {
        for (int q = 0; q < n; q++) Tp[q] = -Tm[q] + (q >= 1 ? 2.0 * Tc[q - 1] : 0.0);
        Tm = Tc;
        Tc = Tp;
      }
    }
    for (int q = 0; q < n; q++) P->horner.c[k][q] = mono[q];
    for (int i = 0; i <= 200; i++) {
      double t = -1.0 + i / 100.0, acc = mono[D];
      for (int q = D - 1; q >= 0; q--) acc = acc * t + mono[q];
      double ex = vp_es((k + 0.5 * (t + 1.0) - 0.5 * W) * 2.0 / W, P->beta);
      maxerr = std::max(maxerr, fabs(acc - ex));
    }
  }
  P->horner_err = maxerr;
  vp_upload_horner(W, P->horner);
  if (!(maxerr <= 0.6 * P->eps)) {  // the fit error floor is the truncated kernel's edge value, ~0.16 eps
    vp_set_last_error("Horner fit of the ES kernel failed");
    throw VpError{VP_ERR_CUDA};
  }
}

// FH <- NH restriction tables (DESIGN.md §NUFFT two-stage FH).  The same host function evaluates
// every weight psi_FH((X1(i) - X2(i')) / (w h2 / 2)) so the prolongation is the exact transpose.
static double rweight(const vp_plan_s *P, int64_t i, int64_t ip) {
  double d = (P->nh.ox - P->fh.ox) + i * P->nh.h - ip * P->fh.h;
  return vp_es(d / (0.5 * P->w * P->fh.h), P->beta);
}
static void setup_restriction(vp_plan_s *P) {
  const double h1 = P->nh.h, h2 = P->fh.h, half = 0.5 * P->w * h2, off = P->nh.ox - P->fh.ox;
  const int64_t n1 = P->nh.nf, n2 = P->fh.nf;
  P->r_ntap = (int)floor(2.0 * half / h1) + 2;
  P->t_ntap = P->w + 1;
  std::vector<int32_t> rlo(n2), tlo(n1);
  std::vector<double> rw((size_t)n2 * P->r_ntap, 0.0), tw((size_t)n1 * P->t_ntap, 0.0);
  int64_t elo = -1, ehi = -1;
  for (int64_t ip = 0; ip < n2; ip++) {
    // NH indices i with |off + i h1 - ip h2| < half
    int64_t lo = (int64_t)ceil((ip * h2 - half - off) / h1);
    rlo[ip] = (int32_t)lo;
    bool any = false;
    for (int t = 0; t < P->r_ntap; t++) {
      int64_t i = lo + t;
      double wv = rweight(P, i, ip);
      rw[(size_t)ip * P->r_ntap + t] = wv;
      if (wv != 0.0 && i >= 0 && i < n1) any = true;
    }
    if (any) {
      if (elo < 0) elo = ip;
      ehi = ip;
    }
  }
  for (int64_t i = 0; i < n1; i++) {
    int64_t lo = (int64_t)ceil((off + i * h1 - half) / h2);
    tlo[i] = (int32_t)lo;
    for (int t = 0; t < P->t_ntap; t++) tw[(size_t)i * P->t_ntap + t] = rweight(P, i, lo + t);
  }
  if (elo < 0) throw VpError{VP_ERR_GEOMETRY};
  P->e_lo = elo;
  P->e_n = ehi - elo + 1;
  // integer ratio: the single tap vector w[q] = psi_FH(2 q / (W m)), |q| < W m / 2, checked against the tables
  {
    const int m = P->fh_ratio;
    const int QH = (P->w * m - 1) / 2;
    bool ok = 2 * QH + 1 <= 192 && fabs(P->fh.h - m * P->nh.h) <= 1e-14 * P->fh.h;
    for (int q = -QH; q <= QH && ok; q++) P->tap_w[q + QH] = vp_es(2.0 * q / (double)(P->w * m), P->beta);
    // spot check: table weight of (i, i') equals w[i + j - m i']
    for (int64_t ip = elo; ip <= ehi && ok; ip += std::max<int64_t>(1, (ehi - elo) / 7)) {
      for (int t = 0; t < P->r_ntap; t++) {
        int64_t i = rlo[ip] + t, q = i + P->fh_shift - m * ip;
        double wt = rw[(size_t)ip * P->r_ntap + t];
        double wq = (q >= -QH && q <= QH) ? P->tap_w[q + QH] : 0.0;
        if (fabs(wt - wq) > 1e-9) ok = false;  // tables carry ~1e-12 rounding of (X1 - X2) at large indices
      }
    }
    P->tap_qh = ok ? QH : 0;
  }
  P->r_lo = vp_alloc<int32_t>(P, n2);
  P->t_lo = vp_alloc<int32_t>(P, n1);
  P->r_w = vp_alloc<double>(P, rw.size());
  P->t_w = vp_alloc<double>(P, tw.size());
  VP_CUDA(cudaMemcpy(P->r_lo, rlo.data(), 4 * n2, cudaMemcpyHostToDevice));
  VP_CUDA(cudaMemcpy(P->t_lo, tlo.data(), 4 * n1, cudaMemcpyHostToDevice));
  VP_CUDA(cudaMemcpy(P->r_w, rw.data(), 8 * rw.size(), cudaMemcpyHostToDevice));
  VP_CUDA(cudaMemcpy(P->t_w, tw.data(), 8 * tw.size(), cudaMemcpyHostToDevice));
  P->scratch = vp_alloc<double>(P, (size_t)n1 * P->e_n);
}

static void make_fft_plans(vp_plan_s *P) {
  size_t ws[4] = {0, 0, 0, 0}, wmax = 0;
  VpGrid *gs[2] = {&P->nh, &P->fh};
  for (int g = 0; g < 2; g++) {
    VpGrid &G = *gs[g];
    vp_fft_setup(P, G);
    if (G.own_fft) continue;
    VP_CUFFT(cufftCreate(&G.fwd));
    VP_CUFFT(cufftCreate(&G.inv));
    VP_CUFFT(cufftSetAutoAllocation(G.fwd, 0));
    VP_CUFFT(cufftSetAutoAllocation(G.inv, 0));
    if (vp_fft4_setup(P, G) && P->opts.fft_rows == 0 && vp_fft4_rows_setup(P, G)) {
      // large grid: own pruned row passes + the four-step column pass (vp_fft.cu); no cuFFT plan
      VP_CUFFT(cufftDestroy(G.fwd));
      VP_CUFFT(cufftDestroy(G.inv));
      G.fwd = G.inv = 0;
      continue;
    }
    if (G.four_step) {  // large grid: cuFFT batched 1D row transforms + the four-step column pass (vp_fft.cu)
      long long n1[1] = {G.nf}, rin1[1] = {G.row}, cin1[1] = {G.crow / 2};
      VP_CUFFT(cufftMakePlanMany64(G.fwd, 1, n1, rin1, 1, G.row, cin1, 1, G.crow / 2, CUFFT_D2Z, G.nf, &ws[2 * g]));
      VP_CUFFT(cufftMakePlanMany64(G.inv, 1, n1, cin1, 1, G.crow / 2, rin1, 1, G.row, CUFFT_Z2D, G.nf,
                                   &ws[2 * g + 1]));
    } else {
      long long n[2] = {G.nf, G.nf};
      long long rin[2] = {G.nf, G.row};         // real layout
      long long cin[2] = {G.nf, G.crow / 2};    // complex layout
      VP_CUFFT(cufftMakePlanMany64(G.fwd, 2, n, rin, 1, G.nf * G.row, cin, 1, G.nf * (G.crow / 2), CUFFT_D2Z, 1,
                                   &ws[2 * g]));
      VP_CUFFT(cufftMakePlanMany64(G.inv, 2, n, cin, 1, G.nf * (G.crow / 2), rin, 1, G.nf * G.row, CUFFT_Z2D, 1,
                                   &ws[2 * g + 1]));
    }
    G.has_plans = true;
  }
  // separate work areas: the NH and FH transforms run concurrently on different streams
  for (int g = 0; g < 2; g++) {
    if (!gs[g]->has_plans) continue;
    void *work = vp_alloc<char>(P, std::max(ws[2 * g], ws[2 * g + 1]) + 256);
    VP_CUFFT(cufftSetWorkArea(gs[g]->fwd, work));
    VP_CUFFT(cufftSetWorkArea(gs[g]->inv, work));
    VP_CUFFT(cufftSetStream(gs[g]->fwd, P->stream));
    VP_CUFFT(cufftSetStream(gs[g]->inv, P->stream));
  }
  (void)wmax;
}


__global__ void k_gather_f64(const double *__restrict__ src, const int32_t *__restrict__ perm, int64_t n,
                             double *__restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}
void vp_gather_f64(const double *src, const int32_t *perm, int64_t n, double *dst, cudaStream_t s) {
  if (n == 0) return;
  k_gather_f64<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(src, perm, n, dst);
  VP_CHECK_LAUNCH();
}

static void free_plan(vp_plan_s *P) {
  if (!P) return;
  for (VpGrid *G : {&P->nh, &P->fh}) {
    if (G->has_plans) {
      cufftDestroy(G->fwd);
      cufftDestroy(G->inv);
    }
  }
  if (P->dlp_has_plans) {
    for (int i = 0; i < 2; i++) {
      if (P->dlp_fwd[i]) cufftDestroy(P->dlp_fwd[i]);
      if (P->dlp_inv[i]) cufftDestroy(P->dlp_inv[i]);
    }
  }
  if (P->bands.has_plans) {
    cufftDestroy(P->bands.fwd);
    cufftDestroy(P->bands.inv);
  }
  if (P->s_h2d) cudaStreamDestroy(P->s_h2d);
  if (P->s_d2h) cudaStreamDestroy(P->s_d2h);
  for (cudaEvent_t e : P->hm_ev)
    if (e) cudaEventDestroy(e);
  if (P->s_fh) cudaStreamDestroy(P->s_fh);
  if (P->s_loc) cudaStreamDestroy(P->s_loc);
  for (cudaEvent_t e : {P->ev_fork, P->ev_fh, P->ev_loc, P->ev_restr})
    if (e) cudaEventDestroy(e);
  for (void *p : P->allocs) cudaFree(p);
  if (P->ev_init)
    for (int i = 0; i < 10; i++) cudaEventDestroy(P->ev[i]);
  delete P;
}

extern "C" vp_status vp_plan(const double *tri_nodes, const double *weights, int64_t M, int32_t p,
                             const double *targets, int64_t T, double tol, const vp_opts *opts, vp_handle *out) {
  if (!out) return VP_ERR_ARG;
  *out = nullptr;
  if (!tri_nodes || !weights || !targets || M <= 0 || p <= 0 || T <= 0) return VP_ERR_ARG;
  if (!(tol >= 1e-14 && tol <= 1e-2)) return VP_ERR_TOL;
  int64_t N = M * (int64_t)p;
  if (N >= ((int64_t)1 << 31) || T >= ((int64_t)1 << 31)) return VP_ERR_UNSUPPORTED;
  vp_plan_s *P = new vp_plan_s();
  auto t0 = std::chrono::steady_clock::now();
  try {
    P->M = M; P->p = p; P->N = N; P->T = T; P->tol = tol;
    if (opts) P->opts = *opts;
    vp_opts &o = P->opts;
    if (o.targets_are_nodes && T < N) throw VpError{VP_ERR_ARG};
    if (o.parts < 0 || o.parts > 3) throw VpError{VP_ERR_ARG};
    if (o.spread_tile < 0 || o.spread_tile > 64 || (o.spread_tile > 0 && o.spread_tile < 8)) throw VpError{VP_ERR_ARG};
    if (o.interp_tile < 0 || o.interp_tile > 128 || (o.interp_tile > 0 && o.interp_tile < 16)) throw VpError{VP_ERR_ARG};
    if (o.interp_tile > 0) P->TSI = o.interp_tile;
    if (o.fft_mode < 0 || o.fft_mode > 1) throw VpError{VP_ERR_ARG};
    if (o.spread_pack < 0 || o.spread_pack > 2) throw VpError{VP_ERR_ARG};
    if (o.fft_rows < 0 || o.fft_rows > 1) throw VpError{VP_ERR_ARG};
    if (o.boundary.kind == VP_BDRY_CIRCLE && !(o.boundary.p[2] > 0)) throw VpError{VP_ERR_GEOMETRY};
    if (o.boundary.kind == VP_BDRY_RECT && !(o.boundary.p[2] > o.boundary.p[0] && o.boundary.p[3] > o.boundary.p[1]))
      throw VpError{VP_ERR_GEOMETRY};
    if (o.boundary.kind < VP_BDRY_NONE || o.boundary.kind > VP_BDRY_CHUNKS) throw VpError{VP_ERR_GEOMETRY};
    o.boundary.pts = nullptr;  // host pointer valid during vp_plan only: read through opts->boundary below
    P->stream = (cudaStream_t)o.cuda_stream;
    P->eps = o.eps_nufft > 0 ? o.eps_nufft : tol;
    // ---- statistics
    const int nblk = 148 * 4;
    double *d_sum, *d_box;
    int *d_bad;
    VP_CUDA(cudaMallocAsync(&d_sum, sizeof(double) * nblk, P->stream));
    VP_CUDA(cudaMallocAsync(&d_box, sizeof(double) * 4 * nblk, P->stream));
    VP_CUDA(cudaMallocAsync(&d_bad, sizeof(int), P->stream));
    VP_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), P->stream));
    k_stats<<<nblk, 256, 0, P->stream>>>(tri_nodes, weights, N, targets, T, d_sum, d_box, d_bad);
    VP_CHECK_LAUNCH();
    std::vector<double> hs(nblk), hb(4 * nblk);
    int hbad = 0;
    VP_CUDA(cudaMemcpyAsync(hs.data(), d_sum, sizeof(double) * nblk, cudaMemcpyDeviceToHost, P->stream));
    VP_CUDA(cudaMemcpyAsync(hb.data(), d_box, sizeof(double) * 4 * nblk, cudaMemcpyDeviceToHost, P->stream));
    VP_CUDA(cudaMemcpyAsync(&hbad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
    VP_CUDA(cudaStreamSynchronize(P->stream));
    VP_CUDA(cudaFree(d_sum)); VP_CUDA(cudaFree(d_box)); VP_CUDA(cudaFree(d_bad));
    if (hbad) throw VpError{VP_ERR_NONFINITE};
    double sumw = 0, x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
    for (int i = 0; i < nblk; i++) {
      sumw += hs[i];
      x0 = std::min(x0, hb[4 * i]); x1 = std::max(x1, hb[4 * i + 1]);
      y0 = std::min(y0, hb[4 * i + 2]); y1 = std::max(y1, hb[4 * i + 3]);
    }
    if (!(sumw > 0)) throw VpError{VP_ERR_ARG};
    // the grid frame also covers a CHUNKS / POLYGON boundary (host array): its nodes are the layer potentials'
    // sources (vp_layer.cu)
    if (opts && opts->boundary.pts && opts->boundary.n > 0 &&
        (opts->boundary.kind == VP_BDRY_CHUNKS || opts->boundary.kind == VP_BDRY_POLYGON)) {
      const vp_boundary &bd = opts->boundary;
      const int64_t np = bd.kind == VP_BDRY_CHUNKS ? bd.n * (int64_t)(bd.q + 1) : bd.n;
      if (bd.kind == VP_BDRY_CHUNKS && (bd.q < 1 || bd.q > VP_CHUNK_MAXQ)) throw VpError{VP_ERR_GEOMETRY};
      for (int64_t i = 0; i < np; i++) {
        const double bx = bd.pts[2 * i], by = bd.pts[2 * i + 1];
        if (!std::isfinite(bx) || !std::isfinite(by)) throw VpError{VP_ERR_NONFINITE};
        x0 = std::min(x0, bx); x1 = std::max(x1, bx);
        y0 = std::min(y0, by); y1 = std::max(y1, by);
      }
    }
    // ---- parameters
    P->dx2 = sumw / (double)N;
    double C = o.C > 0 ? o.C : 3.0;
    double ratio = o.delta2_over_delta1 > 0 ? o.delta2_over_delta1 : 32.0;
    if (ratio <= 1.0) throw VpError{VP_ERR_ARG};
    P->delta1 = o.delta1_override > 0 ? o.delta1_override : C * P->dx2;
    P->delta2 = ratio * P->delta1;
    P->S = std::max(std::max(x1 - x0, y1 - y0), 1e-300);
    P->cx = 0.5 * (x0 + x1);
    P->cy = 0.5 * (y0 + y1);
    double lne = log(1.0 / P->eps);
    P->w = std::min(16, std::max(4, (int)ceil(log10(1.0 / P->eps)) + 1));
    P->beta = 2.30 * P->w;
    P->kmax_nh = sqrt(lne / P->delta1);
    P->kmax_fh = sqrt(lne / P->delta2);
    double zeps = vp_solve_e1(P->eps);
    double m2 = sqrt(4.0 * P->delta2 * lne);
    // margins: the kernel decay and (>= w+4 fine cells) so that spreading never wraps
    double L_nh = P->S + std::max(sqrt(4.0 * P->delta2 * zeps), (P->w + 4) * (VP_PI / P->kmax_nh) / 2.0);
    P->R = sqrt(2.0) * P->S + m2;
    double L_fh = P->S + P->R + m2;
    setup_grid(P, P->nh, 0, L_nh, P->kmax_nh);
    P->nh.delta_a = P->delta1; P->nh.delta_b = P->delta2;
    setup_grid_fh(P, P->fh, L_fh, P->kmax_fh);
    P->fh.delta_a = P->delta2; P->fh.delta_b = P->R;
    {  // boundary geometry of the local part (validated and uploaded; the caller's host array is read here only)
      vp_opts tmp = P->opts;
      if (opts) P->opts.boundary = opts->boundary;
      try {
        vp_build_boundary(P, P->bdev);
      } catch (...) {
        P->opts = tmp;
        throw;
      }
      P->opts = tmp;
    }
    setup_horner(P);
    setup_deconv(P);
    setup_restriction(P);
    // ---- sources and targets sorted by NH tile
    P->sp.det = o.deterministic ? 1 : 0;
    P->bands.sp.det = P->sp.det;
    if (P->sp.det || o.spread_tile > 0)  // tile batches: deterministic colouring, or explicitly requested
      vp_build_spread_order(P, P->sp, tri_nodes, weights, nullptr, N, grid_args(P->nh));
    else
      vp_build_strip_order(P, P->sp, tri_nodes, weights, nullptr, N, grid_args(P->nh));
    P->dmode = o.deriv_mode;
    if (P->dmode == VP_DERIV_AUTO) P->dmode = (o.ref_nodes && N > 10000000) ? VP_DERIV_TRIANGLE : VP_DERIV_KNN;
    vp_build_interp_order(P, targets, T);
    // ---- graded meshes: per-target levels and band boxes (a12)
    int parts = o.parts ? o.parts : VP_PART_ALL;
    if (parts & VP_PART_LOCAL) {
      vp_build_levels(P, tri_nodes, weights);
    } else {
      P->bands.tlev = vp_alloc<int8_t>(P, T);
      VP_CUDA(cudaMemsetAsync(P->bands.tlev, 0, T, P->stream));
    }
    // ---- local part
    if (P->dmode == VP_DERIV_TRIANGLE && (!o.ref_nodes || p < 10 || p > VP_TRI_MAXP || !o.targets_are_nodes))
      throw VpError{VP_ERR_UNSUPPORTED};
    if (P->dmode != VP_DERIV_KNN && P->dmode != VP_DERIV_TRIANGLE) throw VpError{VP_ERR_ARG};
    P->deg = o.deriv_degree > 0 ? o.deriv_degree : (N > 1000000 ? 4 : 6);
    if (P->deg > VP_MAXDEG) throw VpError{VP_ERR_ARG};
    while (P->deg > 0 && 2 * vp_ncoef(P->deg) > N && o.deriv_degree <= 0) P->deg--;  // tiny inputs
    int nc = vp_ncoef(P->deg);
    // K: 2 x #monomials at degree >= 5; degree 4 needs fewer (config 2: 1.30e-9 at K = 17, 20, 24 and 30)
    P->K = o.deriv_k > 0 ? o.deriv_k : (P->deg >= 5 ? 2 * nc : nc + 6);
    if (P->K > 64) P->K = 64;
    if (P->K > N && o.deriv_k <= 0) P->K = (int)N;
    if (P->K < nc) throw VpError{VP_ERR_ARG};
    if (P->K > N) throw VpError{VP_ERR_ARG};
    if (parts & VP_PART_LOCAL) {
      vp_build_local(P, tri_nodes);
      if (P->n_stencil > 0) {
        P->fs = vp_alloc<double>(P, N);
        P->sp.fs_out = P->fs;
        vp_remap_stencils(P);
      }
    } else {
      P->K = 0;
      P->lalpha = vp_alloc<double>(P, 1);
      P->lnode = vp_alloc<int32_t>(P, 1);
      P->lidx = vp_alloc<int32_t>(P, 1);
      P->lw = vp_alloc<double>(P, 1);
      P->lptr = vp_alloc<int32_t>(P, 1);
    }
    // ---- FFT plans, forked streams
    make_fft_plans(P);
    VP_CUDA(cudaStreamCreateWithFlags(&P->s_fh, cudaStreamNonBlocking));
    VP_CUDA(cudaStreamCreateWithFlags(&P->s_loc, cudaStreamNonBlocking));
    VP_CUDA(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
    VP_CUDA(cudaEventCreateWithFlags(&P->ev_fh, cudaEventDisableTiming));
    VP_CUDA(cudaEventCreateWithFlags(&P->ev_loc, cudaEventDisableTiming));
    VP_CUDA(cudaEventCreateWithFlags(&P->ev_restr, cudaEventDisableTiming));
    VP_CUDA(cudaStreamSynchronize(P->stream));
    VP_CUDA(cudaGetLastError());
  } catch (VpError &e) {
    cudaStreamSynchronize(P->stream);
    cudaGetLastError();
    free_plan(P);
    return e.s;
  } catch (...) {
    free_plan(P);
    return VP_ERR_CUDA;
  }
  P->plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  *out = P;
  return VP_OK;
}

// the three transform steps of one history grid: fused kernels (vp_fft.cu) or cuFFT + k_multiply
static void grid_fft_fwd(vp_plan_s *P, VpGrid &G) {
  if (G.own_fft) return vp_fft_forward(P, G);
  if (G.f4_rows) return vp_fft4_rows_fwd(P, G);
  VP_CUFFT(cufftSetStream(G.fwd, P->stream));
  VP_CUFFT(cufftExecD2Z(G.fwd, G.data, (cufftDoubleComplex *)G.cdata));
  P->n_ffts++;
}
static void grid_multiply(vp_plan_s *P, VpGrid &G) {
  if (G.own_fft) return vp_fft_columns(P, G);
  if (G.four_step) return vp_fft4_columns(P, G);  // column FFT + multiply + inverse column FFT
  vp_launch_multiply(P, G);
}
static void grid_fft_inv(vp_plan_s *P, VpGrid &G) {
  if (G.own_fft) return vp_fft_inverse(P, G);
  if (G.f4_rows) return vp_fft4_rows_inv(P, G);
  VP_CUFFT(cufftSetStream(G.inv, P->stream));
  VP_CUFFT(cufftExecZ2D(G.inv, (cufftDoubleComplex *)G.cdata, G.data));
  P->n_ffts++;
}

// inverse transforms of both grids and the far-history prolongation q1 += R^T q2: with own NH row passes the
// prolongation's x pass runs inside the NH inverse row pass (vp_fft4_rows_inv_prolong), after the FH inverse and
// the y pass
static void grids_inverse_prolong(vp_plan_s *P) {
  if (vp_fft4_rows_prolong_ok(P)) {
    grid_fft_inv(P, P->fh);
    vp_launch_prolong(P, 1);
    vp_fft4_rows_inv_prolong(P);
    return;
  }
  grid_fft_inv(P, P->nh);
  grid_fft_inv(P, P->fh);
  vp_launch_prolong(P, 3);
}

static void record(vp_plan_s *P, int i) {
  if (P->profiling) cudaEventRecord(P->ev[i], P->stream);
}

// Fork/join eval (no profiling): after the spread, the far-history chain (restriction, FH transforms,
// prolongation pass B^T) runs on stream B and the local part (stencils, triangle fits) on stream C while
// the near-history transforms run on the caller's stream A; A joins both before the interpolation.
// Cross-eval hazards: B and C start after A's spread of this eval, i.e. after A finished every read of
// the previous eval's scratch (t2), V_L buffers and grids.
struct StreamScope {
  vp_plan_s *P;
  cudaStream_t old;
  StreamScope(vp_plan_s *p, cudaStream_t s) : P(p), old(p->stream) { P->stream = s; }
  ~StreamScope() { P->stream = old; }
};

// everything after the spread (the NH grid already holds this field's spread)
static void eval_concurrent_after_spread(vp_plan_s *P, const double *f, double *out, int parts);

static void eval_concurrent(vp_plan_s *P, const double *f, double *out, int parts) {
  VP_CUDA(cudaMemsetAsync(P->nh.data, 0, sizeof(double) * P->nh.nf * P->nh.row, P->stream));
  vp_launch_spread(P, P->sp, grid_args(P->nh), f);
  eval_concurrent_after_spread(P, f, out, parts);
}

static void eval_concurrent_after_spread(vp_plan_s *P, const double *f, double *out, int parts) {
  cudaStream_t A = P->stream;
  VP_CUDA(cudaEventRecord(P->ev_fork, A));
  {  // B: far history
    StreamScope sc(P, P->s_fh);
    VP_CUDA(cudaStreamWaitEvent(P->s_fh, P->ev_fork, 0));
    VP_CUDA(cudaMemsetAsync(P->fh.data, 0, sizeof(double) * P->fh.nf * P->fh.row, P->s_fh));
    vp_launch_restrict(P);
    VP_CUDA(cudaEventRecord(P->ev_restr, P->s_fh));  // the restriction's last read of the spread NH grid
    grid_fft_fwd(P, P->fh);
    grid_multiply(P, P->fh);
    grid_fft_inv(P, P->fh);
    vp_launch_prolong(P, 1);
    VP_CUDA(cudaEventRecord(P->ev_fh, P->s_fh));
  }
  bool local_forked = false;
  if (parts & VP_PART_LOCAL) {  // C: local part
    StreamScope sc(P, P->s_loc);
    VP_CUDA(cudaStreamWaitEvent(P->s_loc, P->ev_fork, 0));
    vp_launch_tri_local(P, f);
    VP_CUDA(cudaEventRecord(P->ev_loc, P->s_loc));
    local_forked = true;
  }
  // A: near history, join, interpolation
  grid_fft_fwd(P, P->nh);
  grid_multiply(P, P->nh);
  // the NH inverse transform overwrites the NH grid that stream B's restriction reads: wait for it
  VP_CUDA(cudaStreamWaitEvent(A, P->ev_restr, 0));
  grid_fft_inv(P, P->nh);
  VP_CUDA(cudaStreamWaitEvent(A, P->ev_fh, 0));
  vp_launch_prolong(P, 2);
  if (local_forked) VP_CUDA(cudaStreamWaitEvent(A, P->ev_loc, 0));
  vp_launch_interp_local(P, f, out, false);
  if (parts & VP_PART_LOCAL) vp_launch_bands(P, f, out);
}

extern "C" vp_status vp_eval(vp_handle P, const double *f, double *out) {
  if (!P || !f || !out) return VP_ERR_ARG;
  try {
    P->n_kernels = 0;
    P->n_ffts = 0;
    int parts = P->opts.parts ? P->opts.parts : VP_PART_ALL;
    if (P->profiling && !P->ev_init) {
      for (int i = 0; i < 10; i++) VP_CUDA(cudaEventCreate(&P->ev[i]));
      P->ev_init = true;
    }
    // fork/join pays only when the kernels leave the GPU partly idle: measured faster for config 2 (2744^2
    // grids: 0.97 vs 1.03 ms), slower for configs 3-5 (c5: 63.5 vs 58.5 ms)
    if (!P->profiling && P->concurrent && P->nh.nf <= 6000 && (parts & VP_PART_HISTORY)) {
      eval_concurrent(P, f, out, parts);
      return VP_OK;
    }
    record(P, 0);
    if (parts & VP_PART_HISTORY) {
      VP_CUDA(cudaMemsetAsync(P->nh.data, 0, sizeof(double) * P->nh.nf * P->nh.row, P->stream));
      VP_CUDA(cudaMemsetAsync(P->fh.data, 0, sizeof(double) * P->fh.nf * P->fh.row, P->stream));
      record(P, 1);
      vp_launch_spread(P, P->sp, grid_args(P->nh), f);
      record(P, 2);
      vp_launch_restrict(P);
      record(P, 3);
      grid_fft_fwd(P, P->nh);
      grid_fft_fwd(P, P->fh);
      record(P, 4);
      grid_multiply(P, P->nh);
      grid_multiply(P, P->fh);
      record(P, 5);
      if (vp_fft4_rows_prolong_ok(P)) {  // the prolongation's x pass is fused into the NH inverse rows
        grid_fft_inv(P, P->fh);
        vp_launch_prolong(P, 1);
        vp_fft4_rows_inv_prolong(P);
        record(P, 6);
      } else {
        grid_fft_inv(P, P->nh);
        grid_fft_inv(P, P->fh);
        record(P, 6);
        vp_launch_prolong(P, 3);
      }
      record(P, 7);
    } else {
      for (int i = 1; i <= 7; i++) record(P, i);
    }
    vp_launch_interp_local(P, f, out, true);
    record(P, 8);
    if (parts & VP_PART_LOCAL) vp_launch_bands(P, f, out);
    record(P, 9);
    P->n_phase = 9;
  } catch (VpError &e) {
    return e.s;
  }
  return VP_OK;
}

extern "C" vp_status vp_eval_batch(vp_handle P, int32_t K, const double *f, double *out) {
  if (!P || !f || !out || K < 1) return VP_ERR_ARG;
  if (K == 1) return vp_eval(P, f, out);
  try {
    if (!P->sp.strip) throw VpError{VP_ERR_UNSUPPORTED};
    const int parts = P->opts.parts ? P->opts.parts : VP_PART_ALL;
    const size_t gcells = (size_t)P->nh.nf * P->nh.row;
    if (P->bcap < K) {  // plan-owned extra grids (released with the plan); the smaller set is freed first
      VP_CUDA(cudaStreamSynchronize(P->stream));  // no queued work of a previous batch still uses them
      vp_free(P, P->bgrid);
      vp_free(P, P->fs_batch);
      P->bgrid = P->fs_batch = nullptr;
      P->bcap = 1;
      P->bgrid = vp_alloc<double>(P, gcells * (size_t)(K - 1));
      if (P->fs) P->fs_batch = vp_alloc<double>(P, (size_t)P->N * K);
      P->bcap = K;
    }
    P->n_kernels = 0;
    P->n_ffts = 0;
    std::vector<const double *> fk(K);
    std::vector<double *> gk(K), fsk(K, nullptr);
    for (int k = 0; k < K; k++) {
      fk[k] = f + (size_t)k * P->N;
      gk[k] = k == 0 ? P->nh.data : P->bgrid + gcells * (size_t)(k - 1);
      if (P->fs) fsk[k] = P->fs_batch + (size_t)k * P->N;
    }
    double *const data0 = P->nh.data, *const fs0 = P->fs;
    if (parts & VP_PART_HISTORY) {
      for (int k = 0; k < K; k++) VP_CUDA(cudaMemsetAsync(gk[k], 0, sizeof(double) * gcells, P->stream));
      vp_launch_spread_batch(P, P->sp, grid_args(P->nh), K, fk.data(), gk.data(), P->fs ? fsk.data() : nullptr);
    }
    // per field: the fork/join schedule of vp_eval where it pays (small grids), else serial; a field's far-
    // history and local streams start after the caller's stream finished the previous field (ev_fork)
    const bool conc = P->concurrent && P->nh.nf <= 6000 && (parts & VP_PART_HISTORY);
    try {
      for (int k = 0; k < K; k++) {
        P->nh.data = gk[k];
        if (P->fs) P->fs = fsk[k];
        if (conc) {
          eval_concurrent_after_spread(P, fk[k], out + (size_t)k * P->T, parts);
          continue;
        }
        if (parts & VP_PART_HISTORY) {
          VP_CUDA(cudaMemsetAsync(P->fh.data, 0, sizeof(double) * P->fh.nf * P->fh.row, P->stream));
          vp_launch_restrict(P);
          grid_fft_fwd(P, P->nh);
          grid_fft_fwd(P, P->fh);
          grid_multiply(P, P->nh);
          grid_multiply(P, P->fh);
          grids_inverse_prolong(P);
        }
        vp_launch_interp_local(P, fk[k], out + (size_t)k * P->T, true);
        if (parts & VP_PART_LOCAL) vp_launch_bands(P, fk[k], out + (size_t)k * P->T);
      }
    } catch (...) {
      P->nh.data = data0;
      P->fs = fs0;
      throw;
    }
    P->nh.data = data0;
    P->fs = fs0;
    P->n_phase = 0;
  } catch (VpError &e) {
    return e.s;
  }
  return VP_OK;
}

extern "C" vp_status vp_layer_set_levels(vp_handle P, int32_t J) {
  if (!P || J < 0 || J > 8 || P->lay_common) return VP_ERR_ARG;
  P->lay_J = J;
  return VP_OK;
}

extern "C" vp_status vp_slp_prepare(vp_handle P) {
  if (!P) return VP_ERR_ARG;
  try {
    vp_slp_build(P);
  } catch (VpError &e) {
    return e.s;
  }
  return VP_OK;
}

// single-layer potential S[sigma] at the plan's targets (vp_layer.cu): history part through the volume path's
// grids with the boundary nodes as sources, then the local stencils of the targets near the boundary
extern "C" vp_status vp_eval_slp(vp_handle P, const double *sigma, double *out) {
  if (!P || !sigma || !out) return VP_ERR_ARG;
  try {
    if (!P->slp_ready) throw VpError{VP_ERR_ARG};
    P->n_kernels = 0;
    P->n_ffts = 0;
    VP_CUDA(cudaMemsetAsync(P->nh.data, 0, sizeof(double) * P->nh.nf * P->nh.row, P->stream));
    VP_CUDA(cudaMemsetAsync(P->fh.data, 0, sizeof(double) * P->fh.nf * P->fh.row, P->stream));
    VpSpreadSet S = P->bsp;
    S.fs_out = nullptr;
    vp_launch_spread(P, S, grid_args(P->nh), sigma);
    vp_launch_restrict(P);
    grid_fft_fwd(P, P->nh);
    grid_fft_fwd(P, P->fh);
    grid_multiply(P, P->nh);
    grid_multiply(P, P->fh);
    grids_inverse_prolong(P);
    vp_launch_interp_hist(P, out);
    vp_launch_slp_local(P, sigma, out);
  } catch (VpError &e) {
    return e.s;
  }
  return VP_OK;
}

extern "C" vp_status vp_dlp_prepare(vp_handle P) {
  if (!P) return VP_ERR_ARG;
  try {
    vp_dlp_build(P);
  } catch (VpError &e) {
    return e.s;
  }
  return VP_OK;
}

// double-layer potential D[mu] at the plan's targets (vp_layer.cu): the D history is the volume path's history of
// the spectral-derivative source grid g~ = -(d_1 g_1 + d_2 g_2) (lemmas dnearkspace / dfarkspace, reading R20),
// then the local stencils (eq. dlplocO5, reading R21)
extern "C" vp_status vp_eval_dlp(vp_handle P, const double *mu, double *out) {
  if (!P || !mu || !out) return VP_ERR_ARG;
  try {
    if (!P->dlp_ready) throw VpError{VP_ERR_ARG};
    P->n_kernels = 0;
    P->n_ffts = 0;
    vp_dlp_source_grids(P, mu);
    grid_fft_fwd(P, P->nh);
    grid_fft_fwd(P, P->fh);
    grid_multiply(P, P->nh);
    grid_multiply(P, P->fh);
    grids_inverse_prolong(P);
    vp_launch_interp_hist(P, out);
    vp_launch_dlp_local(P, mu, out);
  } catch (VpError &e) {
    return e.s;
  }
  return VP_OK;
}

extern "C" vp_status vp_eval_host(vp_handle P, const double *f_host, double *out_host) {
  if (!P || !f_host || !out_host) return VP_ERR_ARG;
  try {
    if (!P->f_dev) P->f_dev = vp_alloc<double>(P, P->N);
    if (!P->out_dev) P->out_dev = vp_alloc<double>(P, P->T);
    VP_CUDA(cudaMemcpyAsync(P->f_dev, f_host, sizeof(double) * P->N, cudaMemcpyHostToDevice, P->stream));
    vp_status s = vp_eval(P, P->f_dev, P->out_dev);
    if (s != VP_OK) return s;
    VP_CUDA(cudaMemcpyAsync(out_host, P->out_dev, sizeof(double) * P->T, cudaMemcpyDeviceToHost, P->stream));
    VP_CUDA(cudaStreamSynchronize(P->stream));
  } catch (VpError &e) {
    return e.s;
  }
  return VP_OK;
}

// K fields from HOST memory with the transfers overlapped across fields: H2D of field k+1 (stream s_h2d) and
// D2H of field k-1 (stream s_d2h) run while field k is evaluated on the plan's stream (two device slots for f and
// out; PCIe is full duplex).  Ordered after earlier work on the plan's stream; the plan's stream waits for the last
// D2H before the call synchronises it and returns.
extern "C" vp_status vp_eval_host_many(vp_handle P, int32_t K, const double *const *f_host, double *const *out_host) {
  if (!P || K < 1 || !f_host || !out_host) return VP_ERR_ARG;
  for (int32_t k = 0; k < K; k++)
    if (!f_host[k] || !out_host[k]) return VP_ERR_ARG;
  try {
    if (!P->hm_ready) {
      for (int b = 0; b < 2; b++) {
        P->hm_f[b] = vp_alloc<double>(P, P->N);
        P->hm_out[b] = vp_alloc<double>(P, P->T);
      }
      VP_CUDA(cudaStreamCreateWithFlags(&P->s_h2d, cudaStreamNonBlocking));
      VP_CUDA(cudaStreamCreateWithFlags(&P->s_d2h, cudaStreamNonBlocking));
      for (cudaEvent_t &e : P->hm_ev) VP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      P->hm_ready = true;
    }
    cudaEvent_t ev_start = P->hm_ev[0], *ev_in = P->hm_ev + 1, *ev_done = P->hm_ev + 3, *ev_out = P->hm_ev + 5;
    const size_t fb = sizeof(double) * P->N, ob = sizeof(double) * P->T;
    VP_CUDA(cudaEventRecord(ev_start, P->stream));
    VP_CUDA(cudaStreamWaitEvent(P->s_h2d, ev_start, 0));
    VP_CUDA(cudaStreamWaitEvent(P->s_d2h, ev_start, 0));
    auto h2d = [&](int32_t k) {
      const int b = k & 1;
      if (k >= 2) VP_CUDA(cudaStreamWaitEvent(P->s_h2d, ev_done[b], 0));  // eval k-2 has finished reading slot b
      VP_CUDA(cudaMemcpyAsync(P->hm_f[b], f_host[k], fb, cudaMemcpyHostToDevice, P->s_h2d));
      VP_CUDA(cudaEventRecord(ev_in[b], P->s_h2d));
    };
    h2d(0);
    for (int32_t k = 0; k < K; k++) {
      const int b = k & 1;
      if (k + 1 < K) h2d(k + 1);
      VP_CUDA(cudaStreamWaitEvent(P->stream, ev_in[b], 0));
      if (k >= 2) VP_CUDA(cudaStreamWaitEvent(P->stream, ev_out[b], 0));  // D2H of k-2 has read out slot b
      const vp_status st = vp_eval(P, P->hm_f[b], P->hm_out[b]);
      if (st != VP_OK) throw VpError{st};
      VP_CUDA(cudaEventRecord(ev_done[b], P->stream));
      VP_CUDA(cudaStreamWaitEvent(P->s_d2h, ev_done[b], 0));
      VP_CUDA(cudaMemcpyAsync(out_host[k], P->hm_out[b], ob, cudaMemcpyDeviceToHost, P->s_d2h));
      VP_CUDA(cudaEventRecord(ev_out[b], P->s_d2h));
    }
    VP_CUDA(cudaStreamWaitEvent(P->stream, ev_out[(K - 1) & 1], 0));
    VP_CUDA(cudaStreamSynchronize(P->stream));
  } catch (VpError &e) {
    cudaStreamSynchronize(P->stream);
    if (P->s_h2d) cudaStreamSynchronize(P->s_h2d);
    if (P->s_d2h) cudaStreamSynchronize(P->s_d2h);
    return e.s;
  }
  return VP_OK;
}

extern "C" vp_status vp_check_finite(vp_handle P, const double *f) {
  if (!P || !f) return VP_ERR_ARG;
  try {
    int *d_bad, hbad = 0;
    VP_CUDA(cudaMallocAsync(&d_bad, sizeof(int), P->stream));
    VP_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), P->stream));
    k_check_finite<<<148 * 4, 256, 0, P->stream>>>(f, P->N, d_bad);
    VP_CHECK_LAUNCH();
    VP_CUDA(cudaMemcpyAsync(&hbad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
    VP_CUDA(cudaStreamSynchronize(P->stream));
    VP_CUDA(cudaFree(d_bad));
    return hbad ? VP_ERR_NONFINITE : VP_OK;
  } catch (VpError &e) {
    return e.s;
  }
}

extern "C" vp_status vp_destroy(vp_handle P) {
  if (!P) return VP_OK;
  cudaStreamSynchronize(P->stream);
  free_plan(P);
  return VP_OK;
}

extern "C" vp_status vp_get_info(vp_handle P, vp_info *I) {
  if (!P || !I) return VP_ERR_ARG;
  memset(I, 0, sizeof(*I));
  I->M = P->M; I->N = P->N; I->T = P->T; I->p = P->p; I->w_es = P->w; I->beta_es = P->beta;
  I->dx2 = P->dx2; I->delta1 = P->delta1; I->delta2 = P->delta2;
  I->kmax_nh = P->kmax_nh; I->kmax_fh = P->kmax_fh; I->L_nh = P->nh.L; I->L_fh = P->fh.L; I->R_trunc = P->R;
  I->nf_nh = P->nh.nf; I->nf_fh = P->fh.nf; I->nmode_nh = P->nh.nmode; I->nmode_fh = P->fh.nmode;
  I->x0 = P->cx; I->y0 = P->cy; I->S = P->S;
  I->deriv_mode = P->dmode; I->deriv_degree = P->deg; I->deriv_k = P->K;
  I->n_boundary_targets = P->n_bdry;
  I->plan_ms = P->plan_ms;
  I->n_stencil_targets = P->n_stencil;
  I->n_batches = P->sp.n_batches;
  I->horner_err = P->horner_err;
  I->device_bytes = P->device_bytes;
  I->n_levels = P->bands.nlev;
  I->n_boxes = P->bands.nbox;
  I->n_level_targets = P->bands.n_lt;
  I->n_band_pairs = P->bands.n_pairs;
  I->nf_band = P->bands.nfb;
  for (int i = 0; i < 16; i++) I->level_targets[i] = P->bands.lev_count[i];
  I->fft_path_nh = P->nh.own_fft ? 0 : (P->nh.four_step ? (P->nh.f4_rows ? 3 : 2) : 1);
  I->fft_path_fh = P->fh.own_fft ? 0 : (P->fh.four_step ? (P->fh.f4_rows ? 3 : 2) : 1);
  return VP_OK;
}

extern "C" vp_status vp_set_profiling(vp_handle P, int32_t on) {
  if (!P) return VP_ERR_ARG;
  P->profiling = on != 0;
  return VP_OK;
}

static const char *g_phase_names[9] = {"zero",    "spread",  "restrict",     "fft_fwd", "multiply",
                                       "fft_inv", "prolong", "interp_local", "bands"};

extern "C" vp_status vp_get_phase_times(vp_handle P, double *ms, int32_t *n_out, const char **names) {
  if (!P || !ms || !n_out) return VP_ERR_ARG;
  if (!P->profiling || !P->ev_init) return VP_ERR_ARG;
  if (cudaEventSynchronize(P->ev[9]) != cudaSuccess) return VP_ERR_CUDA;
  for (int i = 0; i < 9; i++) {
    float t = 0.f;
    cudaEventElapsedTime(&t, P->ev[i], P->ev[i + 1]);
    ms[i] = t;
    if (names) names[i] = g_phase_names[i];
  }
  *n_out = 9;
  return VP_OK;
}

extern "C" vp_status vp_eval_launch_count(vp_handle P, int32_t *kernels, int32_t *fft_execs) {
  if (!P || !kernels || !fft_execs) return VP_ERR_ARG;
  *kernels = P->n_kernels;
  *fft_execs = P->n_ffts;
  return VP_OK;
}

// ---------------------------------------------------------------------------------------------
// host-callable diagnostics of the method's scalar math (CPU unit tests of host logic)
extern "C" int vp_debug_local_coef(int kind, const double *bp, double x, double y, double delta, int nterms, int deg,
                                   double *coef15) {
  bool b = false;
  if (kind == VP_BDRY_CIRCLE) b = vp_coef_circle(x, y, bp[0], bp[1], bp[2], delta, nterms, deg, coef15);
  else if (kind == VP_BDRY_RECT) b = vp_coef_rect(x, y, bp[0], bp[1], bp[2], bp[3], delta, deg, coef15);
  if (!b) vp_coef_interior(delta, nterms, deg, coef15);
  return b ? 1 : 0;
}
extern "C" double vp_debug_mult(int kind, double k2, double a, double b) {
  return kind == 0 ? vp_mult_nh(k2, a, b) : vp_mult_fh(k2, a, b);
}
extern "C" double vp_debug_e1(double x) { return host_e1(x); }
