// vp_fft.cu -- fused 2D real FFT + spectral multiply for the history grids (
// PAPER.md §3 Steps 2-4, lines 826-893).  Replaces cuFFT D2Z -> k_multiply -> cuFFT Z2D (four to five
// full passes over the half spectrum per transform) by three passes:
//   row pass (forward): one CTA per grid row, the real row read as nf/2 complex values (z[j] = x[2j] +
//       i x[2j+1]), a mixed-radix decimation-in-frequency FFT in shared memory, the real-to-complex split
//       X[k] = Ze[k] + W_nf^k Zo[k], and only the kept columns k <= nmode/2 written;
//   column pass: one CTA per block of kept columns: forward DIF FFT of each column (output in digit-
//       reversed order), the multiplier of k_multiply (NH or FH kernel, ES deconvolution, trapezoid and
//       1/nf^2 scale, truncation |m| <= nmode/2) applied per element, inverse DIT FFT (digit-reversed
//       input, natural output) -- one HBM round trip instead of forward + multiply + inverse;
//   row pass (inverse): the complex-to-real merge Z[k] = Ze[k] + i Zo[k] written to the digit-reversed
//       positions, an inverse DIT FFT, the real row written back.
// Transforms are unnormalised (as cuFFT), so the multiplier tables are shared with the cuFFT path.
// Mixed radix n = r_0 r_1 ... r_{S-1} (r in {2,3,4,5,7,8}), L_s = r_0 ... r_s.  DIT stage s combines r_s
// sub-transforms of length L_{s-1}: positions b L_s + k1 + L_{s-1} t, twiddle W_{L_s}^{t k1}, then an r_s-point
// DFT; DIF runs the transposed stages in reverse order (DFT, then twiddle by the output index).  DIF output /
// DIT input position p = sum_s p_s L_{s-1} holds frequency sigma(p) = sum_s p_s n / L_s.
#include <algorithm>
#include <cmath>
#include <vector>

#include "vp_common.cuh"
#include "vp_math.cuh"

#define VP_FFT_MAXS 16

struct FftStages {
  int n, S;
  int r[VP_FFT_MAXS];
  int Lp[VP_FFT_MAXS];  // L_{s-1}
};

__constant__ double c_dft_c[9][8];  // cos(2 pi j / R), R = 2..8
__constant__ double c_dft_s[9][8];  // sin(2 pi j / R)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// in-place R-point DFT, sign DIR (-1 forward, +1 inverse)
template <int R, int DIR>
__device__ __forceinline__ void dft_small(double2 (&v)[R]) {
  if (R == 2) {
    const double2 a = v[0], b = v[1];
    v[0] = make_double2(a.x + b.x, a.y + b.y);
    v[1] = make_double2(a.x - b.x, a.y - b.y);
  } else if (R == 4) {
    const double2 a0 = make_double2(v[0].x + v[2].x, v[0].y + v[2].y);
    const double2 a1 = make_double2(v[0].x - v[2].x, v[0].y - v[2].y);
    const double2 b0 = make_double2(v[1].x + v[3].x, v[1].y + v[3].y);
    const double2 b1 = make_double2(v[1].x - v[3].x, v[1].y - v[3].y);
    // (-i DIR) b1 for the odd output: forward (DIR = -1) multiplies by -i
    const double2 jb1 = DIR < 0 ? make_double2(b1.y, -b1.x) : make_double2(-b1.y, b1.x);
    v[0] = make_double2(a0.x + b0.x, a0.y + b0.y);
    v[2] = make_double2(a0.x - b0.x, a0.y - b0.y);
    v[1] = make_double2(a1.x + jb1.x, a1.y + jb1.y);
    v[3] = make_double2(a1.x - jb1.x, a1.y - jb1.y);
  } else {
    double2 out[R];
#pragma unroll
    for (int q = 0; q < R; q++) {
      double2 acc = v[0];
#pragma unroll
      for (int t = 1; t < R; t++) {
        const int j = (t * q) % R;
        const double c = c_dft_c[R][j], s = DIR * c_dft_s[R][j];
        acc.x = fma(v[t].x, c, fma(-v[t].y, s, acc.x));
        acc.y = fma(v[t].x, s, fma(v[t].y, c, acc.y));
      }
      out[q] = acc;
    }
#pragma unroll
    for (int q = 0; q < R; q++) v[q] = out[q];
  }
}

// one stage over `batch` independent transforms of length n stored at a + b n
template <int R, int DIR, bool DIT>
__device__ __forceinline__ void fft_stage(double2 *a, int n, int batch, int Lp, const double2 *__restrict__ tw) {
  const int L = Lp * R;
  const int nb = n / R;
  const int tstride = n / L;
  for (int j = threadIdx.x; j < batch * nb; j += blockDim.x) {
    const int col = j / nb, jj = j - col * nb;
    const int b = jj / Lp, k1 = jj - b * Lp;
    double2 *base = a + (size_t)col * n + b * L + k1;
    double2 v[R];
#pragma unroll
    for (int t = 0; t < R; t++) v[t] = base[t * Lp];
    if (DIT) {
#pragma unroll
      for (int t = 1; t < R; t++) {
        double2 w = __ldg(tw + t * k1 * tstride);
        if (DIR > 0) w.y = -w.y;
        v[t] = cmul(v[t], w);
      }
      dft_small<R, DIR>(v);
    } else {
      dft_small<R, DIR>(v);
#pragma unroll
      for (int t = 1; t < R; t++) {
        double2 w = __ldg(tw + t * k1 * tstride);
        if (DIR > 0) w.y = -w.y;
        v[t] = cmul(v[t], w);
      }
    }
#pragma unroll
    for (int t = 0; t < R; t++) base[t * Lp] = v[t];
  }
}

template <int DIR, bool DIT>
__device__ void fft_run(double2 *a, const FftStages &st, int batch, const double2 *__restrict__ tw) {
  for (int i = 0; i < st.S; i++) {
    const int s = DIT ? i : st.S - 1 - i;
    switch (st.r[s]) {
      case 2: fft_stage<2, DIR, DIT>(a, st.n, batch, st.Lp[s], tw); break;
      case 3: fft_stage<3, DIR, DIT>(a, st.n, batch, st.Lp[s], tw); break;
      case 4: fft_stage<4, DIR, DIT>(a, st.n, batch, st.Lp[s], tw); break;
      case 5: fft_stage<5, DIR, DIT>(a, st.n, batch, st.Lp[s], tw); break;
      case 7: fft_stage<7, DIR, DIT>(a, st.n, batch, st.Lp[s], tw); break;
      case 8: fft_stage<8, DIR, DIT>(a, st.n, batch, st.Lp[s], tw); break;
      default: break;
    }
    __syncthreads();
  }
}

// ---- row pass, forward: grid row (real, nf) -> kept half-spectrum columns 0..ncs-1
__global__ void __launch_bounds__(256) k_fft_row_fwd(const double *__restrict__ grid, int64_t row_pitch,
                                                     double2 *__restrict__ spec, int ncs, FftStages st,
                                                     const double2 *__restrict__ tw_r,
                                                     const double2 *__restrict__ tw_c,
                                                     const int32_t *__restrict__ pos_r) {
  extern __shared__ double2 a2[];
  const int nr = st.n;
  const double2 *src = (const double2 *)(grid + (int64_t)blockIdx.x * row_pitch);
  for (int i = threadIdx.x; i < nr; i += blockDim.x) a2[i] = src[i];
  __syncthreads();
  fft_run<-1, false>(a2, st, 1, tw_r);
  double2 *dst = spec + (int64_t)blockIdx.x * ncs;
  for (int k = threadIdx.x; k < ncs; k += blockDim.x) {
    const double2 zk = a2[pos_r[k % nr]], zm = a2[pos_r[(nr - k) % nr]];
    // Ze = (Z[k] + conj Z[nr-k]) / 2, Zo = -i (Z[k] - conj Z[nr-k]) / 2, X = Ze + W_nf^k Zo
    const double2 ze = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    const double2 zo = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
    const double2 w = __ldg(tw_c + k);  // W_nf^k, k <= nr < nf
    const double2 t = cmul(w, zo);
    dst[k] = make_double2(ze.x + t.x, ze.y + t.y);
  }
}

// ---- column pass: forward DIF, multiply, inverse DIT on CB kept columns
__global__ void __launch_bounds__(256) k_fft_col(double2 *__restrict__ spec, int ncs, int CB, FftStages st,
                                                 const double2 *__restrict__ tw_c, const int32_t *__restrict__ sig_c,
                                                 int64_t half_modes, const double *__restrict__ deconv, double dk,
                                                 double scale, int kind, double da, double db) {
  extern __shared__ double2 a2[];
  const int nc = st.n;
  const int c0 = blockIdx.x * CB;
  const int cb_n = min(CB, ncs - c0);
  for (int id = threadIdx.x; id < nc * CB; id += blockDim.x) {
    const int i = id / CB, cb = id - i * CB;
    if (cb < cb_n) a2[cb * nc + i] = spec[(int64_t)i * ncs + c0 + cb];
  }
  __syncthreads();
  fft_run<-1, false>(a2, st, cb_n, tw_c);
  for (int id = threadIdx.x; id < nc * cb_n; id += blockDim.x) {
    const int cb = id / nc, p = id - cb * nc;
    const int64_t m1 = c0 + cb;
    const int f = sig_c[p];
    const int64_t m2 = f <= nc / 2 ? f : f - nc;
    const int64_t a2m = m2 < 0 ? -m2 : m2;
    double fac = 0.0;
    if (m1 <= half_modes && a2m <= half_modes) {
      const double k2 = dk * dk * ((double)m1 * m1 + (double)m2 * m2);
      const double mk = kind == 0 ? vp_mult_nh(k2, da, db) : vp_mult_fh(k2, da, db);
      fac = mk * scale * deconv[m1] * deconv[a2m];
    }
    double2 v = a2[cb * nc + p];
    a2[cb * nc + p] = make_double2(v.x * fac, v.y * fac);
  }
  __syncthreads();
  fft_run<1, true>(a2, st, cb_n, tw_c);
  for (int id = threadIdx.x; id < nc * CB; id += blockDim.x) {
    const int i = id / CB, cb = id - i * CB;
    if (cb < cb_n) spec[(int64_t)i * ncs + c0 + cb] = a2[cb * nc + i];
  }
}

// ---- row pass, inverse: kept half-spectrum columns -> real grid row (unnormalised, as cuFFT Z2D)
__global__ void __launch_bounds__(256) k_fft_row_inv(const double2 *__restrict__ spec, int ncs, double *__restrict__ grid,
                                                     int64_t row_pitch, FftStages st, const double2 *__restrict__ tw_r,
                                                     const double2 *__restrict__ tw_c,
                                                     const int32_t *__restrict__ pos_r) {
  extern __shared__ double2 a2[];
  const int nr = st.n;
  const double2 *src = spec + (int64_t)blockIdx.x * ncs;
  for (int k = threadIdx.x; k < nr; k += blockDim.x) {
    const double2 xk = k < ncs ? src[k] : make_double2(0.0, 0.0);
    const double2 xm = (nr - k) < ncs ? src[nr - k] : make_double2(0.0, 0.0);
    // Ze = (X[k] + conj X[nr-k]) / 2, Zo = W_nf^{-k} (X[k] - conj X[nr-k]) / 2, Z = Ze + i Zo
    const double2 ze = make_double2(0.5 * (xk.x + xm.x), 0.5 * (xk.y - xm.y));
    double2 w = __ldg(tw_c + k);
    w.y = -w.y;
    const double2 zo = cmul(w, make_double2(0.5 * (xk.x - xm.x), 0.5 * (xk.y + xm.y)));
    a2[pos_r[k]] = make_double2(ze.x - zo.y, ze.y + zo.x);
  }
  __syncthreads();
  fft_run<1, true>(a2, st, 1, tw_r);
  double2 *dst = (double2 *)(grid + (int64_t)blockIdx.x * row_pitch);
  for (int i = threadIdx.x; i < nr; i += blockDim.x) {
    const double2 z = a2[i];
    dst[i] = make_double2(2.0 * z.x, 2.0 * z.y);
  }
}

// ---------------------------------------------------------------------------------------------
// host side
static bool factor_stages(int n, FftStages &st) {
  std::vector<int> rs;
  int m = n;
  for (int r : {8, 4, 2}) {
    while (m % r == 0 && (r != 4 || m % 8 != 0) && (r != 2 || m % 4 != 0)) {
      rs.push_back(r);
      m /= r;
    }
  }
  for (int r : {7, 5, 3}) {
    while (m % r == 0) {
      rs.push_back(r);
      m /= r;
    }
  }
  if (m != 1 || rs.empty() || (int)rs.size() > VP_FFT_MAXS) return false;
  // odd radices first: stage 0 (span-1 butterflies, stride r between a thread's elements) then has an odd
  // stride, which spreads a warp over the shared-memory banks
  std::stable_sort(rs.begin(), rs.end(), [](int a, int b) { return (a & 1) > (b & 1); });
  st.n = n;
  st.S = (int)rs.size();
  int L = 1;
  for (int s = 0; s < st.S; s++) {
    st.r[s] = rs[s];
    st.Lp[s] = L;
    L *= rs[s];
  }
  return true;
}

// sigma(p) = sum_s p_s n / L_s for p = sum_s p_s L_{s-1}
static void digit_sigma(const FftStages &st, std::vector<int32_t> &sig) {
  const int n = st.n;
  sig.assign(n, 0);
  for (int p = 0; p < n; p++) {
    int rem = p, L = 1, f = 0;
    for (int s = 0; s < st.S; s++) {
      const int d = rem % st.r[s];
      rem /= st.r[s];
      L *= st.r[s];
      f += d * (n / L);
    }
    sig[p] = f;
  }
}

static double2 *twiddle_table(vp_plan_s *P, int n) {
  std::vector<double2> t(n);
  for (int j = 0; j < n; j++) {
    const long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)j / (long double)n;
    t[j] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  double2 *d = vp_alloc<double2>(P, n);
  VP_CUDA(cudaMemcpy(d, t.data(), sizeof(double2) * n, cudaMemcpyHostToDevice));
  return d;
}

static bool g_dft_uploaded = false;

// decide and build the fused transform for grid G (opts.fft_mode 0: where it fits shared memory)
void vp_fft_setup(vp_plan_s *P, VpGrid &G) {
  G.own_fft = false;
  if (P->opts.fft_mode == 1) return;
  const int nf = (int)G.nf;
  if (nf % 2 || nf > 12800) return;  // column of nf complex values must fit one CTA's shared memory
  FftStages sr, sc;
  if (!factor_stages(nf / 2, sr) || !factor_stages(nf, sc)) return;
  if (!g_dft_uploaded) {
    double hc[9][8] = {}, hs[9][8] = {};
    for (int R = 2; R <= 8; R++)
      for (int j = 0; j < R; j++) {
        const long double ang = 2.0L * 3.141592653589793238462643383279502884L * j / R;
        hc[R][j] = (double)cosl(ang);
        hs[R][j] = (double)sinl(ang);
      }
    VP_CUDA(cudaMemcpyToSymbol(c_dft_c, hc, sizeof(hc)));
    VP_CUDA(cudaMemcpyToSymbol(c_dft_s, hs, sizeof(hs)));
    g_dft_uploaded = true;
  }
  G.fft_ncs = (int)(G.nmode / 2 + 1);
  if (G.fft_ncs > nf / 2 + 1) G.fft_ncs = nf / 2 + 1;
  G.tw_r = twiddle_table(P, nf / 2);
  G.tw_c = twiddle_table(P, nf);
  std::vector<int32_t> sig_r, sig_c, pos_r(nf / 2);
  digit_sigma(sr, sig_r);
  digit_sigma(sc, sig_c);
  for (int p = 0; p < nf / 2; p++) pos_r[sig_r[p]] = p;
  G.pos_r = vp_alloc<int32_t>(P, nf / 2);
  G.sig_c = vp_alloc<int32_t>(P, nf);
  VP_CUDA(cudaMemcpy(G.pos_r, pos_r.data(), 4 * pos_r.size(), cudaMemcpyHostToDevice));
  VP_CUDA(cudaMemcpy(G.sig_c, sig_c.data(), 4 * sig_c.size(), cudaMemcpyHostToDevice));
  static_assert(sizeof(FftStages) <= sizeof(G.fft_st_r), "stage buffer");
  memcpy(G.fft_st_r, &sr, sizeof(sr));
  memcpy(G.fft_st_c, &sc, sizeof(sc));
  // columns per CTA: keep two CTAs per SM where the column block fits ~100 KB
  const size_t col_bytes = sizeof(double2) * (size_t)nf;
  G.fft_cb = (int)std::max<size_t>(1, std::min<size_t>(4, (100 * 1024) / col_bytes));
  const size_t sm_c = col_bytes * G.fft_cb, sm_r = sizeof(double2) * (size_t)(nf / 2);
  VP_CUDA(cudaFuncSetAttribute(k_fft_col, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  VP_CUDA(cudaFuncSetAttribute(k_fft_row_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  VP_CUDA(cudaFuncSetAttribute(k_fft_row_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  if (sm_c > 227 * 1024 || sm_r > 227 * 1024) return;
  G.own_fft = true;
}

void vp_fft_forward(vp_plan_s *P, VpGrid &G) {
  FftStages sr;
  memcpy(&sr, G.fft_st_r, sizeof(sr));
  k_fft_row_fwd<<<(unsigned)G.nf, 256, sizeof(double2) * (G.nf / 2), P->stream>>>(
      G.data, G.row, (double2 *)G.cdata, G.fft_ncs, sr, G.tw_r, G.tw_c, G.pos_r);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

void vp_fft_columns(vp_plan_s *P, VpGrid &G) {
  FftStages sc;
  memcpy(&sc, G.fft_st_c, sizeof(sc));
  const int nblk = (G.fft_ncs + G.fft_cb - 1) / G.fft_cb;
  k_fft_col<<<(unsigned)nblk, 256, sizeof(double2) * G.nf * G.fft_cb, P->stream>>>(
      (double2 *)G.cdata, G.fft_ncs, G.fft_cb, sc, G.tw_c, G.sig_c, G.nmode / 2, G.deconv, 2.0 * VP_PI / G.L,
      G.mult_scale, G.kind, G.delta_a, G.delta_b);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

void vp_fft_inverse(vp_plan_s *P, VpGrid &G) {
  FftStages sr;
  memcpy(&sr, G.fft_st_r, sizeof(sr));
  k_fft_row_inv<<<(unsigned)G.nf, 256, sizeof(double2) * (G.nf / 2), P->stream>>>(
      (const double2 *)G.cdata, G.fft_ncs, G.data, G.row, sr, G.tw_r, G.tw_c, G.pos_r);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}
