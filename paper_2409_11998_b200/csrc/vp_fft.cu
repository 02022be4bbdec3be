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

#include <cuda_pipeline.h>

#include <mutex>
#include <set>

#include "vp_common.cuh"
#include "vp_math.cuh"

#define VP_FFT_MAXS 16

struct FftStages {
  int n, S;
  int r[VP_FFT_MAXS];
  int Lp[VP_FFT_MAXS];      // L_{s-1}
  float invLp[VP_FFT_MAXS];  // 1 / L_{s-1} (butterfly index split without integer division)
};

__constant__ double c_dft_c[10][9];  // cos(2 pi j / R), R = 2..9
__constant__ double c_dft_s[10][9];  // sin(2 pi j / R)

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// in-place R-point DFT, sign DIR (-1 forward, +1 inverse)
template <int R, int DIR>
__device__ __forceinline__ void dft_small(double2 (&v)[R]) {
  if constexpr (R == 2) {
    const double2 a = v[0], b = v[1];
    v[0] = make_double2(a.x + b.x, a.y + b.y);
    v[1] = make_double2(a.x - b.x, a.y - b.y);
  } else if constexpr (R == 4) {
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
  } else if constexpr (R == 8) {  // two radix-4 halves (even, odd inputs) and W_8^q
    double2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    dft_small<4, DIR>(e);
    dft_small<4, DIR>(o);
    const double h = 0.70710678118654752440;
    // W_8^q o[q], W_8 = (1 + DIR i) / sqrt 2
    const double2 o1 = make_double2(h * (o[1].x - DIR * o[1].y), h * (o[1].y + DIR * o[1].x));
    const double2 o2 = DIR < 0 ? make_double2(o[2].y, -o[2].x) : make_double2(-o[2].y, o[2].x);
    const double2 o3 = make_double2(h * (-o[3].x - DIR * o[3].y), h * (-o[3].y + DIR * o[3].x));
    v[0] = make_double2(e[0].x + o[0].x, e[0].y + o[0].y);
    v[4] = make_double2(e[0].x - o[0].x, e[0].y - o[0].y);
    v[1] = make_double2(e[1].x + o1.x, e[1].y + o1.y);
    v[5] = make_double2(e[1].x - o1.x, e[1].y - o1.y);
    v[2] = make_double2(e[2].x + o2.x, e[2].y + o2.y);
    v[6] = make_double2(e[2].x - o2.x, e[2].y - o2.y);
    v[3] = make_double2(e[3].x + o3.x, e[3].y + o3.y);
    v[7] = make_double2(e[3].x - o3.x, e[3].y - o3.y);
  } else {  // odd R: pair t with R - t (a_t = v_t + v_{R-t}, b_t = v_t - v_{R-t})
    constexpr int H = (R - 1) / 2;
    double2 sa[H], sb[H];
    double2 o0 = v[0];
#pragma unroll
    for (int t = 1; t <= H; t++) {
      sa[t - 1] = make_double2(v[t].x + v[R - t].x, v[t].y + v[R - t].y);
      sb[t - 1] = make_double2(v[t].x - v[R - t].x, v[t].y - v[R - t].y);
      o0.x += sa[t - 1].x;
      o0.y += sa[t - 1].y;
    }
    double2 out[R];
    out[0] = o0;
#pragma unroll
    for (int q = 1; q <= H; q++) {
      double2 re = v[0], im = make_double2(0.0, 0.0);
#pragma unroll
      for (int t = 1; t <= H; t++) {
        const int j = (t * q) % R;
        const double c = c_dft_c[R][j], sn = c_dft_s[R][j];
        re.x = fma(sa[t - 1].x, c, re.x);
        re.y = fma(sa[t - 1].y, c, re.y);
        im.x = fma(sb[t - 1].x, sn, im.x);
        im.y = fma(sb[t - 1].y, sn, im.y);
      }
      // out[q] = re + DIR i im, out[R - q] = re - DIR i im
      out[q] = make_double2(re.x - DIR * im.y, re.y + DIR * im.x);
      out[R - q] = make_double2(re.x + DIR * im.y, re.y - DIR * im.x);
    }
#pragma unroll
    for (int q = 0; q < R; q++) v[q] = out[q];
  }
}

// one stage of a length-n transform at a
template <int R, int DIR, bool DIT>
__device__ __forceinline__ void fft_stage(double2 *a, int n, int Lp, float invLp, const double2 *tw) {
  const int L = Lp * R;
  const int nb = n / R;
  const int tstride = n / L;
  for (int j = threadIdx.x; j < nb; j += blockDim.x) {
    int b = __float2int_rz((float)j * invLp), k1 = j - b * Lp;
    if (k1 < 0) {
      b--;
      k1 += Lp;
    } else if (k1 >= Lp) {
      b++;
      k1 -= Lp;
    }
    double2 *base = a + b * L + k1;
    double2 v[R];
#pragma unroll
    for (int t = 0; t < R; t++) v[t] = base[t * Lp];
    // twiddles W_L^{t k1}: one table load (t = 1), higher powers by multiplication (error ~ t eps)
    double2 w1 = make_double2(1.0, 0.0);
    if (k1) {
      w1 = tw[k1 * tstride];  // shared-memory or global table
      if (DIR > 0) w1.y = -w1.y;
    }
    if (!DIT) dft_small<R, DIR>(v);
    if (k1) {
      double2 w = w1;
#pragma unroll
      for (int t = 1; t < R; t++) {
        v[t] = cmul(v[t], w);
        if (t + 1 < R) w = cmul(w, w1);
      }
    }
    if (DIT) dft_small<R, DIR>(v);
#pragma unroll
    for (int t = 0; t < R; t++) base[t * Lp] = v[t];
  }
}

template <int DIR, bool DIT>
__device__ void fft_run(double2 *a, const FftStages &st, const double2 *tw) {
  for (int i = 0; i < st.S; i++) {
    const int s = DIT ? i : st.S - 1 - i;
    switch (st.r[s]) {
      case 2: fft_stage<2, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 3: fft_stage<3, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 4: fft_stage<4, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 5: fft_stage<5, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 7: fft_stage<7, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 8: fft_stage<8, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 9: fft_stage<9, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      default: break;
    }
    __syncthreads();
  }
}

// copy n double2 from global (stride gs) to shared memory with U loads in flight per thread
template <int U>
__device__ __forceinline__ void load_g2s(double2 *dst, const double2 *__restrict__ src, int n, int64_t gs) {
  for (int i0 = threadIdx.x; i0 < n; i0 += U * blockDim.x) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int i = i0 + u * blockDim.x;
      if (i < n) v[u] = src[(int64_t)i * gs];
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int i = i0 + u * blockDim.x;
      if (i < n) dst[i] = v[u];
    }
  }
}

// asynchronous copy of n double2 (16-byte aligned, contiguous) global -> shared (cp.async, 16 B per thread-op)
__device__ __forceinline__ void prefetch_g2s(double2 *dst, const double2 *src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) __pipeline_memcpy_async(dst + i, src + i, sizeof(double2));
}

// ---- row pass, forward: grid rows (real, nf) -> kept half-spectrum columns 0..ncs-1, stored column-major
// (spec[k nf + row]: the column pass then reads contiguous columns; concurrent rows' 16-byte writes meet in
// L2 sectors).  Persistent CTAs: the row twiddles and the digit-reversal map are staged once, and the next
// row is prefetched (cp.async) into a second buffer while the current one is transformed.
__global__ void __launch_bounds__(256) k_fft_row_fwd(const double *__restrict__ grid, int64_t row_pitch,
                                                     double2 *__restrict__ spec, int ncs, int nf, FftStages st,
                                                     const double2 *__restrict__ tw_r,
                                                     const double2 *__restrict__ tw_c,
                                                     const int32_t *__restrict__ pos_r) {
  extern __shared__ double2 sm2[];
  const int nr = st.n;
  double2 *twr = sm2, *buf0 = sm2 + nr, *buf1 = sm2 + 2 * nr;
  int *pos = (int *)(sm2 + 3 * nr);
  for (int i = threadIdx.x; i < nr; i += blockDim.x) {
    twr[i] = tw_r[i];
    pos[i] = pos_r[i];
  }
  int r = blockIdx.x;
  if (r < nf) prefetch_g2s(buf0, (const double2 *)(grid + (int64_t)r * row_pitch), nr);
  __pipeline_commit();
  for (int cur = 0; r < nf; r += gridDim.x, cur ^= 1) {
    double2 *a2 = cur ? buf1 : buf0;
    const int rn = r + gridDim.x;
    if (rn < nf) prefetch_g2s(cur ? buf0 : buf1, (const double2 *)(grid + (int64_t)rn * row_pitch), nr);
    __pipeline_commit();
    __pipeline_wait_prior(1);
    __syncthreads();
    fft_run<-1, false>(a2, st, twr);
    double2 *dst = spec + r;
    for (int k = threadIdx.x; k < ncs; k += blockDim.x) {
      const double2 zk = a2[pos[k % nr]], zm = a2[pos[(nr - k) % nr]];
      // Ze = (Z[k] + conj Z[nr-k]) / 2, Zo = -i (Z[k] - conj Z[nr-k]) / 2, X = Ze + W_nf^k Zo
      const double2 ze = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
      const double2 zo = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
      const double2 w = __ldg(tw_c + k);  // W_nf^k, k <= nr < nf
      const double2 t = cmul(w, zo);
      dst[(int64_t)k * nf] = make_double2(ze.x + t.x, ze.y + t.y);
    }
    __syncthreads();  // buffer a2 is refilled in the next iteration's prefetch of row rn + gridDim.x
  }
}

// multiplier of k_multiply (NH or FH kernel, ES deconvolution, trapezoid and 1/nf^2 scale, truncation) for
// column m1 at DIF output position p (frequency sig_c[p]); tabulated at plan time
__global__ void k_fft_mult_table(double *__restrict__ tab, int ncs, int nc, const int32_t *__restrict__ sig_c,
                                 int64_t half_modes, const double *__restrict__ deconv, double dk, double scale,
                                 int kind, double da, double db) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= (int64_t)ncs * nc) return;
  const int64_t m1 = id / nc;
  const int p = (int)(id - m1 * nc);
  const int f = sig_c[p];
  const int64_t m2 = f <= nc / 2 ? f : f - nc;
  const int64_t a2m = m2 < 0 ? -m2 : m2;
  double fac = 0.0;
  if (m1 <= half_modes && a2m <= half_modes) {
    const double k2 = dk * dk * ((double)m1 * m1 + (double)m2 * m2);
    const double mk = kind == 0 ? vp_mult_nh(k2, da, db) : vp_mult_fh(k2, da, db);
    fac = mk * scale * deconv[m1] * deconv[a2m];
  }
  tab[id] = fac;
}

// ---- column pass: forward DIF, multiply, inverse DIT on kept columns.  Reads the column-major spectrum
// (contiguous columns), writes the result row-major (spec_out[row ncs + m1]; concurrent columns' 16-byte writes
// meet in L2 sectors) so that the inverse row pass reads contiguous rows.  Persistent CTAs, next column
// prefetched (cp.async) while the current one is transformed.
// Several boxes (level bands, §5.6): nbox grids of nc rows stacked (NR = nbox nc spectrum rows), unit u = (box
// b, column m1) with the column at spec + m1 NR + b nc and the multiplier row of the box's level.
__global__ void __launch_bounds__(256) k_fft_col(const double2 *__restrict__ spec, double2 *__restrict__ spec_out,
                                                 int ncs, int nbox, int64_t NR, FftStages st,
                                                 const double2 *__restrict__ tw_c, const double *__restrict__ mult,
                                                 const int32_t *__restrict__ box_level) {
  extern __shared__ double2 sm2[];
  const int nc = st.n;
  const int nu = ncs * nbox;
  double2 *buf0 = sm2, *buf1 = sm2 + nc;
  auto col_of = [&](int u) {
    const int b = u / ncs, m1 = u - b * ncs;
    return spec + (int64_t)m1 * NR + (int64_t)b * nc;
  };
  int u = blockIdx.x;
  if (u < nu) prefetch_g2s(buf0, col_of(u), nc);
  __pipeline_commit();
  for (int cur = 0; u < nu; u += gridDim.x, cur ^= 1) {
    double2 *a2 = cur ? buf1 : buf0;
    const int un = u + gridDim.x;
    if (un < nu) prefetch_g2s(cur ? buf0 : buf1, col_of(un), nc);
    __pipeline_commit();
    __pipeline_wait_prior(1);
    __syncthreads();
    const int b = u / ncs, m1 = u - b * ncs;
    fft_run<-1, false>(a2, st, tw_c);
    const double *mc = mult + ((int64_t)(box_level ? box_level[b] : 0) * ncs + m1) * nc;
    for (int p = threadIdx.x; p < nc; p += blockDim.x) {
      const double fac = __ldg(mc + p);
      const double2 v = a2[p];
      a2[p] = make_double2(v.x * fac, v.y * fac);
    }
    __syncthreads();
    fft_run<1, true>(a2, st, tw_c);
    for (int i = threadIdx.x; i < nc; i += blockDim.x) spec_out[((int64_t)b * nc + i) * ncs + m1] = a2[i];
    __syncthreads();
  }
}

// band multiplier per level l: (e^{-k^2 delta_l} - e^{-k^2 delta_{l-1}}) / k^2, k = dk_l m,
// ES deconvolution and scale_l, in DIF order; level 0 rows are unused (zero)
__global__ void k_fft_mult_table_bands(double *__restrict__ tab, int nlev1, int ncs, int nc,
                                       const int32_t *__restrict__ sig_c, int64_t half_modes,
                                       const double *__restrict__ deconv, const double *__restrict__ lev_par) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= (int64_t)nlev1 * ncs * nc) return;
  const int64_t l = id / ((int64_t)ncs * nc), rem = id - l * ncs * nc;
  const int64_t m1 = rem / nc;
  const int p = (int)(rem - m1 * nc);
  const int f = sig_c[p];
  const int64_t m2 = f <= nc / 2 ? f : f - nc;
  const int64_t a2m = m2 < 0 ? -m2 : m2;
  double fac = 0.0;
  if (l > 0 && m1 <= half_modes && a2m <= half_modes) {
    const double *lp = lev_par + 4 * l;
    const double k2 = lp[2] * lp[2] * ((double)m1 * m1 + (double)m2 * m2);
    fac = vp_mult_nh(k2, lp[0], lp[1]) * lp[3] * deconv[m1] * deconv[a2m];
  }
  tab[id] = fac;
}

// ---- row pass, inverse: kept half-spectrum columns (row-major) -> real grid rows (unnormalised, as cuFFT
// Z2D).  Persistent CTAs with staged row twiddles / digit-reversal map and a prefetched next spectrum row.
__global__ void __launch_bounds__(256) k_fft_row_inv(const double2 *__restrict__ spec, int ncs, int nf,
                                                     double *__restrict__ grid,
                                                     int64_t row_pitch, FftStages st, const double2 *__restrict__ tw_r,
                                                     const double2 *__restrict__ tw_c,
                                                     const int32_t *__restrict__ pos_r) {
  extern __shared__ double2 sm2[];
  const int nr = st.n;
  const int nk = min(ncs, nr + 1);
  const int nkp = (nk + 1) & ~1;
  double2 *twr = sm2, *a2 = sm2 + nr, *xs0 = sm2 + 2 * nr, *xs1 = xs0 + nkp;
  int *pos = (int *)(xs1 + nkp);
  for (int i = threadIdx.x; i < nr; i += blockDim.x) {
    twr[i] = tw_r[i];
    pos[i] = pos_r[i];
  }
  int r = blockIdx.x;
  if (r < nf) prefetch_g2s(xs0, spec + (int64_t)r * ncs, nk);
  __pipeline_commit();
  for (int cur = 0; r < nf; r += gridDim.x, cur ^= 1) {
    const double2 *xs = cur ? xs1 : xs0;
    const int rn = r + gridDim.x;
    if (rn < nf) prefetch_g2s(cur ? xs0 : xs1, spec + (int64_t)rn * ncs, nk);
    __pipeline_commit();
    __pipeline_wait_prior(1);
    __syncthreads();
    for (int k = threadIdx.x; k < nr; k += blockDim.x) {
      const double2 xk = k < nk ? xs[k] : make_double2(0.0, 0.0);
      const double2 xm = (nr - k) < nk ? xs[nr - k] : make_double2(0.0, 0.0);
      // Ze = (X[k] + conj X[nr-k]) / 2, Zo = W_nf^{-k} (X[k] - conj X[nr-k]) / 2, Z = Ze + i Zo
      const double2 ze = make_double2(0.5 * (xk.x + xm.x), 0.5 * (xk.y - xm.y));
      double2 w = __ldg(tw_c + k);
      w.y = -w.y;
      const double2 zo = cmul(w, make_double2(0.5 * (xk.x - xm.x), 0.5 * (xk.y + xm.y)));
      a2[pos[k]] = make_double2(ze.x - zo.y, ze.y + zo.x);
    }
    __syncthreads();
    fft_run<1, true>(a2, st, twr);
    double2 *dst = (double2 *)(grid + (int64_t)r * row_pitch);
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
      const double2 z = a2[i];
      dst[i] = make_double2(2.0 * z.x, 2.0 * z.y);
    }
    __syncthreads();
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
  for (int r : {9, 7, 5, 3}) {  // radix 9 (one in-register stage) before 3 x 3
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
    st.invLp[s] = 1.0f / (float)L;
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

// shared memory of the persistent row kernels: twiddles + 2 buffers (forward) / twiddles + transform buffer +
// 2 staged spectrum rows (inverse), plus the digit-reversal map; the larger of the two
static size_t fft_row_smem(int nr, int ncs) {
  const int nk = std::min(ncs, nr + 1), nkp = (nk + 1) & ~1;
  const size_t fwd = sizeof(double2) * 3 * (size_t)nr + sizeof(int) * nr;
  const size_t inv = sizeof(double2) * (2 * (size_t)nr + 2 * (size_t)nkp) + sizeof(int) * nr;
  return std::max(fwd, inv);
}


// DFT roots of the odd radices in the constant bank (dft_small): uploaded once per device (same values for
// every plan); every transform path that runs dft_small calls this at plan time
static void upload_dft_roots() {
  static std::mutex mu;
  static std::set<int> done;
  const int dev = vp_current_device();
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(dev)) return;
  double hc[10][9] = {}, hs[10][9] = {};
  for (int R = 2; R <= 9; R++)
    for (int j = 0; j < R; j++) {
      const long double ang = 2.0L * 3.141592653589793238462643383279502884L * j / R;
      hc[R][j] = (double)cosl(ang);
      hs[R][j] = (double)sinl(ang);
    }
  VP_CUDA(cudaMemcpyToSymbol(c_dft_c, hc, sizeof(hc)));
  VP_CUDA(cudaMemcpyToSymbol(c_dft_s, hs, sizeof(hs)));
  done.insert(dev);
}

// decide and build the fused transform for grid G (opts.fft_mode 0: where it fits shared memory)
// stage plans, twiddles and digit maps of an nf x nf transform (false: size not supported)
static bool fft_tables(vp_plan_s *P, VpGrid &G) {
  const int nf = (int)G.nf;
  // measured (profiles/r1/probe_fft_*.json): faster than cuFFT + k_multiply up to 6048 (configs 1-2, FH grids of
  // configs 3-4), slower at 12500 (one column fills a CTA's shared memory; load and transform serialise)
  if (nf % 2 || nf > 6400) return false;
  FftStages sr, sc;
  if (!factor_stages(nf / 2, sr) || !factor_stages(nf, sc)) return false;
  upload_dft_roots();
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
  const size_t sm_c = 2 * sizeof(double2) * (size_t)nf, sm_r = fft_row_smem(nf / 2, G.fft_ncs);
  VP_CUDA(cudaFuncSetAttribute(k_fft_col, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  VP_CUDA(cudaFuncSetAttribute(k_fft_row_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  VP_CUDA(cudaFuncSetAttribute(k_fft_row_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  for (const void *k : {(const void *)k_fft_col, (const void *)k_fft_row_fwd, (const void *)k_fft_row_inv})
    VP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  return sm_c <= 227 * 1024 && sm_r <= 227 * 1024;
}

void vp_fft_setup(vp_plan_s *P, VpGrid &G) {
  G.own_fft = false;
  if (P->opts.fft_mode == 1 || !fft_tables(P, G)) return;
  const int nf = (int)G.nf;
  // second spectrum buffer (row-major column-pass output) and the multiplier table (in DIF output order)
  G.spec2 = vp_alloc<double2>(P, (size_t)G.fft_ncs * nf);
  G.fft_mult = vp_alloc<double>(P, (size_t)G.fft_ncs * nf);
  const int64_t nt = (int64_t)G.fft_ncs * nf;
  k_fft_mult_table<<<(unsigned)((nt + 255) / 256), 256, 0, P->stream>>>(G.fft_mult, G.fft_ncs, nf, G.sig_c,
                                                                        G.nmode / 2, G.deconv, 2.0 * VP_PI / G.L,
                                                                        G.mult_scale, G.kind, G.delta_a, G.delta_b);
  VP_CHECK_LAUNCH();
  G.own_fft = true;
}

static int fft_threads(int n) { return n <= 2048 ? 128 : 256; }

static int num_sms() {  // of the current device (asked every time: plans may live on different devices)
  int n = 0;
  VP_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, vp_current_device()));
  return n;
}
// persistent row kernels: CTAs per SM that the shared memory (227 KB) allows, at most 4
static unsigned row_grid(size_t smem, int64_t rows) {
  int per = (int)std::min<size_t>(4, (227 * 1024) / (smem + 1024));
  if (per < 1) per = 1;
  return (unsigned)std::min<int64_t>(rows, (int64_t)per * num_sms());
}

void vp_fft_forward(vp_plan_s *P, VpGrid &G) {
  FftStages sr;
  memcpy(&sr, G.fft_st_r, sizeof(sr));
  const size_t sm = fft_row_smem(sr.n, G.fft_ncs);
  k_fft_row_fwd<<<row_grid(sm, G.nf), 256, sm, P->stream>>>(
      G.data, G.row, (double2 *)G.cdata, G.fft_ncs, (int)G.nf, sr, G.tw_r, G.tw_c, G.pos_r);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

void vp_fft_columns(vp_plan_s *P, VpGrid &G) {
  FftStages sc;
  memcpy(&sc, G.fft_st_c, sizeof(sc));
  const size_t sm = 2 * sizeof(double2) * G.nf;
  k_fft_col<<<row_grid(sm, G.fft_ncs), 256, sm, P->stream>>>(
      (const double2 *)G.cdata, G.spec2, G.fft_ncs, 1, G.nf, sc, G.tw_c, G.fft_mult, nullptr);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

void vp_fft_inverse(vp_plan_s *P, VpGrid &G) {
  FftStages sr;
  memcpy(&sr, G.fft_st_r, sizeof(sr));
  const size_t sm = fft_row_smem(sr.n, G.fft_ncs);
  k_fft_row_inv<<<row_grid(sm, G.nf), 256, sm, P->stream>>>(G.spec2, G.fft_ncs, (int)G.nf, G.data, G.row, sr, G.tw_r,
                                                              G.tw_c, G.pos_r);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

// ---- level bands (vp_levels.cu): nbox boxes of nfb^2 on one virtual grid, same three passes
bool vp_fft_setup_bands(vp_plan_s *P) {
  VpBands &B = P->bands;
  VpGrid &G = B.fg;
  G.nf = B.nfb;
  G.nmode = B.nmode;
  G.row = B.rowb;
  if (P->opts.fft_mode == 1 || !fft_tables(P, G)) return false;
  const int nf = (int)G.nf;
  const int64_t NR = B.nbox * B.nfb;
  G.cdata = (double *)vp_alloc<double2>(P, (size_t)G.fft_ncs * NR);
  G.spec2 = vp_alloc<double2>(P, (size_t)G.fft_ncs * NR);
  const int nlev1 = B.nlev + 1;
  G.fft_mult = vp_alloc<double>(P, (size_t)nlev1 * G.fft_ncs * nf);
  const int64_t nt = (int64_t)nlev1 * G.fft_ncs * nf;
  k_fft_mult_table_bands<<<(unsigned)((nt + 255) / 256), 256, 0, P->stream>>>(G.fft_mult, nlev1, G.fft_ncs, nf, G.sig_c,
                                                                              B.nmode / 2, B.deconv, B.lev_par);
  VP_CHECK_LAUNCH();
  G.own_fft = true;
  return true;
}

void vp_fft_bands(vp_plan_s *P) {
  VpBands &B = P->bands;
  VpGrid &G = B.fg;
  const int64_t NR = B.nbox * B.nfb;
  FftStages sr, sc;
  memcpy(&sr, G.fft_st_r, sizeof(sr));
  memcpy(&sc, G.fft_st_c, sizeof(sc));
  const size_t smr = fft_row_smem(sr.n, G.fft_ncs), smc = 2 * sizeof(double2) * G.nf;
  k_fft_row_fwd<<<row_grid(smr, NR), 256, smr, P->stream>>>(B.grid, B.rowb, (double2 *)G.cdata, G.fft_ncs, (int)NR, sr,
                                                             G.tw_r, G.tw_c, G.pos_r);
  VP_CHECK_LAUNCH();
  k_fft_col<<<row_grid(smc, (int64_t)G.fft_ncs * B.nbox), fft_threads(sc.n), smc, P->stream>>>(
      (const double2 *)G.cdata, G.spec2, G.fft_ncs, (int)B.nbox, NR, sc, G.tw_c, G.fft_mult, B.box_level);
  VP_CHECK_LAUNCH();
  k_fft_row_inv<<<row_grid(smr, NR), 256, smr, P->stream>>>(G.spec2, G.fft_ncs, (int)NR, B.grid, B.rowb, sr, G.tw_r,
                                                             G.tw_c, G.pos_r);
  VP_CHECK_LAUNCH();
  P->n_kernels += 3;
}

// =============================================================================================
// Large grids (nf > 6400, e.g. config 5's 23328^2 NH grid): the row passes are cuFFT batched 1D D2Z / Z2D, the
// column pass (forward FFT, multiply, inverse FFT of the kept columns) is a four-step
// transform over nf = N1 N2 in three streaming kernels, each one HBM round trip over the kept columns (a column of
// nf complex values no longer fits one CTA's shared memory):
//   A: for each n2, the N1-point DIF FFTs over rows n1 N2 + n2 (stride N2), twiddle W_nf^{n2 k1}; in place,
//      position p of the sequence holding k1 = sigma1(p)
//   B: for each p, the N2-point DIF FFT over the contiguous rows p N2 + n2 (frequency k = sigma1(p) +
//      N1 sigma2(p2)), the multiplier of k_multiply (same function, per element on the fly), the inverse N2-point
//      DIT back to natural n2', twiddle W_nf^{-n2' k1}
//   C: for each n2', the inverse N1-point DIT over positions p -> natural n1'; rows n1' N2 + n2'
// (X(k1 + N1 k2) = sum_n2 W_N2^{n2 k2} W_nf^{n2 k1} sum_n1 W_N1^{n1 k1} x(n1 N2 + n2), and its transpose.)
// A CTA owns TC4 consecutive kept columns (256-byte row segments) and transforms TC4 sequences at once.
#define TC4 16
#define VP_FFT4_MIN_NF 10000  // four-step column pass (+ own row passes) above this grid size

// shared layout of a tile: element i of column c at a[i * TC4 + c]; thread (c, q) = (tid % TC4, tid / TC4) works
// on column c, butterflies / elements q, q + 256 / TC4, ...: a row of TC4 columns is one contiguous 256-byte
// segment both in HBM and in shared memory, and no integer division by a runtime length is needed
#define Q4 (256 / TC4)

template <int R, int DIR, bool DIT>
__device__ __forceinline__ void fft_stage_t(double2 *a, int n, int Lp, float invLp, const double2 *__restrict__ tw) {
  const int L = Lp * R;
  const int nb = n / R;
  const int tstride = n / L;
  const int c = threadIdx.x % TC4;
  for (int j = threadIdx.x / TC4; j < nb; j += Q4) {
    int b = __float2int_rz((float)j * invLp), k1 = j - b * Lp;
    if (k1 < 0) {
      b--;
      k1 += Lp;
    } else if (k1 >= Lp) {
      b++;
      k1 -= Lp;
    }
    double2 *base = a + (b * L + k1) * TC4 + c;
    double2 v[R];
#pragma unroll
    for (int t = 0; t < R; t++) v[t] = base[t * Lp * TC4];
    double2 w1 = make_double2(1.0, 0.0);
    if (k1) {
      w1 = __ldg(tw + k1 * tstride);
      if (DIR > 0) w1.y = -w1.y;
    }
    if (!DIT) dft_small<R, DIR>(v);
    if (k1) {
      double2 w = w1;
#pragma unroll
      for (int t = 1; t < R; t++) {
        v[t] = cmul(v[t], w);
        if (t + 1 < R) w = cmul(w, w1);
      }
    }
    if (DIT) dft_small<R, DIR>(v);
#pragma unroll
    for (int t = 0; t < R; t++) base[t * Lp * TC4] = v[t];
  }
}

template <int DIR, bool DIT>
__device__ void fft_run_t(double2 *a, const FftStages &st, const double2 *__restrict__ tw) {
  for (int i = 0; i < st.S; i++) {
    const int s = DIT ? i : st.S - 1 - i;
    switch (st.r[s]) {
      case 2: fft_stage_t<2, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 3: fft_stage_t<3, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 4: fft_stage_t<4, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 5: fft_stage_t<5, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 7: fft_stage_t<7, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 8: fft_stage_t<8, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      case 9: fft_stage_t<9, DIR, DIT>(a, st.n, st.Lp[s], st.invLp[s], tw); break;
      default: break;
    }
    __syncthreads();
  }
}

struct Fft4Args {
  double2 *spec;   // [nf][nc] half spectrum (row stride nc complex), kept columns 0..ncs-1 transformed in place
  int64_t nc;      // nf / 2 + 1
  int ncs, nf, N1, N2;
  FftStages s1, s2;
  const double2 *tw1, *tw2, *twN;  // W_N1^j, W_N2^j, W_nf^j
  const int32_t *sig1, *sig2;      // DIF output position -> frequency
  // multiplier (k_multiply): kind 0 NH / 1 FH, da, db, trapezoid/1/nf^2 scale, deconv[m], dk, truncation
  int kind;
  double da, db, scale, dk;
  int64_t half_modes;
  const double *deconv;
  const double *e1, *e2;  // NH: e^{-dk^2 m^2 delta_1}, e^{-dk^2 m^2 delta_2} for m <= half_modes (separable exponentials)
};

// N rows (global row row0 + i * rstride) x TC4 columns <-> shared a[i * TC4 + c].  The load is asynchronous
// (cp.async, 16 B per element): every element of the tile is in flight at once instead of one dependent
// global load per thread and loop trip (the synchronous copy left the column kernels latency-bound at ~3 TB/s).
__device__ __forceinline__ void fft4_load(double2 *a, const Fft4Args &g, int c0, int ncol, int64_t row0,
                                          int64_t rstride, int N) {
  const int c = threadIdx.x % TC4;
  for (int i = threadIdx.x / TC4; i < N; i += Q4) {
    if (c < ncol) __pipeline_memcpy_async(a + i * TC4 + c, g.spec + (row0 + (int64_t)i * rstride) * g.nc + c0 + c,
                                          sizeof(double2));
    else a[i * TC4 + c] = make_double2(0.0, 0.0);
  }
  __pipeline_commit();
  __pipeline_wait_prior(0);
  __syncthreads();
}

// 1/x to ~1 ulp: hardware approximation + two Newton steps (the multiplier needs ~1e-15 relative, not IEEE
// rounding; the IEEE division costs a long instruction sequence per spectrum element)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  return fma(r, fma(-x, r, 1.0), r);
}
__device__ __forceinline__ void fft4_store(const double2 *a, const Fft4Args &g, int c0, int ncol, int64_t row0,
                                           int64_t rstride, int N) {
  __syncthreads();
  const int c = threadIdx.x % TC4;
  if (c >= ncol) return;
  for (int i = threadIdx.x / TC4; i < N; i += Q4) g.spec[(row0 + (int64_t)i * rstride) * g.nc + c0 + c] = a[i * TC4 + c];
}

// A: blockIdx.x = column tile, blockIdx.y = n2
__global__ void __launch_bounds__(256, 4) k_fft4_a(Fft4Args g) {
  extern __shared__ double2 sm2[];
  const int c0 = blockIdx.x * TC4, ncol = min(TC4, g.ncs - c0), n2 = blockIdx.y;
  fft4_load(sm2, g, c0, ncol, n2, g.N2, g.N1);
  fft_run_t<-1, false>(sm2, g.s1, g.tw1);
  const int c = threadIdx.x % TC4;
  for (int p = threadIdx.x / TC4; p < g.N1; p += Q4)
    sm2[p * TC4 + c] = cmul(sm2[p * TC4 + c], __ldg(g.twN + n2 * __ldg(g.sig1 + p)));  // n2 k1 < N2 N1 = nf
  fft4_store(sm2, g, c0, ncol, n2, g.N2, g.N1);
}

// B: blockIdx.x = column tile, blockIdx.y = p (position of k1)
__global__ void __launch_bounds__(256, 4) k_fft4_b(Fft4Args g) {
  extern __shared__ double2 sm2[];
  const int c0 = blockIdx.x * TC4, ncol = min(TC4, g.ncs - c0), p = blockIdx.y;
  const int64_t row0 = (int64_t)p * g.N2;
  const int k1 = __ldg(g.sig1 + p);
  fft4_load(sm2, g, c0, ncol, row0, 1, g.N2);
  fft_run_t<-1, false>(sm2, g.s2, g.tw2);
  const int c = threadIdx.x % TC4;
  const int m1 = c0 + c;
  const double d1 = m1 <= g.half_modes ? __ldg(g.deconv + m1) * g.scale : 0.0;
  if (g.kind == 0) {
    // NH: per-row factors of the separable form staged once per CTA (the CTA's rows share k1): for row p2,
    // b1 = e^{-k2^2 d_a} deconv(m2), b2 = e^{-k2^2 d_b} deconv(m2) (0 beyond the kept band) and m2^2; an element
    // is then (a1 b1 - a2 b2) / k^2 with the column factors a1, a2 (the small-k^2 branch keeps expm1)
    double *rb = (double *)(sm2 + TC4 * g.N2);  // [N2][3]
    for (int p2 = threadIdx.x; p2 < g.N2; p2 += blockDim.x) {
      const int k = k1 + g.N1 * __ldg(g.sig2 + p2);
      const int m2 = k <= g.nf / 2 ? k : k - g.nf, a2m = m2 < 0 ? -m2 : m2;
      const bool in = a2m <= g.half_modes;
      const double dm = in ? __ldg(g.deconv + a2m) : 0.0;
      rb[3 * p2] = in ? __ldg(g.e1 + a2m) * dm : 0.0;
      rb[3 * p2 + 1] = in ? __ldg(g.e2 + a2m) * dm : 0.0;
      rb[3 * p2 + 2] = in ? (double)m2 * (double)m2 : -1.0;  // -1: outside the band
    }
    __syncthreads();
    const bool col_in = m1 <= g.half_modes;
    const double a1 = col_in ? __ldg(g.e1 + m1) * d1 : 0.0, a2 = col_in ? __ldg(g.e2 + m1) * d1 : 0.0;
    const double dk2 = g.dk * g.dk, m1sq = (double)m1 * m1;
    for (int p2 = threadIdx.x / TC4; p2 < g.N2; p2 += Q4) {
      const double m2sq = rb[3 * p2 + 2];
      double fac = 0.0;
      if (col_in && m2sq >= 0.0) {
        const double k2 = dk2 * (m1sq + m2sq);
        if (k2 * g.db > 0.25) {
          // (e^{-k^2 d1} - e^{-k^2 d2}) / k^2 from the separable exponentials (no cancellation here: the
          // difference is >= 0.2 e^{-k^2 d1} once k^2 d2 > 1/4 with d2 = 32 d1); vp_mult_nh (expm1) below
          fac = fma(a1, rb[3 * p2], -a2 * rb[3 * p2 + 1]) * rcp_nr(k2);
        } else {
          const int a2m = (int)llrint(sqrt(m2sq));
          fac = vp_mult_nh(k2, g.da, g.db) * d1 * __ldg(g.deconv + a2m);
        }
      }
      const double2 v = sm2[p2 * TC4 + c];
      sm2[p2 * TC4 + c] = make_double2(v.x * fac, v.y * fac);
    }
  } else {
    for (int p2 = threadIdx.x / TC4; p2 < g.N2; p2 += Q4) {
      const int k = k1 + g.N1 * __ldg(g.sig2 + p2);
      const int m2 = k <= g.nf / 2 ? k : k - g.nf, a2m = m2 < 0 ? -m2 : m2;
      double fac = 0.0;
      if (m1 <= g.half_modes && a2m <= g.half_modes) {
        const double k2 = g.dk * g.dk * ((double)m1 * m1 + (double)m2 * m2);
        fac = vp_mult_fh(k2, g.da, g.db) * d1 * __ldg(g.deconv + a2m);
      }
      const double2 v = sm2[p2 * TC4 + c];
      sm2[p2 * TC4 + c] = make_double2(v.x * fac, v.y * fac);
    }
  }
  __syncthreads();
  fft_run_t<1, true>(sm2, g.s2, g.tw2);
  for (int n2 = threadIdx.x / TC4; n2 < g.N2; n2 += Q4) {
    double2 w = __ldg(g.twN + n2 * k1);
    w.y = -w.y;
    sm2[n2 * TC4 + c] = cmul(sm2[n2 * TC4 + c], w);
  }
  fft4_store(sm2, g, c0, ncol, row0, 1, g.N2);
}

// C: blockIdx.x = column tile, blockIdx.y = n2'
__global__ void __launch_bounds__(256, 4) k_fft4_c(Fft4Args g) {
  extern __shared__ double2 sm2[];
  const int c0 = blockIdx.x * TC4, ncol = min(TC4, g.ncs - c0), n2 = blockIdx.y;
  fft4_load(sm2, g, c0, ncol, n2, g.N2, g.N1);
  fft_run_t<1, true>(sm2, g.s1, g.tw1);
  fft4_store(sm2, g, c0, ncol, n2, g.N2, g.N1);
}

// nf = N1 N2 with both factors 2,3,5,7-smooth and N1 the divisor closest to sqrt(nf)
static bool fft4_factor(int nf, int &N1, int &N2, FftStages &s1, FftStages &s2) {
  int best = -1;
  for (int d = 2; d * d <= nf * 4 && d < nf; d++) {
    if (nf % d) continue;
    FftStages a, b;
    if (!factor_stages(d, a) || !factor_stages(nf / d, b)) continue;
    if (d > 512 || nf / d > 512) continue;
    if (best < 0 || std::abs(d - std::sqrt((double)nf)) < std::abs(best - std::sqrt((double)nf))) best = d;
  }
  if (best < 0) return false;
  N1 = best;
  N2 = nf / best;
  return factor_stages(N1, s1) && factor_stages(N2, s2);
}

bool vp_fft4_setup(vp_plan_s *P, VpGrid &G) {
  // measured crossover: cuFFT 2D D2Z + multiply + Z2D is faster up to ~10^4 (config 3, n_f = 8640: 2.4 vs 2.9 ms
  // for transforms, multiply and prolongation), the four-step pass with own rows above (config 4, 12500: 5.5 vs
  // 7.2 ms; config 5, 23328: 14.7 vs 25.1 ms)
  if (P->opts.fft_mode != 0 || G.nf <= VP_FFT4_MIN_NF || G.nf > (1 << 30)) return false;
  int N1, N2;
  FftStages s1, s2;
  if (!fft4_factor((int)G.nf, N1, N2, s1, s2)) return false;
  upload_dft_roots();  // odd-radix butterflies read the constant-bank roots
  G.f4_N1 = N1;
  G.f4_N2 = N2;
  static_assert(sizeof(FftStages) <= sizeof(G.fft_st_r), "stage buffer");
  memcpy(G.fft_st_r, &s1, sizeof(s1));
  memcpy(G.fft_st_c, &s2, sizeof(s2));
  G.f4_tw1 = twiddle_table(P, N1);
  G.f4_tw2 = twiddle_table(P, N2);
  G.f4_twN = twiddle_table(P, (int)G.nf);
  std::vector<int32_t> g1, g2;
  digit_sigma(s1, g1);
  digit_sigma(s2, g2);
  G.f4_sig1 = vp_alloc<int32_t>(P, N1);
  G.f4_sig2 = vp_alloc<int32_t>(P, N2);
  VP_CUDA(cudaMemcpy(G.f4_sig1, g1.data(), 4 * N1, cudaMemcpyHostToDevice));
  VP_CUDA(cudaMemcpy(G.f4_sig2, g2.data(), 4 * N2, cudaMemcpyHostToDevice));
  G.fft_ncs = (int)std::min<int64_t>(G.nmode / 2 + 1, G.nf / 2 + 1);
  if (G.kind == 0) {  // separable exponentials of the NH multiplier (k_fft4_b)
    const int64_t nh = G.nmode / 2 + 1;
    const double dk = 2.0 * VP_PI / G.L;
    std::vector<double> a(nh), b(nh);
    for (int64_t m = 0; m < nh; m++) {
      a[m] = std::exp(-dk * dk * (double)m * (double)m * G.delta_a);
      b[m] = std::exp(-dk * dk * (double)m * (double)m * G.delta_b);
    }
    G.f4_e1 = vp_alloc<double>(P, nh);
    G.f4_e2 = vp_alloc<double>(P, nh);
    VP_CUDA(cudaMemcpy(G.f4_e1, a.data(), sizeof(double) * nh, cudaMemcpyHostToDevice));
    VP_CUDA(cudaMemcpy(G.f4_e2, b.data(), sizeof(double) * nh, cudaMemcpyHostToDevice));
  }
  G.four_step = true;
  return true;
}

void vp_fft4_columns(vp_plan_s *P, VpGrid &G) {
  Fft4Args g;
  g.spec = (double2 *)G.cdata;
  g.nc = G.nf / 2 + 1;
  g.ncs = G.fft_ncs;
  g.nf = (int)G.nf;
  g.N1 = G.f4_N1;
  g.N2 = G.f4_N2;
  memcpy(&g.s1, G.fft_st_r, sizeof(g.s1));
  memcpy(&g.s2, G.fft_st_c, sizeof(g.s2));
  g.tw1 = G.f4_tw1;
  g.tw2 = G.f4_tw2;
  g.twN = G.f4_twN;
  g.sig1 = G.f4_sig1;
  g.sig2 = G.f4_sig2;
  g.kind = G.kind;
  g.da = G.delta_a;
  g.db = G.delta_b;
  g.scale = G.mult_scale;
  g.dk = 2.0 * VP_PI / G.L;
  g.half_modes = G.nmode / 2;
  g.deconv = G.deconv;
  g.e1 = G.f4_e1;
  g.e2 = G.f4_e2;
  const unsigned ntile = (unsigned)((g.ncs + TC4 - 1) / TC4);
  const size_t sm1 = sizeof(double2) * (size_t)TC4 * g.N1, sm2 = sizeof(double2) * (size_t)TC4 * g.N2 + 24 * (size_t)g.N2;
  vp_smem_attr((const void *)k_fft4_a, sm1);
  vp_smem_attr((const void *)k_fft4_b, sm2);
  vp_smem_attr((const void *)k_fft4_c, sm1);
  k_fft4_a<<<dim3(ntile, g.N2), 256, sm1, P->stream>>>(g);
  VP_CHECK_LAUNCH();
  k_fft4_b<<<dim3(ntile, g.N1), 256, sm2, P->stream>>>(g);
  VP_CHECK_LAUNCH();
  k_fft4_c<<<dim3(ntile, g.N2), 256, sm1, P->stream>>>(g);
  VP_CHECK_LAUNCH();
  // cuFFT's inverse row transforms read the whole half spectrum: the columns beyond the kept band are zero (the
  // own row passes read only the kept columns)
  const int64_t nz = g.nc - g.ncs;
  if (nz > 0 && !G.f4_rows)
    VP_CUDA(cudaMemset2DAsync(g.spec + g.ncs, sizeof(double2) * g.nc, 0, sizeof(double2) * nz, G.nf, P->stream));
  P->n_kernels += 3;
}

// ---- large-grid row passes (four-step grids with nf % 4 == 0): pruned real FFT by radix-4 decimation in time.
// Q = nf/4, y_r[m] = x[4m + r], Y_r = FFT_Q(y_r); X[k] = sum_r W_nf^{rk} Y_r[k mod Q] for the kept k < ncs <= Q + 1.
// Two complex Q-point FFTs per row (z_h = y_{2h} + i y_{2h+1}, h = 0, 1: Y_{2h}[j] = (Z_h[j] + conj Z_h[Q-j]) / 2,
// Y_{2h+1}[j] = -i (Z_h[j] - conj Z_h[Q-j]) / 2).  One CTA holds a whole row: both Q-length sequences in shared
// memory (2 Q x 16 B, 187 KB at config 5), loaded by cp.async (16-byte chunk c of the row = (x[2c], x[2c+1]) is
// z_{c & 1}[c >> 1]: every chunk of the row is in flight at once, each byte read once), both transforms advanced
// stage by stage with one barrier per stage, X[k] combined from both in shared memory and written once; only the
// kept columns are written (the inverse reads only them: no zeroing of the rest).  Measured at config 5 (NH):
// the first form (halves one after the other in 93 KB, X accumulated through global memory, 16 warps/SM) 5.1 ms;
// a cluster of two CTAs per row (one half each, X combined through distributed shared memory) 5.4 ms (the
// interleaved 16-byte halves of a row were read / written twice as often from HBM); this form 4.1 ms at 512
// threads.
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}

template <int DIR, bool DIT>
__device__ void fft_run2(double2 *a0, double2 *a1, const FftStages &st, const double2 *tw) {
  for (int i = 0; i < st.S; i++) {
    const int s = DIT ? i : st.S - 1 - i;
    switch (st.r[s]) {
#define VP_RUN2(R)                                                \
  case R:                                                         \
    fft_stage<R, DIR, DIT>(a0, st.n, st.Lp[s], st.invLp[s], tw); \
    fft_stage<R, DIR, DIT>(a1, st.n, st.Lp[s], st.invLp[s], tw); \
    break;
      VP_RUN2(2) VP_RUN2(3) VP_RUN2(4) VP_RUN2(5) VP_RUN2(7) VP_RUN2(8) VP_RUN2(9)
#undef VP_RUN2
      default: break;
    }
    __syncthreads();
  }
}

#ifndef VP_ROWQ_THREADS
#define VP_ROWQ_THREADS 1024
#endif
__global__ void __launch_bounds__(VP_ROWQ_THREADS, 1) k_row4_fwd(const double *__restrict__ grid, int64_t row_pitch,
                                                                 double2 *__restrict__ spec, int64_t nc, int ncs, int nf,
                                                                 FftStages st, const double2 *__restrict__ twQ,
                                                                 const double2 *__restrict__ twN,
                                                                 const int32_t *__restrict__ posQ) {
  extern __shared__ double2 z[];
  const int Q = st.n;
  double2 *z0 = z, *z1 = z + Q;
  for (int r = blockIdx.x; r < nf; r += gridDim.x) {
    const double2 *x2 = (const double2 *)(grid + (int64_t)r * row_pitch);
    for (int c = threadIdx.x; c < 2 * Q; c += blockDim.x) cp_async16(((c & 1) ? z1 : z0) + (c >> 1), x2 + c);
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    fft_run2<-1, false>(z0, z1, st, twQ);
    double2 *X = spec + (int64_t)r * nc;
    for (int k = threadIdx.x; k < ncs; k += blockDim.x) {
      const int j = k < Q ? k : 0;
      const int pj = __ldg(posQ + j), pm = __ldg(posQ + (j ? Q - j : 0));
      const double2 w1 = __ldg(twN + k);  // W_nf^k; W^{2k}, W^{3k} by multiplication
      const double2 w2 = cmul(w1, w1), w3 = cmul(w2, w1);
      double2 v;
      {
        const double2 zj = z0[pj], zm = z0[pm];
        const double2 ya = make_double2(0.5 * (zj.x + zm.x), 0.5 * (zj.y - zm.y));   // Y_0[j]
        const double2 yb = make_double2(0.5 * (zj.y + zm.y), -0.5 * (zj.x - zm.x));  // Y_1[j]
        const double2 b = cmul(w1, yb);
        v = make_double2(ya.x + b.x, ya.y + b.y);
      }
      {
        const double2 zj = z1[pj], zm = z1[pm];
        const double2 ya = make_double2(0.5 * (zj.x + zm.x), 0.5 * (zj.y - zm.y));   // Y_2[j]
        const double2 yb = make_double2(0.5 * (zj.y + zm.y), -0.5 * (zj.x - zm.x));  // Y_3[j]
        const double2 a = cmul(w2, ya), b = cmul(w3, yb);
        v.x += a.x + b.x;
        v.y += a.y + b.y;
      }
      X[k] = v;
    }
    __syncthreads();  // z0 / z1 are refilled for the next row
  }
}

// inverse: x[4m + r] = sum_{k in band} X[k] W_nf^{-(4m + r) k} (unnormalised, as cuFFT Z2D) = IFFT_Q(S_r)[m] with
// S_r[j] = ([j < ncs] X[j] + [Q - j < ncs] conj(X[Q - j]) (-i)^r) W_nf^{-rj} for j >= 1 and
// S_r[0] = X[0] + [ncs > Q] (conj(X[Q]) (-i)^r + X[Q] i^r); S_r is Hermitian, so IFFT(S_{2h} + i S_{2h+1}) =
// y_{2h} + i y_{2h+1} with real y.  Both h in one CTA: X is read once, the real row written as 32-byte groups
// (x[4m .. 4m + 3] = z0[m], z1[m]).
// PM > 0 fuses the x pass of the far-history prolongation (k_prolong_x_fix: q1[r][i] += sum_{i'} w[i + j - PM i']
// t2[r][i' - e_lo]) for grid ratio PM: the CTA adds it to its row in shared memory before the row
// is written, so the NH grid is written once instead of written, read and written again (8.7 GB at config 5).
struct RowProlong {
  const double *t2;    // [nf rows][ne] y-prolongated far-history field (vp_launch_prolong pass 1)
  int64_t ne, e_lo;    // t2 column range [e_lo, e_lo + ne)
  int64_t c_lo;        // first FH column whose images i = PM c + k - j reach the row
  int nc, QH, j;
};

// taps of the fused prolongation (grid ratio 5): w[q + QH] = psi_FH(2q / (5w)), |q| <= QH = (5w - 1) / 2, one slot
// per QH in {22, 24, 27} (w = 9, 10, 11); the values depend on w only (beta = 2.30 w), so a slot is written once
// per device, synchronously, with identical bytes for every plan
__constant__ double c_ptap[3][56];
static int ptap_slot(int QH) { return QH == 22 ? 0 : (QH == 24 ? 1 : (QH == 27 ? 2 : -1)); }
static void upload_ptap(int QH, const double *w) {
  static std::mutex mu;
  static std::set<std::pair<int, int>> done;
  const int dev = vp_current_device();
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(std::make_pair(dev, QH))) return;
  VP_CUDA(cudaMemcpyToSymbol(c_ptap, w, sizeof(double) * (2 * QH + 1), sizeof(double) * 56 * ptap_slot(QH)));
  done.insert(std::make_pair(dev, QH));
}

template <int PM, int QH>
__global__ void __launch_bounds__(VP_ROWQ_THREADS, 1) k_row4_inv(const double2 *__restrict__ spec, int64_t nc, int ncs,
                                                                 int nf, double *__restrict__ grid, int64_t row_pitch,
                                                                 FftStages st, const double2 *__restrict__ twQ,
                                                                 const double2 *__restrict__ twN,
                                                                 const int32_t *__restrict__ posQ, RowProlong pr) {
  extern __shared__ double2 z[];
  const int Q = st.n;
  double2 *z0 = z, *z1 = z + Q;
  for (int r = blockIdx.x; r < nf; r += gridDim.x) {
    const double2 *X = spec + (int64_t)r * nc;
    for (int j = threadIdx.x; j < Q; j += blockDim.x) {
      const double2 xj = j < ncs ? X[j] : make_double2(0.0, 0.0);
      const int jm = j ? Q - j : Q;  // partner frequency k = j - Q
      const double2 xm = jm < ncs ? X[jm] : make_double2(0.0, 0.0);
      const double2 xq = (j == 0 && ncs > Q) ? X[Q] : make_double2(0.0, 0.0);  // k = +Q (j = 0 only)
      double2 w1 = __ldg(twN + j);  // W_nf^{j}; conjugated powers W^{-rj} by multiplication
      w1.y = -w1.y;
      const double2 w2 = cmul(w1, w1), w3 = cmul(w2, w1);
      double2 sv[4];
#pragma unroll
      for (int rr = 0; rr < 4; rr++) {  // (-i)^rr conj(X[Q-j]) + i^rr X[Q]
        double2 c = make_double2(xm.x, -xm.y), d = xq;
#pragma unroll
        for (int t = 0; t < rr; t++) {
          c = make_double2(c.y, -c.x);
          d = make_double2(-d.y, d.x);
        }
        const double2 acc = make_double2(xj.x + c.x + d.x, xj.y + c.y + d.y);
        sv[rr] = rr == 0 ? acc : cmul(acc, rr == 1 ? w1 : (rr == 2 ? w2 : w3));
      }
      const int pj = __ldg(posQ + j);
      z0[pj] = make_double2(sv[0].x - sv[1].y, sv[0].y + sv[1].x);  // S_0 + i S_1
      z1[pj] = make_double2(sv[2].x - sv[3].y, sv[2].y + sv[3].x);  // S_2 + i S_3
    }
    __syncthreads();
    fft_run2<1, true>(z0, z1, st, twQ);
    if constexpr (PM > 0) {
      // a thread owns FH column c and the PM row elements i = PM c + k - j it reaches (disjoint across threads);
      // compile-time taps (constant-bank DFMA operands)
      constexpr int SL = QH == 22 ? 0 : (QH == 24 ? 1 : 2);
      constexpr int DLO = -(QH / PM), DHI = (PM - 1 + QH) / PM;
      const double *t2r = pr.t2 + r * pr.ne - pr.e_lo;
      for (int cc = threadIdx.x; cc < pr.nc; cc += blockDim.x) {
        const int64_t c = pr.c_lo + cc;
        double acc[PM];
#pragma unroll
        for (int k = 0; k < PM; k++) acc[k] = 0.0;
#pragma unroll
        for (int d = DLO; d <= DHI; d++) {
          const int64_t ip = c + d;
          const double x = (ip >= pr.e_lo && ip < pr.e_lo + pr.ne) ? __ldg(t2r + ip) : 0.0;
#pragma unroll
          for (int k = 0; k < PM; k++) {
            const int q = k - PM * d;
            if (q >= -QH && q <= QH) acc[k] = fma(c_ptap[SL][q + QH], x, acc[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < PM; k++) {
          const int64_t i = PM * c + k - pr.j;
          if (i >= 0 && i < nf) ((double *)((i & 2) ? z1 : z0))[2 * (i >> 2) + (i & 1)] += acc[k];
        }
      }
      __syncthreads();
    }
    double2 *x2 = (double2 *)(grid + (int64_t)r * row_pitch);
    for (int c = threadIdx.x; c < 2 * Q; c += blockDim.x) x2[c] = ((c & 1) ? z1 : z0)[c >> 1];
    __syncthreads();
  }
}

bool vp_fft4_rows_setup(vp_plan_s *P, VpGrid &G) {
  if (G.nf % 4) return false;
  const int Q = (int)(G.nf / 4);
  FftStages st;
  if (!factor_stages(Q, st)) return false;
  const size_t sm = 2 * sizeof(double2) * (size_t)Q;  // both half-sequences of a row
  if (sm > 220 * 1024) return false;
  if (G.fft_ncs > Q + 1) return false;
  std::vector<int32_t> sig, pos(Q);
  digit_sigma(st, sig);
  for (int p = 0; p < Q; p++) pos[sig[p]] = p;
  G.f4_posQ = vp_alloc<int32_t>(P, Q);
  VP_CUDA(cudaMemcpy(G.f4_posQ, pos.data(), 4 * (size_t)Q, cudaMemcpyHostToDevice));
  G.f4_twQ = twiddle_table(P, Q);
  static_assert(sizeof(FftStages) <= sizeof(G.f4_stQ), "stage buffer");
  memcpy(G.f4_stQ, &st, sizeof(st));
  vp_smem_attr((const void *)k_row4_fwd, sm);
  vp_smem_attr((const void *)k_row4_inv<0, 0>, sm);
  G.f4_rows = true;
  return true;
}

static unsigned row4_grid(size_t smem, int64_t rows) {
  int per = (int)std::min<size_t>(2, (227 * 1024) / (smem + 2048));
  if (per < 1) per = 1;
  return (unsigned)std::min<int64_t>(rows, (int64_t)per * num_sms());
}

void vp_fft4_rows_fwd(vp_plan_s *P, VpGrid &G) {
  FftStages st;
  memcpy(&st, G.f4_stQ, sizeof(st));
  const size_t sm = 2 * sizeof(double2) * (size_t)st.n;
  k_row4_fwd<<<row4_grid(sm, G.nf), VP_ROWQ_THREADS, sm, P->stream>>>(G.data, G.row, (double2 *)G.cdata, G.nf / 2 + 1, G.fft_ncs,
                                                          (int)G.nf, st, G.f4_twQ, G.f4_twN, G.f4_posQ);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

// inverse row pass; pr.t2 != nullptr fuses the prolongation's x pass for grid ratio 5 (the caller checked
// vp_fft4_rows_prolong_ok)
void vp_fft4_rows_inv(vp_plan_s *P, VpGrid &G, const RowProlong *pr) {
  FftStages st;
  memcpy(&st, G.f4_stQ, sizeof(st));
  const size_t sm = 2 * sizeof(double2) * (size_t)st.n;
  RowProlong none;
  memset(&none, 0, sizeof(none));
  const unsigned nb = row4_grid(sm, G.nf);
  const double2 *spec = (const double2 *)G.cdata;
#define VP_ROWINV(PM, QH, ARG)                                                                                  \
  {                                                                                                           \
    vp_smem_attr((const void *)k_row4_inv<PM, QH>, sm);                                                       \
    k_row4_inv<PM, QH><<<nb, VP_ROWQ_THREADS, sm, P->stream>>>(spec, G.nf / 2 + 1, G.fft_ncs, (int)G.nf, G.data, \
                                                               G.row, st, G.f4_twQ, G.f4_twN, G.f4_posQ, ARG);  \
  }
  if (pr && pr->t2 && pr->QH == 22) VP_ROWINV(5, 22, *pr)
  else if (pr && pr->t2 && pr->QH == 24) VP_ROWINV(5, 24, *pr)
  else if (pr && pr->t2 && pr->QH == 27) VP_ROWINV(5, 27, *pr)
  else VP_ROWINV(0, 0, none)
#undef VP_ROWINV
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

// the fused prolongation needs the NH grid on own row passes, integer ratio 5 with tabulated taps, and shared
// memory for the taps next to the row
bool vp_fft4_rows_prolong_ok(vp_plan_s *P) {
  if (!P->nh.f4_rows || P->tap_qh <= 0 || P->fh_ratio != 5 || ptap_slot(P->tap_qh) < 0) return false;
  upload_ptap(P->tap_qh, P->tap_w);  // once per (device, QH)
  return true;
}

void vp_fft4_rows_inv_prolong(vp_plan_s *P) {
  RowProlong pr;
  memset(&pr, 0, sizeof(pr));
  const int M = 5;
  const int64_t j = P->fh_shift;
  pr.t2 = P->scratch;
  pr.ne = P->e_n;
  pr.e_lo = P->e_lo;
  pr.c_lo = (j >= 0) ? j / M : -((-j + M - 1) / M);
  const int64_t c_hi = (P->nh.nf - 1 + j) / M;
  pr.nc = (int)(c_hi - pr.c_lo + 1);
  pr.QH = P->tap_qh;
  pr.j = (int)j;
  vp_fft4_rows_inv(P, P->nh, &pr);
}
