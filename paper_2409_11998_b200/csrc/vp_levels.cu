// vp_levels.cu -- plan-time construction of the level-band corrections for graded meshes
// (DESIGN.md §5.6 and reading R15).
//
// The paper's method is "suitable only for quasi-uniform triangulations":
// with one global delta_1 = C Dx^2 the local expansion V_L[delta_1] fails where the mesh (and f) vary
// on scales below sqrt(delta_1).  The telescoping identity of §4.1 (lines 1200-1252, "extends
// naturally to the ... volume heat potential") splits the local time interval dyadically:
//
//   V_L[delta_0](x) = sum_{l=1}^{l(x)} B_l(x) + V_L[delta_{l(x)}](x),   delta_l = delta_0 / 4^l,
//   B_l(x) = int_{delta_l}^{delta_{l-1}} int_Omega K_t(x - y) f(y) dy dt = sum_j c_j K_l(x - x_j),
//   K_l(r) = (1/4pi) [E1(r^2 / 4 delta_{l-1}) - E1(r^2 / 4 delta_l)]      (the paper's K_j, eq. eiformula)
//
// with Fourier transform (e^{-k^2 delta_l} - e^{-k^2 delta_{l-1}}) / k^2 -- a near-history multiplier
// with (delta_l, delta_{l-1}).  Each band is evaluated by a box-local NUFFT: level-l targets are
// grouped into square core boxes of side core * h_l; every box gets its own periodic fine grid of
// nfb^2 points (spacing h_l = pi / (2 k_l), k_l = sqrt(ln(1/eps) / delta_l)) holding the sources
// within r_eps = sqrt(4 delta_{l-1} z_eps) (E1(z_eps) = eps) of the core; the margin keeps both the
// aliased images (period nfb h_l >= core + 2 r_eps) and the spreading footprints inside the box.
// All boxes of all levels live in one "virtual" grid (box b = rows [b nfb, (b+1) nfb)), so the
// eval is one spread, one batched D2Z, one multiply, one batched Z2D and one interpolation.
//
// Level of a target (plan time): node y carries lambda(y) = floor(log4(delta_0 / (C_min Dx_loc^2(y))))
// with Dx_loc^2 the larger of its triangle's mean weight (the paper's Dx^2 = sum w / N, P:1352,
// taken locally) and diam^2 / 48; l(x) = the largest l such that every node within the 3 x 3 cells
// of side rho sqrt(delta_l) around x has lambda >= l (and so for all coarser levels).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "vp_common.cuh"
#include "vp_math.cuh"

__global__ void k_node_lambda(const double *__restrict__ nodes, const double *__restrict__ w, int64_t M, int p,
                              double delta0, double cmin, int lcap, int8_t *__restrict__ lam, int *__restrict__ lmax) {
  int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int l = 0;
  if (m < M) {
    const double *nd = nodes + m * (int64_t)p * 2;
    const double *ww = w + m * (int64_t)p;
    double sw = 0.0, d2 = 0.0;
    for (int k = 0; k < p; k++) {
      sw += ww[k];
      for (int j = 0; j < k; j++) {
        double dx = nd[2 * k] - nd[2 * j], dy = nd[2 * k + 1] - nd[2 * j + 1];
        d2 = fmax(d2, dx * dx + dy * dy);
      }
    }
    // node spread of the 12-point rule = 0.8107 x triangle diameter; diam^2 / 48 = mean weight for a
    // right isosceles triangle, and larger for slivers (whose nodes resolve only along the long side)
    double dx2 = sw / p;
    if (p == 12) dx2 = fmax(dx2, d2 / (0.8107329565254939 * 0.8107329565254939 * 48.0));
    if (dx2 > 0.0) {
      double r = delta0 / (cmin * dx2);
      l = r >= 1.0 ? (int)floor(log(r) / log(4.0)) : 0;
    } else {
      l = lcap;  // zero-weight (degenerate) triangle: no constraint
    }
    l = l < 0 ? 0 : (l > lcap ? lcap : l);
    for (int k = 0; k < p; k++) lam[m * p + k] = (int8_t)l;
  }
  typedef cub::BlockReduce<int, 256> BR;
  __shared__ typename BR::TempStorage ts;
  int bm = BR(ts).Reduce(m < M ? l : 0, cub::Max());
  if (threadIdx.x == 0) atomicMax(lmax, bm);
}

__global__ void k_cell_keys(const double *__restrict__ xy, int64_t n, double ox, double oy, double inv_c, int64_t ncx,
                            int64_t ncy, const int8_t *__restrict__ lam, uint64_t *__restrict__ keys,
                            int32_t *__restrict__ vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t cx = (int64_t)floor((xy[2 * i] - ox) * inv_c), cy = (int64_t)floor((xy[2 * i + 1] - oy) * inv_c);
  cx = cx < 0 ? 0 : (cx >= ncx ? ncx - 1 : cx);
  cy = cy < 0 ? 0 : (cy >= ncy ? ncy - 1 : cy);
  keys[i] = (uint64_t)(cy * ncx + cx);
  vals[i] = lam[i];
}

__device__ __forceinline__ int64_t bsearch_u64(const uint64_t *__restrict__ a, int64_t n, uint64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return (lo < n && a[lo] == key) ? lo : -1;
}

__global__ void k_level_test(const double *__restrict__ tx, const double *__restrict__ ty, int64_t T,
                             int8_t *__restrict__ tlev, int l, double ox, double oy, double inv_c, int64_t ncx,
                             int64_t ncy, const uint64_t *__restrict__ ukeys, const int32_t *__restrict__ umin,
                             int64_t nu) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T || tlev[t] != l - 1) return;
  int64_t cx = (int64_t)floor((tx[t] - ox) * inv_c), cy = (int64_t)floor((ty[t] - oy) * inv_c);
  bool any = false, ok = true;
  for (int dy = -1; dy <= 1 && ok; dy++)
    for (int dx = -1; dx <= 1 && ok; dx++) {
      int64_t x = cx + dx, y = cy + dy;
      if (x < 0 || y < 0 || x >= ncx || y >= ncy) continue;
      int64_t i = bsearch_u64(ukeys, nu, (uint64_t)(y * ncx + x));
      if (i >= 0) {
        any = true;
        if (umin[i] < l) ok = false;
      }
    }
  if (ok && any) tlev[t] = (int8_t)l;
}

// ---------------------------------------------------------------------------------------------
// boxes: key = level << 58 | by << 29 | bx
struct BoxGeom {
  double x_lo, y_lo;
  double h[16], C[16], r[16];  // per level: fine spacing, core side, source reach
  int margin, nfb;
};

__device__ __forceinline__ uint64_t box_key(int l, int64_t bx, int64_t by) {
  return ((uint64_t)l << 58) | ((uint64_t)by << 29) | (uint64_t)bx;
}

__global__ void k_entry_keys(const double *__restrict__ tx, const double *__restrict__ ty,
                             const int32_t *__restrict__ lt_t, const int32_t *__restrict__ lt_off, int64_t n_lt,
                             const int8_t *__restrict__ tlev, BoxGeom bg, uint64_t *__restrict__ ekeys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_lt) return;
  const int32_t t = lt_t[i];
  const double x = tx[t], y = ty[t];
  for (int l = 1; l <= tlev[t]; l++) {
    int64_t bx = (int64_t)floor((x - bg.x_lo) / bg.C[l]), by = (int64_t)floor((y - bg.y_lo) / bg.C[l]);
    bx = bx < 0 ? 0 : bx;
    by = by < 0 ? 0 : by;
    ekeys[lt_off[i] + l - 1] = box_key(l, bx, by);
  }
}

__device__ __forceinline__ void box_origin(const BoxGeom &bg, uint64_t key, int *l, double *ox, double *oy) {
  int lv = (int)(key >> 58);
  int64_t by = (int64_t)((key >> 29) & ((1ull << 29) - 1)), bx = (int64_t)(key & ((1ull << 29) - 1));
  *l = lv;
  *ox = bg.x_lo + bx * bg.C[lv] - bg.margin * bg.h[lv];
  *oy = bg.y_lo + by * bg.C[lv] - bg.margin * bg.h[lv];
}

__global__ void k_entry_coords(const double *__restrict__ tx, const double *__restrict__ ty,
                               const int32_t *__restrict__ lt_t, const int32_t *__restrict__ lt_off, int64_t n_lt,
                               const int8_t *__restrict__ tlev, const uint64_t *__restrict__ ekeys,
                               const uint64_t *__restrict__ ubox, int64_t nbox, BoxGeom bg, double *__restrict__ ex,
                               double *__restrict__ ey) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_lt) return;
  const int32_t t = lt_t[i];
  const double x = tx[t], y = ty[t];
  for (int l = 1; l <= tlev[t]; l++) {
    int64_t e = lt_off[i] + l - 1;
    int64_t b = bsearch_u64(ubox, nbox, ekeys[e]);
    int lv;
    double ox, oy;
    box_origin(bg, ubox[b], &lv, &ox, &oy);
    ex[e] = (x - ox) / bg.h[lv];
    ey[e] = (y - oy) / bg.h[lv] + (double)b * bg.nfb;
  }
}

__global__ void k_box_levels(const uint64_t *__restrict__ ubox, int64_t nbox, int32_t *__restrict__ blev) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b < nbox) blev[b] = (int32_t)(ubox[b] >> 58);
}

// (box, source) pairs: every source within reach r_l of an active level-l box core
template <bool FILL>
__global__ void k_src_pairs(const double *__restrict__ xy, const double *__restrict__ w, int64_t N, int nlev,
                            const uint64_t *__restrict__ ubox, int64_t nbox, BoxGeom bg,
                            int64_t *__restrict__ count, const int64_t *__restrict__ off, double *__restrict__ pxy,
                            double *__restrict__ pw, int32_t *__restrict__ pnode) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= N) return;
  const double x = xy[2 * j], y = xy[2 * j + 1], wj = w[j];
  int64_t c = 0, o = FILL ? off[j] : 0;
  if (wj != 0.0) {
    for (int l = 1; l <= nlev; l++) {
      const double C = bg.C[l], r = bg.r[l];
      int64_t bx0 = (int64_t)floor((x - bg.x_lo - r) / C), bx1 = (int64_t)floor((x - bg.x_lo + r) / C);
      int64_t by0 = (int64_t)floor((y - bg.y_lo - r) / C), by1 = (int64_t)floor((y - bg.y_lo + r) / C);
      bx0 = bx0 < 0 ? 0 : bx0;
      by0 = by0 < 0 ? 0 : by0;
      for (int64_t by = by0; by <= by1; by++)
        for (int64_t bx = bx0; bx <= bx1; bx++) {
          int64_t b = bsearch_u64(ubox, nbox, box_key(l, bx, by));
          if (b < 0) continue;
          if (FILL) {
            int lv;
            double ox, oy;
            box_origin(bg, ubox[b], &lv, &ox, &oy);
            pxy[2 * (o + c)] = (x - ox) / bg.h[lv];
            pxy[2 * (o + c) + 1] = (y - oy) / bg.h[lv] + (double)b * bg.nfb;
            pw[o + c] = wj;
            pnode[o + c] = (int32_t)j;
          }
          c++;
        }
    }
  }
  if (!FILL) count[j] = c;
}

__global__ void k_interleave(const double *__restrict__ x, const double *__restrict__ y, int64_t n,
                             double *__restrict__ xy) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    xy[2 * i] = x[i];
    xy[2 * i + 1] = y[i];
  }
}

__global__ void k_lev_flag(const int8_t *__restrict__ tlev, int64_t T, int32_t *__restrict__ flag,
                           int32_t *__restrict__ val) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  flag[t] = tlev[t] > 0 ? 1 : 0;
  val[t] = tlev[t];
}

__global__ void k_gather_i32(const int32_t *__restrict__ src, const int32_t *__restrict__ idx, int64_t n,
                             int32_t *__restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

template <typename T>
static T *tmp_alloc(size_t n, cudaStream_t s) {
  void *p = nullptr;
  VP_CUDA(cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), s));
  return (T *)p;
}

static int64_t fetch_i64(const int64_t *d, cudaStream_t s) {
  int64_t h = 0;
  VP_CUDA(cudaMemcpyAsync(&h, d, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  VP_CUDA(cudaStreamSynchronize(s));
  return h;
}

void vp_build_levels(vp_plan_s *P, const double *nodes, const double *weights) {
  VpBands &B = P->bands;
  cudaStream_t s = P->stream;
  const int64_t N = P->N, T = P->T;
  B.tlev = vp_alloc<int8_t>(P, T);
  VP_CUDA(cudaMemsetAsync(B.tlev, 0, T, s));
  const vp_opts &o = P->opts;
  if (o.levels < 0) return;
  const int lcap = o.levels > 0 ? std::min(o.levels, 12) : 12;
  const double cmin = o.level_cmin > 0 ? o.level_cmin : 1.5;
  const double rho = o.level_rho > 0 ? o.level_rho : 4.0;
  const double d0 = P->delta1;
  // ---- lambda per node
  int8_t *lam = tmp_alloc<int8_t>(N, s);
  int *d_lmax = tmp_alloc<int>(1, s);
  VP_CUDA(cudaMemsetAsync(d_lmax, 0, sizeof(int), s));
  k_node_lambda<<<(unsigned)((P->M + 255) / 256), 256, 0, s>>>(nodes, weights, P->M, P->p, d0, cmin, lcap, lam, d_lmax);
  VP_CHECK_LAUNCH();
  int lmax = 0;
  VP_CUDA(cudaMemcpyAsync(&lmax, d_lmax, sizeof(int), cudaMemcpyDeviceToHost, s));
  VP_CUDA(cudaStreamSynchronize(s));
  const double x_lo = P->cx - 0.5 * P->S, y_lo = P->cy - 0.5 * P->S;
  // ---- per-target level by the neighbourhood test, level by level
  if (lmax > 0) {
    uint64_t *keys = tmp_alloc<uint64_t>(N, s), *keys2 = tmp_alloc<uint64_t>(N, s), *ukeys = tmp_alloc<uint64_t>(N, s);
    int32_t *vals = tmp_alloc<int32_t>(N, s), *vals2 = tmp_alloc<int32_t>(N, s), *umin = tmp_alloc<int32_t>(N, s);
    int64_t *d_nu = tmp_alloc<int64_t>(1, s);
    size_t tb1 = 0, tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb1, keys, keys2, vals, vals2, (int)N, 0, 64, s);
    cub::DeviceReduce::ReduceByKey(nullptr, tb2, keys2, ukeys, vals2, umin, d_nu, cub::Min(), (int)N, s);
    void *tmp = tmp_alloc<char>(std::max(tb1, tb2) + 16, s);
    for (int l = 1; l <= lmax; l++) {
      double c = rho * sqrt(d0 / pow(4.0, l));
      int64_t ncx = (int64_t)ceil(P->S / c) + 3;
      if ((double)ncx * (double)ncx > 9e18) break;
      double ox = x_lo - c, oy = y_lo - c;
      k_cell_keys<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(nodes, N, ox, oy, 1.0 / c, ncx, ncx, lam, keys, vals);
      VP_CHECK_LAUNCH();
      int eb = 1;
      while (eb < 64 && ((uint64_t)1 << eb) < (uint64_t)(ncx * ncx)) eb++;
      VP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb1, keys, keys2, vals, vals2, (int)N, 0, eb, s));
      VP_CUDA(cub::DeviceReduce::ReduceByKey(tmp, tb2, keys2, ukeys, vals2, umin, d_nu, cub::Min(), (int)N, s));
      int64_t nu = fetch_i64(d_nu, s);
      k_level_test<<<(unsigned)((T + 255) / 256), 256, 0, s>>>(P->tx, P->ty, T, B.tlev, l, ox, oy, 1.0 / c, ncx, ncx,
                                                              ukeys, umin, nu);
      VP_CHECK_LAUNCH();
    }
    for (void *q : {(void *)keys, (void *)keys2, (void *)ukeys, (void *)vals, (void *)vals2, (void *)umin,
                    (void *)d_nu, tmp})
      VP_CUDA(cudaFreeAsync(q, s));
  }
  VP_CUDA(cudaFreeAsync(lam, s));
  VP_CUDA(cudaFreeAsync(d_lmax, s));
  // ---- targets with level >= 1, their entries (one per level 1..l(x))
  int32_t *flag = tmp_alloc<int32_t>(T, s), *val = tmp_alloc<int32_t>(T, s);
  k_lev_flag<<<(unsigned)((T + 255) / 256), 256, 0, s>>>(B.tlev, T, flag, val);
  VP_CHECK_LAUNCH();
  {
    int32_t *hist = tmp_alloc<int32_t>(16, s);
    size_t tb = 0;
    cub::DeviceHistogram::HistogramEven(nullptr, tb, val, hist, 17, 0, 16, (int)T, s);
    void *tmp = tmp_alloc<char>(tb + 16, s);
    VP_CUDA(cub::DeviceHistogram::HistogramEven(tmp, tb, val, hist, 17, 0, 16, (int)T, s));
    int32_t hh[16];
    VP_CUDA(cudaMemcpyAsync(hh, hist, sizeof(hh), cudaMemcpyDeviceToHost, s));
    VP_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < 16; i++) B.lev_count[i] = hh[i];
    VP_CUDA(cudaFreeAsync(tmp, s));
    VP_CUDA(cudaFreeAsync(hist, s));
  }
  B.nlev = 0;
  for (int i = 1; i < 16; i++)
    if (B.lev_count[i] > 0) B.nlev = i;
  B.n_lt = T - B.lev_count[0];
  if (B.nlev == 0) {
    VP_CUDA(cudaFreeAsync(flag, s));
    VP_CUDA(cudaFreeAsync(val, s));
    return;
  }
  // ---- geometry of the boxes
  const double lne = log(1.0 / P->eps), zeps = vp_solve_e1(P->eps);
  BoxGeom bg;
  memset(&bg, 0, sizeof(bg));
  bg.x_lo = x_lo;
  bg.y_lo = y_lo;
  double r_over_h = 8.0 * sqrt(zeps * lne) / VP_PI;  // sqrt(4 delta_{l-1} z) / h_l, level independent
  B.margin = (int)ceil(r_over_h) + P->w / 2 + 2;
  B.nfb = vp_next_smooth(8 * (int64_t)B.margin);  // core = nfb - 2 margin ~ 3/4 nfb: ~1.8x box overlap
  B.core = (int)(B.nfb - 2 * B.margin);
  B.rowb = 2 * (B.nfb / 2 + 1);
  B.nmode = B.nfb / 2;
  bg.margin = B.margin;
  bg.nfb = (int)B.nfb;
  std::vector<double> lp(4 * (B.nlev + 1), 0.0);
  for (int l = 1; l <= B.nlev; l++) {
    double dl = d0 / pow(4.0, l), dlm = d0 / pow(4.0, l - 1);
    double kl = sqrt(lne / dl);
    bg.h[l] = VP_PI / (2.0 * kl);
    bg.C[l] = B.core * bg.h[l];
    bg.r[l] = sqrt(4.0 * dlm * zeps);
    lp[4 * l] = dl;
    lp[4 * l + 1] = dlm;
    lp[4 * l + 2] = 2.0 * VP_PI / (B.nfb * bg.h[l]);
    lp[4 * l + 3] = 1.0 / (bg.h[l] * bg.h[l] * (double)B.nfb * (double)B.nfb);
  }
  // ---- entries and boxes
  B.lt_t = vp_alloc<int32_t>(P, B.n_lt);
  B.lt_off = vp_alloc<int32_t>(P, B.n_lt + 1);
  {
    int32_t *d_n = tmp_alloc<int32_t>(1, s);
    size_t tb = 0;
    cub::CountingInputIterator<int32_t> cnt(0);
    cub::DeviceSelect::Flagged(nullptr, tb, cnt, flag, B.lt_t, d_n, (int)T, s);
    void *tmp = tmp_alloc<char>(tb + 16, s);
    VP_CUDA(cub::DeviceSelect::Flagged(tmp, tb, cnt, flag, B.lt_t, d_n, (int)T, s));
    VP_CUDA(cudaFreeAsync(tmp, s));
    VP_CUDA(cudaFreeAsync(d_n, s));
    int32_t *lv = tmp_alloc<int32_t>(B.n_lt + 1, s);
    VP_CUDA(cudaMemsetAsync(lv, 0, sizeof(int32_t) * (B.n_lt + 1), s));
    k_gather_i32<<<(unsigned)((B.n_lt + 255) / 256), 256, 0, s>>>(val, B.lt_t, B.n_lt, lv);
    VP_CHECK_LAUNCH();
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, lv, B.lt_off, (int)(B.n_lt + 1), s);
    tmp = tmp_alloc<char>(tb + 16, s);
    VP_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, lv, B.lt_off, (int)(B.n_lt + 1), s));
    VP_CUDA(cudaFreeAsync(tmp, s));
    VP_CUDA(cudaFreeAsync(lv, s));
    int32_t ne = 0;
    VP_CUDA(cudaMemcpyAsync(&ne, B.lt_off + B.n_lt, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    VP_CUDA(cudaStreamSynchronize(s));
    B.n_ent = ne;
  }
  VP_CUDA(cudaFreeAsync(flag, s));
  VP_CUDA(cudaFreeAsync(val, s));
  uint64_t *ekeys = tmp_alloc<uint64_t>(B.n_ent, s), *ekeys2 = tmp_alloc<uint64_t>(B.n_ent, s);
  uint64_t *ubox_t = tmp_alloc<uint64_t>(B.n_ent, s);
  k_entry_keys<<<(unsigned)((B.n_lt + 255) / 256), 256, 0, s>>>(P->tx, P->ty, B.lt_t, B.lt_off, B.n_lt, B.tlev, bg,
                                                               ekeys);
  VP_CHECK_LAUNCH();
  {
    size_t tb1 = 0, tb2 = 0;
    int64_t *d_nb = tmp_alloc<int64_t>(1, s);
    cub::DeviceRadixSort::SortKeys(nullptr, tb1, ekeys, ekeys2, (int)B.n_ent, 0, 64, s);
    cub::DeviceSelect::Unique(nullptr, tb2, ekeys2, ubox_t, d_nb, (int)B.n_ent, s);
    void *tmp = tmp_alloc<char>(std::max(tb1, tb2) + 16, s);
    VP_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb1, ekeys, ekeys2, (int)B.n_ent, 0, 64, s));
    VP_CUDA(cub::DeviceSelect::Unique(tmp, tb2, ekeys2, ubox_t, d_nb, (int)B.n_ent, s));
    B.nbox = fetch_i64(d_nb, s);
    VP_CUDA(cudaFreeAsync(tmp, s));
    VP_CUDA(cudaFreeAsync(d_nb, s));
  }
  if ((double)B.nbox * B.nfb * B.rowb * 8.0 > 60e9) throw VpError{VP_ERR_OOM};
  uint64_t *ubox = vp_alloc<uint64_t>(P, B.nbox);
  VP_CUDA(cudaMemcpyAsync(ubox, ubox_t, sizeof(uint64_t) * B.nbox, cudaMemcpyDeviceToDevice, s));
  B.box_level = vp_alloc<int32_t>(P, B.nbox);
  k_box_levels<<<(unsigned)((B.nbox + 255) / 256), 256, 0, s>>>(ubox, B.nbox, B.box_level);
  VP_CHECK_LAUNCH();
  B.ent_x = vp_alloc<double>(P, B.n_ent);
  B.ent_y = vp_alloc<double>(P, B.n_ent);
  k_entry_coords<<<(unsigned)((B.n_lt + 255) / 256), 256, 0, s>>>(P->tx, P->ty, B.lt_t, B.lt_off, B.n_lt, B.tlev,
                                                                 ekeys, ubox, B.nbox, bg, B.ent_x, B.ent_y);
  VP_CHECK_LAUNCH();
  for (void *q : {(void *)ekeys, (void *)ekeys2, (void *)ubox_t}) VP_CUDA(cudaFreeAsync(q, s));
  // (the staged entry order is built below, once the virtual grid exists)
  // ---- (box, source) pairs
  int64_t *cnt = tmp_alloc<int64_t>(N + 1, s), *off = tmp_alloc<int64_t>(N + 1, s);
  VP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (N + 1), s));
  k_src_pairs<false><<<(unsigned)((N + 255) / 256), 256, 0, s>>>(nodes, weights, N, B.nlev, ubox, B.nbox, bg, cnt,
                                                                nullptr, nullptr, nullptr, nullptr);
  VP_CHECK_LAUNCH();
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int)(N + 1), s);
    void *tmp = tmp_alloc<char>(tb + 16, s);
    VP_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, (int)(N + 1), s));
    VP_CUDA(cudaFreeAsync(tmp, s));
  }
  B.n_pairs = fetch_i64(off + N, s);
  if (B.n_pairs >= ((int64_t)1 << 31)) throw VpError{VP_ERR_UNSUPPORTED};
  double *pxy = tmp_alloc<double>(2 * B.n_pairs, s), *pw = tmp_alloc<double>(B.n_pairs, s);
  int32_t *pnode = tmp_alloc<int32_t>(B.n_pairs, s);
  k_src_pairs<true><<<(unsigned)((N + 255) / 256), 256, 0, s>>>(nodes, weights, N, B.nlev, ubox, B.nbox, bg, nullptr,
                                                               off, pxy, pw, pnode);
  VP_CHECK_LAUNCH();
  // ---- virtual grid, spreading order, FFT plans, multiplier tables
  B.grid = vp_alloc<double>(P, (size_t)B.nbox * B.nfb * B.rowb);
  GridArgs gb{B.grid, B.nfb, B.nbox * B.nfb, B.rowb, 0.0, 0.0, 1.0, 1.0};
  {  // entries ordered for the shared-memory-staged interpolation on the virtual grid
    double *exy = tmp_alloc<double>(2 * B.n_ent, s);
    k_interleave<<<(unsigned)((B.n_ent + 255) / 256), 256, 0, s>>>(B.ent_x, B.ent_y, B.n_ent, exy);
    VP_CHECK_LAUNCH();
    vp_build_interp_order_g(P, exy, B.n_ent, gb, &B.e_x, &B.e_y, &B.e_perm, &B.e_items, &B.e_n_items);
    B.ent_val = vp_alloc<double>(P, B.n_ent);
    VP_CUDA(cudaFreeAsync(exy, s));
  }
  if (B.sp.det || P->opts.spread_tile > 0)
    vp_build_spread_order(P, B.sp, pxy, pw, pnode, B.n_pairs, gb);
  else
    vp_build_strip_order(P, B.sp, pxy, pw, pnode, B.n_pairs, gb);
  for (void *q : {(void *)cnt, (void *)off, (void *)pxy, (void *)pw, (void *)pnode}) VP_CUDA(cudaFreeAsync(q, s));
  B.lev_par = vp_alloc<double>(P, lp.size());
  VP_CUDA(cudaMemcpyAsync(B.lev_par, lp.data(), sizeof(double) * lp.size(), cudaMemcpyHostToDevice, s));
  std::vector<double> dg;
  vp_es_deconv_table(P, 1.0, (double)B.nfb, B.nmode / 2, dg);
  B.deconv = vp_alloc<double>(P, dg.size());
  VP_CUDA(cudaMemcpyAsync(B.deconv, dg.data(), sizeof(double) * dg.size(), cudaMemcpyHostToDevice, s));
  if (!vp_fft_setup_bands(P)) {  // cuFFT batched over the boxes where the fused transform does not apply
    long long n[2] = {B.nfb, B.nfb};
    long long rin[2] = {B.nfb, B.rowb}, cin[2] = {B.nfb, B.rowb / 2};
    size_t w1 = 0, w2 = 0;
    VP_CUFFT(cufftCreate(&B.fwd));
    VP_CUFFT(cufftCreate(&B.inv));
    B.has_plans = true;
    VP_CUFFT(cufftSetAutoAllocation(B.fwd, 0));
    VP_CUFFT(cufftSetAutoAllocation(B.inv, 0));
    VP_CUFFT(cufftMakePlanMany64(B.fwd, 2, n, rin, 1, B.nfb * B.rowb, cin, 1, B.nfb * (B.rowb / 2), CUFFT_D2Z,
                                 B.nbox, &w1));
    VP_CUFFT(cufftMakePlanMany64(B.inv, 2, n, cin, 1, B.nfb * (B.rowb / 2), rin, 1, B.nfb * B.rowb, CUFFT_Z2D,
                                 B.nbox, &w2));
    void *work = vp_alloc<char>(P, std::max(w1, w2) + 256);
    VP_CUFFT(cufftSetWorkArea(B.fwd, work));
    VP_CUFFT(cufftSetWorkArea(B.inv, work));
    VP_CUFFT(cufftSetStream(B.fwd, s));
    VP_CUFFT(cufftSetStream(B.inv, s));
  }
  VP_CUDA(cudaStreamSynchronize(s));
}
