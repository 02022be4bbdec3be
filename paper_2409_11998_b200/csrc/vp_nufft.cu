// vp_nufft.cu -- sm_100a kernels of the history part (§3, Steps 2-4, lines 826-898):
//   spread  : type-1 spreading of c_j = f_j w_j onto the near-history (NH) and far-history (FH)
//             fine grids with the ES kernel, one CTA per (NH tile, point chunk), shared-memory tile
//             accumulation, one global fp64 RED per touched tile cell;
//   multiply: Fourier-space multiplication by the split kernel's transform (NH: (vnearkspace),
//             FH: e^{-k^2 delta2} W_R(k), (vfarkspace)/(Wdef)), deconvolution by the ES kernel's
//             transform (twice: spread and interpolation), trapezoid weight (Dk/2pi)^2 and cuFFT's
//             1/nf^2 normalisation, with |m_i| <= nmode/2 truncation (k_max, (fouriernhtrunc));
//   interp  : type-2 interpolation of both grids at the targets, fused with the local part
//             V_L = alpha f_t + sum_k omega_k f[idx_k] and the scatter to the user's target order.
#include <cub/cub.cuh>

#include "vp_common.cuh"
#include "vp_math.cuh"

#define VP_MAXW 16

struct GridArgs {
  double *data;
  int64_t nf, row;
  double ox, oy, h;
};
static GridArgs grid_args(const VpGrid &G) { return GridArgs{G.data, G.nf, G.row, G.ox, G.oy, G.h}; }

// fractional grid coordinate of x (identical expression in binning, spreading and interpolation)
__device__ __forceinline__ double gcoord(double x, double o, double h) { return (x - o) / h; }

// ES weights for the W grid points i0 .. i0+W-1 around fractional coordinate g
template <int W>
__device__ __forceinline__ int es_weights(double g, double beta, double *wts) {
  int i0 = (int)ceil(g - 0.5 * W);
  const double s = 2.0 / W;
#pragma unroll
  for (int k = 0; k < W; k++) wts[k] = vp_es((i0 + k - g) * s, beta);
  return i0;
}

__device__ __forceinline__ int64_t wrapi(int64_t i, int64_t n) {
  i %= n;
  return i < 0 ? i + n : i;
}

// ---------------------------------------------------------------------------------------------
// spreading: one CTA per sub-problem (tile_x, tile_y, start, count)
template <int W>
__global__ void __launch_bounds__(256) k_spread(const int4 *__restrict__ sub, const double *__restrict__ sx,
                                                const double *__restrict__ sy, const double *__restrict__ sw,
                                                const int32_t *__restrict__ sperm, const double *__restrict__ f,
                                                GridArgs g1, GridArgs g2, int TS, int fhw, double beta) {
  extern __shared__ double smem[];
  const int nw = TS + W + 1;            // NH smem tile width
  double *s1 = smem;                    // nw * nw
  double *s2 = smem + nw * nw;          // fhw * fhw
  const int4 sp = sub[blockIdx.x];
  const int64_t t1x = (int64_t)sp.x * TS - (W / 2 + 1), t1y = (int64_t)sp.y * TS - (W / 2 + 1);
  // FH tile origin covering this NH tile's spatial extent
  const double xlo = g1.ox + (double)sp.x * TS * g1.h, ylo = g1.oy + (double)sp.y * TS * g1.h;
  const int64_t t2x = (int64_t)floor(gcoord(xlo, g2.ox, g2.h)) - (W / 2 + 1);
  const int64_t t2y = (int64_t)floor(gcoord(ylo, g2.oy, g2.h)) - (W / 2 + 1);
  for (int i = threadIdx.x; i < nw * nw + fhw * fhw; i += blockDim.x) smem[i] = 0.0;
  __syncthreads();
  for (int j = sp.z + threadIdx.x; j < sp.z + sp.w; j += blockDim.x) {
    const double x = sx[j], y = sy[j];
    const double c = f[sperm[j]] * sw[j];
    double wx[W], wy[W];
    {
      int ix = es_weights<W>(gcoord(x, g1.ox, g1.h), beta, wx);
      int iy = es_weights<W>(gcoord(y, g1.oy, g1.h), beta, wy);
      int lx = (int)(ix - t1x), ly = (int)(iy - t1y);
#pragma unroll
      for (int b = 0; b < W; b++) {
        double cy = c * wy[b];
        double *rowp = s1 + (ly + b) * nw + lx;
#pragma unroll
        for (int a = 0; a < W; a++) atomicAdd(rowp + a, cy * wx[a]);
      }
    }
    {
      int ix = es_weights<W>(gcoord(x, g2.ox, g2.h), beta, wx);
      int iy = es_weights<W>(gcoord(y, g2.oy, g2.h), beta, wy);
      int lx = (int)(ix - t2x), ly = (int)(iy - t2y);
#pragma unroll
      for (int b = 0; b < W; b++) {
        double cy = c * wy[b];
        double *rowp = s2 + (ly + b) * fhw + lx;
#pragma unroll
        for (int a = 0; a < W; a++) atomicAdd(rowp + a, cy * wx[a]);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nw * nw; i += blockDim.x) {
    double v = s1[i];
    if (v != 0.0) {
      int64_t gx = wrapi(t1x + i % nw, g1.nf), gy = wrapi(t1y + i / nw, g1.nf);
      atomicAdd(g1.data + gy * g1.row + gx, v);
    }
  }
  for (int i = threadIdx.x; i < fhw * fhw; i += blockDim.x) {
    double v = s2[i];
    if (v != 0.0) {
      int64_t gx = wrapi(t2x + i % fhw, g2.nf), gy = wrapi(t2y + i / fhw, g2.nf);
      atomicAdd(g2.data + gy * g2.row + gx, v);
    }
  }
}

template <int W>
static void launch_spread_w(vp_plan_s *P, const double *f) {
  int nw = P->tiles.TS + W + 1;
  size_t sm = sizeof(double) * ((size_t)nw * nw + (size_t)P->fh_tile_w * P->fh_tile_w);
  static bool attr = false;
  if (!attr) {
    VP_CUDA(cudaFuncSetAttribute(k_spread<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  if (P->tiles.nsub == 0) return;
  k_spread<W><<<(unsigned)P->tiles.nsub, 256, sm, P->stream>>>(P->tiles.sub, P->sx, P->sy, P->sw, P->sperm, f,
                                                              grid_args(P->nh), grid_args(P->fh), P->tiles.TS,
                                                              P->fh_tile_w, P->beta);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

void vp_launch_spread(vp_plan_s *P, const double *f) {
  switch (P->w) {
#define CASE(W) \
  case W: launch_spread_w<W>(P, f); break;
    CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: throw VpError{VP_ERR_UNSUPPORTED};
  }
}

// ---------------------------------------------------------------------------------------------
// multiply the half spectrum (in-place R2C layout: row r holds nf/2+1 complex values)
__global__ void k_multiply(double *__restrict__ data, int64_t nf, int64_t row, int64_t half_modes,
                           const double *__restrict__ deconv, double dk, double scale, int kind, double da,
                           double db) {
  const int64_t ncol = nf / 2 + 1;
  const int64_t total = nf * ncol;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = id / ncol, c = id - r * ncol;
    int64_t m2 = r <= nf / 2 ? r : r - nf;
    int64_t m1 = c;
    double *z = data + r * row + 2 * c;
    int64_t a2 = m2 < 0 ? -m2 : m2;
    if (m1 > half_modes || a2 > half_modes) {
      z[0] = 0.0;
      z[1] = 0.0;
      continue;
    }
    double k2 = dk * dk * ((double)m1 * m1 + (double)m2 * m2);
    double mk = kind == 0 ? vp_mult_nh(k2, da, db) : vp_mult_fh(k2, da, db);
    double fac = mk * scale * deconv[m1] * deconv[a2];
    z[0] *= fac;
    z[1] *= fac;
  }
}

void vp_launch_multiply(vp_plan_s *P, VpGrid &G) {
  int64_t ncol = G.nf / 2 + 1;
  int64_t total = G.nf * ncol;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  double dk = 2.0 * VP_PI / G.L;
  // M(k) h^2 / (nf^2 Phi(k1)^2 Phi(k2)^2): deconv holds 1/Phi^2
  double scale = G.h * G.h / ((double)G.nf * (double)G.nf);
  k_multiply<<<blocks, 256, 0, P->stream>>>(G.data, G.nf, G.row, G.nmode / 2, G.deconv, dk, scale, G.kind,
                                            G.delta_a, G.delta_b);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

// ---------------------------------------------------------------------------------------------
// interpolation + local part + scatter to user order
template <int W>
__device__ __forceinline__ double interp_one(const GridArgs &g, double x, double y, double beta) {
  double wx[W], wy[W];
  int ix = es_weights<W>(gcoord(x, g.ox, g.h), beta, wx);
  int iy = es_weights<W>(gcoord(y, g.oy, g.h), beta, wy);
  double acc = 0.0;
  bool inside = ix >= 0 && iy >= 0 && ix + W <= g.nf && iy + W <= g.nf;
#pragma unroll
  for (int b = 0; b < W; b++) {
    double racc = 0.0;
    if (inside) {
      const double *rp = g.data + (int64_t)(iy + b) * g.row + ix;
#pragma unroll
      for (int a = 0; a < W; a++) racc += wx[a] * __ldg(rp + a);
    } else {
      int64_t yy = wrapi(iy + b, g.nf);
#pragma unroll
      for (int a = 0; a < W; a++) racc += wx[a] * __ldg(g.data + yy * g.row + wrapi(ix + a, g.nf));
    }
    acc += wy[b] * racc;
  }
  return acc;
}

template <int W>
__global__ void __launch_bounds__(256) k_interp_local(const double *__restrict__ tx, const double *__restrict__ ty,
                                                      const int64_t *__restrict__ tperm, int64_t T, GridArgs g1,
                                                      GridArgs g2, double beta, int do_hist,
                                                      const double *__restrict__ f, const double *__restrict__ lalpha,
                                                      const int32_t *__restrict__ lnode,
                                                      const int32_t *__restrict__ lidx, const double *__restrict__ lw,
                                                      int K, int do_local, double *__restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  double v = 0.0;
  if (do_hist) {
    double x = tx[t], y = ty[t];
    v = interp_one<W>(g1, x, y, beta) + interp_one<W>(g2, x, y, beta);
  }
  if (do_local) {
    double vl = 0.0;
    int32_t nd = lnode[t];
    if (nd >= 0) vl = lalpha[t] * f[nd];
    const int32_t *ip = lidx + t * (int64_t)K;
    const double *wp = lw + t * (int64_t)K;
    for (int k = 0; k < K; k++) vl += wp[k] * f[ip[k]];
    v += vl;
  }
  out[tperm[t]] = v;
}

template <int W>
static void launch_interp_w(vp_plan_s *P, const double *f, double *out) {
  int parts = P->opts.parts ? P->opts.parts : VP_PART_ALL;
  unsigned blocks = (unsigned)((P->T + 255) / 256);
  if (!blocks) return;
  k_interp_local<W><<<blocks, 256, 0, P->stream>>>(P->tx, P->ty, P->tperm, P->T, grid_args(P->nh), grid_args(P->fh),
                                                   P->beta, (parts & VP_PART_HISTORY) ? 1 : 0, f, P->lalpha,
                                                   P->lnode, P->lidx, P->lw, P->K,
                                                   (parts & VP_PART_LOCAL) ? 1 : 0, out);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

void vp_launch_interp_local(vp_plan_s *P, const double *f, double *out) {
  switch (P->w) {
#define CASE(W) \
  case W: launch_interp_w<W>(P, f, out); break;
    CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: throw VpError{VP_ERR_UNSUPPORTED};
  }
}

// ---------------------------------------------------------------------------------------------
// binning + sort of points into a uniform grid of bins (plan time)
__global__ void k_bin_keys(const double *__restrict__ xy, int64_t n, double ox, double oy, double cell, int64_t nbx,
                           int64_t nby, uint32_t *__restrict__ keys, int32_t *__restrict__ idx,
                           unsigned long long *__restrict__ counts) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = xy[2 * i], y = xy[2 * i + 1];
  int64_t bx = (int64_t)floor((x - ox) / cell), by = (int64_t)floor((y - oy) / cell);
  bx = bx < 0 ? 0 : (bx >= nbx ? nbx - 1 : bx);
  by = by < 0 ? 0 : (by >= nby ? nby - 1 : by);
  uint32_t k = (uint32_t)(by * nbx + bx);
  keys[i] = k;
  idx[i] = (int32_t)i;
  atomicAdd(counts + k, 1ULL);
}

__global__ void k_gather_xy(const double *__restrict__ xy, const int32_t *__restrict__ idx, int64_t n,
                            double *__restrict__ xs, double *__restrict__ ys, int64_t *__restrict__ p64,
                            int32_t *__restrict__ p32) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t j = idx[i];
  xs[i] = xy[2 * (int64_t)j];
  ys[i] = xy[2 * (int64_t)j + 1];
  if (p64) p64[i] = j;
  if (p32) p32[i] = j;
}

// Sort n points (interleaved xy, device) into bins (row-major by, bx); returns sorted coordinates
// and the permutation (sorted -> input index).  bin_start (device, nbins+1, caller-owned via
// plan allocs) is returned if bin_start_out != NULL.  Uses CUB radix sort (stable).
int64_t vp_sort_points(vp_plan_s *P, const double *xy, int64_t n, double ox, double oy, double cell, int64_t nbx,
                       int64_t nby, double *xs, double *ys, int64_t *perm64, int32_t *perm32,
                       int64_t **bin_start_out) {
  int64_t nb = nbx * nby;
  if (nb >= (int64_t)1 << 32) throw VpError{VP_ERR_OOM};
  cudaStream_t s = P->stream;
  uint32_t *keys = nullptr, *keys2 = nullptr;
  int32_t *idx = nullptr, *idx2 = nullptr;
  unsigned long long *counts = nullptr;
  VP_CUDA(cudaMallocAsync(&keys, sizeof(uint32_t) * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&keys2, sizeof(uint32_t) * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&idx, sizeof(int32_t) * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&idx2, sizeof(int32_t) * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&counts, sizeof(unsigned long long) * (nb + 1), s));
  VP_CUDA(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * (nb + 1), s));
  if (n > 0) {
    k_bin_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(xy, n, ox, oy, cell, nbx, nby, keys, idx, counts);
    VP_CHECK_LAUNCH();
  }
  int end_bit = 1;
  while (end_bit < 32 && ((uint64_t)1 << end_bit) < (uint64_t)nb) end_bit++;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, idx, idx2, (int)n, 0, end_bit, s);
  void *tmp = nullptr;
  VP_CUDA(cudaMallocAsync(&tmp, tmp_bytes + 16, s));
  if (n > 0) VP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, idx, idx2, (int)n, 0, end_bit, s));
  if (n > 0) {
    k_gather_xy<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(xy, idx2, n, xs, ys, perm64, perm32);
    VP_CHECK_LAUNCH();
  }
  if (bin_start_out) {
    int64_t *bs = vp_alloc<int64_t>(P, nb + 1);
    // exclusive scan of counts (as int64) -> bin_start
    {
      size_t tb2 = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb2, (const unsigned long long *)counts, (unsigned long long *)bs,
                                    (int)(nb + 1), s);
      void *tmp2 = nullptr;
      VP_CUDA(cudaMallocAsync(&tmp2, tb2 + 16, s));
      VP_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, tb2, (const unsigned long long *)counts, (unsigned long long *)bs,
                                            (int)(nb + 1), s));
      VP_CUDA(cudaFreeAsync(tmp2, s));
    }
    *bin_start_out = bs;
  }
  VP_CUDA(cudaFreeAsync(tmp, s));
  VP_CUDA(cudaFreeAsync(keys, s));
  VP_CUDA(cudaFreeAsync(keys2, s));
  VP_CUDA(cudaFreeAsync(idx, s));
  VP_CUDA(cudaFreeAsync(idx2, s));
  VP_CUDA(cudaFreeAsync(counts, s));
  return nb;
}
