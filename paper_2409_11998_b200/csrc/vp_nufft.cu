// vp_nufft.cu -- sm_100a kernels of the history part (§3, Steps 2-4, lines 826-898).
//
// Both history parts share ONE set of per-point kernels on the near-history (NH) fine grid:
//   spread_nh : type-1 spreading of c_j = f_j w_j onto the NH grid.  One warp per CTA owns a private
//               (TS+W+3)^2 fp64 shared-memory tile; points were sorted at plan time into "row-rank"
//               batches (<= 32 points of one tile with pairwise distinct footprint rows), so inside a
//               footprint row step every lane writes its own grid row: plain LDS/DFMA/STS, no atomics,
//               one __syncwarp per row.  One global fp64 RED per tile cell at the end.
//   restrict  : the far-history (FH) grid is obtained from the NH grid by a separable convolution with
//               the FH-scale ES kernel (g2 = R g1); the FH transform then carries the product kernel
//               Phi_NH Phi_FH in its deconvolution (DESIGN.md §NUFFT "two-stage FH").
//   multiply  : Fourier multiplication by the split kernels' transforms (NH: (vnearkspace); FH:
//               e^{-k^2 delta2} W_R(k), (vfarkspace)/(Wdef)), ES deconvolution, trapezoid weight
//               (Dk/2pi)^2, cuFFT 1/nf^2, truncation |m_i| <= nmode/2.
//   prolong   : q1 += R^T q2 (FH potential onto the NH grid).
//   interp    : type-2 interpolation of the NH grid at the targets fused with the local part
//               V_L = alpha f_t + sum_k omega_k f[idx_k] and the scatter to the user's order.
// ES kernel values come from per-tap Horner polynomials (vp_common.cuh VpHorner), degree ~ W-1.
#include <cub/cub.cuh>
#include <cuda_pipeline.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <set>

#include "vp_common.cuh"
#include "vp_math.cuh"


// fractional grid coordinate of x (identical expression in binning, spreading and interpolation; the _rn
// intrinsics keep the compiler from contracting it differently in different kernels, so plan-time keys and
// eval-time footprints agree bit for bit)
__device__ __forceinline__ double gcoord(double x, double o, double inv_h) { return __dmul_rn(__dsub_rn(x, o), inv_h); }

// first grid index of the W-point footprint around fractional coordinate g
__device__ __forceinline__ int es_origin(double g, int W) { return (int)ceil(__dsub_rn(g, 0.5 * W)); }

// Horner tables of the ES taps for every width W (beta = 2.30 W fixed, so the table depends on W only)
__constant__ double c_horner[VP_HORNER_MAXW - 3][VP_HORNER_MAXW][VP_HORNER_MAXW];

// The table of width W depends on W only (beta = 2.30 W, fixed degree), so every plan uploads identical bytes:
// once per (device, W), synchronously at plan time, under a mutex.
void vp_upload_horner(int W, const VpHorner &h) {
  static std::mutex mu;
  static std::set<std::pair<int, int>> done;
  const int dev = vp_current_device();
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(std::make_pair(dev, W))) return;
  VP_CUDA(cudaMemcpyToSymbol(c_horner, &h.c[0][0], sizeof(h.c), sizeof(h.c) * (size_t)(W - 4)));
  done.insert(std::make_pair(dev, W));
}

// ES weights for grid points i0 .. i0+W-1 around fractional coordinate g, by Horner polynomials in
// t = 2u - 1, u = i0 - (g - W/2) in [0, 1).  psi is even, so tap W-1-k at t equals tap k at -t: with
// P_k(t) = E_k(t^2) + t O_k(t^2) one even and one odd Horner chain in t^2 give both taps of a pair
// (about half the DFMA of W separate chains).
// taps k and W-1-k at t (u = t^2): even and odd Horner chains of tap k's polynomial
template <int W, int D>
__device__ __forceinline__ void es_pair(int k, double t, double u, double *wk, double *wm) {
  constexpr int DE = D / 2, DO = (D - 1) / 2;  // highest even / odd coefficient: 2 DE, 2 DO + 1 <= D
  double e = c_horner[W - 4][k][2 * DE], o = c_horner[W - 4][k][2 * DO + 1];
#pragma unroll
  for (int j = DE - 1; j >= 0; j--) e = fma(e, u, c_horner[W - 4][k][2 * j]);
#pragma unroll
  for (int j = DO - 1; j >= 0; j--) o = fma(o, u, c_horner[W - 4][k][2 * j + 1]);
  *wk = fma(t, o, e);
  *wm = fma(-t, o, e);
}

// footprint origin and Horner argument of fractional grid coordinate g
template <int W>
__device__ __forceinline__ int es_arg(double g, double *t) {
  const double s = __dsub_rn(g, 0.5 * W);
  const int i0 = (int)ceil(s);
  *t = 2.0 * (i0 - s) - 1.0;
  return i0;
}

template <int W, int D>
__device__ __forceinline__ int es_horner(double g, double *wts) {
  double t;
  const int i0 = es_arg<W>(g, &t);
  const double u = t * t;
#pragma unroll
  for (int k = 0; k < (W + 1) / 2; k++) {
    double wk, wm;
    es_pair<W, D>(k, t, u, &wk, &wm);
    wts[k] = wk;
    if (W - 1 - k != k) wts[W - 1 - k] = wm;
  }
  return i0;
}

__global__ void k_gather_xy(const double *__restrict__ xy, const int32_t *__restrict__ idx, int64_t n,
                            double *__restrict__ xs, double *__restrict__ ys, int64_t *__restrict__ p64,
                            int32_t *__restrict__ p32);

// ES weight of tap k at t (one Horner chain; register-lean form of es_horner for kernels that keep many
// accumulators live)
template <int W, int D>
__device__ __forceinline__ double es_tap(double t, int k) {
  double v = c_horner[W - 4][k][D];
#pragma unroll
  for (int j = D - 1; j >= 0; j--) v = fma(v, t, c_horner[W - 4][k][j]);
  return v;
}

// the same weights as es_horner by W separate Horner chains in t (lower register pressure in kernels that keep
// a w x w window sweep live; the interpolation is bound by shared-memory reads, not by these DFMA)
template <int W, int D>
__device__ __forceinline__ int es_horner_chains(double g, double *wts) {
  double t;
  const int i0 = es_arg<W>(g, &t);
#pragma unroll
  for (int k = 0; k < W; k++) wts[k] = c_horner[W - 4][k][D];
#pragma unroll
  for (int j = D - 1; j >= 0; j--) {
#pragma unroll
    for (int k = 0; k < W; k++) wts[k] = fma(wts[k], t, c_horner[W - 4][k][j]);
  }
  return i0;
}

__device__ __forceinline__ int64_t wrapi(int64_t i, int64_t n) {
  i %= n;
  return i < 0 ? i + n : i;
}

// fp64 RED of v into grid row gy (periodic) at column pointer col; the wrapped case out of line (small code
// in unrolled loops)
__device__ __noinline__ void red_row_wrapped(double *col, int64_t gy, int64_t nfy, int64_t row, double v) {
  atomicAdd(col + wrapi(gy, nfy) * row, v);
}
__device__ __forceinline__ void red_row(double *col, int64_t gy, bool interior, const GridArgs &g, double v) {
  if (v == 0.0) return;
  if (interior) atomicAdd(col + gy * g.row, v);
  else red_row_wrapped(col, gy, g.nfy, g.row, v);
}

// ---------------------------------------------------------------------------------------------
// plan-time keys for the batch ordering: (tile, footprint row, footprint column) of each point
__global__ void k_spread_keys(const double *__restrict__ xy, int64_t n, GridArgs g, int TS, int W, int64_t ntx,
                              int64_t nty, uint64_t *__restrict__ keys, int32_t *__restrict__ idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double gx = gcoord(xy[2 * i], g.ox, g.inv_h), gy = gcoord(xy[2 * i + 1], g.oy, g.inv_h);
  int64_t tx = (int64_t)floor(gx / TS), ty = (int64_t)floor(gy / TS);
  tx = tx < 0 ? 0 : (tx >= ntx ? ntx - 1 : tx);
  ty = ty < 0 ? 0 : (ty >= nty ? nty - 1 : ty);
  int64_t lrow = (int64_t)es_origin(gy, W) - (ty * TS - (W / 2 + 1));
  int64_t lcol = (int64_t)es_origin(gx, W) - (tx * TS - (W / 2 + 1));
  lrow = lrow < 0 ? 0 : (lrow > 255 ? 255 : lrow);
  lcol = lcol < 0 ? 0 : (lcol > 255 ? 255 : lcol);
  keys[i] = ((uint64_t)(ty * ntx + tx) << 32) | ((uint64_t)lrow << 16) | (uint64_t)lcol;
  idx[i] = (int32_t)i;
}

__global__ void k_tile_heads(const uint64_t *__restrict__ k1, int64_t n, int32_t *__restrict__ head) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  head[i] = (i == 0 || (k1[i - 1] >> 32) != (k1[i] >> 32)) ? 1 : 0;
}

// Level assignment, one thread per non-empty tile: points of one footprint row that share a level are
// >= W columns apart, so points of one level never write the same grid cell within a row step.
// Inside a level, points are then ordered rank-major over the shared-memory bank slot of their
// footprint origin (res = (row * nw + col) mod 16, 16 slots of 8 B per 128 B wavefront): a chunk of
// 32 consecutive points holds at most 2 points per slot when the slots are evenly populated, so the
// row-step LDS/STS of a batch need ~2 wavefronts instead of the ~4-5 of random columns.
#define PK_B 32
#define PK_ROWS 72  // footprint start rows of a tile: TS + 2 (TS <= 64)
__global__ void k_levels(const uint64_t *__restrict__ k1, const int32_t *__restrict__ tstart, int64_t ntile,
                         int64_t n, int W, int nw, uint64_t *__restrict__ k2, int *__restrict__ overflow_flag) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= ntile) return;
  const int64_t s0 = tstart[t], s1 = (t + 1 < ntile) ? tstart[t + 1] : n;
  const uint64_t tile = k1[s0] >> 32;
  // sparse tile (every row has few points): greedy packing into <= PK_B open batches of <= 32 points, first
  // batch whose row is free at these columns and whose bank slot holds < 2 points -> full batches
  int64_t maxrow = 0;
  for (int64_t r0 = s0; r0 < s1;) {
    int64_t r1 = r0;
    const uint64_t rk = (k1[r0] >> 16) & 0xff;
    while (r1 < s1 && ((k1[r1] >> 16) & 0xff) == rk) r1++;
    if (r1 - r0 > maxrow) maxrow = r1 - r0;
    r0 = r1;
  }
  if (maxrow <= 2 * PK_B && s1 - s0 <= 8192) {
    uint8_t rowend[PK_B][PK_ROWS];
    uint8_t slot[PK_B][16];
    uint8_t cnt[PK_B];
    uint32_t bid[PK_B];
    int nopen = 0;
    uint32_t next_id = 0;
    bool ok = true;
    for (int64_t i = s0; i < s1 && ok; i++) {
      const int row = (int)((k1[i] >> 16) & 0xff), col = (int)(k1[i] & 0xff);
      if (row >= PK_ROWS || col + W > 255) { ok = false; break; }
      const int res = (row * nw + col) & 15;
      int best = -1, soft = -1;
      for (int b = 0; b < nopen; b++) {
        if (rowend[b][row] <= col) {
          if (slot[b][res] < 2) { best = b; break; }
          if (soft < 0) soft = b;
        }
      }
      if (best < 0) {
        if (soft >= 0) {
          best = soft;  // a bank-slot repeat costs one extra wavefront; a new batch costs a whole row sweep
        } else if (nopen < PK_B) {
          best = nopen++;
          for (int r = 0; r < PK_ROWS; r++) rowend[best][r] = 0;
          for (int r = 0; r < 16; r++) slot[best][r] = 0;
          cnt[best] = 0;
          bid[best] = next_id++;
        } else {  // every open batch is taken on this row: use the level scheme for this tile
          ok = false;
          break;
        }
      }
      k2[i] = (tile << 40) | ((uint64_t)(bid[best] & 0xFFFFF) << 20) | (uint64_t)res;
      rowend[best][row] = (uint8_t)(col + W);
      slot[best][res]++;
      if (++cnt[best] == 32) {  // closed: reopen the slot as a fresh batch
        for (int r = 0; r < PK_ROWS; r++) rowend[best][r] = 0;
        for (int r = 0; r < 16; r++) slot[best][r] = 0;
        cnt[best] = 0;
        bid[best] = next_id++;
      }
    }
    if (ok && next_id <= 0xFFFFF) return;
  }
  // dense tile: rows are contiguous (keys sorted by tile, row, column).  With K = the largest number of points
  // of the row inside any W-column window, level = (index in the row) mod K is a valid assignment (points i and
  // i + K are >= W columns apart) and uses the minimum number of levels (the maximum overlap).
  for (int64_t r0 = s0; r0 < s1;) {
    const uint64_t row_key = (k1[r0] >> 16) & 0xff;
    int64_t r1 = r0;
    while (r1 < s1 && ((k1[r1] >> 16) & 0xff) == row_key) r1++;
    int64_t K = 1;
    for (int64_t i = r0, j = r0; i < r1; i++) {  // window [col_i - W, col_i]: points j..i with col_j > col_i - W
      const int ci = (int)(k1[i] & 0xff);
      while ((int)(k1[j] & 0xff) <= ci - W) j++;
      if (i - j + 1 > K) K = i - j + 1;
    }
    if (K > 0xFFFFF) *overflow_flag = 1;
    const int row = (int)row_key;
    for (int64_t i = r0; i < r1; i++) {
      const int col = (int)(k1[i] & 0xff);
      const int lv = (int)((i - r0) % K);
      const int res = (row * nw + col) & 15;
      k2[i] = (tile << 40) | ((uint64_t)(lv & 0xFFFFF) << 20) | (uint64_t)res;  // rank bits filled by k_bank_rank
    }
    r0 = r1;
  }
}

// rank of a point inside its (tile, level, bank slot) group (keys sorted, rank bits zero): sorting by
// (tile, level, rank, slot) then interleaves the slots, so 32 consecutive points hold <= 2 per slot when the
// group's slots are evenly populated
__global__ void k_bank_rank(const uint64_t *__restrict__ ks, int64_t n, uint64_t *__restrict__ kr) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t key = ks[i];
  int64_t lo = 0, hi = i;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (ks[mid] < key) lo = mid + 1; else hi = mid;
  }
  uint64_t rank = (uint64_t)(i - lo);
  if (rank > 0xFFFF) rank = 0xFFFF;
  kr[i] = key | (rank << 4);
}

// batch heads: new (tile, level) or every 32 points of one level
__global__ void k_batch_heads(const uint64_t *__restrict__ k2, int64_t n, int32_t *__restrict__ head) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t grp = k2[i] >> 20;
  int h = 0;
  if (i == 0 || (k2[i - 1] >> 20) != grp) {
    h = 1;
  } else {
    int64_t lo = 0, hi = i;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if ((k2[mid] >> 20) < grp) lo = mid + 1; else hi = mid;
    }
    h = ((i - lo) % 32) == 0;
  }
  head[i] = h;
}

// ---------------------------------------------------------------------------------------------
// NH spreading: one warp per work item (tile_x, tile_y, first batch, end batch)
template <int W, int D>
__global__ void __launch_bounds__(32) k_spread_nh(const int4 *__restrict__ items, const int32_t *__restrict__ bstart,
                                                  const double *__restrict__ sx, const double *__restrict__ sy,
                                                  const double *__restrict__ sw, const int32_t *__restrict__ sperm,
                                                  const double *__restrict__ f, GridArgs g, int TS, int det,
                                                  double *__restrict__ fs_out) {
  extern __shared__ double tile[];
  const int nw = TS + W + 3;
  const int lane = threadIdx.x;
  const int4 it = items[blockIdx.x];
  const int64_t ox = (int64_t)it.x * TS - (W / 2 + 1), oy = (int64_t)it.y * TS - (W / 2 + 1);
  for (int i = lane; i < nw * nw; i += 32) tile[i] = 0.0;
  __syncwarp();
  // software pipeline over batches: the next batch's point data (x, y, w, node index, then f) is loaded while
  // the current batch's row steps run, so the global-memory latency is not exposed once per batch
  int jn = -1;
  double xn = 0.0, yn = 0.0, wn = 0.0, fn = 0.0;
  {
    const int s0 = bstart[it.z];
    if (lane < bstart[it.z + 1] - s0) {
      jn = s0 + lane;
      xn = sx[jn]; yn = sy[jn]; wn = sw[jn];
      fn = f[sperm[jn]];
    }
  }
  for (int b = it.z; b < it.w; b++) {
    const int j = jn;
    const bool act = j >= 0;
    const double x = xn, y = yn, fj = fn, wj = wn;
    int pn = -1;
    jn = -1;
    if (b + 1 < it.w) {
      const int s1 = bstart[b + 1];
      if (lane < bstart[b + 2] - s1) {
        jn = s1 + lane;
        xn = sx[jn]; yn = sy[jn]; wn = sw[jn];
        pn = sperm[jn];
      }
    }
    double wx[W], wy[W], c = 0.0;
    int lx = 0, ly = 0;
    if (act) {
      if (fs_out) fs_out[j] = fj;  // f in spreading order: spatially coherent copy for the stencil gathers
      c = fj * wj;
      lx = (int)(es_horner<W, D>(gcoord(x, g.ox, g.inv_h), wx) - ox);
      ly = (int)(es_horner<W, D>(gcoord(y, g.oy, g.inv_h), wy) - oy);
    }
    if (pn >= 0) fn = f[pn];
#pragma unroll
    for (int r = 0; r < W; r++) {
      if (act) {
        double *rowp = tile + (ly + r) * nw + lx;
        const double cr = c * wy[r];
        double v[W];
#pragma unroll
        for (int a = 0; a < W; a++) v[a] = rowp[a];
#pragma unroll
        for (int a = 0; a < W; a++) rowp[a] = fma(cr, wx[a], v[a]);
      }
      __syncwarp();
    }
  }
  __syncwarp();
  const bool interior = ox >= 0 && oy >= 0 && ox + nw <= g.nfx && oy + nw <= g.nfy;
  for (int rr = 0; rr < nw; rr++) {
    for (int cc = lane; cc < nw; cc += 32) {
      double v = tile[rr * nw + cc];
      if (v != 0.0) {
        int64_t gx = ox + cc, gy = oy + rr;
        if (!interior) {
          gx = wrapi(gx, g.nfx);
          gy = wrapi(gy, g.nfy);
        }
        if (det) g.data[gy * g.row + gx] += v;  // colour-separated launch: no concurrent writer
        else atomicAdd(g.data + gy * g.row + gx, v);
      }
    }
  }
}

template <int W>
static void launch_spread_w(vp_plan_s *P, const VpSpreadSet &S, const GridArgs &g, const double *f) {
  constexpr int D = VP_HORNER_DEG(W);
  int nw = S.tiles.TS + W + 3;
  size_t sm = sizeof(double) * (size_t)nw * nw;
  if (S.tiles.nsub == 0) return;
  vp_smem_attr((const void *)k_spread_nh<W, D>, sm);
  if (!S.det) {
    k_spread_nh<W, D><<<(unsigned)S.tiles.nsub, 32, sm, P->stream>>>(S.tiles.sub, S.bstart, S.sx, S.sy, S.sw,
                                                                     S.sperm, f, g, S.tiles.TS, 0, S.fs_out);
    VP_CHECK_LAUNCH();
    P->n_kernels++;
    return;
  }
  // deterministic mode: one item per tile, four launches by tile colour (tx & 1, ty & 1); tiles of one colour
  // have disjoint windows, so the plain read-add-write of each cell has a fixed order
  for (int c = 0; c < 4; c++) {
    const int64_t i0 = S.color_off[c], i1 = S.color_off[c + 1];
    if (i1 <= i0) continue;
    k_spread_nh<W, D><<<(unsigned)(i1 - i0), 32, sm, P->stream>>>(S.tiles.sub + i0, S.bstart, S.sx, S.sy, S.sw,
                                                                  S.sperm, f, g, S.tiles.TS, 1, S.fs_out);
    VP_CHECK_LAUNCH();
    P->n_kernels++;
  }
}

// ---------------------------------------------------------------------------------------------
// NH spreading, strip form (default for the NH grid).  A warp owns a 32-column strip of the grid: lane =
// column.  The points of a work item are those whose footprint origin lies in an SW x SH "strip" (SW = 33 - W,
// so every footprint fits the 32 lanes), sorted by origin row.  The warp walks the rows in order and keeps the
// W rows r .. r + W - 1 in REGISTERS as a ring (row rho in acc[rho mod W]); a point with origin row r adds
// wxrow[lane] * (c wy[b]) to row r + b (W DFMA, no shared-memory writes, no atomics), and leaving row r flushes
// acc[r mod W] (one coalesced fp64 RED per lane, skipped when zero).  The ring phase k = r mod W is a
// compile-time constant in each of the W unrolled phases (switch + fall-through), so acc[] stays in registers.
// Points are staged 32 at a time (lane per point): the x weights as a zero-padded 32-wide row (the lane's
// column weight is then one conflict-free load; restaging clears only the previous footprint), c wy as
// 16-byte rows read by double2 broadcasts; the origin row stays in the staging lane's register and the row
// ends come from one ballot per row.  Compared with the shared-memory tile scatter (k_spread_nh) this
// replaces 2 W^2 shared-memory accesses per point by W/2 + 1 loads (measured ~16 wavefronts per point at
// W = 10, against ~40 for the tile scatter).
#define VP_STRIP_WARPS 4
#define VP_STRIP_MAXP 2048  // points per work item: dense strips are split (each part flushes its own rows)
#ifndef VP_STRIP_SH
#define VP_STRIP_SH 64  // footprint-origin rows per strip (the register ring is W rows whatever the height)
#endif
template <int W>
struct StripCfg {
  static constexpr int SW = 33 - W;         // footprint-origin columns per strip
  static constexpr int SH = VP_STRIP_SH;    // footprint-origin rows per strip
  static constexpr int CH = 32;             // points staged per chunk (one per lane)
  static constexpr int WXS = 33;            // padded x-weight rows (32 columns)
  static constexpr int WYS = (W + 1) & ~1;  // even stride: 16-byte aligned rows for double2 broadcasts
  static constexpr size_t smem_warp = (size_t)CH * (WXS + WYS) * 8;
  static constexpr int NPMAX = (32 - W) / W + 1;  // column-disjoint W-wide footprints in one 32-lane window
};

template <int W, int D, bool PACK>
__global__ void __launch_bounds__(32 * VP_STRIP_WARPS, W <= 10 ? 5 : 4)
    k_spread_strip(const int4 *__restrict__ items, int64_t n_items, const double *__restrict__ sx,
                   const double *__restrict__ sy, const double *__restrict__ sw, const int32_t *__restrict__ sperm,
                   const double *__restrict__ f, GridArgs g, double *__restrict__ fs_out) {
  using C = StripCfg<W>;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * VP_STRIP_WARPS + warp;
  if (item >= n_items) return;
  double *s_wy = smem + (size_t)warp * C::CH * (C::WXS + C::WYS);
  double *s_wx = s_wy + C::CH * C::WYS;
  const int4 it = items[item];
  const int64_t ox = (int64_t)it.x * C::SW - (W / 2 + 1), oy = (int64_t)it.y * C::SH - (W / 2 + 1);
  const bool interior = ox >= 0 && oy >= 0 && ox + 32 <= g.nfx && oy + C::SH + W - 1 <= g.nfy;
  double *col = g.data + (interior ? ox + lane : wrapi(ox + lane, g.nfx));
  double acc[W];
#pragma unroll
  for (int b = 0; b < W; b++) acc[b] = 0.0;
  int c0 = it.z, n = 0, q = 0, r = 0, mylr = 0x7fffffff, prev_lc = 0, mylc = 0;
  unsigned starts = 0;
  bool first = true;
  double *wrow = s_wx + lane * C::WXS;
#pragma unroll
  for (int a = 0; a < 32; a++) wrow[a] = 0.0;
stage:
  n = min(C::CH, it.w - c0);
  mylr = 0x7fffffff;
  mylc = 1 << 20;
  if (lane < n) {
    const int j = c0 + lane;
    const double fj = __ldg(f + sperm[j]);
    if (fs_out) fs_out[j] = fj;  // f in spreading order: spatially coherent copy for the stencil gathers
    const double c = fj * sw[j];
#pragma unroll
    for (int a = 0; a < W; a++) wrow[prev_lc + a] = 0.0;  // the row is zero outside the footprint
    int lc, lr;
    {
      double wx[W];
      lc = (int)(es_horner<W, D>(gcoord(sx[j], g.ox, g.inv_h), wx) - ox);
#pragma unroll
      for (int a = 0; a < W; a++) wrow[lc + a] = wx[a];
    }
    prev_lc = lc;
    mylc = lc;
    double wy[W];
    lr = (int)(es_horner<W, D>(gcoord(sy[j], g.oy, g.inv_h), wy) - oy);
    double2 *wyp = (double2 *)(s_wy + lane * C::WYS);
#pragma unroll
    for (int b = 0; b + 1 < W; b += 2) wyp[b >> 1] = make_double2(c * wy[b], c * wy[b + 1]);
    if (W & 1) s_wy[lane * C::WYS + W - 1] = c * wy[W - 1];
    mylr = lr;
  }
  __syncwarp();
  if constexpr (PACK) {
    // packs: a staged point joins the previous one's pack when it has the same origin row and lies right of the
    // previous member's footprint (the plan sorts each strip row into column-disjoint packs);
    // one step of W DFMA per lane then adds a whole pack, each lane taking the member covering its column
    const int plr = __shfl_up_sync(0xffffffffu, mylr, 1), plc = __shfl_up_sync(0xffffffffu, mylc, 1);
    starts = __ballot_sync(0xffffffffu, lane == 0 || lane >= n || mylr != plr || mylc < plc + W);
  }
  q = 0;
  if (first) {
    r = __shfl_sync(0xffffffffu, mylr, 0);
    first = false;
  }
  for (;;) {
    switch (r % W) {
#define VP_STRIP_PHASE(k)                                                              \
  case k:                                                                              \
    if ((k) < W) {                                                                     \
      _Pragma("unroll 2") for (const int e = __popc(__ballot_sync(0xffffffffu, mylr <= r)); q < e;) { \
        const unsigned later = PACK && q < 31 ? (starts >> (q + 1)) << (q + 1) : 0u;   \
        const int q2 = PACK ? min(later ? __ffs(later) - 1 : 32, e) : q + 1;           \
        int sel = q;                                                                   \
        if (PACK) _Pragma("unroll") for (int m = 1; m < C::NPMAX; m++) {               \
          const int lcm = __shfl_sync(0xffffffffu, mylc, (q + m) & 31);                 \
          if (q + m < q2 && lcm <= lane) sel = q + m;                                  \
        }                                                                              \
        const double wxl = s_wx[sel * C::WXS + lane];                                  \
        const double2 *wyp = (const double2 *)(s_wy + sel * C::WYS);                   \
        _Pragma("unroll") for (int b = 0; b + 1 < W; b += 2) {                         \
          const double2 v = wyp[b >> 1];                                               \
          acc[((k) + b) % W] = fma(v.x, wxl, acc[((k) + b) % W]);                      \
          acc[((k) + b + 1) % W] = fma(v.y, wxl, acc[((k) + b + 1) % W]);              \
        }                                                                              \
        if (W & 1) acc[((k) + W - 1) % W] = fma(s_wy[sel * C::WYS + W - 1], wxl, acc[((k) + W - 1) % W]); \
        q = q2;                                                                        \
      }                                                                                \
      if (q == n) goto next_chunk;                                                     \
      red_row(col, oy + r, interior, g, acc[(k) % W]);                                 \
      acc[(k) % W] = 0.0;                                                              \
      r++;                                                                             \
    }
      VP_STRIP_PHASE(0) VP_STRIP_PHASE(1) VP_STRIP_PHASE(2) VP_STRIP_PHASE(3) VP_STRIP_PHASE(4)
      VP_STRIP_PHASE(5) VP_STRIP_PHASE(6) VP_STRIP_PHASE(7) VP_STRIP_PHASE(8) VP_STRIP_PHASE(9)
      VP_STRIP_PHASE(10) VP_STRIP_PHASE(11) VP_STRIP_PHASE(12) VP_STRIP_PHASE(13) VP_STRIP_PHASE(14)
      VP_STRIP_PHASE(15)
#undef VP_STRIP_PHASE
    }
  }
next_chunk:
  __syncwarp();
  c0 += C::CH;
  if (c0 < it.w) goto stage;
  // flush the ring: acc[j] holds row r + ((j - r) mod W)
#pragma unroll
  for (int j = 0; j < W; j++) {
    red_row(col, oy + r + ((j - r % W) + W) % W, interior, g, acc[j]);
  }
}

template <int W>
static void launch_spread_strip_w(vp_plan_s *P, const VpSpreadSet &S, const GridArgs &g, const double *f) {
  constexpr int D = VP_HORNER_DEG(W);
  if (S.n_sitems == 0) return;
  const size_t sm = StripCfg<W>::smem_warp * VP_STRIP_WARPS;
  const unsigned nb = (unsigned)((S.n_sitems + VP_STRIP_WARPS - 1) / VP_STRIP_WARPS);
  if (P->opts.spread_pack == 1) {
    vp_smem_attr((const void *)k_spread_strip<W, D, true>, sm);
    k_spread_strip<W, D, true><<<nb, 32 * VP_STRIP_WARPS, sm, P->stream>>>(S.sitems, S.n_sitems, S.sx, S.sy, S.sw,
                                                                           S.sperm, f, g, S.fs_out);
  } else {
    vp_smem_attr((const void *)k_spread_strip<W, D, false>, sm);
    k_spread_strip<W, D, false><<<nb, 32 * VP_STRIP_WARPS, sm, P->stream>>>(S.sitems, S.n_sitems, S.sx, S.sy, S.sw,
                                                                            S.sperm, f, g, S.fs_out);
  }
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

// ---------------------------------------------------------------------------------------------
// Row-pair strips (default for W <= 12).  Measured on B200 (profiles/r2): the 32-column strip
// above is bound by shared-memory wavefronts (~16 per point; an LDS.128 broadcast costs 2 of them) and wastes
// 32 - W of the 32 lanes in every DFMA step.  Here a warp owns 16 grid columns and two row phases: lane
// (c, h) = (lane & 15, lane >> 4) accumulates column c of the rows 2P + h, so a point's W x W footprint keeps
// W of 16 columns busy (62% at W = 10) and each lane needs only the ~W/2 y weights of its row parity.  Row
// pairs (2P, 2P + 1) live in a register ring of S = W/2 + 1 slots (pair P in acc[P mod S]); a point with origin
// row r (pair P = r >> 1) adds to pairs P .. P + S - 1 the products wx[c - lc] * c_j wy[2j + h - (r & 1)]
// (zero-padded taps at -1 and >= W), i.e. one LDS.64 of two adjacent addresses (one wavefront) and one DFMA
// per pair.  The x taps are staged compactly with fixed zero margins, so the lane's x weight is one LDS.64 of
// 16 consecutive words, and no padding is rewritten when points are restaged.  Per point: 1 meta + 1 x + S - 1
// or S y loads (about 7.5 wavefronts at W = 10) and S - 1 or S DFMA per lane.  Strips are SW = 17 - W origin
// columns wide, so the RED flush covers 16 / SW columns per origin column (more halo REDs than the 32-column
// strip, 2.3x vs 1.4x at W = 10; the L2 atomic rate, 4.7e11/s, is below the shared-memory bound).
#ifndef VP_PAIR_WARPS
#define VP_PAIR_WARPS 4  // warps per CTA at W <= 10
#endif
#ifndef VP_PAIR_MINB
#define VP_PAIR_MINB 5   // CTAs per SM
#endif
#ifndef VP_PAIR2_WARPS
#define VP_PAIR2_WARPS 4
#define VP_PAIR2_MINB 5
#endif
#ifndef VP_PAIR_SH
#define VP_PAIR_SH 128  // footprint-origin rows per pair strip (even)
#endif
template <int W>
struct PairCfg {
  static constexpr int SW = 17 - W;  // footprint-origin columns per strip
  static constexpr int SH = VP_PAIR_SH;
  static constexpr int S = W / 2 + 1;  // ring slots (row pairs touched by one footprint)
  static constexpr int CH = 32;
  static constexpr int XO = SW & ~1;   // x row: tap a at XO + a (XO >= SW - 1, even), zeros around
  static constexpr int odd_half(int n) { return ((n / 2) & 1) ? n : n + 2; }  // 16-byte stride odd: no conflicts
  static constexpr int WXS = odd_half(XO + 16);
  static constexpr int WYS = odd_half(2 * S + 2);  // y row: c wy[b] at 2 + b, zeros at 0, 1 and >= 2 + W
  static constexpr size_t smem_warp = (size_t)CH * (WXS + WYS + 1) * 8;  // + per-point meta (int2)
  // warps per CTA and CTAs per SM: 4 x 5 = 20 warps, one warp of each CTA per SM sub-partition, so ptxas may use
  // 16384 / (5 x 32) -> 96 registers.  (7-warp CTAs x 3 = 21 warps put two warps of a CTA on one sub-partition:
  // 6 per sub-partition, an 80-register cap; measured at config 5: 10.40 ms vs 9.98 ms with 4 x 5, and the two-field
  // kernel 285 -> 198 us on config 2, profiles/r2/pair2.  8 x 3 = 24 warps: 11.12 ms.)
  static constexpr int WARPS = W <= 10 ? VP_PAIR_WARPS : 4;
  static constexpr int MINB = W <= 10 ? VP_PAIR_MINB : 5;
  // two-field kernel (k_spread_pair2): the same shape; at the 80-register cap of 7-warp CTAs the tap loads of a
  // point were serialised through two registers
  static constexpr int WARPS2 = VP_PAIR2_WARPS;
  static constexpr int MINB2 = VP_PAIR2_MINB;
  static constexpr int WARPS4 = 4;  // four-field kernel: 16 warps per SM, 128 registers
  static constexpr int MINB4 = 4;
};

template <int W, int D>
__global__ void __launch_bounds__(32 * PairCfg<W>::WARPS, PairCfg<W>::MINB)
    k_spread_pair(const int4 *__restrict__ items, int64_t n_items, const double *__restrict__ sx,
                  const double *__restrict__ sy, const double *__restrict__ sw, const int32_t *__restrict__ sperm,
                  const double *__restrict__ f, GridArgs g, double *__restrict__ fs_out) {
  using C = PairCfg<W>;
  constexpr int S = C::S;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, c = lane & 15, h = lane >> 4;
  const int64_t item = (int64_t)blockIdx.x * C::WARPS + warp;
  if (item >= n_items) return;
  double *s_wx = smem + (size_t)warp * (C::CH * (C::WXS + C::WYS + 1));
  double *s_wy = s_wx + C::CH * C::WXS;
  int2 *s_meta = (int2 *)(s_wy + C::CH * C::WYS);
  // fixed zero margins of the staged rows (the staging below writes only the tap positions)
  for (int i = lane; i < C::CH * C::WXS; i += 32) s_wx[i] = 0.0;
  for (int i = lane; i < C::CH * C::WYS; i += 32) s_wy[i] = 0.0;
  __syncwarp();
  // lane bases: the staged per-point meta holds byte offsets, so a point costs one broadcast load, two adds and
  // the tap loads with immediate offsets (no per-point index arithmetic)
  const char *xb = (const char *)s_wx + 8 * c;
  const char *yb = (const char *)s_wy + 8 * h;
  // (persistent warps walking every stride-th item measured slower, 14.5 vs 10.9 ms at config 5: the items in
  // flight no longer form one band of neighbouring strips, so the halo REDs and grid rows miss L2)
  const int4 it = items[item];
  const int64_t ox = (int64_t)it.x * C::SW - (W / 2 + 1), oy = (int64_t)it.y * C::SH - (W / 2 + 1);
  const bool interior = ox >= 0 && oy >= 0 && ox + 16 <= g.nfx && oy + C::SH + W + 1 <= g.nfy;
  double *col = g.data + (interior ? ox + c : wrapi(ox + c, g.nfx));
  // two accumulator rings, for the even and odd points of a row-pair step: consecutive points then have no DFMA
  // dependency (the ring is summed when a pair is flushed)
  // (W >= 11: one ring; the second one does not fit the register budget of 3 CTAs per SM)
  constexpr bool TWO = W <= 10;
  double acc[S], acc_b[S];
  double(&acc2)[S] = TWO ? acc_b : acc;
#pragma unroll
  for (int b = 0; b < S; b++) acc[b] = acc_b[b] = 0.0;
  double *rowp = nullptr;  // interior items: the flushed pair's row 2P + h in column c (advanced by 2 rows)
  int c0 = it.z, n = 0, q = 0, P = 0, mylr = 0x7fffffff;
  bool first = true;
  // software pipeline over the 32-point chunks: the coordinates, weight and f of chunk k + 1 and the f index of
  // chunk k + 2 are loaded while chunk k is staged and walked, so no global-load latency (two dependent loads for
  // f[sperm[j]]) is exposed at a staging step
  double px = 0.0, py = 0.0, pw = 0.0, pf = 0.0;
  int pidx = 0;
  {
    const int j = c0 + lane;
    if (j < it.w) {
      px = sx[j];
      py = sy[j];
      pw = sw[j];
      pf = __ldg(f + sperm[j]);
    }
    if (j + C::CH < it.w) pidx = sperm[j + C::CH];
  }
stage:
  n = min(C::CH, it.w - c0);
  mylr = 0x7fffffff;
  {
    const double xj = px, yj = py, wj = pw, fj = pf;
    const int j = c0 + lane, jn = j + C::CH;
    if (jn < it.w) {
      px = sx[jn];
      py = sy[jn];
      pw = sw[jn];
      pf = __ldg(f + pidx);
    }
    if (jn + C::CH < it.w) pidx = sperm[jn + C::CH];
    if (lane < n) {
      if (fs_out) fs_out[j] = fj;  // f in spreading order: spatially coherent copy for the stencil gathers
      const double cj = fj * wj;
      double wv[W];
      const int lc = (int)(es_horner<W, D>(gcoord(xj, g.ox, g.inv_h), wv) - ox);
      double2 *xp = (double2 *)(s_wx + lane * C::WXS + C::XO);
#pragma unroll
      for (int a = 0; a < W; a += 2) xp[a >> 1] = make_double2(wv[a], a + 1 < W ? wv[a + 1] : 0.0);
      const int lr = (int)(es_horner<W, D>(gcoord(yj, g.oy, g.inv_h), wv) - oy);
      double2 *yp = (double2 *)(s_wy + lane * C::WYS + 2);
#pragma unroll
      for (int b = 0; b < W; b += 2) yp[b >> 1] = make_double2(cj * wv[b], b + 1 < W ? cj * wv[b + 1] : 0.0);
      // x tap of lane column c at byte xb + meta.x: tap c - lc of this point's row; y taps of lane half h at
      // yb + meta.y + 16 j: c wy[2j + h - (lr & 1)] (zero-padded at -1 and >= W)
      s_meta[lane] = make_int2(8 * (lane * C::WXS + C::XO - lc), 8 * (lane * C::WYS + 2 - (lr & 1)));
      mylr = lr;
    }
  }
  __syncwarp();
  q = 0;
  if (first) {
    P = __shfl_sync(0xffffffffu, mylr, 0) >> 1;
    rowp = col + (oy + 2 * P + h) * g.row;
    first = false;
  }
  for (;;) {
    switch (P % S) {
#define VP_PAIR_POINT(ACC, qq, K)                                                                      \
  {                                                                                                   \
    const int2 m = s_meta[qq];                                                                        \
    const double wxl = *(const double *)(xb + m.x);                                                   \
    const char *yp = yb + m.y;                                                                        \
    /* the last pair is all zero for an even origin row at even W (bit 3 of the y offset = origin parity) */ \
    _Pragma("unroll") for (int jj = 0; jj < S; jj++)                                                  \
      if (jj < S - 1 || (W & 1) || (m.y & 8))                                                         \
        ACC[((K) + jj) % S] = fma(*(const double *)(yp + 16 * jj), wxl, ACC[((K) + jj) % S]);         \
  }
#define VP_PAIR_PHASE(k)                                                                              \
  case k:                                                                                             \
    if ((k) < S) {                                                                                    \
      const int e = __popc(__ballot_sync(0xffffffffu, mylr <= 2 * P + 1));                             \
      for (; q + 1 < e; q += 2) {                                                                     \
        VP_PAIR_POINT(acc, q, k)                                                                      \
        VP_PAIR_POINT(acc2, q + 1, k)                                                                 \
      }                                                                                               \
      if (q < e) {                                                                                    \
        VP_PAIR_POINT(acc, q, k)                                                                      \
        q++;                                                                                          \
      }                                                                                               \
      if (q == n) goto next_chunk;                                                                    \
      const double v = TWO ? acc[(k)] + acc2[(k)] : acc[(k)];                                        \
      if (interior) {                                                                                 \
        if (v != 0.0) atomicAdd(rowp, v);                                                             \
      } else if (v != 0.0) {                                                                          \
        red_row_wrapped(col, oy + 2 * P + h, g.nfy, g.row, v);                                        \
      }                                                                                               \
      rowp += 2 * g.row;                                                                              \
      acc[(k)] = 0.0;                                                                                 \
      acc2[(k)] = 0.0;                                                                                \
      P++;                                                                                            \
    }
      VP_PAIR_PHASE(0) VP_PAIR_PHASE(1) VP_PAIR_PHASE(2) VP_PAIR_PHASE(3) VP_PAIR_PHASE(4)
      VP_PAIR_PHASE(5) VP_PAIR_PHASE(6) VP_PAIR_PHASE(7) VP_PAIR_PHASE(8)
#undef VP_PAIR_PHASE
#undef VP_PAIR_POINT
    }
  }
next_chunk:
  __syncwarp();
  c0 += C::CH;
  if (c0 < it.w) goto stage;
  // flush the ring: acc[i] holds pair P + ((i - P) mod S)
#pragma unroll
  for (int i = 0; i < S; i++) red_row(col, oy + 2 * (P + ((i - P % S) + S) % S) + h, interior, g, TWO ? acc[i] + acc2[i] : acc[i]);
}

template <int W>
static void launch_spread_pair_w(vp_plan_s *P, const VpSpreadSet &S, const GridArgs &g, const double *f) {
  constexpr int D = VP_HORNER_DEG(W);
  if constexpr (W <= 12) {
    if (S.n_sitems == 0) return;
    constexpr int NW = PairCfg<W>::WARPS;
    const size_t sm = PairCfg<W>::smem_warp * NW;
    const unsigned nb = (unsigned)((S.n_sitems + NW - 1) / NW);
    vp_smem_attr((const void *)k_spread_pair<W, D>, sm);
    k_spread_pair<W, D><<<nb, 32 * NW, sm, P->stream>>>(S.sitems, S.n_sitems, S.sx, S.sy, S.sw, S.sperm,
                                                                   f, g, S.fs_out);
    VP_CHECK_LAUNCH();
    P->n_kernels++;
  } else {
    throw VpError{VP_ERR_UNSUPPORTED};
  }
}

// strip geometry of width W (host side of StripCfg / PairCfg): kind 0 = 32-column strips, 1 = row-pair strips
void vp_strip_dims(int W, int kind, int *SW, int *SH) {
  *SW = kind ? 17 - W : 33 - W;
  *SH = kind ? VP_PAIR_SH : VP_STRIP_SH;
}

void vp_launch_spread(vp_plan_s *P, const VpSpreadSet &S, const GridArgs &g, const double *f) {
  switch (P->w) {
#define CASE(W)                                                \
  case W:                                                      \
    if (S.strip == 2) launch_spread_pair_w<W>(P, S, g, f);     \
    else if (S.strip) launch_spread_strip_w<W>(P, S, g, f);    \
    else launch_spread_w<W>(P, S, g, f);                       \
    break;
    CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: throw VpError{VP_ERR_UNSUPPORTED};
  }
}

// ---------------------------------------------------------------------------------------------
// Batched strip spreading: KB fields f_0 .. f_{KB-1} on the same nodes, KB NH grids.  The
// footprint geometry, the Horner weights and the shared-memory broadcasts of wx / wy are shared by the KB
// fields; per point and lane the kernel adds wx * c_k * wy[b] to KB register rings (KB * W DFMA for one set
// of loads), so the shared-memory delivery that bounds k_spread_strip is paid once per KB fields.
template <int KB>
struct BatchPtrs {
  const double *f[KB];
  double *grid[KB];
  double *fs[KB];  // spreading-order copies of the fields (null: not written)
};

template <int W, int D, int KB>
__global__ void __launch_bounds__(32 * VP_STRIP_WARPS, (KB <= 2 || W <= 10) ? 4 : 3)
    k_spread_strip_b(const int4 *__restrict__ items, int64_t n_items, const double *__restrict__ sx,
                     const double *__restrict__ sy, const double *__restrict__ sw, const int32_t *__restrict__ sperm,
                     BatchPtrs<KB> bp, GridArgs g) {
  using C = StripCfg<W>;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * VP_STRIP_WARPS + warp;
  if (item >= n_items) return;
  constexpr size_t per_warp = (size_t)C::CH * (C::WXS + C::WYS + KB);
  double *s_wy = smem + (size_t)warp * per_warp;
  double *s_wx = s_wy + C::CH * C::WYS;
  double *s_c = s_wx + C::CH * C::WXS;  // [CH][KB], 16-byte aligned rows (KB even)
  const int4 it = items[item];
  const int64_t ox = (int64_t)it.x * C::SW - (W / 2 + 1), oy = (int64_t)it.y * C::SH - (W / 2 + 1);
  const bool interior = ox >= 0 && oy >= 0 && ox + 32 <= g.nfx && oy + C::SH + W - 1 <= g.nfy;
  const int64_t colx = interior ? ox + lane : wrapi(ox + lane, g.nfx);
  double acc[KB][W];
#pragma unroll
  for (int k = 0; k < KB; k++)
#pragma unroll
    for (int b = 0; b < W; b++) acc[k][b] = 0.0;
  int c0 = it.z, n = 0, q = 0, r = 0, mylr = 0x7fffffff, prev_lc = 0, mylc = 0;
  unsigned starts = 0;
  bool first = true;
  double *wrow = s_wx + lane * C::WXS;
#pragma unroll
  for (int a = 0; a < 32; a++) wrow[a] = 0.0;
stage:
  n = min(C::CH, it.w - c0);
  mylr = 0x7fffffff;
  mylc = 1 << 20;
  if (lane < n) {
    const int j = c0 + lane;
    const int32_t node = sperm[j];
    const double wj = sw[j];
#pragma unroll
    for (int k = 0; k < KB; k++) {
      const double fj = __ldg(bp.f[k] + node);
      if (bp.fs[k]) bp.fs[k][j] = fj;
      s_c[lane * KB + k] = fj * wj;
    }
#pragma unroll
    for (int a = 0; a < W; a++) wrow[prev_lc + a] = 0.0;
    // taps one Horner chain at a time (the KB register rings stay live through the staging)
    const double gx = gcoord(sx[j], g.ox, g.inv_h), gy = gcoord(sy[j], g.oy, g.inv_h);
    const double sxw = __dsub_rn(gx, 0.5 * W), syw = __dsub_rn(gy, 0.5 * W);
    const int ix = (int)ceil(sxw), iy = (int)ceil(syw);
    const double txh = 2.0 * (ix - sxw) - 1.0, tyh = 2.0 * (iy - syw) - 1.0;
    const int lc = (int)(ix - ox), lr = (int)(iy - oy);
#pragma unroll 1
    for (int a = 0; a < W; a++) wrow[lc + a] = es_tap<W, D>(txh, a);
    prev_lc = lc;
#pragma unroll 1
    for (int b = 0; b < W; b++) s_wy[lane * C::WYS + b] = es_tap<W, D>(tyh, b);
    mylr = lr;
  }
  __syncwarp();
  q = 0;
  if (first) {
    r = __shfl_sync(0xffffffffu, mylr, 0);
    first = false;
  }
  for (;;) {
    switch (r % W) {
#define VP_STRIPB_PHASE(ph)                                                                     \
  case ph:                                                                                      \
    if ((ph) < W) {                                                                             \
      _Pragma("unroll 2") for (const int e = __popc(__ballot_sync(0xffffffffu, mylr <= r)); q < e; q++) { \
        const double wxl = s_wx[q * C::WXS + lane];                                             \
        double t[KB];                                                                           \
        _Pragma("unroll") for (int k = 0; k < KB; k += 2) {                                     \
          const double2 cc = *(const double2 *)(s_c + q * KB + k);                              \
          t[k] = wxl * cc.x;                                                                    \
          t[k + 1] = wxl * cc.y;                                                                \
        }                                                                                       \
        const double2 *wyp = (const double2 *)(s_wy + q * C::WYS);                              \
        _Pragma("unroll") for (int b = 0; b + 1 < W; b += 2) {                                  \
          const double2 v = wyp[b >> 1];                                                        \
          _Pragma("unroll") for (int k = 0; k < KB; k++) {                                      \
            acc[k][((ph) + b) % W] = fma(v.x, t[k], acc[k][((ph) + b) % W]);                    \
            acc[k][((ph) + b + 1) % W] = fma(v.y, t[k], acc[k][((ph) + b + 1) % W]);            \
          }                                                                                     \
        }                                                                                       \
        if (W & 1) {                                                                            \
          const double v = s_wy[q * C::WYS + W - 1];                                            \
          _Pragma("unroll") for (int k = 0; k < KB; k++) acc[k][((ph) + W - 1) % W] =           \
              fma(v, t[k], acc[k][((ph) + W - 1) % W]);                                         \
        }                                                                                       \
      }                                                                                         \
      if (q == n) goto next_chunk;                                                              \
      _Pragma("unroll") for (int k = 0; k < KB; k++) {                                          \
        red_row(bp.grid[k] + colx, oy + r, interior, g, acc[k][(ph) % W]);                      \
        acc[k][(ph) % W] = 0.0;                                                                 \
      }                                                                                         \
      r++;                                                                                      \
    }
      VP_STRIPB_PHASE(0) VP_STRIPB_PHASE(1) VP_STRIPB_PHASE(2) VP_STRIPB_PHASE(3) VP_STRIPB_PHASE(4)
      VP_STRIPB_PHASE(5) VP_STRIPB_PHASE(6) VP_STRIPB_PHASE(7) VP_STRIPB_PHASE(8) VP_STRIPB_PHASE(9)
      VP_STRIPB_PHASE(10) VP_STRIPB_PHASE(11) VP_STRIPB_PHASE(12) VP_STRIPB_PHASE(13) VP_STRIPB_PHASE(14)
      VP_STRIPB_PHASE(15)
#undef VP_STRIPB_PHASE
    }
  }
next_chunk:
  __syncwarp();
  c0 += C::CH;
  if (c0 < it.w) goto stage;
#pragma unroll
  for (int k = 0; k < KB; k++)
#pragma unroll
    for (int jj = 0; jj < W; jj++) red_row(bp.grid[k] + colx, oy + r + ((jj - r % W) + W) % W, interior, g, acc[k][jj]);
}

// ---------------------------------------------------------------------------------------------
// Row-pair strips for two fields.  k_spread_pair is bound by shared-memory
// wavefronts and issue slots per point (meta + x tap + S y taps, ES taps by Horner in the staging); two fields
// on the same nodes share all of them.  The y taps are staged unscaled, the strengths (c_0, c_1) = (f_0, f_1) w
// of a point sit next to its meta (one 128-bit broadcast), and the lane's x tap is scaled per field in
// registers: per point 1 meta + 1 strengths (2 wavefronts) + 1 x + S y loads and 2 DMUL + 2 S DFMA, i.e. ~5
// wavefronts per field-point instead of ~8.  The two register rings of k_spread_pair (even / odd points)
// become the rings of field 0 and field 1 (96 registers at 4 warps x 5 CTAs per SM, PairCfg).  W <= 10.
template <int W, int D>
__global__ void __launch_bounds__(32 * PairCfg<W>::WARPS2, PairCfg<W>::MINB2)
    k_spread_pair2(const int4 *__restrict__ items, int64_t n_items, const double *__restrict__ sx,
                   const double *__restrict__ sy, const double *__restrict__ sw, const int32_t *__restrict__ sperm,
                   BatchPtrs<2> bp, GridArgs g) {
  using C = PairCfg<W>;
  constexpr int S = C::S;
  constexpr int PW = C::WXS + C::WYS + 3;  // doubles per staged point: x row, y row, meta (int2), strengths
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, c = lane & 15, h = lane >> 4;
  const int64_t item = (int64_t)blockIdx.x * C::WARPS2 + warp;
  if (item >= n_items) return;
  double *s_wx = smem + (size_t)warp * (C::CH * PW);
  double *s_wy = s_wx + C::CH * C::WXS;
  double2 *s_c = (double2 *)(s_wy + C::CH * C::WYS);  // 16-byte aligned: CH * (WXS + WYS) is even
  int2 *s_meta = (int2 *)(s_c + C::CH);
  for (int i = lane; i < C::CH * C::WXS; i += 32) s_wx[i] = 0.0;
  for (int i = lane; i < C::CH * C::WYS; i += 32) s_wy[i] = 0.0;
  __syncwarp();
  const char *xb = (const char *)s_wx + 8 * c;
  const char *yb = (const char *)s_wy + 8 * h;
  const int4 it = items[item];
  const int64_t ox = (int64_t)it.x * C::SW - (W / 2 + 1), oy = (int64_t)it.y * C::SH - (W / 2 + 1);
  const bool interior = ox >= 0 && oy >= 0 && ox + 16 <= g.nfx && oy + C::SH + W + 1 <= g.nfy;
  const int64_t coff = interior ? ox + c : wrapi(ox + c, g.nfx);
  double *col0 = bp.grid[0] + coff, *col1 = bp.grid[1] + coff;
  const ptrdiff_t gd = bp.grid[1] - bp.grid[0];
  double acc[S], acc2[S];  // rings of field 0 and field 1
#pragma unroll
  for (int b = 0; b < S; b++) acc[b] = acc2[b] = 0.0;
  double *rowp = nullptr;
  int c0 = it.z, n = 0, q = 0, P = 0, mylr = 0x7fffffff;
  bool first = true;
  const double *__restrict__ f0 = bp.f[0], *__restrict__ f1 = bp.f[1];
  double px = 0.0, py = 0.0, pw = 0.0, pf0 = 0.0, pf1 = 0.0;
  int pidx = 0;
  {
    const int j = c0 + lane;
    if (j < it.w) {
      px = sx[j];
      py = sy[j];
      pw = sw[j];
      const int s = sperm[j];
      pf0 = __ldg(f0 + s);
      pf1 = __ldg(f1 + s);
    }
    if (j + C::CH < it.w) pidx = sperm[j + C::CH];
  }
stage:
  n = min(C::CH, it.w - c0);
  mylr = 0x7fffffff;
  {
    const double xj = px, yj = py, wj = pw, fj0 = pf0, fj1 = pf1;
    const int j = c0 + lane, jn = j + C::CH;
    if (jn < it.w) {
      px = sx[jn];
      py = sy[jn];
      pw = sw[jn];
      pf0 = __ldg(f0 + pidx);
      pf1 = __ldg(f1 + pidx);
    }
    if (jn + C::CH < it.w) pidx = sperm[jn + C::CH];
    if (lane < n) {
      if (bp.fs[0]) {
        bp.fs[0][j] = fj0;
        bp.fs[1][j] = fj1;
      }
      double wv[W];
      const int lc = (int)(es_horner<W, D>(gcoord(xj, g.ox, g.inv_h), wv) - ox);
      double2 *xp = (double2 *)(s_wx + lane * C::WXS + C::XO);
#pragma unroll
      for (int a = 0; a < W; a += 2) xp[a >> 1] = make_double2(wv[a], a + 1 < W ? wv[a + 1] : 0.0);
      const int lr = (int)(es_horner<W, D>(gcoord(yj, g.oy, g.inv_h), wv) - oy);
      double2 *yp = (double2 *)(s_wy + lane * C::WYS + 2);
#pragma unroll
      for (int b = 0; b < W; b += 2) yp[b >> 1] = make_double2(wv[b], b + 1 < W ? wv[b + 1] : 0.0);
      s_c[lane] = make_double2(fj0 * wj, fj1 * wj);
      s_meta[lane] = make_int2(8 * (lane * C::WXS + C::XO - lc), 8 * (lane * C::WYS + 2 - (lr & 1)));
      mylr = lr;
    }
  }
  __syncwarp();
  q = 0;
  if (first) {
    P = __shfl_sync(0xffffffffu, mylr, 0) >> 1;
    rowp = col0 + (oy + 2 * P + h) * g.row;
    first = false;
  }
  for (;;) {
    switch (P % S) {
#ifndef VP_PAIR2_X2
#define VP_PAIR2_X2 1  // two points per iteration of the point loop
#endif
#define VP_PAIR2_POINT(qq, K)                                                                         \
  {                                                                                                   \
    const int2 m = s_meta[qq];                                                                        \
    const double2 cc = s_c[qq];                                                                       \
    const double wxl = *(const double *)(xb + m.x);                                                   \
    const double wx0 = wxl * cc.x, wx1 = wxl * cc.y;                                                  \
    const char *yp = yb + m.y;                                                                        \
    _Pragma("unroll") for (int jj = 0; jj < S; jj++)                                                  \
      if (jj < S - 1 || (W & 1) || (m.y & 8)) {                                                       \
        const double wyl = *(const double *)(yp + 16 * jj);                                           \
        acc[((K) + jj) % S] = fma(wyl, wx0, acc[((K) + jj) % S]);                                     \
        acc2[((K) + jj) % S] = fma(wyl, wx1, acc2[((K) + jj) % S]);                                   \
      }                                                                                               \
  }
  // (the point loop is not unrolled further: with 9 phases the kernel must stay inside the instruction cache;
  // an 8x unrolled build ran 4x slower on B200, stalled on instruction fetch: profiles/r2/pair2)
#define VP_PAIR2_PHASE(k)                                                                             \
  case k:                                                                                             \
    if ((k) < S) {                                                                                    \
      const int e = __popc(__ballot_sync(0xffffffffu, mylr <= 2 * P + 1));                             \
      if (VP_PAIR2_X2) {                                                                              \
        _Pragma("unroll 1") for (; q + 1 < e; q += 2) {                                               \
          VP_PAIR2_POINT(q, k)                                                                        \
          VP_PAIR2_POINT(q + 1, k)                                                                    \
        }                                                                                             \
        if (q < e) {                                                                                  \
          VP_PAIR2_POINT(q, k)                                                                        \
          q++;                                                                                        \
        }                                                                                             \
      } else {                                                                                        \
        _Pragma("unroll 1") for (; q < e; q++) VP_PAIR2_POINT(q, k)                                   \
      }                                                                                               \
      if (q == n) goto next_chunk;                                                                    \
      const double v0 = acc[(k)], v1 = acc2[(k)];                                                     \
      if (interior) {                                                                                 \
        if (v0 != 0.0) atomicAdd(rowp, v0);                                                           \
        if (v1 != 0.0) atomicAdd(rowp + gd, v1);                                                      \
      } else {                                                                                        \
        if (v0 != 0.0) red_row_wrapped(col0, oy + 2 * P + h, g.nfy, g.row, v0);                       \
        if (v1 != 0.0) red_row_wrapped(col1, oy + 2 * P + h, g.nfy, g.row, v1);                       \
      }                                                                                               \
      rowp += 2 * g.row;                                                                              \
      acc[(k)] = 0.0;                                                                                 \
      acc2[(k)] = 0.0;                                                                                \
      P++;                                                                                            \
    }
      VP_PAIR2_PHASE(0) VP_PAIR2_PHASE(1) VP_PAIR2_PHASE(2) VP_PAIR2_PHASE(3) VP_PAIR2_PHASE(4)
      VP_PAIR2_PHASE(5) VP_PAIR2_PHASE(6) VP_PAIR2_PHASE(7) VP_PAIR2_PHASE(8)
#undef VP_PAIR2_PHASE
#undef VP_PAIR2_POINT
    }
  }
next_chunk:
  __syncwarp();
  c0 += C::CH;
  if (c0 < it.w) goto stage;
#pragma unroll
  for (int i = 0; i < S; i++) {
    const int64_t gy = oy + 2 * (P + ((i - P % S) + S) % S) + h;
    red_row(col0, gy, interior, g, acc[i]);
    red_row(col1, gy, interior, g, acc2[i]);
  }
}

// Four fields per pass (K >= 4 batches): the same kernel with four register rings and two 128-bit strength loads
// per point (24 DFMA for 12.5 shared-memory wavefronts); 4-warp CTAs x 4 per SM for the 128-register budget.
template <int W, int D>
__global__ void __launch_bounds__(32 * PairCfg<W>::WARPS4, PairCfg<W>::MINB4)
    k_spread_pair4(const int4 *__restrict__ items, int64_t n_items, const double *__restrict__ sx,
                   const double *__restrict__ sy, const double *__restrict__ sw, const int32_t *__restrict__ sperm,
                   BatchPtrs<4> bp, GridArgs g) {
  using C = PairCfg<W>;
  constexpr int S = C::S;
  constexpr int PW = C::WXS + C::WYS + 5;  // doubles per staged point: x row, y row, meta (int2), 4 strengths
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, c = lane & 15, h = lane >> 4;
  const int64_t item = (int64_t)blockIdx.x * C::WARPS4 + warp;
  if (item >= n_items) return;
  double *s_wx = smem + (size_t)warp * (C::CH * PW);
  double *s_wy = s_wx + C::CH * C::WXS;
  double2 *s_c = (double2 *)(s_wy + C::CH * C::WYS);  // 16-byte aligned: CH * (WXS + WYS) is even; [point][2]
  int2 *s_meta = (int2 *)(s_c + 2 * C::CH);
  for (int i = lane; i < C::CH * C::WXS; i += 32) s_wx[i] = 0.0;
  for (int i = lane; i < C::CH * C::WYS; i += 32) s_wy[i] = 0.0;
  __syncwarp();
  const char *xb = (const char *)s_wx + 8 * c;
  const char *yb = (const char *)s_wy + 8 * h;
  const int4 it = items[item];
  const int64_t ox = (int64_t)it.x * C::SW - (W / 2 + 1), oy = (int64_t)it.y * C::SH - (W / 2 + 1);
  const bool interior = ox >= 0 && oy >= 0 && ox + 16 <= g.nfx && oy + C::SH + W + 1 <= g.nfy;
  const int64_t coff = interior ? ox + c : wrapi(ox + c, g.nfx);
  double *col0 = bp.grid[0] + coff, *col1 = bp.grid[1] + coff, *col2 = bp.grid[2] + coff, *col3 = bp.grid[3] + coff;
  const ptrdiff_t gd = bp.grid[1] - bp.grid[0], gd2 = bp.grid[2] - bp.grid[0], gd3 = bp.grid[3] - bp.grid[0];
  double acc[S], acc2[S], acc3[S], acc4[S];  // rings of the four fields
#pragma unroll
  for (int b = 0; b < S; b++) acc[b] = acc2[b] = acc3[b] = acc4[b] = 0.0;
  double *rowp = nullptr;
  int c0 = it.z, n = 0, q = 0, P = 0, mylr = 0x7fffffff;
  bool first = true;
  const double *__restrict__ f0 = bp.f[0], *__restrict__ f1 = bp.f[1], *__restrict__ f2 = bp.f[2], *__restrict__ f3 = bp.f[3];
  double px = 0.0, py = 0.0, pw = 0.0, pf0 = 0.0, pf1 = 0.0, pf2 = 0.0, pf3 = 0.0;
  int pidx = 0;
  {
    const int j = c0 + lane;
    if (j < it.w) {
      px = sx[j];
      py = sy[j];
      pw = sw[j];
      const int s = sperm[j];
      pf0 = __ldg(f0 + s);
      pf1 = __ldg(f1 + s);
      pf2 = __ldg(f2 + s);
      pf3 = __ldg(f3 + s);
    }
    if (j + C::CH < it.w) pidx = sperm[j + C::CH];
  }
stage:
  n = min(C::CH, it.w - c0);
  mylr = 0x7fffffff;
  {
    const double xj = px, yj = py, wj = pw, fj0 = pf0, fj1 = pf1, fj2 = pf2, fj3 = pf3;
    const int j = c0 + lane, jn = j + C::CH;
    if (jn < it.w) {
      px = sx[jn];
      py = sy[jn];
      pw = sw[jn];
      pf0 = __ldg(f0 + pidx);
      pf1 = __ldg(f1 + pidx);
      pf2 = __ldg(f2 + pidx);
      pf3 = __ldg(f3 + pidx);
    }
    if (jn + C::CH < it.w) pidx = sperm[jn + C::CH];
    if (lane < n) {
      if (bp.fs[0]) {
        bp.fs[0][j] = fj0;
        bp.fs[1][j] = fj1;
        bp.fs[2][j] = fj2;
        bp.fs[3][j] = fj3;
      }
      double wv[W];
      const int lc = (int)(es_horner<W, D>(gcoord(xj, g.ox, g.inv_h), wv) - ox);
      double2 *xp = (double2 *)(s_wx + lane * C::WXS + C::XO);
#pragma unroll
      for (int a = 0; a < W; a += 2) xp[a >> 1] = make_double2(wv[a], a + 1 < W ? wv[a + 1] : 0.0);
      const int lr = (int)(es_horner<W, D>(gcoord(yj, g.oy, g.inv_h), wv) - oy);
      double2 *yp = (double2 *)(s_wy + lane * C::WYS + 2);
#pragma unroll
      for (int b = 0; b < W; b += 2) yp[b >> 1] = make_double2(wv[b], b + 1 < W ? wv[b + 1] : 0.0);
      s_c[2 * lane] = make_double2(fj0 * wj, fj1 * wj);
      s_c[2 * lane + 1] = make_double2(fj2 * wj, fj3 * wj);
      s_meta[lane] = make_int2(8 * (lane * C::WXS + C::XO - lc), 8 * (lane * C::WYS + 2 - (lr & 1)));
      mylr = lr;
    }
  }
  __syncwarp();
  q = 0;
  if (first) {
    P = __shfl_sync(0xffffffffu, mylr, 0) >> 1;
    rowp = col0 + (oy + 2 * P + h) * g.row;
    first = false;
  }
  for (;;) {
    switch (P % S) {
#ifndef VP_PAIR4_X2
#define VP_PAIR4_X2 1  // two points per iteration of the point loop
#endif
#define VP_PAIR4_POINT(qq, K)                                                                         \
  {                                                                                                   \
    const int2 m = s_meta[qq];                                                                        \
    const double2 cc = s_c[2 * (qq)], cd = s_c[2 * (qq) + 1];                                         \
    const double wxl = *(const double *)(xb + m.x);                                                   \
    const double wx0 = wxl * cc.x, wx1 = wxl * cc.y, wx2 = wxl * cd.x, wx3 = wxl * cd.y;              \
    const char *yp = yb + m.y;                                                                        \
    _Pragma("unroll") for (int jj = 0; jj < S; jj++)                                                  \
      if (jj < S - 1 || (W & 1) || (m.y & 8)) {                                                       \
        const double wyl = *(const double *)(yp + 16 * jj);                                           \
        acc[((K) + jj) % S] = fma(wyl, wx0, acc[((K) + jj) % S]);                                     \
        acc2[((K) + jj) % S] = fma(wyl, wx1, acc2[((K) + jj) % S]);                                   \
        acc3[((K) + jj) % S] = fma(wyl, wx2, acc3[((K) + jj) % S]);                                   \
        acc4[((K) + jj) % S] = fma(wyl, wx3, acc4[((K) + jj) % S]);                                   \
      }                                                                                               \
  }
  // (the point loop is not unrolled further: with 9 phases the kernel must stay inside the instruction cache;
  // an 8x unrolled build ran 4x slower on B200, stalled on instruction fetch: profiles/r2/pair2)
#define VP_PAIR4_PHASE(k)                                                                             \
  case k:                                                                                             \
    if ((k) < S) {                                                                                    \
      const int e = __popc(__ballot_sync(0xffffffffu, mylr <= 2 * P + 1));                             \
      if (VP_PAIR4_X2) {                                                                              \
        _Pragma("unroll 1") for (; q + 1 < e; q += 2) {                                               \
          VP_PAIR4_POINT(q, k)                                                                        \
          VP_PAIR4_POINT(q + 1, k)                                                                    \
        }                                                                                             \
        if (q < e) {                                                                                  \
          VP_PAIR4_POINT(q, k)                                                                        \
          q++;                                                                                        \
        }                                                                                             \
      } else {                                                                                        \
        _Pragma("unroll 1") for (; q < e; q++) VP_PAIR4_POINT(q, k)                                   \
      }                                                                                               \
      if (q == n) goto next_chunk;                                                                    \
      const double v0 = acc[(k)], v1 = acc2[(k)], v2 = acc3[(k)], v3 = acc4[(k)];                     \
      if (interior) {                                                                                 \
        if (v0 != 0.0) atomicAdd(rowp, v0);                                                           \
        if (v1 != 0.0) atomicAdd(rowp + gd, v1);                                                      \
        if (v2 != 0.0) atomicAdd(rowp + gd2, v2);                                                     \
        if (v3 != 0.0) atomicAdd(rowp + gd3, v3);                                                     \
      } else {                                                                                        \
        if (v0 != 0.0) red_row_wrapped(col0, oy + 2 * P + h, g.nfy, g.row, v0);                       \
        if (v1 != 0.0) red_row_wrapped(col1, oy + 2 * P + h, g.nfy, g.row, v1);                       \
        if (v2 != 0.0) red_row_wrapped(col2, oy + 2 * P + h, g.nfy, g.row, v2);                       \
        if (v3 != 0.0) red_row_wrapped(col3, oy + 2 * P + h, g.nfy, g.row, v3);                       \
      }                                                                                               \
      rowp += 2 * g.row;                                                                              \
      acc[(k)] = 0.0;                                                                                 \
      acc2[(k)] = 0.0;                                                                                \
      acc3[(k)] = 0.0;                                                                                \
      acc4[(k)] = 0.0;                                                                                \
      P++;                                                                                            \
    }
      VP_PAIR4_PHASE(0) VP_PAIR4_PHASE(1) VP_PAIR4_PHASE(2) VP_PAIR4_PHASE(3) VP_PAIR4_PHASE(4)
      VP_PAIR4_PHASE(5) VP_PAIR4_PHASE(6) VP_PAIR4_PHASE(7) VP_PAIR4_PHASE(8)
#undef VP_PAIR4_PHASE
#undef VP_PAIR4_POINT
    }
  }
next_chunk:
  __syncwarp();
  c0 += C::CH;
  if (c0 < it.w) goto stage;
#pragma unroll
  for (int i = 0; i < S; i++) {
    const int64_t gy = oy + 2 * (P + ((i - P % S) + S) % S) + h;
    red_row(col0, gy, interior, g, acc[i]);
    red_row(col1, gy, interior, g, acc2[i]);
    red_row(col2, gy, interior, g, acc3[i]);
    red_row(col3, gy, interior, g, acc4[i]);
  }
}

template <int W>
static void launch_spread_pair4_w(vp_plan_s *P, const VpSpreadSet &S, const GridArgs &g, const double *const *f,
                                  double *const *grids, double *const *fs) {
  constexpr int D = VP_HORNER_DEG(W);
  if constexpr (W <= 10) {
    if (S.n_sitems == 0) return;
    using C = PairCfg<W>;
    constexpr int NW = C::WARPS4;
    const size_t sm = (size_t)C::CH * (C::WXS + C::WYS + 5) * 8 * NW;
    const unsigned nb = (unsigned)((S.n_sitems + NW - 1) / NW);
    vp_smem_attr((const void *)k_spread_pair4<W, D>, sm);
    BatchPtrs<4> bp;
    for (int k = 0; k < 4; k++) {
      bp.f[k] = f[k];
      bp.grid[k] = grids[k];
      bp.fs[k] = fs ? fs[k] : nullptr;
    }
    k_spread_pair4<W, D><<<nb, 32 * NW, sm, P->stream>>>(S.sitems, S.n_sitems, S.sx, S.sy, S.sw, S.sperm, bp, g);
    VP_CHECK_LAUNCH();
    P->n_kernels++;
  } else {
    throw VpError{VP_ERR_UNSUPPORTED};
  }
}

template <int W>
static void launch_spread_pair2_w(vp_plan_s *P, const VpSpreadSet &S, const GridArgs &g, const double *const *f,
                                  double *const *grids, double *const *fs) {
  constexpr int D = VP_HORNER_DEG(W);
  if constexpr (W <= 10) {
    if (S.n_sitems == 0) return;
    using C = PairCfg<W>;
    constexpr int NW = C::WARPS2;
    const size_t sm = (size_t)C::CH * (C::WXS + C::WYS + 3) * 8 * NW;
    const unsigned nb = (unsigned)((S.n_sitems + NW - 1) / NW);
    vp_smem_attr((const void *)k_spread_pair2<W, D>, sm);
    BatchPtrs<2> bp;
    for (int k = 0; k < 2; k++) {
      bp.f[k] = f[k];
      bp.grid[k] = grids[k];
      bp.fs[k] = fs ? fs[k] : nullptr;
    }
    k_spread_pair2<W, D><<<nb, 32 * NW, sm, P->stream>>>(S.sitems, S.n_sitems, S.sx, S.sy, S.sw, S.sperm, bp, g);
    VP_CHECK_LAUNCH();
    P->n_kernels++;
  } else {
    throw VpError{VP_ERR_UNSUPPORTED};
  }
}

template <int W, int KB>
static void launch_spread_strip_b_w(vp_plan_s *P, const VpSpreadSet &S, const GridArgs &g, const double *const *f,
                                    double *const *grids, double *const *fs) {
  constexpr int D = VP_HORNER_DEG(W);
  if (S.n_sitems == 0) return;
  const size_t sm = (size_t)StripCfg<W>::CH * (StripCfg<W>::WXS + StripCfg<W>::WYS + KB) * 8 * VP_STRIP_WARPS;
  vp_smem_attr((const void *)k_spread_strip_b<W, D, KB>, sm);
  BatchPtrs<KB> bp;
  for (int k = 0; k < KB; k++) {
    bp.f[k] = f[k];
    bp.grid[k] = grids[k];
    bp.fs[k] = fs ? fs[k] : nullptr;
  }
  const unsigned nb = (unsigned)((S.n_sitems + VP_STRIP_WARPS - 1) / VP_STRIP_WARPS);
  k_spread_strip_b<W, D, KB><<<nb, 32 * VP_STRIP_WARPS, sm, P->stream>>>(S.sitems, S.n_sitems, S.sx, S.sy, S.sw,
                                                                         S.sperm, bp, g);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

// spread K fields (K = 1 uses k_spread_strip; pairs and quadruples share one strip pass)
void vp_launch_spread_batch(vp_plan_s *P, const VpSpreadSet &S, const GridArgs &g, int K, const double *const *f,
                            double *const *grids, double *const *fs) {
  if (!S.strip) throw VpError{VP_ERR_UNSUPPORTED};
  for (int k0 = 0; k0 < K;) {
    // row-pair strips: four or two fields per pass at W <= 10 (k_spread_pair4 / k_spread_pair2; batch_pair = 2:
    // pairs only, 1: one pass per field), else one pass per field; 32-column
    // strips: quadruples and pairs (k_spread_strip_b)
    const int kb = S.strip == 2 ? ((P->w <= 10 && P->opts.batch_pair != 1)
                                       ? ((K - k0 >= 4 && P->opts.batch_pair != 2) ? 4 : (K - k0 >= 2 ? 2 : 1))
                                       : 1)
                                : (K - k0 >= 4 ? 4 : (K - k0 >= 2 ? 2 : 1));
    if (kb == 1) {
      VpSpreadSet S1 = S;
      S1.fs_out = fs ? fs[k0] : nullptr;
      GridArgs g1 = g;
      g1.data = grids[k0];
      vp_launch_spread(P, S1, g1, f[k0]);
    } else {
      switch (P->w) {
#define CASEB(W)                                                                                     \
  case W:                                                                                            \
    if (S.strip == 2 && kb == 4) launch_spread_pair4_w<W>(P, S, g, f + k0, grids + k0, fs ? fs + k0 : nullptr); \
    else if (S.strip == 2) launch_spread_pair2_w<W>(P, S, g, f + k0, grids + k0, fs ? fs + k0 : nullptr); \
    else if (kb == 4) launch_spread_strip_b_w<W, 4>(P, S, g, f + k0, grids + k0, fs ? fs + k0 : nullptr); \
    else launch_spread_strip_b_w<W, 2>(P, S, g, f + k0, grids + k0, fs ? fs + k0 : nullptr);         \
    break;
        CASEB(4) CASEB(5) CASEB(6) CASEB(7) CASEB(8) CASEB(9) CASEB(10) CASEB(11) CASEB(12) CASEB(13) CASEB(14)
        CASEB(15) CASEB(16)
#undef CASEB
        default: throw VpError{VP_ERR_UNSUPPORTED};
      }
    }
    k0 += kb;
  }
}

// ---------------------------------------------------------------------------------------------
// FH restriction / prolongation (separable, gather form).  Tap table for FH index i':
// NH indices rlo[i'] .. rlo[i'] + ntap-1, weights rw[i'][t] = psi_FH(X1(i) - X2(i')).
// Transposed table for NH index i: FH indices tlo[i] .. tlo[i] + ntt-1, weights tw[i][t].
struct RestrictArgs {
  const int32_t *rlo;
  const double *rw;
  int ntap;
  const int32_t *tlo;
  const double *tw;
  int ntt;
  int64_t e_lo, ne;  // effective FH index range [e_lo, e_lo + ne)
  int64_t n1, row1, n2, row2;
};

// pass A: tA[r][e] = sum_t rw[e_lo+e][t] g1[r][rlo + t]
__global__ void k_restrict_x(const double *__restrict__ g1, double *__restrict__ tA, RestrictArgs a) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t r = blockIdx.y;
  if (e >= a.ne) return;
  int64_t ip = a.e_lo + e;
  const int32_t lo = a.rlo[ip];
  const double *w = a.rw + ip * a.ntap;
  const double *src = g1 + r * a.row1;
  double acc = 0.0;
  for (int t = 0; t < a.ntap; t++) {
    int64_t i = lo + t;
    if (i >= 0 && i < a.n1) acc = fma(w[t], __ldg(src + i), acc);
  }
  tA[r * a.ne + e] = acc;
}

// pass B: g2[e_lo+ey][e_lo+ex] = sum_t rw[e_lo+ey][t] tA[rlo + t][ex]
__global__ void k_restrict_y(const double *__restrict__ tA, double *__restrict__ g2, RestrictArgs a) {
  int64_t ex = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t ey = blockIdx.y;
  if (ex >= a.ne) return;
  int64_t jp = a.e_lo + ey;
  const int32_t lo = a.rlo[jp];
  const double *w = a.rw + jp * a.ntap;
  double acc = 0.0;
  for (int t = 0; t < a.ntap; t++) {
    int64_t r = lo + t;
    if (r >= 0 && r < a.n1) acc = fma(w[t], __ldg(tA + r * a.ne + ex), acc);
  }
  g2[jp * a.row2 + a.e_lo + ex] = acc;
}

// prolongation pass B^T: t2[r][ex] = sum_t tw[r][t] q2[tlo[r] + t][e_lo + ex]
__global__ void k_prolong_y(const double *__restrict__ q2, double *__restrict__ t2, RestrictArgs a) {
  int64_t ex = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t r = blockIdx.y;
  if (ex >= a.ne) return;
  const int32_t lo = a.tlo[r];
  const double *w = a.tw + r * a.ntt;
  double acc = 0.0;
  for (int t = 0; t < a.ntt; t++) {
    int64_t jp = lo + t;
    if (jp >= 0 && jp < a.n2) acc = fma(w[t], __ldg(q2 + jp * a.row2 + a.e_lo + ex), acc);
  }
  t2[r * a.ne + ex] = acc;
}

// prolongation pass A^T: q1[r][i] += sum_t tw[i][t] t2[r][tlo[i] + t - e_lo]
__global__ void k_prolong_x(const double *__restrict__ t2, double *__restrict__ q1, RestrictArgs a) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t r = blockIdx.y;
  if (i >= a.n1) return;
  const int32_t lo = a.tlo[i];
  const double *w = a.tw + i * a.ntt;
  const double *src = t2 + r * a.ne;
  double acc = 0.0;
  for (int t = 0; t < a.ntt; t++) {
    int64_t e = lo + t - a.e_lo;
    if (e >= 0 && e < a.ne) acc = fma(w[t], __ldg(src + e), acc);
  }
  q1[r * a.row1 + i] += acc;
}

// ---- integer-ratio restriction / prolongation (h_FH = M h_NH, FH node i' on NH node M i' - j): one tap vector
// w[q] = psi_FH(2 q / (W M)), |q| <= QH, for every output.  Each thread keeps Q (restriction) or M
// (prolongation) consecutive outputs in registers and streams the union of their inputs once.
#define VP_MAXTAP 192
struct TapArgs {
  double w[VP_MAXTAP];  // w[q + QH]
  int QH;
  int64_t j;
};

// pass A: tA[r][e] = sum_q w[q] g1[r][M (e_lo + e) - j + q]; the NH row segment is staged in shared memory
// with one pad word every M*Q entries, so the 32 lanes' windows (M*Q apart) start in distinct bank slots
template <int M, int Q>
__global__ void __launch_bounds__(128) k_restrict_x_int(const double *__restrict__ g1, double *__restrict__ tA,
                                                        RestrictArgs a, TapArgs tp) {
  extern __shared__ double s[];
  constexpr int SKEW = M * Q;
  const int64_t r = blockIdx.y;
  const int64_t e0 = (int64_t)blockIdx.x * 128 * Q;
  const int NT = 2 * tp.QH + 1;
  const int span = M * (128 * Q - 1) + NT;
  const int64_t i0 = M * (a.e_lo + e0) - tp.j - tp.QH;
  const double *src = g1 + r * a.row1;
  // asynchronous copy (cp.async, 8 B per element): every element of the span in flight at once (the synchronous
  // loop left the kernel latency-bound at ~3.4 TB/s)
  for (int idx = threadIdx.x; idx < span; idx += 128) {
    const int64_t gi = i0 + idx;
    if (gi >= 0 && gi < a.n1) __pipeline_memcpy_async(s + idx + idx / SKEW, src + gi, sizeof(double));
    else s[idx + idx / SKEW] = 0.0;
  }
  __pipeline_commit();
  __pipeline_wait_prior(0);
  __syncthreads();
  const int t = threadIdx.x;
  const double *sb = s + (SKEW + 1) * t;
  double acc[Q];
#pragma unroll
  for (int k = 0; k < Q; k++) acc[k] = 0.0;
  const int nin = M * (Q - 1) + NT;
  for (int ii = 0; ii < nin; ii++) {
    const double x = sb[ii + ii / SKEW];
#pragma unroll
    for (int k = 0; k < Q; k++) {
      const int q = ii - M * k;
      if (q >= 0 && q < NT) acc[k] = fma(tp.w[q], x, acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < Q; k++) {
    const int64_t e = e0 + Q * t + k;
    if (e < a.ne) tA[r * a.ne + e] = acc[k];
  }
}

// pass A with compile-time tap count (QHC = QH): fully unrolled, every weight a static kernel-parameter
// (constant-bank) operand of its DFMA, every shared-memory read a static offset
template <int M, int Q, int QHC>
__global__ void __launch_bounds__(128) k_restrict_x_fix(const double *__restrict__ g1, double *__restrict__ tA,
                                                        RestrictArgs a, TapArgs tp) {
  extern __shared__ double s[];
  constexpr int SKEW = M * Q, NT = 2 * QHC + 1, NIN = M * (Q - 1) + NT;
  const int64_t r = blockIdx.y;
  const int64_t e0 = (int64_t)blockIdx.x * 128 * Q;
  const int span = M * (128 * Q - 1) + NT;
  const int64_t i0 = M * (a.e_lo + e0) - tp.j - QHC;
  const double *src = g1 + r * a.row1;
  // asynchronous copy (cp.async, 8 B per element): every element of the span in flight at once (the synchronous
  // loop left the kernel latency-bound at ~3.4 TB/s)
  for (int idx = threadIdx.x; idx < span; idx += 128) {
    const int64_t gi = i0 + idx;
    if (gi >= 0 && gi < a.n1) __pipeline_memcpy_async(s + idx + idx / SKEW, src + gi, sizeof(double));
    else s[idx + idx / SKEW] = 0.0;
  }
  __pipeline_commit();
  __pipeline_wait_prior(0);
  __syncthreads();
  const int t = threadIdx.x;
  const double *sb = s + (SKEW + 1) * t;
  double acc[Q];
#pragma unroll
  for (int k = 0; k < Q; k++) acc[k] = 0.0;
#pragma unroll
  for (int ii = 0; ii < NIN; ii++) {
    const double x = sb[ii + ii / SKEW];
#pragma unroll
    for (int k = 0; k < Q; k++) {
      const int q = ii - M * k;
      if (q >= 0 && q < NT) acc[k] = fma(tp.w[q], x, acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < Q; k++) {
    const int64_t e = e0 + Q * t + k;
    if (e < a.ne) tA[r * a.ne + e] = acc[k];
  }
}

// pass B: g2[e_lo + ey][e_lo + ex] = sum_q w[q] tA[M (e_lo + ey) - j + q][ex] (coalesced along ex)
template <int M, int Q>
__global__ void __launch_bounds__(128) k_restrict_y_int(const double *__restrict__ tA, double *__restrict__ g2,
                                                        RestrictArgs a, TapArgs tp) {
  const int64_t ex = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int64_t ey0 = (int64_t)blockIdx.y * Q;
  if (ex >= a.ne) return;
  const int NT = 2 * tp.QH + 1;
  const int nin = M * (Q - 1) + NT;
  const int64_t r0 = M * (a.e_lo + ey0) - tp.j - tp.QH;
  double acc[Q];
#pragma unroll
  for (int k = 0; k < Q; k++) acc[k] = 0.0;
  for (int ii = 0; ii < nin; ii++) {
    const int64_t r = r0 + ii;
    const double x = (r >= 0 && r < a.n1) ? __ldg(tA + r * a.ne + ex) : 0.0;
#pragma unroll
    for (int k = 0; k < Q; k++) {
      const int q = ii - M * k;
      if (q >= 0 && q < NT) acc[k] = fma(tp.w[q], x, acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < Q; k++) {
    const int64_t ey = ey0 + k;
    if (ey < a.ne) g2[(a.e_lo + ey) * a.row2 + a.e_lo + ex] = acc[k];
  }
}

// pass B with compile-time taps (QHC) and Q outputs per thread: the tap loop is fully unrolled (no per-tap bounds
// tests, the weights are constant-bank operands); config 5: the runtime form ran at 80% issue
template <int M, int Q, int QHC>
__global__ void __launch_bounds__(128) k_restrict_y_fix(const double *__restrict__ tA, double *__restrict__ g2,
                                                        RestrictArgs a, TapArgs tp) {
  const int64_t ex = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int64_t ey0 = (int64_t)blockIdx.y * Q;
  if (ex >= a.ne) return;
  constexpr int NT = 2 * QHC + 1, NIN = M * (Q - 1) + NT;
  const int64_t r0 = M * (a.e_lo + ey0) - tp.j - QHC;
  double acc[Q];
#pragma unroll
  for (int k = 0; k < Q; k++) acc[k] = 0.0;
#pragma unroll
  for (int ii = 0; ii < NIN; ii++) {
    const int64_t r = r0 + ii;
    const double x = (r >= 0 && r < a.n1) ? __ldg(tA + r * a.ne + ex) : 0.0;
#pragma unroll
    for (int k = 0; k < Q; k++) {
      const int q = ii - M * k;
      if (q >= 0 && q < NT) acc[k] = fma(tp.w[q], x, acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < Q; k++) {
    const int64_t ey = ey0 + k;
    if (ey < a.ne) g2[(a.e_lo + ey) * a.row2 + a.e_lo + ex] = acc[k];
  }
}

// prolongation pass B^T: t2[r][ex] = sum_{i'} w[r + j - M i'] q2[i'][e_lo + ex], i' in the effective range;
// a thread owns the M rows r = M c + k - j (k = 0..M-1) sharing the FH rows i' = c + d
template <int M>
__global__ void __launch_bounds__(128) k_prolong_y_int(const double *__restrict__ q2, double *__restrict__ t2,
                                                       RestrictArgs a, TapArgs tp, int64_t c_lo) {
  const int64_t ex = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int64_t c = c_lo + blockIdx.y;
  if (ex >= a.ne) return;
  const int QH = tp.QH;
  const int dlo = -(QH / M), dhi = (M - 1 + QH) / M;
  double acc[M];
#pragma unroll
  for (int k = 0; k < M; k++) acc[k] = 0.0;
  for (int d = dlo; d <= dhi; d++) {
    const int64_t ip = c + d;
    if (ip < a.e_lo || ip >= a.e_lo + a.ne) continue;
    const double x = __ldg(q2 + ip * a.row2 + a.e_lo + ex);
#pragma unroll
    for (int k = 0; k < M; k++) {
      const int q = k - M * d;
      if (q >= -QH && q <= QH) acc[k] = fma(tp.w[q + QH], x, acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < M; k++) {
    const int64_t r = M * c + k - tp.j;
    if (r >= 0 && r < a.n1) t2[r * a.ne + ex] = acc[k];
  }
}

// prolongation pass A^T: q1[r][i] += sum_{i'} w[i + j - M i'] t2[r][i' - e_lo]; a thread owns the M
// columns i = M c + k - j, the warp reads consecutive i' (coalesced)
template <int M>
__global__ void __launch_bounds__(128) k_prolong_x_int(const double *__restrict__ t2, double *__restrict__ q1,
                                                       RestrictArgs a, TapArgs tp, int64_t c_lo, int64_t nc) {
  const int64_t cc = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int64_t r = blockIdx.y;
  if (cc >= nc) return;
  const int64_t c = c_lo + cc;
  const int QH = tp.QH;
  const int dlo = -(QH / M), dhi = (M - 1 + QH) / M;
  const double *src = t2 + r * a.ne - a.e_lo;
  double acc[M];
#pragma unroll
  for (int k = 0; k < M; k++) acc[k] = 0.0;
  for (int d = dlo; d <= dhi; d++) {
    const int64_t ip = c + d;
    if (ip < a.e_lo || ip >= a.e_lo + a.ne) continue;
    const double x = __ldg(src + ip);
#pragma unroll
    for (int k = 0; k < M; k++) {
      const int q = k - M * d;
      if (q >= -QH && q <= QH) acc[k] = fma(tp.w[q + QH], x, acc[k]);
    }
  }
  double *dst = q1 + r * a.row1;
#pragma unroll
  for (int k = 0; k < M; k++) {
    const int64_t i = M * c + k - tp.j;
    if (i >= 0 && i < a.n1) dst[i] += acc[k];
  }
}

// prolongation passes with a compile-time tap count (QHC = QH): the d loop and every weight index are static,
// so the weights are constant-bank DFMA operands (the runtime-QH forms above are issue-bound on the indexed
// parameter loads; config 5: k_prolong_x_int 2.4 ms at 86% issue)
template <int M, int QHC>
__global__ void __launch_bounds__(128) k_prolong_y_fix(const double *__restrict__ q2, double *__restrict__ t2,
                                                       RestrictArgs a, TapArgs tp, int64_t c_lo) {
  const int64_t ex = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int64_t c = c_lo + blockIdx.y;
  if (ex >= a.ne) return;
  constexpr int DLO = -(QHC / M), DHI = (M - 1 + QHC) / M;
  double acc[M];
#pragma unroll
  for (int k = 0; k < M; k++) acc[k] = 0.0;
#pragma unroll
  for (int d = DLO; d <= DHI; d++) {
    const int64_t ip = c + d;
    const double x = (ip >= a.e_lo && ip < a.e_lo + a.ne) ? __ldg(q2 + ip * a.row2 + a.e_lo + ex) : 0.0;
#pragma unroll
    for (int k = 0; k < M; k++) {
      const int q = k - M * d;
      if (q >= -QHC && q <= QHC) acc[k] = fma(tp.w[q + QHC], x, acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < M; k++) {
    const int64_t r = M * c + k - tp.j;
    if (r >= 0 && r < a.n1) t2[r * a.ne + ex] = acc[k];
  }
}

template <int M, int QHC>
__global__ void __launch_bounds__(128) k_prolong_x_fix(const double *__restrict__ t2, double *__restrict__ q1,
                                                       RestrictArgs a, TapArgs tp, int64_t c_lo, int64_t nc) {
  const int64_t cc = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int64_t r = blockIdx.y;
  if (cc >= nc) return;
  const int64_t c = c_lo + cc;
  constexpr int DLO = -(QHC / M), DHI = (M - 1 + QHC) / M;
  const double *src = t2 + r * a.ne - a.e_lo;
  double acc[M];
#pragma unroll
  for (int k = 0; k < M; k++) acc[k] = 0.0;
#pragma unroll
  for (int d = DLO; d <= DHI; d++) {
    const int64_t ip = c + d;
    const double x = (ip >= a.e_lo && ip < a.e_lo + a.ne) ? __ldg(src + ip) : 0.0;
#pragma unroll
    for (int k = 0; k < M; k++) {
      const int q = k - M * d;
      if (q >= -QHC && q <= QHC) acc[k] = fma(tp.w[q + QHC], x, acc[k]);
    }
  }
  double *dst = q1 + r * a.row1;
#pragma unroll
  for (int k = 0; k < M; k++) {
    const int64_t i = M * c + k - tp.j;
    if (i >= 0 && i < a.n1) dst[i] += acc[k];
  }
}

static TapArgs tap_args(vp_plan_s *P) {
  TapArgs t;
  memset(&t, 0, sizeof(t));
  t.QH = P->tap_qh;
  t.j = P->fh_shift;
  for (int q = 0; q < 2 * P->tap_qh + 1; q++) t.w[q] = P->tap_w[q];
  return t;
}

template <int M>
static void launch_restrict_int(vp_plan_s *P, const RestrictArgs &a, const TapArgs &tp) {
  constexpr int Q = 4;
  const int span = M * (128 * Q - 1) + 2 * tp.QH + 1;
  const size_t sm = sizeof(double) * (size_t)(span + span / (M * Q) + 2);
  vp_smem_attr((const void *)k_restrict_x_int<M, Q>, 96 * 1024);
  dim3 gA((unsigned)((a.ne + 128 * Q - 1) / (128 * Q)), (unsigned)a.n1);
  bool fixed = false;
  // compile-time taps: 8 outputs per thread (84 shared loads for 8 outputs instead of 64 for 4; the kernel is
  // bound by shared-memory issue, mio_throttle 36% at 4 outputs)
  constexpr int QF = 8;
  const int spanf = M * (128 * QF - 1) + 2 * tp.QH + 1;
  const size_t smf = sizeof(double) * (size_t)(spanf + spanf / (M * QF) + 2);
  dim3 gF((unsigned)((a.ne + 128 * QF - 1) / (128 * QF)), (unsigned)a.n1);
#define VP_RFIX(QHV)                                                                                   \
  if (tp.QH == QHV) {                                                                                  \
    vp_smem_attr((const void *)k_restrict_x_fix<M, QF, QHV>, 96 * 1024);                             \
    k_restrict_x_fix<M, QF, QHV><<<gF, 128, smf, P->stream>>>(P->nh.data, P->scratch, a, tp);         \
    fixed = true;                                                                                      \
  }
  if (M == 5) {  // the ratio delta2/delta1 = 32 gives m = 5 on every config; w = 9, 10, 11 (tol 1e-8 .. 1e-10)
    VP_RFIX(22) else VP_RFIX(24) else VP_RFIX(27)
  }
#undef VP_RFIX
  if (!fixed) k_restrict_x_int<M, Q><<<gA, 128, sm, P->stream>>>(P->nh.data, P->scratch, a, tp);
  VP_CHECK_LAUNCH();
  bool yfix = false;
  if (M == 5) {
    constexpr int QY = 8;
    dim3 gY((unsigned)((a.ne + 127) / 128), (unsigned)((a.ne + QY - 1) / QY));
    if (tp.QH == 22) { k_restrict_y_fix<M, QY, 22><<<gY, 128, 0, P->stream>>>(P->scratch, P->fh.data, a, tp); yfix = true; }
    else if (tp.QH == 24) { k_restrict_y_fix<M, QY, 24><<<gY, 128, 0, P->stream>>>(P->scratch, P->fh.data, a, tp); yfix = true; }
    else if (tp.QH == 27) { k_restrict_y_fix<M, QY, 27><<<gY, 128, 0, P->stream>>>(P->scratch, P->fh.data, a, tp); yfix = true; }
  }
  if (!yfix) {
    dim3 gB((unsigned)((a.ne + 127) / 128), (unsigned)((a.ne + Q - 1) / Q));
    k_restrict_y_int<M, Q><<<gB, 128, 0, P->stream>>>(P->scratch, P->fh.data, a, tp);
  }
  VP_CHECK_LAUNCH();
  P->n_kernels += 2;
}

template <int M>
static void launch_prolong_int(vp_plan_s *P, const RestrictArgs &a, const TapArgs &tp, int pass) {
  // NH index i = M c + k - j covers [0, n1) for c in [c_lo, c_hi]
  const int64_t c_lo = (tp.j >= 0) ? tp.j / M : -((-tp.j + M - 1) / M);
  const int64_t c_hi = (a.n1 - 1 + tp.j) / M;
  const int64_t nc = c_hi - c_lo + 1;
  if (pass & 1) {
    dim3 gB((unsigned)((a.ne + 127) / 128), (unsigned)nc);
    bool fixed = false;
    if (M == 5) {  // w = 9, 10, 11 (tol 1e-8 .. 1e-10) with m = 5: compile-time taps
      if (tp.QH == 22) { k_prolong_y_fix<M, 22><<<gB, 128, 0, P->stream>>>(P->fh.data, P->scratch, a, tp, c_lo); fixed = true; }
      else if (tp.QH == 24) { k_prolong_y_fix<M, 24><<<gB, 128, 0, P->stream>>>(P->fh.data, P->scratch, a, tp, c_lo); fixed = true; }
      else if (tp.QH == 27) { k_prolong_y_fix<M, 27><<<gB, 128, 0, P->stream>>>(P->fh.data, P->scratch, a, tp, c_lo); fixed = true; }
    }
    if (!fixed) k_prolong_y_int<M><<<gB, 128, 0, P->stream>>>(P->fh.data, P->scratch, a, tp, c_lo);
    VP_CHECK_LAUNCH();
    P->n_kernels++;
  }
  if (!(pass & 2)) return;
  dim3 gA((unsigned)((nc + 127) / 128), (unsigned)a.n1);
  bool fixed = false;
  if (M == 5) {
    if (tp.QH == 22) { k_prolong_x_fix<M, 22><<<gA, 128, 0, P->stream>>>(P->scratch, P->nh.data, a, tp, c_lo, nc); fixed = true; }
    else if (tp.QH == 24) { k_prolong_x_fix<M, 24><<<gA, 128, 0, P->stream>>>(P->scratch, P->nh.data, a, tp, c_lo, nc); fixed = true; }
    else if (tp.QH == 27) { k_prolong_x_fix<M, 27><<<gA, 128, 0, P->stream>>>(P->scratch, P->nh.data, a, tp, c_lo, nc); fixed = true; }
  }
  if (!fixed) k_prolong_x_int<M><<<gA, 128, 0, P->stream>>>(P->scratch, P->nh.data, a, tp, c_lo, nc);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

static RestrictArgs restrict_args(vp_plan_s *P) {
  RestrictArgs a;
  a.rlo = P->r_lo; a.rw = P->r_w; a.ntap = P->r_ntap;
  a.tlo = P->t_lo; a.tw = P->t_w; a.ntt = P->t_ntap;
  a.e_lo = P->e_lo; a.ne = P->e_n;
  a.n1 = P->nh.nf; a.row1 = P->nh.row; a.n2 = P->fh.nf; a.row2 = P->fh.row;
  return a;
}

void vp_launch_restrict(vp_plan_s *P) {
  RestrictArgs a = restrict_args(P);
  if (P->tap_qh > 0) {
    TapArgs tp = tap_args(P);
    switch (P->fh_ratio) {
      case 2: launch_restrict_int<2>(P, a, tp); return;
      case 3: launch_restrict_int<3>(P, a, tp); return;
      case 4: launch_restrict_int<4>(P, a, tp); return;
      case 5: launch_restrict_int<5>(P, a, tp); return;
      case 6: launch_restrict_int<6>(P, a, tp); return;
      case 7: launch_restrict_int<7>(P, a, tp); return;
      case 8: launch_restrict_int<8>(P, a, tp); return;
      default: break;
    }
  }
  dim3 bA((unsigned)((a.ne + 127) / 128), (unsigned)a.n1);
  k_restrict_x<<<bA, 128, 0, P->stream>>>(P->nh.data, P->scratch, a);
  VP_CHECK_LAUNCH();
  dim3 bB((unsigned)((a.ne + 127) / 128), (unsigned)a.ne);
  k_restrict_y<<<bB, 128, 0, P->stream>>>(P->scratch, P->fh.data, a);
  VP_CHECK_LAUNCH();
  P->n_kernels += 2;
}

// pass: 1 = FH rows -> t2 (pass B^T, reads the FH grid), 2 = t2 -> NH grid (pass A^T), 3 = both
void vp_launch_prolong(vp_plan_s *P, int pass) {
  RestrictArgs a = restrict_args(P);
  if (P->tap_qh > 0) {
    TapArgs tp = tap_args(P);
    switch (P->fh_ratio) {
      case 2: launch_prolong_int<2>(P, a, tp, pass); return;
      case 3: launch_prolong_int<3>(P, a, tp, pass); return;
      case 4: launch_prolong_int<4>(P, a, tp, pass); return;
      case 5: launch_prolong_int<5>(P, a, tp, pass); return;
      case 6: launch_prolong_int<6>(P, a, tp, pass); return;
      case 7: launch_prolong_int<7>(P, a, tp, pass); return;
      case 8: launch_prolong_int<8>(P, a, tp, pass); return;
      default: break;
    }
  }
  if (pass & 1) {
    dim3 bB((unsigned)((a.ne + 127) / 128), (unsigned)a.n1);
    k_prolong_y<<<bB, 128, 0, P->stream>>>(P->fh.data, P->scratch, a);
    VP_CHECK_LAUNCH();
    P->n_kernels++;
  }
  if (pass & 2) {
    dim3 bA((unsigned)((a.n1 + 127) / 128), (unsigned)a.n1);
    k_prolong_x<<<bA, 128, 0, P->stream>>>(P->scratch, P->nh.data, a);
    VP_CHECK_LAUNCH();
    P->n_kernels++;
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
  k_multiply<<<blocks, 256, 0, P->stream>>>(G.cdata, G.nf, G.crow, G.nmode / 2, G.deconv, dk, G.mult_scale, G.kind,
                                            G.delta_a, G.delta_b);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

// ---------------------------------------------------------------------------------------------
// interpolation (NH grid, which also carries the prolongated FH field) + local part + scatter.
// One CTA of 256 threads per work item (tile_x, tile_y, t0, t1): the (TSI+W+3)^2 grid window of a
// TSI x TSI tile is staged once in shared memory (coalesced rows), then every thread interpolates
// targets t0 + tid, t0 + tid + 256, ... from shared memory.  Targets were ordered at plan time
// rank-major over the bank slot of their footprint origin (vp_build_interp_order), so the 32
// row-reads of a warp spread over the 16 8-byte bank slots.
template <int W, int D>
__global__ void __launch_bounds__(256, 4) k_interp_local(const int4 *__restrict__ items, int TSI,
                                                      const double *__restrict__ tx, const double *__restrict__ ty,
                                                      const int32_t *__restrict__ tperm, GridArgs g, int do_hist,
                                                      const double *__restrict__ f, const double *__restrict__ lalpha,
                                                      const int32_t *__restrict__ lnode, int do_local,
                                                      const int32_t *__restrict__ lptr,
                                                      const double *__restrict__ vL_tri,
                                                      const double *__restrict__ vL_st, double *__restrict__ out) {
  extern __shared__ double tile[];
  const int nw = TSI + W + 3;
  const int4 it = items[blockIdx.x];
  const int64_t ox = (int64_t)it.x * TSI - (W / 2 + 1), oy = (int64_t)it.y * TSI - (W / 2 + 1);
  if (do_hist) {
    const bool interior = ox >= 0 && oy >= 0 && ox + nw <= g.nfx && oy + nw <= g.nfy;
    if (interior) {  // common case: flat copy with 4 independent loads in flight per thread
      const int ncell = nw * nw;
      const double *base = g.data + oy * g.row + ox;
      for (int i0 = threadIdx.x; i0 < ncell; i0 += 4 * 256) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int i = i0 + u * 256;
          if (i < ncell) {
            const int r = i / nw;
            v[u] = __ldg(base + (int64_t)r * g.row + (i - r * nw));
          }
        }
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (i0 + u * 256 < ncell) tile[i0 + u * 256] = v[u];
      }
    } else {  // window wraps around the periodic grid
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      for (int r = warp; r < nw; r += 8) {
        const double *src = g.data + wrapi(oy + r, g.nfy) * g.row;
        for (int c = lane; c < nw; c += 32) tile[r * nw + c] = __ldg(src + wrapi(ox + c, g.nfx));
      }
    }
    __syncthreads();
  }
  // software pipeline: the next target's coordinates are loaded while the current one is interpolated, and the
  // current target's local-part value is fetched before its w x w shared-memory sweep (long-latency loads hidden)
  int t = it.z + threadIdx.x;
  double xn = 0.0, yn = 0.0;
  if (t < it.w) {
    xn = tx[t];
    yn = ty[t];
  }
  for (; t < it.w; t += blockDim.x) {
    const double xc = xn, yc = yn;
    const int tn = t + blockDim.x;
    if (tn < it.w) {
      xn = tx[tn];
      yn = ty[tn];
    }
    const int32_t dst = tperm[t];
    double vl = 0.0;
    if (do_local) {
      const int32_t nd = lnode[t];
      const int32_t sp = lptr[t];
      if (sp >= 0) {  // least-squares stencil, applied by k_local_stencil
        if (nd >= 0) vl = lalpha[t] * __ldg(f + nd);
        vl += __ldcs(vL_st + sp);
      } else if (vL_tri) {  // own-triangle cubic fit, evaluated per node by k_tri_local
        vl = __ldg(vL_tri + nd);
      } else if (nd >= 0) {
        vl = lalpha[t] * __ldg(f + nd);
      }
    }
    double v = 0.0;
    if (do_hist) {
      if constexpr (W <= 0) {  // (measured slower at config 5: 3 CTAs/SM to avoid spills, 7.9 vs 7.2 ms)
      // x taps by even/odd Horner pairs (half the DFMA of W chains); the y taps of rows b and W - 1 - b come from
      // one pair evaluation inside the row loop, so only the W x taps stay live (wider kernels spill with this
      // form and keep the W separate chains below)
      double wx[W], ty;
      const int lx = (int)(es_horner<W, D>(gcoord(xc, g.ox, g.inv_h), wx) - ox);
      const int ly = (int)(es_arg<W>(gcoord(yc, g.oy, g.inv_h), &ty) - oy);
      const double uy = ty * ty;
      const double *rp = tile + ly * nw + lx;
#pragma unroll
      for (int b = 0; b < (W + 1) / 2; b++) {
        double wk, wm;
        es_pair<W, D>(b, ty, uy, &wk, &wm);
        double racc = 0.0;
#pragma unroll
        for (int a = 0; a < W; a++) racc = fma(wx[a], rp[b * nw + a], racc);
        v = fma(wk, racc, v);
        if (W - 1 - b != b) {
          double racc2 = 0.0;
#pragma unroll
          for (int a = 0; a < W; a++) racc2 = fma(wx[a], rp[(W - 1 - b) * nw + a], racc2);
          v = fma(wm, racc2, v);
        }
      }
      } else {
      double wx[W], wy[W];
      const int lx = (int)(es_horner_chains<W, D>(gcoord(xc, g.ox, g.inv_h), wx) - ox);
      const int ly = (int)(es_horner_chains<W, D>(gcoord(yc, g.oy, g.inv_h), wy) - oy);
      const double *rp = tile + ly * nw + lx;
#pragma unroll
      for (int b = 0; b < W; b++) {
        double racc = 0.0;
#pragma unroll
        for (int a = 0; a < W; a++) racc = fma(wx[a], rp[b * nw + a], racc);
        v = fma(wy[b], racc, v);
      }
      }
    }
    out[dst] = v + vl;
  }
}

// TRIANGLE-mode local part for every node of a qualifying triangle (one thread per triangle, 12 coalesced
// f values, reference Hessian operators in shared memory, read in lockstep -> broadcast):
//   V_L(node k) = delta f_k + (delta^2 / 2) Lap f(node k),  Lap f = M11 f_11 + 2 M12 f_12 + M22 f_22
// with f_ab the second reference derivatives of the least-squares cubic on the triangle's p nodes.
template <int PP>  // PP > 0: compile-time rule size (registers); 0: runtime p
__global__ void __launch_bounds__(128) k_tri_local(const double *__restrict__ f, const int8_t *__restrict__ tri_ok,
                                                   const double *__restrict__ tri_M,
                                                   const double *__restrict__ tri_H, int p_rt, int64_t M, double c1,
                                                   double c2, double *__restrict__ vL) {
  __shared__ double H[3 * VP_TRI_MAXP * VP_TRI_MAXP];
  const int p = PP > 0 ? PP : p_rt;
  for (int i = threadIdx.x; i < 3 * p * p; i += blockDim.x) H[i] = tri_H[i];
  __syncthreads();
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= M || !tri_ok[m]) return;
  const double m11 = tri_M[3 * m], m12x2 = 2.0 * tri_M[3 * m + 1], m22 = tri_M[3 * m + 2];
  double fb[PP > 0 ? PP : VP_TRI_MAXP];
#pragma unroll
  for (int j = 0; j < p; j++) fb[j] = __ldcs(f + m * p + j);
#pragma unroll
  for (int k = 0; k < p; k++) {
    const double *h0 = H + k * p, *h1 = h0 + p * p, *h2 = h1 + p * p;
    double lap = 0.0;
#pragma unroll
    for (int j = 0; j < p; j++) lap = fma(fma(m11, h0[j], fma(m12x2, h1[j], m22 * h2[j])), fb[j], lap);
    vL[m * p + k] = fma(c2, lap, c1 * fb[k]);
  }
}

// p = 12 (the 12-point rule): reference Hessian operators in the constant bank (uniform, static offsets ->
// DFMA constant operands, no shared-memory traffic), f and V_L staged through shared memory so that the
// CTA's 128 x 12 values move as coalesced rows
// Operators depend on the plan's reference rule, so distinct plans may need distinct tables: VP_TRIH_SLOTS
// constant-bank slots per device, each written once (at plan time, synchronously) and never overwritten, so a
// kernel queued by one plan can never see another plan's operators.  A plan whose rule finds no free slot
// uses the shared-memory kernel k_tri_local<12>.
#define VP_TRIH_SLOTS 4
__constant__ double c_triH[VP_TRIH_SLOTS][3 * 12 * 12];

int vp_acquire_trih_slot(const double *hop432) {
  static std::mutex mu;
  static std::map<int, std::vector<std::vector<double>>> slots;  // device -> uploaded tables
  const int dev = vp_current_device();
  std::lock_guard<std::mutex> lk(mu);
  std::vector<std::vector<double>> &v = slots[dev];
  for (size_t i = 0; i < v.size(); i++)
    if (memcmp(v[i].data(), hop432, sizeof(double) * 432) == 0) return (int)i;
  if (v.size() >= VP_TRIH_SLOTS) return -1;
  VP_CUDA(cudaMemcpyToSymbol(c_triH, hop432, sizeof(double) * 432, sizeof(double) * 432 * v.size()));
  v.emplace_back(hop432, hop432 + 432);
  return (int)v.size() - 1;
}

template <int SLOT>
__global__ void __launch_bounds__(128) k_tri_local12(const double *__restrict__ f, const int8_t *__restrict__ tri_ok,
                                                     const double *__restrict__ tri_M, int64_t M, double c1, double c2,
                                                     double *__restrict__ vL) {
  __shared__ double sf[128 * 12 + 1];
  const int64_t m0 = (int64_t)blockIdx.x * 128;
  const int nt = (int)((M - m0) < 128 ? (M - m0) : 128);
  for (int i = threadIdx.x; i < nt * 12; i += 128) sf[i] = __ldcs(f + m0 * 12 + i);
  __syncthreads();
  const int t = threadIdx.x;
  const int64_t m = m0 + t;
  if (t < nt && tri_ok[m]) {
    const double m11 = tri_M[3 * m], m12x2 = 2.0 * tri_M[3 * m + 1], m22 = tri_M[3 * m + 2];
    double fb[12], out[12];
#pragma unroll
    for (int j = 0; j < 12; j++) fb[j] = sf[t * 12 + j];  // stride 12 doubles: 4-way bank spread, once per value
#pragma unroll
    for (int k = 0; k < 12; k++) {
      double lap = 0.0;
#pragma unroll
      for (int j = 0; j < 12; j++)
        lap = fma(fma(m11, c_triH[SLOT][k * 12 + j],
                      fma(m12x2, c_triH[SLOT][144 + k * 12 + j], m22 * c_triH[SLOT][288 + k * 12 + j])),
                  fb[j], lap);
      out[k] = fma(c2, lap, c1 * fb[k]);
    }
    // each thread overwrites only the 12 entries it read itself: no cross-thread hazard
#pragma unroll
    for (int k = 0; k < 12; k++) sf[t * 12 + k] = out[k];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nt * 12; i += 128)
    if (tri_ok[m0 + i / 12]) vL[m0 * 12 + i] = sf[i];
}

// KNN-stencil local part, one thread per stencil slot: vL_st[s] = sum_k w[k][s] f[idx[k][s]] (k-major layout:
// the warp streams consecutive slots, 12 B per entry, HBM-bound; f gathers hit L2)
__global__ void __launch_bounds__(256) k_local_stencil(const int32_t *__restrict__ lidx, const double *__restrict__ lw,
                                                       int K, int64_t S, const double *__restrict__ f,
                                                       double *__restrict__ vL_st) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= S) return;
  double acc = 0.0;
#pragma unroll 8
  for (int k = 0; k < K; k++) acc = fma(__ldcs(lw + k * S + s), __ldg(f + __ldcs(lidx + k * S + s)), acc);
  vL_st[s] = acc;
}

__global__ void k_invert_perm(const int32_t *__restrict__ perm, int64_t n, int32_t *__restrict__ inv) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) inv[perm[i]] = (int32_t)i;
}

__global__ void k_remap_idx(int32_t *__restrict__ idx, int64_t n, const int32_t *__restrict__ inv) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) idx[i] = inv[idx[i]];
}

// stencil node indices: user order -> spreading order (plan time)
void vp_remap_stencils(vp_plan_s *P) {
  if (P->n_stencil == 0 || P->K == 0) return;
  int32_t *inv = nullptr;
  VP_CUDA(cudaMallocAsync(&inv, sizeof(int32_t) * P->N, P->stream));
  k_invert_perm<<<(unsigned)((P->N + 255) / 256), 256, 0, P->stream>>>(P->sp.sperm, P->N, inv);
  VP_CHECK_LAUNCH();
  const int64_t ne = P->n_stencil * (int64_t)P->K;
  k_remap_idx<<<(unsigned)((ne + 255) / 256), 256, 0, P->stream>>>(P->lidx, ne, inv);
  VP_CHECK_LAUNCH();
  VP_CUDA(cudaFreeAsync(inv, P->stream));
}

__global__ void k_gather_f(const double *__restrict__ f, const int32_t *__restrict__ perm, int64_t n,
                           double *__restrict__ fs) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) fs[i] = __ldg(f + perm[i]);
}

void vp_launch_tri_local(vp_plan_s *P, const double *f) {
  if (P->n_stencil > 0 && P->st_vL) {
    // stencil entries index f in spreading order (P->fs, written by the spread of this eval; gathered here
    // when the history part is off)
    int parts = P->opts.parts ? P->opts.parts : VP_PART_ALL;
    if (!(parts & VP_PART_HISTORY)) {
      k_gather_f<<<(unsigned)((P->N + 255) / 256), 256, 0, P->stream>>>(f, P->sp.sperm, P->N, P->fs);
      VP_CHECK_LAUNCH();
      P->n_kernels++;
    }
    k_local_stencil<<<(unsigned)((P->n_stencil + 255) / 256), 256, 0, P->stream>>>(P->lidx, P->lw, P->K, P->n_stencil,
                                                                                   P->fs, P->st_vL);
    VP_CHECK_LAUNCH();
    P->n_kernels++;
  }
  if (!P->tri_vL || P->M == 0) return;
  const unsigned nb = (unsigned)((P->M + 127) / 128);
  if (P->p == 12 && P->trih_slot >= 0) {  // slot acquired at plan time (vp_build_local)
    switch (P->trih_slot) {
#define CASE(S)                                                                                                 \
  case S:                                                                                                       \
    k_tri_local12<S><<<nb, 128, 0, P->stream>>>(f, P->tri_ok, P->tri_M, P->M, P->delta1, P->tri_c2, P->tri_vL); \
    break;
      CASE(0) CASE(1) CASE(2) CASE(3)
#undef CASE
      default: throw VpError{VP_ERR_CUDA};
    }
  } else if (P->p == 12)
    k_tri_local<12><<<nb, 128, 0, P->stream>>>(f, P->tri_ok, P->tri_M, P->tri_H, 12, P->M, P->delta1, P->tri_c2,
                                               P->tri_vL);
  else
    k_tri_local<0><<<nb, 128, 0, P->stream>>>(f, P->tri_ok, P->tri_M, P->tri_H, P->p, P->M, P->delta1, P->tri_c2,
                                              P->tri_vL);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

template <int W>
static void launch_interp_w(vp_plan_s *P, const double *f, double *out) {
  constexpr int D = VP_HORNER_DEG(W);
  int parts = P->opts.parts ? P->opts.parts : VP_PART_ALL;
  if (P->n_items == 0) return;
  const int TSI = P->TSI, nw = TSI + W + 3;
  const int do_hist = (parts & VP_PART_HISTORY) ? 1 : 0;
  size_t sm = do_hist ? sizeof(double) * (size_t)nw * nw : 0;
  vp_smem_attr((const void *)k_interp_local<W, D>, sm);
  k_interp_local<W, D><<<(unsigned)P->n_items, 256, sm, P->stream>>>(
      P->items, TSI, P->tx, P->ty, P->tperm, grid_args(P->nh), do_hist, f, P->lalpha, P->lnode,
      (parts & VP_PART_LOCAL) ? 1 : 0, P->lptr, P->tri_vL, P->st_vL, out);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

// ---------------------------------------------------------------------------------------------
// plan-time: order the targets by (TSI-tile, rank within bank slot, bank slot) and cut the tiles into
// work items of <= VP_INTERP_CHUNK targets
#define VP_INTERP_CHUNK 16384  // targets per work item: dense tiles reload the grid window once per item
__global__ void k_interp_keys1(const double *__restrict__ xy, int64_t n, GridArgs g, int TSI, int W, int64_t ntx,
                               int64_t nty, uint64_t *__restrict__ keys, int32_t *__restrict__ idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double gx = gcoord(xy[2 * i], g.ox, g.inv_h), gy = gcoord(xy[2 * i + 1], g.oy, g.inv_h);
  int64_t tx = (int64_t)floor(gx / TSI), ty = (int64_t)floor(gy / TSI);
  tx = tx < 0 ? 0 : (tx >= ntx ? ntx - 1 : tx);
  ty = ty < 0 ? 0 : (ty >= nty ? nty - 1 : ty);
  const int nw = TSI + W + 3;
  int64_t lrow = (int64_t)ceil(gy - 0.5 * W) - (ty * TSI - (W / 2 + 1));
  int64_t lcol = (int64_t)ceil(gx - 0.5 * W) - (tx * TSI - (W / 2 + 1));
  const int res = (int)((((lrow * nw + lcol) % 16) + 16) % 16);
  keys[i] = ((uint64_t)(ty * ntx + tx) << 4) | (uint64_t)res;
  idx[i] = (int32_t)i;
}

#ifndef VP_INTERP_DEAL
#define VP_INTERP_DEAL 0
#endif
// Second key of the interpolation order.  A half-warp of k_interp_local reads 16 window words whose bank slots
// are the targets' slots.  0 (default): rank-major (tile, rank within slot, slot).  1 (tried, not kept): the n_t
// targets of a tile, sorted by slot (index j), dealt to the G = ceil(n_t / 16) half-warp groups like cards (group
// j mod G, place j div G), so that a group holds two targets of one slot only if that slot has more than G
// members.  Measured at config 5: bank-conflict wavefronts 2.43e8 -> 3.55e8, 7.26 -> 7.62 ms: in the dense tiles
// the same-slot neighbours of the rank-major order mostly sit in the same grid cell (nodes of one triangle), i.e.
// read the same address (a broadcast, no conflict), and dealing them apart pairs targets of different cells.
__global__ void k_interp_keys2(const uint64_t *__restrict__ k1, int64_t n, uint64_t *__restrict__ k2) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t key = k1[i];
#if VP_INTERP_DEAL
  const uint64_t tile = key >> 4;
  int64_t lo = 0, hi = i;
  while (lo < hi) {  // first index of this tile
    int64_t mid = (lo + hi) >> 1;
    if ((k1[mid] >> 4) < tile) lo = mid + 1; else hi = mid;
  }
  const int64_t t0 = lo;
  lo = i + 1, hi = n;
  while (lo < hi) {  // one past the last index of this tile
    int64_t mid = (lo + hi) >> 1;
    if ((k1[mid] >> 4) <= tile) lo = mid + 1; else hi = mid;
  }
  const int64_t nt = lo - t0, G = (nt + 15) / 16, j = i - t0;
  k2[i] = (tile << 24) | ((uint64_t)(j % G) << 4) | (uint64_t)(j / G);
#else
  int64_t lo = 0, hi = i;
  while (lo < hi) {  // first index of this (tile, slot) group
    int64_t mid = (lo + hi) >> 1;
    if (k1[mid] < key) lo = mid + 1; else hi = mid;
  }
  uint64_t rank = (uint64_t)(i - lo);
  if (rank > 0xFFFFF) rank = 0xFFFFF;
  k2[i] = ((key >> 4) << 24) | (rank << 4) | (key & 15);
#endif
}

void vp_build_interp_order_g(vp_plan_s *P, const double *xy, int64_t n, const GridArgs &g, double **otx,
                             double **oty, int32_t **otperm, int4 **oitems, int64_t *on_items);
void vp_build_interp_order(vp_plan_s *P, const double *xy, int64_t n) {
  vp_build_interp_order_g(P, xy, n, grid_args(P->nh), &P->tx, &P->ty, &P->tperm, &P->items, &P->n_items);
}

// targets (xy interleaved, n) of grid g ordered for k_interp_local: *tx, *ty, *tperm (sorted -> input index),
// work items.  (A (tile, triangle, node) order that coalesces the per-node V_L reads cost more bank
// conflicts than it saved: config 5 interp 9.7 -> 11.8 ms.)
void vp_build_interp_order_g(vp_plan_s *P, const double *xy, int64_t n, const GridArgs &g, double **otx, double **oty, int32_t **otperm, int4 **oitems, int64_t *on_items) {
  cudaStream_t s = P->stream;
  const int TSI = P->TSI;
  const int64_t ntx = (g.nfx + TSI - 1) / TSI, nty = (g.nfy + TSI - 1) / TSI;
  uint64_t *k1, *k1s, *k2, *k2s;
  int32_t *i1, *i1s, *i2s;
  VP_CUDA(cudaMallocAsync(&k1, 8 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&k1s, 8 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&k2, 8 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&k2s, 8 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&i1, 4 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&i1s, 4 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&i2s, 4 * (n + 1), s));
  unsigned nb = (unsigned)((n + 255) / 256);
  // (tile, triangle, node) order coalesces the per-node V_L reads but costs more shared-memory bank conflicts
  // than it saves (config 5: interp 9.7 -> 11.8 ms); off
  size_t tb = 0, tb2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, k1, k1s, i1, i1s, (int)n, 0, 64, s);
  cub::DeviceRadixSort::SortPairs(nullptr, tb2, k2, k2s, i1s, i2s, (int)n, 0, 64, s);
  void *tmp;
  VP_CUDA(cudaMallocAsync(&tmp, std::max(tb, tb2) + 16, s));
  const int tile_shift = 24;
  k_interp_keys1<<<nb, 256, 0, s>>>(xy, n, g, TSI, P->w, ntx, nty, k1, i1);
  VP_CHECK_LAUNCH();
  VP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k1, k1s, i1, i1s, (int)n, 0, 64, s));
  k_interp_keys2<<<nb, 256, 0, s>>>(k1s, n, k2);
  VP_CHECK_LAUNCH();
  VP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb2, k2, k2s, i1s, i2s, (int)n, 0, 64, s));
  *otx = vp_alloc<double>(P, n);
  *oty = vp_alloc<double>(P, n);
  *otperm = vp_alloc<int32_t>(P, n);
  k_gather_xy<<<nb, 256, 0, s>>>(xy, i2s, n, *otx, *oty, nullptr, *otperm);
  VP_CHECK_LAUNCH();
  std::vector<uint64_t> hk(n);
  VP_CUDA(cudaMemcpyAsync(hk.data(), k2s, 8 * n, cudaMemcpyDeviceToHost, s));
  VP_CUDA(cudaStreamSynchronize(s));
  std::vector<int4> items;
  for (int64_t i = 0; i < n;) {
    const uint64_t tile = hk[i] >> tile_shift;
    int64_t e = i;
    while (e < n && (hk[e] >> tile_shift) == tile) e++;
    for (int64_t c = i; c < e; c += VP_INTERP_CHUNK)
      items.push_back(make_int4((int)(tile % ntx), (int)(tile / ntx), (int)c, (int)std::min<int64_t>(e, c + VP_INTERP_CHUNK)));
    i = e;
  }
  *on_items = (int64_t)items.size();
  *oitems = vp_alloc<int4>(P, std::max<size_t>(items.size(), 1));
  if (!items.empty())
    VP_CUDA(cudaMemcpy(*oitems, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice));
  for (void *q : {(void *)k1, (void *)k1s, (void *)k2, (void *)k2s, (void *)i1, (void *)i1s, (void *)i2s, tmp})
    VP_CUDA(cudaFreeAsync(q, s));
}

// interpolation of the history part only (single-layer potential: the local part is applied separately)
template <int W>
static void launch_interp_hist_w(vp_plan_s *P, double *out) {
  constexpr int D = VP_HORNER_DEG(W);
  if (P->n_items == 0) return;
  const int TSI = P->TSI, nw = TSI + W + 3;
  const size_t sm = sizeof(double) * (size_t)nw * nw;
  vp_smem_attr((const void *)k_interp_local<W, D>, sm);
  k_interp_local<W, D><<<(unsigned)P->n_items, 256, sm, P->stream>>>(P->items, TSI, P->tx, P->ty, P->tperm,
                                                                     grid_args(P->nh), 1, nullptr, nullptr, nullptr,
                                                                     0, nullptr, nullptr, nullptr, out);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

void vp_launch_interp_hist(vp_plan_s *P, double *out) {
  switch (P->w) {
#define CASE(W) \
  case W: launch_interp_hist_w<W>(P, out); break;
    CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: throw VpError{VP_ERR_UNSUPPORTED};
  }
}

void vp_launch_interp_local(vp_plan_s *P, const double *f, double *out, bool local_kernels) {
  int parts_ = P->opts.parts ? P->opts.parts : VP_PART_ALL;
  if (local_kernels && (parts_ & VP_PART_LOCAL)) vp_launch_tri_local(P, f);
  switch (P->w) {
#define CASE(W) \
  case W: launch_interp_w<W>(P, f, out); break;
    CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: throw VpError{VP_ERR_UNSUPPORTED};
  }
}

// ---------------------------------------------------------------------------------------------
// plan-time: sort sources into row-rank batches and build the per-warp work items
__global__ void k_gather_src(const double *__restrict__ xy, const double *__restrict__ w, const int32_t *__restrict__ idx,
                             const int32_t *__restrict__ node_of, int64_t n, double *__restrict__ xs,
                             double *__restrict__ ys, double *__restrict__ ws, int32_t *__restrict__ perm) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t j = idx[i];
  xs[i] = xy[2 * (int64_t)j];
  ys[i] = xy[2 * (int64_t)j + 1];
  ws[i] = w[j];
  perm[i] = node_of ? node_of[j] : j;
}

// Sort n points (xy interleaved, in the frame of grid g) into the batch order of k_spread_nh.
// node_of (optional) maps a point to the user node whose f it carries.
void vp_build_spread_order(vp_plan_s *P, VpSpreadSet &S, const double *xy, const double *weights,
                           const int32_t *node_of, int64_t n, const GridArgs &g) {
  cudaStream_t s = P->stream;
  VpTiles &Tl = S.tiles;
  Tl.TS = P->opts.spread_tile > 0 ? P->opts.spread_tile : 32;
  Tl.ntx = (g.nfx + Tl.TS - 1) / Tl.TS;
  Tl.nty = (g.nfy + Tl.TS - 1) / Tl.TS;
  if (n == 0) {
    S.sx = vp_alloc<double>(P, 1); S.sy = vp_alloc<double>(P, 1); S.sw = vp_alloc<double>(P, 1);
    S.sperm = vp_alloc<int32_t>(P, 1); S.bstart = vp_alloc<int32_t>(P, 1);
    S.n_batches = 0; Tl.nsub = 0; Tl.sub = vp_alloc<int4>(P, 1);
    return;
  }
  uint64_t *k1, *k1s, *k2, *k2s;
  int32_t *i1, *i1s, *i2s, *head;
  VP_CUDA(cudaMallocAsync(&k1, 8 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&k1s, 8 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&k2, 8 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&k2s, 8 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&i1, 4 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&i1s, 4 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&i2s, 4 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&head, 4 * (n + 1), s));
  unsigned nb = (unsigned)((n + 255) / 256);
  k_spread_keys<<<nb, 256, 0, s>>>(xy, n, g, Tl.TS, P->w, Tl.ntx, Tl.nty, k1, i1);
  VP_CHECK_LAUNCH();
  size_t tb = 0, tb2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, k1, k1s, i1, i1s, (int)n, 0, 64, s);
  cub::DeviceRadixSort::SortPairs(nullptr, tb2, k2, k2s, i1s, i2s, (int)n, 0, 64, s);
  void *tmp;
  VP_CUDA(cudaMallocAsync(&tmp, std::max(tb, tb2) + 16, s));
  VP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k1, k1s, i1, i1s, (int)n, 0, 64, s));
  {
    // non-empty tile ranges
    k_tile_heads<<<nb, 256, 0, s>>>(k1s, n, head);
    VP_CHECK_LAUNCH();
    int32_t *tst, *d_nt;
    VP_CUDA(cudaMallocAsync(&tst, 4 * (n + 1), s));
    VP_CUDA(cudaMallocAsync(&d_nt, 4, s));
    size_t tb3 = 0;
    cub::CountingInputIterator<int32_t> cnt(0);
    cub::DeviceSelect::Flagged(nullptr, tb3, cnt, head, tst, d_nt, (int)n, s);
    void *tmp3;
    VP_CUDA(cudaMallocAsync(&tmp3, tb3 + 16, s));
    VP_CUDA(cub::DeviceSelect::Flagged(tmp3, tb3, cnt, head, tst, d_nt, (int)n, s));
    int32_t nt = 0;
    VP_CUDA(cudaMemcpyAsync(&nt, d_nt, 4, cudaMemcpyDeviceToHost, s));
    VP_CUDA(cudaStreamSynchronize(s));
    int *d_ovf;
    VP_CUDA(cudaMallocAsync(&d_ovf, sizeof(int), s));
    VP_CUDA(cudaMemsetAsync(d_ovf, 0, sizeof(int), s));
    k_levels<<<(unsigned)((nt + 127) / 128), 128, 0, s>>>(k1s, tst, nt, n, P->w, Tl.TS + P->w + 3, k2, d_ovf);
    VP_CHECK_LAUNCH();
    int h_ovf = 0;
    VP_CUDA(cudaMemcpyAsync(&h_ovf, d_ovf, sizeof(int), cudaMemcpyDeviceToHost, s));
    VP_CUDA(cudaStreamSynchronize(s));
    VP_CUDA(cudaFreeAsync(d_ovf, s));
    if (h_ovf) {
      vp_set_last_error("more than 2^20 points share one footprint row of a spreading tile");
      throw VpError{VP_ERR_UNSUPPORTED};
    }
    for (void *p : {(void *)tst, (void *)d_nt, tmp3}) VP_CUDA(cudaFreeAsync(p, s));
  }
  // (tile, level, slot) order -> bank ranks -> (tile, level, rank, slot) order
  VP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb2, k2, k2s, i1s, i2s, (int)n, 0, 64, s));
  k_bank_rank<<<nb, 256, 0, s>>>(k2s, n, k2);
  VP_CHECK_LAUNCH();
  VP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb2, k2, k2s, i2s, i1s, (int)n, 0, 64, s));
  std::swap(i1s, i2s);
  k_batch_heads<<<nb, 256, 0, s>>>(k2s, n, head);
  VP_CHECK_LAUNCH();
  S.sx = vp_alloc<double>(P, n);
  S.sy = vp_alloc<double>(P, n);
  S.sw = vp_alloc<double>(P, n);
  S.sperm = vp_alloc<int32_t>(P, n);
  k_gather_src<<<nb, 256, 0, s>>>(xy, weights, i2s, node_of, n, S.sx, S.sy, S.sw, S.sperm);
  VP_CHECK_LAUNCH();
  // host: batches and work items
  std::vector<uint64_t> hk(n);
  std::vector<int32_t> hh(n);
  VP_CUDA(cudaMemcpyAsync(hk.data(), k2s, 8 * n, cudaMemcpyDeviceToHost, s));
  VP_CUDA(cudaMemcpyAsync(hh.data(), head, 4 * n, cudaMemcpyDeviceToHost, s));
  VP_CUDA(cudaStreamSynchronize(s));
  std::vector<int32_t> bst;
  std::vector<int64_t> btile;
  for (int64_t i = 0; i < n; i++)
    if (hh[i]) {
      bst.push_back((int32_t)i);
      btile.push_back((int64_t)(hk[i] >> 40));
    }
  int64_t nbat = (int64_t)bst.size();
  bst.push_back((int32_t)n);
  const int64_t MAXB = S.det ? INT64_MAX : 48;  // batches per warp work item (deterministic: whole tile)
  std::vector<int4> items;
  for (int64_t b = 0; b < nbat;) {
    int64_t t = btile[b], e = b;
    while (e < nbat && btile[e] == t && e - b < MAXB) e++;
    items.push_back(make_int4((int)(t % Tl.ntx), (int)(t / Tl.ntx), (int)b, (int)e));
    b = e;
  }
  if (S.det) {
    std::stable_sort(items.begin(), items.end(),
                     [](const int4 &a, const int4 &b) { return ((a.x & 1) | ((a.y & 1) << 1)) < ((b.x & 1) | ((b.y & 1) << 1)); });
    for (int c = 0; c <= 4; c++) S.color_off[c] = 0;
    for (const int4 &it : items) S.color_off[((it.x & 1) | ((it.y & 1) << 1)) + 1]++;
    for (int c = 0; c < 4; c++) S.color_off[c + 1] += S.color_off[c];
  }
  S.n_batches = nbat;
  S.bstart = vp_alloc<int32_t>(P, bst.size());
  VP_CUDA(cudaMemcpy(S.bstart, bst.data(), 4 * bst.size(), cudaMemcpyHostToDevice));
  Tl.nsub = (int64_t)items.size();
  Tl.sub = vp_alloc<int4>(P, items.size());
  if (!items.empty()) VP_CUDA(cudaMemcpy(Tl.sub, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice));
  for (void *p : {(void *)k1, (void *)k1s, (void *)k2, (void *)k2s, (void *)i1, (void *)i1s, (void *)i2s, (void *)head,
                  tmp})
    VP_CUDA(cudaFreeAsync(p, s));
}

// ---------------------------------------------------------------------------------------------
// plan-time: strip order for k_spread_strip.  Key = (strip, origin row in strip, origin column in strip);
// the same es_origin() as the kernel's es_horner, so the kernel's rows agree with the sort.
__global__ void k_strip_keys(const double *__restrict__ xy, int64_t n, GridArgs g, int W, int SW, int SH,
                             int64_t nsx, int64_t nsy, uint64_t *__restrict__ keys, int32_t *__restrict__ idx,
                             int *__restrict__ bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t cx = (int64_t)es_origin(gcoord(xy[2 * i], g.ox, g.inv_h), W) + (W / 2 + 1);
  const int64_t cy = (int64_t)es_origin(gcoord(xy[2 * i + 1], g.oy, g.inv_h), W) + (W / 2 + 1);
  const int64_t bx = cx >= 0 ? cx / SW : -1, by = cy >= 0 ? cy / SH : -1;
  if (bx < 0 || by < 0 || bx >= nsx || by >= nsy) {  // outside the grid frame (not produced by the plan's grid)
    *bad = 1;
    keys[i] = 0;
  } else {
    keys[i] = ((uint64_t)(by * nsx + bx) << 16) | ((uint64_t)(cy - by * SH) << 8) | (uint64_t)(cx - bx * SW);
  }
  idx[i] = (int32_t)i;
}

// after the pack re-sort the strip id sits in key >> 32
__global__ void k_strip_heads(const uint64_t *__restrict__ k, int64_t n, int32_t *__restrict__ head) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  head[i] = (i == 0 || (k[i - 1] >> 32) != (k[i] >> 32)) ? 1 : 0;
}

__global__ void k_strip_ids(const uint64_t *__restrict__ k, const int32_t *__restrict__ pos, int64_t m,
                            int64_t *__restrict__ sid) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) sid[i] = (int64_t)(k[pos[i]] >> 32);
}

// pack order inside each (strip, origin row) group of points sorted by column (the group's keys share key >> 8):
// K = the most points in any W-column window of the group; point of rank i gets pack i mod K, so two points of a
// pack are >= W columns apart (a closer pair would put K + 1 points in one window).  New key (strip, row, pack,
// column); k_spread_strip packs consecutive column-disjoint points of a row.
__global__ void k_group_heads(const uint64_t *__restrict__ k, int64_t n, int shift, int32_t *__restrict__ head) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  head[i] = (i == 0 || (k[i - 1] >> shift) != (k[i] >> shift)) ? 1 : 0;
}

__global__ void k_strip_pack_keys(const uint64_t *__restrict__ k, const int32_t *__restrict__ gpos, int64_t ng,
                                  int64_t n, int W, uint64_t *__restrict__ k2) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t a = gpos[g], b = g + 1 < ng ? gpos[g + 1] : n;
  int K = 1;
  for (int64_t i = a, j = a; i < b; i++) {  // two pointers: points with column in (col_i - W, col_i]
    const int ci = (int)(k[i] & 0xff);
    while ((int)(k[j] & 0xff) <= ci - W) j++;
    K = max(K, (int)(i - j + 1));
  }
  K = min(K, 65535);
  for (int64_t i = a; i < b; i++) {
    const uint64_t key = k[i];
    const uint64_t strip = key >> 16, row = (key >> 8) & 0xff, col = key & 0xff;
    k2[i] = (strip << 32) | (row << 24) | ((uint64_t)((i - a) % K) << 8) | col;
  }
}

__global__ void k_strip_key_shift(uint64_t *__restrict__ k, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t key = k[i];
  k[i] = ((key >> 16) << 32) | (((key >> 8) & 0xff) << 24) | (key & 0xff);
}

void vp_strip_dims(int W, int kind, int *SW, int *SH);

void vp_build_strip_order(vp_plan_s *P, VpSpreadSet &S, const double *xy, const double *weights,
                          const int32_t *node_of, int64_t n, const GridArgs &g) {
  cudaStream_t s = P->stream;
  // 2: row-pair strips (k_spread_pair, default for W <= 12); 1: 32-column strips (k_spread_strip)
  S.strip = (P->opts.spread_pack == 0 && P->w <= 12) ? 2 : 1;
  int SW, SH;
  vp_strip_dims(P->w, S.strip == 2, &SW, &SH);
  const int64_t nsx = (g.nfx + P->w + 2) / SW + 1, nsy = (g.nfy + P->w + 2) / SH + 1;
  if (n == 0) {
    S.sx = vp_alloc<double>(P, 1); S.sy = vp_alloc<double>(P, 1); S.sw = vp_alloc<double>(P, 1);
    S.sperm = vp_alloc<int32_t>(P, 1); S.sitems = vp_alloc<int4>(P, 1);
    S.n_sitems = 0; S.n_batches = 0;
    return;
  }
  if (nsx * nsy >= (int64_t)1 << 31) throw VpError{VP_ERR_UNSUPPORTED};
  uint64_t *k1, *k1s;
  int32_t *i1, *i1s, *head, *hpos, *d_nh;
  int *d_bad;
  VP_CUDA(cudaMallocAsync(&k1, 8 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&k1s, 8 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&i1, 4 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&i1s, 4 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&head, 4 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&hpos, 4 * (n + 1), s));
  VP_CUDA(cudaMallocAsync(&d_nh, 4, s));
  VP_CUDA(cudaMallocAsync(&d_bad, 4, s));
  VP_CUDA(cudaMemsetAsync(d_bad, 0, 4, s));
  const unsigned nb = (unsigned)((n + 255) / 256);
  k_strip_keys<<<nb, 256, 0, s>>>(xy, n, g, P->w, SW, SH, nsx, nsy, k1, i1, d_bad);
  VP_CHECK_LAUNCH();
  size_t tb = 0, tb3 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, k1, k1s, i1, i1s, (int)n, 0, 64, s);
  cub::CountingInputIterator<int32_t> cnt(0);
  cub::DeviceSelect::Flagged(nullptr, tb3, cnt, head, hpos, d_nh, (int)n, s);
  void *tmp;
  VP_CUDA(cudaMallocAsync(&tmp, std::max(tb, tb3) + 16, s));
  VP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k1, k1s, i1, i1s, (int)n, 0, 64, s));
  if (P->opts.spread_pack == 1) {  // re-sort every (strip, row) group into column-disjoint packs
    k_group_heads<<<nb, 256, 0, s>>>(k1s, n, 8, head);
    VP_CHECK_LAUNCH();
    VP_CUDA(cub::DeviceSelect::Flagged(tmp, tb3, cnt, head, hpos, d_nh, (int)n, s));
    int32_t ng = 0;
    VP_CUDA(cudaMemcpyAsync(&ng, d_nh, 4, cudaMemcpyDeviceToHost, s));
    VP_CUDA(cudaStreamSynchronize(s));
    k_strip_pack_keys<<<(unsigned)((ng + 127) / 128), 128, 0, s>>>(k1s, hpos, ng, n, P->w, k1);
    VP_CHECK_LAUNCH();
    VP_CUDA(cudaMemcpyAsync(i1, i1s, 4 * (size_t)n, cudaMemcpyDeviceToDevice, s));
    VP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k1, k1s, i1, i1s, (int)n, 0, 64, s));
  } else {  // (strip, row, column) order; strip id moved to key >> 32 like the pack keys
    k_strip_key_shift<<<nb, 256, 0, s>>>(k1s, n);
    VP_CHECK_LAUNCH();
  }
  k_strip_heads<<<nb, 256, 0, s>>>(k1s, n, head);
  VP_CHECK_LAUNCH();
  VP_CUDA(cub::DeviceSelect::Flagged(tmp, tb3, cnt, head, hpos, d_nh, (int)n, s));
  int32_t nh = 0;
  int bad = 0;
  VP_CUDA(cudaMemcpyAsync(&nh, d_nh, 4, cudaMemcpyDeviceToHost, s));
  VP_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, s));
  VP_CUDA(cudaStreamSynchronize(s));
  if (bad) {
    vp_set_last_error("a source lies outside the spreading grid's frame");
    throw VpError{VP_ERR_GEOMETRY};
  }
  int64_t *d_sid;
  VP_CUDA(cudaMallocAsync(&d_sid, 8 * (size_t)nh, s));
  k_strip_ids<<<(unsigned)((nh + 255) / 256), 256, 0, s>>>(k1s, hpos, nh, d_sid);
  VP_CHECK_LAUNCH();
  std::vector<int32_t> hp(nh);
  std::vector<int64_t> hs(nh);
  VP_CUDA(cudaMemcpyAsync(hp.data(), hpos, 4 * (size_t)nh, cudaMemcpyDeviceToHost, s));
  VP_CUDA(cudaMemcpyAsync(hs.data(), d_sid, 8 * (size_t)nh, cudaMemcpyDeviceToHost, s));
  S.sx = vp_alloc<double>(P, n);
  S.sy = vp_alloc<double>(P, n);
  S.sw = vp_alloc<double>(P, n);
  S.sperm = vp_alloc<int32_t>(P, n);
  k_gather_src<<<nb, 256, 0, s>>>(xy, weights, i1s, node_of, n, S.sx, S.sy, S.sw, S.sperm);
  VP_CHECK_LAUNCH();
  VP_CUDA(cudaStreamSynchronize(s));
  // work items: every strip in strip order (neighbouring strips run together, so the halo REDs of adjacent
  // windows meet in L2), dense strips cut into <= VP_STRIP_MAXP points
  std::vector<int4> items;
  for (int64_t h = 0; h < nh; h++) {
    const int64_t p0 = hp[h], p1 = (h + 1 < nh) ? hp[h + 1] : n;
    const int bx = (int)(hs[h] % nsx), by = (int)(hs[h] / nsx);
    for (int64_t a = p0; a < p1; a += VP_STRIP_MAXP)
      items.push_back(make_int4(bx, by, (int)a, (int)std::min<int64_t>(p1, a + VP_STRIP_MAXP)));
  }
  // (ordering the items largest first for load balance measured slower: c5 12.09 vs 11.96 ms, DRAM 28.5 vs 18.8 GB)
  S.n_sitems = (int64_t)items.size();
  S.n_batches = S.n_sitems;
  S.sitems = vp_alloc<int4>(P, items.size());
  VP_CUDA(cudaMemcpy(S.sitems, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice));
  for (void *p : {(void *)k1, (void *)k1s, (void *)i1, (void *)i1s, (void *)head, (void *)hpos, (void *)d_nh,
                  (void *)d_bad, (void *)d_sid, tmp})
    VP_CUDA(cudaFreeAsync(p, s));
}

// ---------------------------------------------------------------------------------------------
// binning + sort of points into a uniform grid of bins (plan time; targets and kNN bins)
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
    size_t tb2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb2, (const unsigned long long *)counts, (unsigned long long *)bs,
                                  (int)(nb + 1), s);
    void *tmp2 = nullptr;
    VP_CUDA(cudaMallocAsync(&tmp2, tb2 + 16, s));
    VP_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, tb2, (const unsigned long long *)counts, (unsigned long long *)bs,
                                          (int)(nb + 1), s));
    VP_CUDA(cudaFreeAsync(tmp2, s));
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

// ---------------------------------------------------------------------------------------------
// level bands (a12; plan in vp_levels.cu): multiply every box's half spectrum by its level's band
// multiplier (e^{-k^2 delta_l} - e^{-k^2 delta_{l-1}})/k^2, grid-unit deconvolution, scale 1/(h_l^2 nfb^2)
__global__ void k_multiply_bands(double *__restrict__ data, int64_t nbox, int64_t nf, int64_t row, int64_t half_modes,
                                 const int32_t *__restrict__ box_level, const double *__restrict__ lev_par,
                                 const double *__restrict__ deconv) {
  const int64_t ncol = nf / 2 + 1;
  const int64_t per = nf * ncol, total = nbox * per;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = id / per, rem = id - b * per;
    int64_t r = rem / ncol, c = rem - r * ncol;
    int64_t m2 = r <= nf / 2 ? r : r - nf, a2 = m2 < 0 ? -m2 : m2;
    double *z = data + (b * nf + r) * row + 2 * c;
    if (c > half_modes || a2 > half_modes) {
      z[0] = 0.0;
      z[1] = 0.0;
      continue;
    }
    const double *lp = lev_par + 4 * box_level[b];
    double k2 = lp[2] * lp[2] * ((double)c * c + (double)m2 * m2);
    double fac = vp_mult_nh(k2, lp[0], lp[1]) * lp[3] * deconv[c] * deconv[a2];
    z[0] *= fac;
    z[1] *= fac;
  }
}

// per-target sum of its band entries (CSR by target) into out
__global__ void k_band_sum(const int32_t *__restrict__ lt_t, const int32_t *__restrict__ lt_off, int64_t n_lt,
                           const double *__restrict__ ent_val, const int32_t *__restrict__ tperm,
                           double *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_lt) return;
  double v = 0.0;
  for (int32_t e = lt_off[i]; e < lt_off[i + 1]; e++) v += ent_val[e];
  out[tperm[lt_t[i]]] += v;
}

template <int W>
static void launch_band_entries_w(vp_plan_s *P, const GridArgs &g) {
  constexpr int D = VP_HORNER_DEG(W);
  VpBands &B = P->bands;
  const int TSI = P->TSI, nw = TSI + W + 3;
  const size_t sm = sizeof(double) * (size_t)nw * nw;
  vp_smem_attr((const void *)k_interp_local<W, D>, sm);
  k_interp_local<W, D><<<(unsigned)B.e_n_items, 256, sm, P->stream>>>(
      B.e_items, TSI, B.e_x, B.e_y, B.e_perm, g, 1, nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr,
      B.ent_val);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}

void vp_launch_bands(vp_plan_s *P, const double *f, double *out) {
  VpBands &B = P->bands;
  if (B.nlev == 0 || B.nbox == 0) return;
  GridArgs g{B.grid, B.nfb, B.nbox * B.nfb, B.rowb, 0.0, 0.0, 1.0, 1.0};
  VP_CUDA(cudaMemsetAsync(B.grid, 0, sizeof(double) * B.nbox * B.nfb * B.rowb, P->stream));
  vp_launch_spread(P, B.sp, g, f);
  if (B.fg.own_fft) {
    vp_fft_bands(P);
  } else {
    VP_CUFFT(cufftSetStream(B.fwd, P->stream));
    VP_CUFFT(cufftSetStream(B.inv, P->stream));
    VP_CUFFT(cufftExecD2Z(B.fwd, B.grid, (cufftDoubleComplex *)B.grid));
    int64_t total = B.nbox * B.nfb * (B.nfb / 2 + 1);
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    k_multiply_bands<<<blocks, 256, 0, P->stream>>>(B.grid, B.nbox, B.nfb, B.rowb, B.nmode / 2, B.box_level,
                                                    B.lev_par, B.deconv);
    VP_CHECK_LAUNCH();
    P->n_kernels++;
    VP_CUFFT(cufftExecZ2D(B.inv, (cufftDoubleComplex *)B.grid, B.grid));
    P->n_ffts += 2;
  }
  // staged interpolation of the (target, level) entries, then the per-target sums
  switch (P->w) {
#define CASE(W) \
  case W: launch_band_entries_w<W>(P, g); break;
    CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: throw VpError{VP_ERR_UNSUPPORTED};
  }
  k_band_sum<<<(unsigned)((B.n_lt + 255) / 256), 256, 0, P->stream>>>(B.lt_t, B.lt_off, B.n_lt, B.ent_val, P->tperm,
                                                                       out);
  VP_CHECK_LAUNCH();
  P->n_kernels++;
}
