// vp_local.cu -- plan-time construction of the local-part stencils (§4).
//
// V_L at a target needs the Taylor jet of f there (eq. (vplocO5) and its interior/on-boundary forms,
// PAPER.md lines 1061-1127); the paper does not say how the jet is obtained from nodal data
// (reading R6).  Here: a least-squares polynomial fit of degree q over the K nearest
// quadrature nodes (kNN by ring search over a uniform bin grid), solved by Householder QR.  Because
// V_L is LINEAR in the jet, and the jet is linear in the nodal f, the whole local part collapses
// at plan time to one stencil per target:
//
//     V_L(t) = alpha_t f(node_t) + sum_k omega_{t,k} f[idx_{t,k}]
//
// with omega = Q R^{-T} ell, ell_ab = coef_ab / h^{a+b} the geometry-only coefficient vector of
// vp_math.cuh (interior series / circle formula / rectangle product form).  For node targets the
// a_00 coefficient goes to alpha_t and multiplies the exact nodal value.  Eval reads K (idx, omega)
// pairs per target.
#include <cub/cub.cuh>

#include "vp_common.cuh"
#include "vp_math.cuh"

#define KNN_MAX 64
#define NC_MAX 28  // degree 6

struct LocalArgs {
  const double *kx, *ky;          // nodes sorted by kNN bin
  const int32_t *kperm;           // sorted -> user node index
  const int64_t *bstart;          // bin CSR
  double bo_x, bo_y, bcell;
  int64_t nbx, nby;
  const double *tx, *ty;          // sorted targets
  const int64_t *tperm;
  int64_t T;
  int K, deg, nterms, node_targets;
  double delta;
  vp_boundary bd;
  int32_t *lidx;
  double *lw, *lalpha;
  int32_t *lnode;
  int32_t *is_bdry;
  double *scratch;                // per-thread LSQ scratch: K*nc + K doubles
};

__device__ void heap_sift_down(double *d, int32_t *id, int n, int i) {
  while (true) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && d[l] > d[m]) m = l;
    if (r < n && d[r] > d[m]) m = r;
    if (m == i) return;
    double td = d[i]; d[i] = d[m]; d[m] = td;
    int32_t ti = id[i]; id[i] = id[m]; id[m] = ti;
    i = m;
  }
}
__device__ void heap_sift_up(double *d, int32_t *id, int i) {
  while (i > 0) {
    int p = (i - 1) / 2;
    if (d[p] >= d[i]) return;
    double td = d[i]; d[i] = d[p]; d[p] = td;
    int32_t ti = id[i]; id[i] = id[p]; id[p] = ti;
    i = p;
  }
}

__global__ void k_build_local(LocalArgs a) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= a.T) return;
  const double x = a.tx[t], y = a.ty[t];
  const int K = a.K, nc = vp_ncoef(a.deg);
  // ---- kNN by ring search
  double hd[KNN_MAX];
  int32_t hi[KNN_MAX];
  int cnt = 0;
  double fx = (x - a.bo_x) / a.bcell, fy = (y - a.bo_y) / a.bcell;
  int64_t bx = (int64_t)floor(fx), by = (int64_t)floor(fy);
  bx = bx < 0 ? 0 : (bx >= a.nbx ? a.nbx - 1 : bx);
  by = by < 0 ? 0 : (by >= a.nby ? a.nby - 1 : by);
  int64_t rmax = a.nbx > a.nby ? a.nbx : a.nby;
  for (int64_t r = 0; r <= rmax; r++) {
    for (int64_t yy = by - r; yy <= by + r; yy++) {
      if (yy < 0 || yy >= a.nby) continue;
      bool edge_row = (yy == by - r) || (yy == by + r);
      for (int64_t xx = bx - r; xx <= bx + r; xx += (edge_row ? 1 : 2 * r > 0 ? 2 * r : 1)) {
        if (xx < 0 || xx >= a.nbx) continue;
        int64_t b = yy * a.nbx + xx;
        for (int64_t j = a.bstart[b]; j < a.bstart[b + 1]; j++) {
          double dx = a.kx[j] - x, dy = a.ky[j] - y, d2 = dx * dx + dy * dy;
          if (cnt < K) {
            hd[cnt] = d2; hi[cnt] = (int32_t)j;
            heap_sift_up(hd, hi, cnt);
            cnt++;
          } else if (d2 < hd[0]) {
            hd[0] = d2; hi[0] = (int32_t)j;
            heap_sift_down(hd, hi, K, 0);
          }
        }
      }
    }
    // all unscanned points are at least this far
    double gap = fmin(fmin(fx - (bx - r), (bx + r + 1) - fx), fmin(fy - (by - r), (by + r + 1) - fy)) * a.bcell;
    if (cnt == K && gap * gap >= hd[0]) break;
  }
  // ---- least squares: A (K x nc) column-major in scratch, Householder QR
  double *A = a.scratch + t * (int64_t)(K * nc + K + nc);
  double *yv = A + K * nc;
  double *diag = yv + K;
  double h = sqrt(hd[0]);
  if (h <= 0.0) h = 1.0;
  for (int k = 0; k < K; k++) {
    int32_t j = hi[k];
    double dx = (a.kx[j] - x) / h, dy = (a.ky[j] - y) / h;
    for (int d = 0; d <= a.deg; d++) {
      for (int p = d; p >= 0; p--) {
        int q = d - p;
        double v = 1.0;
        for (int e = 0; e < p; e++) v *= dx;
        for (int e = 0; e < q; e++) v *= dy;
        A[vp_mono_index(p, q) * K + k] = v;
      }
    }
  }
  for (int j = 0; j < nc; j++) {
    double *col = A + j * K;
    double nrm = 0.0;
    for (int i = j; i < K; i++) nrm += col[i] * col[i];
    nrm = sqrt(nrm);
    double alpha = col[j] > 0 ? -nrm : nrm;
    diag[j] = alpha;
    col[j] -= alpha;  // v = x - alpha e1 stored in col[j..K-1]
    double vv = 0.0;
    for (int i = j; i < K; i++) vv += col[i] * col[i];
    double beta = vv > 0 ? 2.0 / vv : 0.0;
    for (int c = j + 1; c < nc; c++) {
      double *cc = A + c * K;
      double s = 0.0;
      for (int i = j; i < K; i++) s += col[i] * cc[i];
      s *= beta;
      for (int i = j; i < K; i++) cc[i] -= s * col[i];
    }
  }
  // ---- geometry coefficients of V_L in the Taylor basis
  double coef[VP_NTAYLOR];
  bool bdry = false;
  if (a.bd.kind == VP_BDRY_CIRCLE)
    bdry = vp_coef_circle(x, y, a.bd.p[0], a.bd.p[1], a.bd.p[2], a.delta, a.nterms, a.deg, coef);
  else if (a.bd.kind == VP_BDRY_RECT)
    bdry = vp_coef_rect(x, y, a.bd.p[0], a.bd.p[1], a.bd.p[2], a.bd.p[3], a.delta, a.deg, coef);
  if (!bdry) vp_coef_interior(a.delta, a.nterms, a.deg, coef);
  a.is_bdry[t] = bdry ? 1 : 0;
  double alpha = 0.0;
  int32_t node = a.node_targets ? (int32_t)a.tperm[t] : -1;
  if (node >= 0) {
    alpha = coef[0];
    coef[0] = 0.0;
  }
  // ell in the scaled monomial basis: coefficient a_ab = c_ab / h^{a+b}
  double ell[NC_MAX];
  for (int i = 0; i < nc; i++) ell[i] = 0.0;
  int dm = a.deg < 4 ? a.deg : 4;
  for (int d = 0; d <= dm; d++)
    for (int p = d; p >= 0; p--) {
      int idx = vp_mono_index(p, d - p);
      ell[idx] = coef[idx] / pow(h, (double)d);
    }
  // z = R^{-T} ell  (R[i][j] = A[j*K + i] for j > i, R[i][i] = diag[i])
  double z[NC_MAX];
  for (int j = 0; j < nc; j++) {
    double s = ell[j];
    for (int i = 0; i < j; i++) s -= A[j * K + i] * z[i];
    z[j] = s / diag[j];
  }
  // omega = Q [z; 0] = H_0 ... H_{nc-1} [z; 0]
  for (int i = 0; i < K; i++) yv[i] = i < nc ? z[i] : 0.0;
  for (int j = nc - 1; j >= 0; j--) {
    const double *v = A + j * K;
    double vv = 0.0, s = 0.0;
    // v_j holds (col[j] - alpha, col[j+1..]) ; recompute |v|^2
    for (int i = j; i < K; i++) { vv += v[i] * v[i]; s += v[i] * yv[i]; }
    if (vv > 0) {
      s *= 2.0 / vv;
      for (int i = j; i < K; i++) yv[i] -= s * v[i];
    }
  }
  int32_t *op = a.lidx + t * (int64_t)K;
  double *ow = a.lw + t * (int64_t)K;
  for (int k = 0; k < K; k++) {
    op[k] = a.kperm[hi[k]];
    ow[k] = yv[k];
  }
  a.lalpha[t] = alpha;
  a.lnode[t] = node;
}

void vp_build_local(vp_plan_s *P, const double *nodes_dev) {
  int deg = P->deg, K = P->K;
  int nc = vp_ncoef(deg);
  // kNN bins: about 8 nodes per bin over the bounding square
  double S = P->S;
  double cell = sqrt(8.0 * S * S / (double)P->N);
  int64_t nb = (int64_t)ceil(S / cell) + 1;
  if (nb < 1) nb = 1;
  if (nb > 40000) { nb = 40000; cell = S / (nb - 1); }
  double ox = P->cx - 0.5 * S - 0.5 * cell, oy = P->cy - 0.5 * S - 0.5 * cell;
  double *kx = vp_alloc<double>(P, P->N), *ky = vp_alloc<double>(P, P->N);
  int32_t *kperm = vp_alloc<int32_t>(P, P->N);
  int64_t *bstart = nullptr;
  vp_sort_points(P, nodes_dev, P->N, ox, oy, cell, nb, nb, kx, ky, nullptr, kperm, &bstart);
  P->lidx = vp_alloc<int32_t>(P, (size_t)P->T * K);
  P->lw = vp_alloc<double>(P, (size_t)P->T * K);
  P->lalpha = vp_alloc<double>(P, P->T);
  P->lnode = vp_alloc<int32_t>(P, P->T);
  int32_t *isb = vp_alloc<int32_t>(P, P->T);
  // scratch in chunks of targets to bound memory
  int64_t per = (int64_t)(K * nc + K + nc);
  int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(P->T, (int64_t)(2e9 / 8) / per));
  double *scratch = nullptr;
  VP_CUDA(cudaMallocAsync(&scratch, sizeof(double) * per * chunk, P->stream));
  for (int64_t s0 = 0; s0 < P->T; s0 += chunk) {
    int64_t n = std::min(chunk, P->T - s0);
    LocalArgs a;
    a.kx = kx; a.ky = ky; a.kperm = kperm; a.bstart = bstart;
    a.bo_x = ox; a.bo_y = oy; a.bcell = cell; a.nbx = nb; a.nby = nb;
    a.tx = P->tx + s0; a.ty = P->ty + s0; a.tperm = P->tperm + s0; a.T = n;
    a.K = K; a.deg = deg; a.nterms = P->opts.series_order > 0 ? P->opts.series_order : 3;
    a.node_targets = P->opts.targets_are_nodes ? 1 : 0;
    a.delta = P->delta1;
    a.bd = P->opts.boundary;
    a.lidx = P->lidx + s0 * K; a.lw = P->lw + s0 * K; a.lalpha = P->lalpha + s0; a.lnode = P->lnode + s0;
    a.is_bdry = isb + s0;
    a.scratch = scratch;
    k_build_local<<<(unsigned)((n + 127) / 128), 128, 0, P->stream>>>(a);
    VP_CHECK_LAUNCH();
  }
  VP_CUDA(cudaFreeAsync(scratch, P->stream));
  // count boundary targets
  int64_t *d_cnt = nullptr;
  VP_CUDA(cudaMallocAsync(&d_cnt, sizeof(int64_t), P->stream));
  size_t tb = 0;
  cub::DeviceReduce::Sum(nullptr, tb, isb, d_cnt, (int)P->T, P->stream);
  void *tmp = nullptr;
  VP_CUDA(cudaMallocAsync(&tmp, tb + 16, P->stream));
  VP_CUDA(cub::DeviceReduce::Sum(tmp, tb, isb, d_cnt, (int)P->T, P->stream));
  VP_CUDA(cudaMemcpyAsync(&P->n_bdry, d_cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, P->stream));
  VP_CUDA(cudaStreamSynchronize(P->stream));
  VP_CUDA(cudaFree(tmp));
  VP_CUDA(cudaFree(d_cnt));
}
