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

#include "vp_boundary.cuh"
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
  const int32_t *tperm;
  const int32_t *list;            // targets (sorted index) that get a stencil; slot i -> target list[i]
  int64_t T;                      // number of list entries
  int K, deg, nterms;
  int64_t node_targets;           // targets with user index < node_targets are the nodes themselves
  double delta;
  VpBdryDev bd;
  int32_t *lidx;                  // stencils, k-major: entry k of slot s at [k * stride + s]
  double *lw, *lalpha;
  int64_t slot0, stride;          // global slot of list entry 0; number of stencil slots
  int32_t *lnode;
  int32_t *is_bdry;
  double *scratch;                // per-thread LSQ scratch: K*nc + K doubles
  const int8_t *tlev;             // [T] band level of the sorted target: V_L uses delta / 4^level
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
  int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (slot >= a.T) return;
  const int64_t t = a.list[slot];
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
  double *A = a.scratch + slot * (int64_t)(K * nc + K + nc);
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
  const double delta = a.tlev ? a.delta * pow(0.25, (double)a.tlev[t]) : a.delta;
  bdry = vp_bdry_coef(a.bd, x, y, delta, a.nterms, a.deg, coef) == 1;  // -1 (geometry error) flags bd.err
  if (!bdry) vp_coef_interior(delta, a.nterms, a.deg, coef);
  a.is_bdry[t] = bdry ? 1 : 0;
  // a target farther than 12 sqrt(delta) from every node sees no local part (the short-time kernel is below
  // 1e-14 there): f is not extrapolated outside the mesh
  {
    double d2min = hd[0];
    for (int k = 1; k < K; k++) d2min = fmin(d2min, hd[k]);
    if (d2min > 144.0 * delta) vp_coef_clear(coef);
  }
  double alpha = 0.0;
  int32_t node = a.tperm[t] < a.node_targets ? (int32_t)a.tperm[t] : -1;
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
  const int64_t gs = a.slot0 + slot;
  for (int k = 0; k < K; k++) {
    a.lidx[k * a.stride + gs] = a.kperm[hi[k]];
    a.lw[k * a.stride + gs] = yv[k];
  }
  a.lalpha[t] = alpha;
  a.lnode[t] = node;
}

// ---------------------------------------------------------------------------------------------
// TRIANGLE mode: per-triangle affine map from the reference rule, aspect test, metric M = A^-1 A^-T
struct TriArgs {
  const double *nodes;   // [M][p][2] user order
  int64_t M;
  int p;
  double pinv[3][VP_TRI_MAXP];  // affine LSQ: (A row x | A row y | b) = nodes * pinv^T
  double ref[VP_TRI_MAXP][2];   // reference coordinates of the rule's nodes
  double amax;
  int8_t *ok;
  double *Mm;            // [M][3]: M11, M12, M22
};

__global__ void k_tri_classify(TriArgs a) {
  int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= a.M) return;
  const double *nd = a.nodes + m * (int64_t)a.p * 2;
  double c[2][3] = {{0, 0, 0}, {0, 0, 0}};
  for (int k = 0; k < a.p; k++)
    for (int r = 0; r < 3; r++) {
      c[0][r] += a.pinv[r][k] * nd[2 * k];
      c[1][r] += a.pinv[r][k] * nd[2 * k + 1];
    }
  // x = A xi + b with A = [[c00, c01], [c10, c11]], b = (c02, c12); residual must vanish (straight)
  double A00 = c[0][0], A01 = c[0][1], A10 = c[1][0], A11 = c[1][1];
  double det = A00 * A11 - A01 * A10;
  double fro = A00 * A00 + A01 * A01 + A10 * A10 + A11 * A11;
  bool ok = fabs(det) > 1e-300 && isfinite(det);
  // aspect = sigma_max / sigma_min of A
  double disc = sqrt(fmax(fro * fro - 4.0 * det * det, 0.0));
  double s2max = 0.5 * (fro + disc), s2min = 0.5 * (fro - disc);
  if (!(s2min > 0.0) || s2max > a.amax * a.amax * s2min) ok = false;
  // the map must reproduce every node (straight triangle carrying this rule)
  double res = 0.0;
  for (int k = 0; k < a.p; k++) {
    double ex = A00 * a.ref[k][0] + A01 * a.ref[k][1] + c[0][2] - nd[2 * k];
    double ey = A10 * a.ref[k][0] + A11 * a.ref[k][1] + c[1][2] - nd[2 * k + 1];
    res = fmax(res, fabs(ex) + fabs(ey));
  }
  if (!(res <= 1e-10 * sqrt(fro))) ok = false;
  double Mm11 = 0, Mm12 = 0, Mm22 = 0;
  if (ok) {
    // A^-1 = [[A11, -A01], [-A10, A00]] / det ; M = A^-1 A^-T
    double i00 = A11 / det, i01 = -A01 / det, i10 = -A10 / det, i11 = A00 / det;
    Mm11 = i00 * i00 + i01 * i01;
    Mm12 = i00 * i10 + i01 * i11;
    Mm22 = i10 * i10 + i11 * i11;
  }
  a.ok[m] = ok ? 1 : 0;
  a.Mm[3 * m] = Mm11;
  a.Mm[3 * m + 1] = Mm12;
  a.Mm[3 * m + 2] = Mm22;
}

// Hessian operators of the least-squares cubic fit on the reference rule (host, once per plan):
// Hop[ab][k][j], ab in {xi1 xi1, xi1 xi2, xi2 xi2}: second derivative of the fit at node k per f_j.
void vp_cubic_hessian_ops(const double *ref, int p, std::vector<double> &Hop) {
  const int nc = 10;
  std::vector<double> V((size_t)p * nc);
  auto mono = [](double u, double v, int m, int du, int dv) {
    static const int ea[10] = {0, 1, 0, 2, 1, 0, 3, 2, 1, 0}, eb[10] = {0, 0, 1, 0, 1, 2, 0, 1, 2, 3};
    int a = ea[m], b = eb[m];
    if (du > a || dv > b) return 0.0;
    double c = 1.0;
    for (int i = 0; i < du; i++) c *= (a - i);
    for (int i = 0; i < dv; i++) c *= (b - i);
    return c * pow(u, a - du) * pow(v, b - dv);
  };
  const double c0 = 1.0 / 3.0;
  for (int k = 0; k < p; k++)
    for (int m = 0; m < nc; m++) V[(size_t)k * nc + m] = mono(ref[2 * k] - c0, ref[2 * k + 1] - c0, m, 0, 0);
  // P = (V^T V)^-1 V^T by Gauss-Jordan on the 10x10 normal matrix (long double)
  long double G[10][20];
  for (int i = 0; i < nc; i++)
    for (int j = 0; j < 2 * nc; j++) {
      long double s = 0;
      if (j < nc)
        for (int k = 0; k < p; k++) s += (long double)V[(size_t)k * nc + i] * V[(size_t)k * nc + j];
      else
        s = (j - nc == i) ? 1.0L : 0.0L;
      G[i][j] = s;
    }
  for (int c = 0; c < nc; c++) {
    int piv = c;
    for (int r = c + 1; r < nc; r++)
      if (fabsl(G[r][c]) > fabsl(G[piv][c])) piv = r;
    for (int j = 0; j < 2 * nc; j++) std::swap(G[c][j], G[piv][j]);
    long double d = G[c][c];
    for (int j = 0; j < 2 * nc; j++) G[c][j] /= d;
    for (int r = 0; r < nc; r++)
      if (r != c) {
        long double f = G[r][c];
        for (int j = 0; j < 2 * nc; j++) G[r][j] -= f * G[c][j];
      }
  }
  std::vector<double> Pm((size_t)nc * p);
  for (int m = 0; m < nc; m++)
    for (int k = 0; k < p; k++) {
      long double s = 0;
      for (int i = 0; i < nc; i++) s += G[m][nc + i] * (long double)V[(size_t)k * nc + i];
      Pm[(size_t)m * p + k] = (double)s;
    }
  Hop.assign((size_t)3 * p * p, 0.0);
  const int dd[3][2] = {{2, 0}, {1, 1}, {0, 2}};
  for (int h = 0; h < 3; h++)
    for (int k = 0; k < p; k++)
      for (int j = 0; j < p; j++) {
        double s = 0;
        for (int m = 0; m < nc; m++) s += mono(ref[2 * k] - c0, ref[2 * k + 1] - c0, m, dd[h][0], dd[h][1]) * Pm[(size_t)m * p + j];
        Hop[((size_t)h * p + k) * p + j] = s;
      }
}

// per sorted target: triangle mode (interior node of an ok triangle) or stencil
__global__ void k_target_mode(const double *tx, const double *ty, const int32_t *tperm, int64_t T, int p,
                              const int8_t *tri_ok, int64_t node_targets, VpBdryDev bd, double delta, double c1,
                              const int8_t *tlev, int32_t *need, double *lalpha, int32_t *lnode) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= T) return;
  int nd = tperm[t] < node_targets ? (int)tperm[t] : -1;
  bool tri = nd >= 0 && tri_ok && tri_ok[nd / p] && !(tlev && tlev[t] > 0);
  if (tri && bd.kind != VP_BDRY_NONE) {
    double coef[VP_NTAYLOR];
    double x = tx[t], y = ty[t];
    if (vp_bdry_coef(bd, x, y, delta, 1, 0, coef) != 0) tri = false;  // near the boundary: stencil path
  }
  need[t] = tri ? 0 : 1;
  if (tri) {
    lalpha[t] = c1;
    lnode[t] = nd;
  }
}

__global__ void k_fill_ptr(const int32_t *list, int64_t n, int32_t *lptr) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) lptr[list[i]] = (int32_t)i;
}

void vp_build_local(vp_plan_s *P, const double *nodes_dev) {
  int deg = P->deg, K = P->K;
  int nc = vp_ncoef(deg);
  cudaStream_t st = P->stream;
  const int nterms = P->opts.series_order > 0 ? P->opts.series_order : 3;
  P->lalpha = vp_alloc<double>(P, P->T);
  P->lnode = vp_alloc<int32_t>(P, P->T);
  P->lptr = vp_alloc<int32_t>(P, P->T);
  VP_CUDA(cudaMemsetAsync(P->lptr, 0xff, sizeof(int32_t) * P->T, st));
  int32_t *need = nullptr;
  VP_CUDA(cudaMallocAsync(&need, sizeof(int32_t) * (P->T + 1), st));
  unsigned tb_t = (unsigned)((P->T + 255) / 256);
  if (P->dmode == VP_DERIV_TRIANGLE) {
    // reference-rule operators on the host: affine pseudo-inverse and cubic-fit Hessian operators
    const int p = P->p;
    const double *ref = P->opts.ref_nodes;
    TriArgs ta;
    memset(&ta, 0, sizeof(ta));
    {
      // normal equations of [xi1 xi2 1] (p x 3): pinv = (V^T V)^-1 V^T
      double G[3][3] = {{0}}, V[VP_TRI_MAXP][3];
      for (int k = 0; k < p; k++) {
        V[k][0] = ref[2 * k]; V[k][1] = ref[2 * k + 1]; V[k][2] = 1.0;
        for (int i = 0; i < 3; i++)
          for (int j = 0; j < 3; j++) G[i][j] += V[k][i] * V[k][j];
      }
      double Gi[3][3];
      double d = G[0][0] * (G[1][1] * G[2][2] - G[1][2] * G[2][1]) - G[0][1] * (G[1][0] * G[2][2] - G[1][2] * G[2][0]) +
                 G[0][2] * (G[1][0] * G[2][1] - G[1][1] * G[2][0]);
      for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
          int i1 = (j + 1) % 3, i2 = (j + 2) % 3, j1 = (i + 1) % 3, j2 = (i + 2) % 3;
          Gi[i][j] = (G[i1][j1] * G[i2][j2] - G[i1][j2] * G[i2][j1]) / d;
        }
      for (int r = 0; r < 3; r++)
        for (int k = 0; k < p; k++) {
          double s = 0;
          for (int j = 0; j < 3; j++) s += Gi[r][j] * V[k][j];
          ta.pinv[r][k] = s;
        }
    }
    ta.nodes = nodes_dev; ta.M = P->M; ta.p = p;
    for (int k = 0; k < p; k++) { ta.ref[k][0] = ref[2 * k]; ta.ref[k][1] = ref[2 * k + 1]; }
    ta.amax = P->opts.tri_max_aspect > 0 ? P->opts.tri_max_aspect : 3.0;
    P->tri_ok = vp_alloc<int8_t>(P, P->M);
    P->tri_M = vp_alloc<double>(P, 3 * P->M);
    ta.ok = P->tri_ok; ta.Mm = P->tri_M;
    k_tri_classify<<<(unsigned)((P->M + 127) / 128), 128, 0, st>>>(ta);
    VP_CHECK_LAUNCH();
    // Hessian operators of the reference cubic fit: H_ab[k][j] = d2/dxi_a dxi_b of the fit at node k
    std::vector<double> Hop;
    vp_cubic_hessian_ops(ref, p, Hop);
    P->tri_H = vp_alloc<double>(P, Hop.size());
    P->tri_H_host = Hop;
    if (p == 12) P->trih_slot = vp_acquire_trih_slot(Hop.data());
    VP_CUDA(cudaMemcpy(P->tri_H, Hop.data(), sizeof(double) * Hop.size(), cudaMemcpyHostToDevice));
    double c1 = P->delta1;
    k_target_mode<<<tb_t, 256, 0, st>>>(P->tx, P->ty, P->tperm, P->T, p, P->tri_ok, P->opts.targets_are_nodes ? P->N : 0,
                                       P->bdev, P->delta1, c1, P->bands.tlev, need, P->lalpha, P->lnode);
    VP_CHECK_LAUNCH();
    P->tri_c2 = nterms >= 2 ? 0.5 * P->delta1 * P->delta1 : 0.0;
    P->tri_vL = vp_alloc<double>(P, P->N);
  } else {
    k_target_mode<<<tb_t, 256, 0, st>>>(P->tx, P->ty, P->tperm, P->T, 1, nullptr, 0, P->bdev, P->delta1, 0.0,
                                       P->bands.tlev, need, P->lalpha, P->lnode);
    VP_CHECK_LAUNCH();
  }
  // compact the stencil targets
  int32_t *list = nullptr, *d_n = nullptr;
  VP_CUDA(cudaMallocAsync(&list, sizeof(int32_t) * (P->T + 1), st));
  VP_CUDA(cudaMallocAsync(&d_n, sizeof(int32_t), st));
  {
    size_t tb = 0;
    cub::CountingInputIterator<int32_t> cnt(0);
    cub::DeviceSelect::Flagged(nullptr, tb, cnt, need, list, d_n, (int)P->T, st);
    void *tmp;
    VP_CUDA(cudaMallocAsync(&tmp, tb + 16, st));
    VP_CUDA(cub::DeviceSelect::Flagged(tmp, tb, cnt, need, list, d_n, (int)P->T, st));
    VP_CUDA(cudaFreeAsync(tmp, st));
  }
  int32_t nst = 0;
  VP_CUDA(cudaMemcpyAsync(&nst, d_n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  VP_CUDA(cudaStreamSynchronize(st));
  P->n_stencil = nst;
  if (nst > 0) {
    k_fill_ptr<<<(unsigned)((nst + 255) / 256), 256, 0, st>>>(list, nst, P->lptr);
    VP_CHECK_LAUNCH();
  }
  P->st_vL = vp_alloc<double>(P, (size_t)std::max<int64_t>(nst, 1));
  P->lidx = vp_alloc<int32_t>(P, (size_t)std::max<int64_t>(nst, 1) * K);
  P->lw = vp_alloc<double>(P, (size_t)std::max<int64_t>(nst, 1) * K);
  int32_t *isb = nullptr;
  VP_CUDA(cudaMallocAsync(&isb, sizeof(int32_t) * (P->T + 1), st));
  VP_CUDA(cudaMemsetAsync(isb, 0, sizeof(int32_t) * (P->T + 1), st));
  if (nst > 0) {
    // kNN bins: about 8 nodes per bin over the bounding square
    double S = P->S;
    double cell = sqrt(8.0 * S * S / (double)P->N);
    int64_t nb = (int64_t)ceil(S / cell) + 1;
    if (nb < 1) nb = 1;
    if (nb > 40000) { nb = 40000; cell = S / (nb - 1); }
    double ox = P->cx - 0.5 * S - 0.5 * cell, oy = P->cy - 0.5 * S - 0.5 * cell;
    double *kx = nullptr, *ky = nullptr;
    int32_t *kperm = nullptr;
    VP_CUDA(cudaMallocAsync(&kx, sizeof(double) * P->N, st));
    VP_CUDA(cudaMallocAsync(&ky, sizeof(double) * P->N, st));
    VP_CUDA(cudaMallocAsync(&kperm, sizeof(int32_t) * P->N, st));
    int64_t *bstart = nullptr;
    vp_sort_points(P, nodes_dev, P->N, ox, oy, cell, nb, nb, kx, ky, nullptr, kperm, &bstart);
    int64_t per = (int64_t)(K * nc + K + nc);
    int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(nst, (int64_t)(2e9 / 8) / per));
    double *scratch = nullptr;
    VP_CUDA(cudaMallocAsync(&scratch, sizeof(double) * per * chunk, st));
    for (int64_t s0 = 0; s0 < nst; s0 += chunk) {
      int64_t n = std::min<int64_t>(chunk, nst - s0);
      LocalArgs a;
      a.kx = kx; a.ky = ky; a.kperm = kperm; a.bstart = bstart;
      a.bo_x = ox; a.bo_y = oy; a.bcell = cell; a.nbx = nb; a.nby = nb;
      a.tx = P->tx; a.ty = P->ty; a.tperm = P->tperm; a.list = list + s0; a.T = n;
      a.K = K; a.deg = deg; a.nterms = nterms;
      a.node_targets = P->opts.targets_are_nodes ? P->N : 0;
      a.delta = P->delta1;
      a.bd = P->bdev;
      a.lidx = P->lidx; a.lw = P->lw; a.slot0 = s0; a.stride = nst; a.lalpha = P->lalpha; a.lnode = P->lnode;
      a.is_bdry = isb;
      a.scratch = scratch;
      a.tlev = P->bands.tlev;
      k_build_local<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(a);
      VP_CHECK_LAUNCH();
    }
    for (void *q : {(void *)scratch, (void *)kx, (void *)ky, (void *)kperm}) VP_CUDA(cudaFreeAsync(q, st));
  }
  // count boundary targets
  int64_t *d_cnt = nullptr;
  VP_CUDA(cudaMallocAsync(&d_cnt, sizeof(int64_t), st));
  size_t tb = 0;
  cub::DeviceReduce::Sum(nullptr, tb, isb, d_cnt, (int)P->T, st);
  void *tmp = nullptr;
  VP_CUDA(cudaMallocAsync(&tmp, tb + 16, st));
  VP_CUDA(cub::DeviceReduce::Sum(tmp, tb, isb, d_cnt, (int)P->T, st));
  VP_CUDA(cudaMemcpyAsync(&P->n_bdry, d_cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  int gerr = 0;
  if (P->bdev.err) VP_CUDA(cudaMemcpyAsync(&gerr, P->bdev.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  VP_CUDA(cudaStreamSynchronize(st));
  if (gerr) {
    vp_set_last_error("boundary: ambiguous closest point (medial axis) or unsupported local geometry within "
                      "12 sqrt(delta_1) of a target");
    throw VpError{VP_ERR_GEOMETRY};
  }
  for (void *q : {(void *)tmp, (void *)d_cnt, (void *)need, (void *)list, (void *)d_n, (void *)isb})
    VP_CUDA(cudaFree(q));
}
