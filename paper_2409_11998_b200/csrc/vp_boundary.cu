// vp_boundary.cu -- plan-time validation and upload of the boundary descriptor (include/vp.h vp_boundary;
// PAPER.md §2.2).  Device-side use: vp_boundary.cuh vp_bdry_coef.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "vp_boundary.cuh"

void vp_gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w);  // vp_api.cu, on [-1, 1]

// CSR bins of items (bounding boxes expanded by `pad`) over [x0, x0 + nbx cell) x [y0, y0 + nby cell)
static void build_bins(vp_plan_s *P, VpBdryDev &B, const std::vector<double> &bb /* [m][4] xlo xhi ylo yhi */,
                       double pad, double cell) {
  double xlo = 1e300, xhi = -1e300, ylo = 1e300, yhi = -1e300;
  const size_t m = bb.size() / 4;
  for (size_t i = 0; i < m; i++) {
    xlo = std::min(xlo, bb[4 * i]); xhi = std::max(xhi, bb[4 * i + 1]);
    ylo = std::min(ylo, bb[4 * i + 2]); yhi = std::max(yhi, bb[4 * i + 3]);
  }
  xlo -= pad; ylo -= pad; xhi += pad; yhi += pad;
  // at most ~4M bins
  const double span = std::max(xhi - xlo, yhi - ylo);
  if (span / cell > 2048.0) cell = span / 2048.0;
  B.bcell = cell;
  B.bx0 = xlo;
  B.by0 = ylo;
  B.nbx = (int64_t)std::ceil((xhi - xlo) / cell) + 1;
  B.nby = (int64_t)std::ceil((yhi - ylo) / cell) + 1;
  std::vector<int32_t> cnt((size_t)(B.nbx * B.nby + 1), 0);
  auto range = [&](size_t i, int64_t &ax, int64_t &bx, int64_t &ay, int64_t &by) {
    ax = std::max<int64_t>(0, (int64_t)std::floor((bb[4 * i] - pad - B.bx0) / cell));
    bx = std::min<int64_t>(B.nbx - 1, (int64_t)std::floor((bb[4 * i + 1] + pad - B.bx0) / cell));
    ay = std::max<int64_t>(0, (int64_t)std::floor((bb[4 * i + 2] - pad - B.by0) / cell));
    by = std::min<int64_t>(B.nby - 1, (int64_t)std::floor((bb[4 * i + 3] + pad - B.by0) / cell));
  };
  for (size_t i = 0; i < m; i++) {
    int64_t ax, bx, ay, by;
    range(i, ax, bx, ay, by);
    for (int64_t y = ay; y <= by; y++)
      for (int64_t x = ax; x <= bx; x++) cnt[(size_t)(y * B.nbx + x) + 1]++;
  }
  for (size_t i = 1; i < cnt.size(); i++) cnt[i] += cnt[i - 1];
  std::vector<int32_t> idx((size_t)cnt.back()), fill(cnt.begin(), cnt.end() - 1);
  for (size_t i = 0; i < m; i++) {
    int64_t ax, bx, ay, by;
    range(i, ax, bx, ay, by);
    for (int64_t y = ay; y <= by; y++)
      for (int64_t x = ax; x <= bx; x++) idx[(size_t)fill[(size_t)(y * B.nbx + x)]++] = (int32_t)i;
  }
  int32_t *bs = vp_alloc<int32_t>(P, cnt.size());
  int32_t *bi = vp_alloc<int32_t>(P, std::max<size_t>(1, idx.size()));
  VP_CUDA(cudaMemcpy(bs, cnt.data(), 4 * cnt.size(), cudaMemcpyHostToDevice));
  if (!idx.empty()) VP_CUDA(cudaMemcpy(bi, idx.data(), 4 * idx.size(), cudaMemcpyHostToDevice));
  B.bstart = bs;
  B.bidx = bi;
}

static double cross2(double ax, double ay, double bx, double by) { return ax * by - ay * bx; }

// proper intersection of segments p1p2 and p3p4 (shared endpoints excluded by the caller)
static bool seg_cross(const double *p1, const double *p2, const double *p3, const double *p4) {
  const double d1 = cross2(p4[0] - p3[0], p4[1] - p3[1], p1[0] - p3[0], p1[1] - p3[1]);
  const double d2 = cross2(p4[0] - p3[0], p4[1] - p3[1], p2[0] - p3[0], p2[1] - p3[1]);
  const double d3 = cross2(p2[0] - p1[0], p2[1] - p1[1], p3[0] - p1[0], p3[1] - p1[1]);
  const double d4 = cross2(p2[0] - p1[0], p2[1] - p1[1], p4[0] - p1[0], p4[1] - p1[1]);
  return ((d1 > 0) != (d2 > 0)) && ((d3 > 0) != (d4 > 0)) && d1 != 0 && d2 != 0 && d3 != 0 && d4 != 0;
}

void vp_build_boundary(vp_plan_s *P, VpBdryDev &B) {
  const vp_boundary &bd = P->opts.boundary;
  B = VpBdryDev();
  B.kind = bd.kind;
  for (int i = 0; i < 4; i++) B.p[i] = bd.p[i];
  B.reach = 12.0 * std::sqrt(P->delta1);
  if (bd.kind == VP_BDRY_NONE || bd.kind == VP_BDRY_CIRCLE || bd.kind == VP_BDRY_RECT) return;
  int *err = vp_alloc<int>(P, 1);
  VP_CUDA(cudaMemset(err, 0, sizeof(int)));
  B.err = err;
  if (!bd.pts || bd.n < 1) throw VpError{VP_ERR_GEOMETRY};
  if (bd.kind == VP_BDRY_POLYGON) {
    const int64_t n0 = bd.n;
    if (n0 < 3) throw VpError{VP_ERR_GEOMETRY};
    for (int64_t i = 0; i < 2 * n0; i++)
      if (!std::isfinite(bd.pts[i])) throw VpError{VP_ERR_NONFINITE};
    // signed area (CCW required)
    double area = 0;
    for (int64_t i = 0; i < n0; i++) {
      const double *a = bd.pts + 2 * i, *b = bd.pts + 2 * ((i + 1) % n0);
      area += cross2(a[0], a[1], b[0], b[1]);
    }
    if (!(area > 0)) throw VpError{VP_ERR_GEOMETRY};
    // drop straight (180 degree) vertices, classify the rest: convex / reflex right angles only
    std::vector<double> v;
    std::vector<int8_t> kind;
    for (int64_t i = 0; i < n0; i++) {
      const double *a = bd.pts + 2 * ((i - 1 + n0) % n0), *p = bd.pts + 2 * i, *c = bd.pts + 2 * ((i + 1) % n0);
      const double ux = p[0] - a[0], uy = p[1] - a[1], wx = c[0] - p[0], wy = c[1] - p[1];
      const double lu = std::hypot(ux, uy), lw = std::hypot(wx, wy);
      if (!(lu > 0) || !(lw > 0)) throw VpError{VP_ERR_GEOMETRY};  // repeated vertex
      const double cr = cross2(ux, uy, wx, wy) / (lu * lw), dt = (ux * wx + uy * wy) / (lu * lw);
      if (std::fabs(cr) <= 1e-12 && dt > 0) continue;  // straight: merged into one edge
      if (std::fabs(dt) > 1e-9) throw VpError{VP_ERR_UNSUPPORTED};  // not a right angle (R8)
      v.push_back(p[0]);
      v.push_back(p[1]);
      kind.push_back(cr > 0 ? 1 : 2);
    }
    const int64_t n = (int64_t)kind.size();
    if (n < 4) throw VpError{VP_ERR_GEOMETRY};
    // simple polygon: no two non-adjacent edges cross (O(n^2), small n)
    if (n <= 4096)
      for (int64_t i = 0; i < n; i++)
        for (int64_t j = i + 2; j < n; j++) {
          if (i == 0 && j == n - 1) continue;
          if (seg_cross(&v[2 * i], &v[2 * ((i + 1) % n)], &v[2 * j], &v[2 * ((j + 1) % n)]))
            throw VpError{VP_ERR_GEOMETRY};
        }
    B.n = n;
    double *dv = vp_alloc<double>(P, 2 * n);
    int8_t *dk = vp_alloc<int8_t>(P, n);
    VP_CUDA(cudaMemcpy(dv, v.data(), sizeof(double) * 2 * n, cudaMemcpyHostToDevice));
    VP_CUDA(cudaMemcpy(dk, kind.data(), n, cudaMemcpyHostToDevice));
    B.pts = dv;
    B.vkind = dk;
    std::vector<double> bb(4 * n);
    for (int64_t i = 0; i < n; i++) {
      const double *a = &v[2 * i], *b = &v[2 * ((i + 1) % n)];
      bb[4 * i] = std::min(a[0], b[0]); bb[4 * i + 1] = std::max(a[0], b[0]);
      bb[4 * i + 2] = std::min(a[1], b[1]); bb[4 * i + 3] = std::max(a[1], b[1]);
    }
    build_bins(P, B, bb, B.reach * (1 + 1e-9), std::max(B.reach, 1e-300));
    return;
  }
  if (bd.kind != VP_BDRY_CHUNKS) throw VpError{VP_ERR_GEOMETRY};
  const int q = bd.q;
  if (q < 2 || q > VP_CHUNK_MAXQ) throw VpError{VP_ERR_UNSUPPORTED};
  const int64_t n = bd.n, qp = q + 1;
  for (int64_t i = 0; i < 2 * n * qp; i++)
    if (!std::isfinite(bd.pts[i])) throw VpError{VP_ERR_NONFINITE};
  std::vector<double> s, w;
  vp_gauss_legendre(q + 1, s, w);  // increasing nodes on [-1, 1]
  // Legendre coefficients c_m = (2m+1)/2 sum_k w_k P_m(s_k) gamma_k (exact for the degree-q interpolant)
  std::vector<double> coef((size_t)n * qp * 2, 0.0);
  for (int64_t c = 0; c < n; c++)
    for (int k = 0; k < qp; k++) {
      double P0 = 1.0, P1 = s[k];
      for (int m = 0; m <= q; m++) {
        const double Pm = m == 0 ? 1.0 : P1;
        const double f = 0.5 * (2 * m + 1) * w[k] * Pm;
        coef[((size_t)c * qp + m) * 2] += f * bd.pts[(c * qp + k) * 2];
        coef[((size_t)c * qp + m) * 2 + 1] += f * bd.pts[(c * qp + k) * 2 + 1];
        if (m >= 1) {
          const double Pn = ((2 * m + 1) * s[k] * P1 - m * P0) / (m + 1);
          P0 = P1;
          P1 = Pn;
        }
      }
    }
  auto evalc = [&](int64_t c, double t, double *g, double *g1) {
    double P0 = 1.0, P1 = t, D0 = 0.0, D1 = 1.0;
    g[0] = coef[(size_t)c * qp * 2]; g[1] = coef[(size_t)c * qp * 2 + 1];
    g1[0] = g1[1] = 0.0;
    for (int m = 1; m <= q; m++) {
      g[0] += coef[((size_t)c * qp + m) * 2] * P1; g[1] += coef[((size_t)c * qp + m) * 2 + 1] * P1;
      g1[0] += coef[((size_t)c * qp + m) * 2] * D1; g1[1] += coef[((size_t)c * qp + m) * 2 + 1] * D1;
      const double Pn = ((2 * m + 1) * t * P1 - m * P0) / (m + 1), Dn = D0 + (2 * m + 1) * P1;
      P0 = P1; P1 = Pn; D0 = D1; D1 = Dn;
    }
  };
  // closed curve: each chunk's end meets the next chunk's start; CCW (positive enclosed area); gap between nodes
  double area = 0.0, gap = 0.0, len_min = 1e300, len_max = 0.0;
  for (int64_t c = 0; c < n; c++) {
    double e1[2], e0[2], d[2], len = 0.0;
    evalc(c, 1.0, e1, d);
    evalc((c + 1) % n, -1.0, e0, d);
    for (int k = 0; k < qp; k++) {
      double g[2], g1[2];
      evalc(c, s[k], g, g1);
      area += w[k] * (g[0] * g1[1] - g[1] * g1[0]) * 0.5;
      len += w[k] * std::hypot(g1[0], g1[1]);
      const double *a = bd.pts + (c * qp + k) * 2;
      const double *b = k + 1 < qp ? a + 2 : bd.pts + (((c + 1) % n) * qp) * 2;
      gap = std::max(gap, std::hypot(b[0] - a[0], b[1] - a[1]));
    }
    len_min = std::min(len_min, len);
    len_max = std::max(len_max, len);
    if (std::hypot(e1[0] - e0[0], e1[1] - e0[1]) > 1e-6 * len) throw VpError{VP_ERR_GEOMETRY};
  }
  if (!(area > 0) || !(len_min > 0)) throw VpError{VP_ERR_GEOMETRY};
  B.n = n;
  B.q = q;
  B.gap = gap;
  B.len_max = len_max;
  double *dp = vp_alloc<double>(P, 2 * n * qp), *dc = vp_alloc<double>(P, 2 * n * qp), *ds = vp_alloc<double>(P, qp);
  VP_CUDA(cudaMemcpy(dp, bd.pts, sizeof(double) * 2 * n * qp, cudaMemcpyHostToDevice));
  VP_CUDA(cudaMemcpy(dc, coef.data(), sizeof(double) * 2 * n * qp, cudaMemcpyHostToDevice));
  VP_CUDA(cudaMemcpy(ds, s.data(), sizeof(double) * qp, cudaMemcpyHostToDevice));
  B.pts = dp;
  B.coef = dc;
  B.snode = ds;
  std::vector<double> bb(4 * n * qp);
  for (int64_t i = 0; i < n * qp; i++) {
    bb[4 * i] = bb[4 * i + 1] = bd.pts[2 * i];
    bb[4 * i + 2] = bb[4 * i + 3] = bd.pts[2 * i + 1];
  }
  // every node within reach + gap of a point is in that point's 3 x 3 bin neighbourhood
  build_bins(P, B, bb, 0.0, B.reach + gap);
}
