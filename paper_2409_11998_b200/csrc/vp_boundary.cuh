// vp_boundary.cuh -- boundary geometry of the local part V_L (§2.2; §4 eq. (vplocO5)).
//
// A target x within reach = 12 sqrt(delta) of the boundary gets the boundary form of V_L (PAPER.md lines 665-667:
// "the local part of the heat kernel has decayed to less than 1e-14 at that distance"):
//   CHUNKS  (smooth closed curve as n chunks of degree q): the closest point b is found
//           as the paper does (lines 668-674): the nearest discretisation node as the initial guess, then Newton
//           steps on (gamma(s) - x) . gamma'(s) = 0 along the chunk's Legendre interpolant (stepping into the
//           neighbouring chunk when s leaves [-1, 1]); V_L = eq. (vplocO5) with kappa_b, the inward normal at b.
//           An ambiguous closest point (a second, non-adjacent piece of the curve as close, or x beyond the
//           centre of curvature: the medial axis) is VP_ERR_GEOMETRY (the paper assumes uniqueness, lines 660-665).
//   POLYGON (straight edges, right-angle corners; R8): the exact product form over the local model
//           region seen within reach -- a half plane (one edge), a quadrant (convex corner) or the plane minus a
//           quadrant (reflex corner) -- in the edge frame, rotated to the global Taylor basis.  Anything else
//           within reach (two edges that do not meet, three edges) is VP_ERR_GEOMETRY.
//   CIRCLE / RECT: analytic special cases (vp_math.cuh).
#pragma once
#include "vp_common.cuh"
#include "vp_math.cuh"

// Legendre interpolant of chunk c at s: position, first and second derivative in s
__device__ __forceinline__ void vp_chunk_eval(const VpBdryDev &B, int64_t c, double s, double *g, double *g1,
                                              double *g2) {
  const double *cf = B.coef + c * (int64_t)(B.q + 1) * 2;
  double P0 = 1.0, P1 = s, D0 = 0.0, D1 = 1.0, E0 = 0.0, E1 = 0.0;
  g[0] = cf[0]; g[1] = cf[1];
  g1[0] = g1[1] = g2[0] = g2[1] = 0.0;
  for (int m = 1; m <= B.q; m++) {
    // (P, D, E) = (P_m, P_m', P_m'') at s
    const double P = P1, D = D1, E = E1;
    g[0] += cf[2 * m] * P; g[1] += cf[2 * m + 1] * P;
    g1[0] += cf[2 * m] * D; g1[1] += cf[2 * m + 1] * D;
    g2[0] += cf[2 * m] * E; g2[1] += cf[2 * m + 1] * E;
    const double Pn = ((2 * m + 1) * s * P1 - m * P0) / (m + 1);
    const double Dn = D0 + (2 * m + 1) * P1;
    const double En = E0 + (2 * m + 1) * D1;
    P0 = P1; P1 = Pn; D0 = D1; D1 = Dn; E0 = E1; E1 = En;
  }
}

// Newton from (chunk c, parameter s) to the local minimiser of |gamma(s) - x|; returns the distance, the chunk
// and parameter reached, the inward normal and the signed curvature there.
__device__ inline double vp_chunk_closest(const VpBdryDev &B, double x, double y, int64_t c, double s, int64_t *oc,
                                          double *os, double *nx, double *ny, double *kap) {
  double g[2], g1[2], g2[2];
  for (int it = 0; it < 24; it++) {
    vp_chunk_eval(B, c, s, g, g1, g2);
    const double ex = g[0] - x, ey = g[1] - y;
    const double phi = ex * g1[0] + ey * g1[1];
    const double dphi = g1[0] * g1[0] + g1[1] * g1[1] + ex * g2[0] + ey * g2[1];
    double ds = dphi > 0 ? -phi / dphi : -phi / (g1[0] * g1[0] + g1[1] * g1[1]);
    if (ds > 0.5) ds = 0.5;
    if (ds < -0.5) ds = -0.5;
    s += ds;
    if (s > 1.0) {  // continue on the next chunk (CCW order); parameters of neighbours are comparable in speed
      c = (c + 1) % B.n;
      s -= 2.0;
    } else if (s < -1.0) {
      c = (c - 1 + B.n) % B.n;
      s += 2.0;
    }
    if (fabs(ds) < 1e-15) break;
  }
  vp_chunk_eval(B, c, s, g, g1, g2);
  const double sp = sqrt(g1[0] * g1[0] + g1[1] * g1[1]);
  // CCW curve: the interior lies to the left of the tangent
  *nx = -g1[1] / sp;
  *ny = g1[0] / sp;
  *kap = (g1[0] * g2[1] - g1[1] * g2[0]) / (sp * sp * sp);
  *oc = c;
  *os = s;
  return sqrt((g[0] - x) * (g[0] - x) + (g[1] - y) * (g[1] - y));
}

__device__ __forceinline__ double vp_seg_dist(double x, double y, const double *a, const double *b, double *t) {
  const double dx = b[0] - a[0], dy = b[1] - a[1];
  double u = ((x - a[0]) * dx + (y - a[1]) * dy) / (dx * dx + dy * dy);
  u = u < 0 ? 0 : (u > 1 ? 1 : u);
  *t = u;
  const double ex = a[0] + u * dx - x, ey = a[1] + u * dy - y;
  return sqrt(ex * ex + ey * ey);
}

__device__ __forceinline__ bool vp_chunks_adjacent(int64_t a, int64_t b, int64_t n) {
  const int64_t d = a > b ? a - b : b - a;
  return d <= 1 || d == n - 1;
}

// Boundary form of V_L at (x, y) for local time delta (<= delta_1): 1 = coef filled, 0 = interior (caller uses the
// interior series), -1 = geometry error (flagged in B.err).
__device__ inline int vp_bdry_coef(const VpBdryDev &B, double x, double y, double delta, int nterms, int deg,
                                   double *coef) {
  if (B.kind == VP_BDRY_NONE) return 0;
  if (B.kind == VP_BDRY_CIRCLE) return vp_coef_circle(x, y, B.p[0], B.p[1], B.p[2], delta, nterms, deg, coef) ? 1 : 0;
  if (B.kind == VP_BDRY_RECT) return vp_coef_rect(x, y, B.p[0], B.p[1], B.p[2], B.p[3], delta, deg, coef) ? 1 : 0;
  const double reach = 12.0 * sqrt(delta);
  int64_t bx = (int64_t)floor((x - B.bx0) / B.bcell), by = (int64_t)floor((y - B.by0) / B.bcell);
  if (B.kind == VP_BDRY_POLYGON) {
    // edges within reach (the bins hold every edge within B.reach >= reach of the bin)
    if (bx < 0 || by < 0 || bx >= B.nbx || by >= B.nby) return 0;
    const int64_t b = by * B.nbx + bx;
    int64_t e_in[3];
    int ne = 0;
    for (int32_t k = B.bstart[b]; k < B.bstart[b + 1]; k++) {
      const int64_t e = B.bidx[k];
      double t;
      if (vp_seg_dist(x, y, B.pts + 2 * e, B.pts + 2 * ((e + 1) % B.n), &t) < reach) {
        if (ne < 3) e_in[ne] = e;
        ne++;
      }
    }
    if (ne == 0) return 0;
    double cloc[VP_NTAYLOR];
    if (ne == 1) {  // half plane in the edge frame: a = tangent, b = inward normal
      const double *A = B.pts + 2 * e_in[0], *C = B.pts + 2 * ((e_in[0] + 1) % B.n);
      double tx = C[0] - A[0], ty = C[1] - A[1], L = sqrt(tx * tx + ty * ty);
      tx /= L; ty /= L;
      const double nx = -ty, ny = tx;
      const double lo2 = (A[0] - x) * nx + (A[1] - y) * ny;  // edge at s2 = lo2 (<= 0 inside)
      vp_coef_box(-INFINITY, INFINITY, lo2, INFINITY, delta, deg, cloc);
      vp_coef_rotate(cloc, tx, ty, nx, ny, deg, coef);
      return 1;
    }
    if (ne == 2) {
      int64_t e0 = e_in[0], e1 = e_in[1];
      if ((e0 + 1) % B.n != e1) {  // order so that e1 follows e0
        const int64_t t = e0; e0 = e1; e1 = t;
      }
      if ((e0 + 1) % B.n == e1) {
        const int64_t v = e1;  // shared vertex
        const double *V = B.pts + 2 * v, *A = B.pts + 2 * e0, *C = B.pts + 2 * ((e1 + 1) % B.n);
        // incoming edge direction u (A -> V), outgoing w (V -> C); right angle
        double ux = V[0] - A[0], uy = V[1] - A[1], lu = sqrt(ux * ux + uy * uy);
        double wx = C[0] - V[0], wy = C[1] - V[1], lw = sqrt(wx * wx + wy * wy);
        ux /= lu; uy /= lu; wx /= lw; wy /= lw;
        const double sx = (V[0] - x), sy = (V[1] - y);
        if (B.vkind[v] == 1) {
          // convex corner: interior = {(y - V) . w >= 0 along ... } -- in the frame (a, b) = (w, -u): the quadrant
          // s1 >= (V - x) . w, s2 >= (V - x) . (-u)
          const double ax = wx, ay = wy, bxx = -ux, byy = -uy;
          vp_coef_box(sx * ax + sy * ay, INFINITY, sx * bxx + sy * byy, INFINITY, delta, deg, cloc);
          vp_coef_rotate(cloc, ax, ay, bxx, byy, deg, coef);
          return 1;
        }
        if (B.vkind[v] == 2) {
          // reflex corner (right turn): the same frame (a, b) = (w, -u) now bounds the EXTERIOR quadrant
          // s1 >= (V - x) . a, s2 >= (V - x) . b; V_L = plane - exterior quadrant
          const double ax = wx, ay = wy, bxx = -ux, byy = -uy;
          double cq[VP_NTAYLOR], cg[VP_NTAYLOR], cp[VP_NTAYLOR];
          vp_coef_box(sx * ax + sy * ay, INFINITY, sx * bxx + sy * byy, INFINITY, delta, deg, cq);
          vp_coef_rotate(cq, ax, ay, bxx, byy, deg, cg);
          vp_coef_box(-INFINITY, INFINITY, -INFINITY, INFINITY, delta, deg, cp);  // plane: frame-independent
          for (int i = 0; i < VP_NTAYLOR; i++) coef[i] = cp[i] - cg[i];
          return 1;
        }
      }
    }
    if (B.err) atomicExch(B.err, 1);
    return -1;
  }
  // CHUNKS: nearest node in the 3 x 3 bins (cell >= reach + gap), then Newton from it
  const int qp = B.q + 1;
  double dn = 1e300;
  int64_t nid = -1;
  for (int64_t yy = by - 1; yy <= by + 1; yy++) {
    if (yy < 0 || yy >= B.nby) continue;
    for (int64_t xx = bx - 1; xx <= bx + 1; xx++) {
      if (xx < 0 || xx >= B.nbx) continue;
      const int64_t b = yy * B.nbx + xx;
      for (int32_t k = B.bstart[b]; k < B.bstart[b + 1]; k++) {
        const int64_t id = B.bidx[k];
        const double px = B.pts[2 * id] - x, py = B.pts[2 * id + 1] - y;
        const double d = px * px + py * py;
        if (d < dn) { dn = d; nid = id; }
      }
    }
  }
  if (nid < 0 || sqrt(dn) >= reach + B.gap) return 0;
  int64_t bch;
  double bs, bnx, bny, bkap;
  double best = vp_chunk_closest(B, x, y, nid / qp, B.snode[nid % qp], &bch, &bs, &bnx, &bny, &bkap);
  double g[2], g1[2], g2[2];
  vp_chunk_eval(B, bch, bs, g, g1, g2);
  double bpx = g[0], bpy = g[1];
  // another piece of the curve nearly as close (a second local minimum of the distance: the medial axis)?  Newton
  // from nodes of chunks not adjacent to the closest point's chunk that lie within best + gap
  int tries = 0;
  for (int64_t yy = by - 1; yy <= by + 1 && best < reach; yy++) {
    if (yy < 0 || yy >= B.nby) continue;
    for (int64_t xx = bx - 1; xx <= bx + 1; xx++) {
      if (xx < 0 || xx >= B.nbx) continue;
      const int64_t b = yy * B.nbx + xx;
      for (int32_t k = B.bstart[b]; k < B.bstart[b + 1]; k++) {
        const int64_t id = B.bidx[k];
        if (vp_chunks_adjacent(id / qp, bch, B.n)) continue;
        const double px = B.pts[2 * id] - x, py = B.pts[2 * id + 1] - y;
        if (sqrt(px * px + py * py) >= best + B.gap) continue;
        if (++tries > 16) {  // many distant pieces of the curve within reach: not a unique closest point
          if (B.err) atomicExch(B.err, 1);
          return -1;
        }
        int64_t c2;
        double s2, nx2, ny2, k2;
        const double d2 = vp_chunk_closest(B, x, y, id / qp, B.snode[id % qp], &c2, &s2, &nx2, &ny2, &k2);
        double h[2], h1[2], h2[2];
        vp_chunk_eval(B, c2, s2, h, h1, h2);
        const double sep = sqrt((h[0] - bpx) * (h[0] - bpx) + (h[1] - bpy) * (h[1] - bpy));
        if (sep <= B.gap) continue;  // converged to the same closest point
        if (d2 <= best * (1.0 + 1e-6) + 1e-300) {  // a second, distinct minimiser as close (or closer)
          if (B.err) atomicExch(B.err, 1);
          return -1;
        }
      }
    }
  }
  if (best >= reach) return 0;
  // inside / outside: the target lies on the interior side when (x - b) . n >= 0; outside -> on the boundary
  const double side = (x - bpx) * bnx + (y - bpy) * bny;
  const double r = side > 0 ? best : 0.0;
  if (bkap > 0 && r * bkap >= 0.9) {  // at or beyond the centre of curvature: the medial axis
    if (B.err) atomicExch(B.err, 1);
    return -1;
  }
  vp_coef_smooth(r, bnx, bny, bkap, delta, nterms, deg, coef);
  return 1;
}

// host side (vp_boundary.cu): validate the descriptor, upload the geometry and bins (plan-owned)
void vp_build_boundary(vp_plan_s *P, VpBdryDev &B);
