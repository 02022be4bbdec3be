// vp_common.cuh -- plan layout and shared device/host helpers of libvp.so (product path).
// No code here is shared with oracle/ (test infrastructure).
#pragma once
#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/vp.h"

#define VP_PI 3.14159265358979323846
#define VP_TRI_MAXP 32

// ---------------------------------------------------------------------------------------------
// error plumbing: every CUDA / cuFFT call inside the library goes through these
struct VpError {
  vp_status s;
};
#define VP_CUDA(x)                                                 \
  do {                                                             \
    cudaError_t e_ = (x);                                          \
    if (e_ != cudaSuccess) {                                       \
      vp_set_last_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
      throw VpError{e_ == cudaErrorMemoryAllocation ? VP_ERR_OOM : VP_ERR_CUDA}; \
    }                                                              \
  } while (0)
#define VP_CUFFT(x)                                                \
  do {                                                             \
    cufftResult r_ = (x);                                          \
    if (r_ != CUFFT_SUCCESS) {                                     \
      vp_set_last_error(std::string(#x) + ": cufft error " + std::to_string((int)r_)); \
      throw VpError{r_ == CUFFT_ALLOC_FAILED ? VP_ERR_OOM : VP_ERR_CUFFT}; \
    }                                                              \
  } while (0)
#define VP_CHECK_LAUNCH() VP_CUDA(cudaGetLastError())

void vp_set_last_error(const std::string &s);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel) and size; thread safe (a mutex-
// guarded cache keyed by the current device, so a plan on a second device sets its own attribute)
void vp_smem_attr(const void *func, size_t bytes);
// current device (cached per call site is not safe across devices: always ask the runtime)
int vp_current_device();
// SM count of the current device (plans may live on different devices)
inline int vp_num_sms() {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, vp_current_device());
  return n > 0 ? n : 1;
}

// ---------------------------------------------------------------------------------------------
// ES kernel taps as Horner polynomials: psi(z_k(t)), z_k = (k + (t+1)/2 - W/2) 2/W, t in [-1, 1]
#define VP_HORNER_MAXW 16
#define VP_HORNER_DEG(W) ((W) <= 8 ? ((W) + 1) : ((W)-1))  // fit error ~0.16 x 10^-(W-1): the kernel's edge value
struct VpHorner {
  double c[VP_HORNER_MAXW][VP_HORNER_MAXW];  // c[k][j]: coefficient of t^j for tap k
};

// ---------------------------------------------------------------------------------------------
// One uniform periodic fine grid of the NUFFT (§3).
// Point x lies at fractional grid coordinate g = (x - o)/h; grid node i sits at o + i h.
struct VpGrid {
  int64_t nf = 0;     // fine points per dimension (even, 2,3,5,7-smooth)
  int64_t nmode = 0;  // kept modes per dimension (even); |m| <= nmode/2
  int64_t row = 0;    // real grid row length in doubles (nf)
  int64_t crow = 0;   // half-spectrum row length in doubles: 2 (nf/2 + 1)
  double L = 0, h = 0, ox = 0, oy = 0;
  double delta_a = 0, delta_b = 0;  // NH: (delta1, delta2); FH: (delta2, R)
  int kind = 0;                     // 0 = near history, 1 = far history
  double *data = nullptr;           // nf * row doubles (real grid)
  double *cdata = nullptr;          // nf * crow doubles (half spectrum; out-of-place D2Z / Z2D)
  double *deconv = nullptr;         // [nmode/2+1]: 1 / Phi(k_m)^2 (1D kernel transform, squared inverse)
  double mult_scale = 0;            // h^2 / nf^2 (NH);  h2^2 h1^4 / nf2^2 (FH, two-stage kernel)
  cufftHandle fwd = 0, inv = 0;
  bool has_plans = false;
  // fused transform (vp_fft.cu): row pass, column pass with the multiply, inverse row pass
  bool own_fft = false;
  int fft_ncs = 0;                                 // kept columns (nmode/2 + 1)
  double2 *tw_r = nullptr, *tw_c = nullptr;        // W_{nf/2}^j, W_nf^j
  int32_t *pos_r = nullptr, *sig_c = nullptr;      // digit-reversal maps (row: frequency -> position)
  double2 *spec2 = nullptr;                        // column-pass output, row-major [nf][ncs]
  double *fft_mult = nullptr;                      // multiplier table [ncs][nf] in DIF output order
  alignas(8) char fft_st_r[256] = {}, fft_st_c[256] = {};  // FftStages (row length nf/2, column length nf)
  // four-step column pass for large grids (vp_fft.cu, nf = f4_N1 f4_N2; fft_st_r / fft_st_c hold the N1 / N2
  // stages): rows by cuFFT batched 1D plans (rfwd / rinv)
  bool four_step = false;
  int f4_N1 = 0, f4_N2 = 0;
  double2 *f4_tw1 = nullptr, *f4_tw2 = nullptr, *f4_twN = nullptr;
  int32_t *f4_sig1 = nullptr, *f4_sig2 = nullptr;
  double *f4_e1 = nullptr, *f4_e2 = nullptr;  // NH: e^{-dk^2 m^2 delta_a}, e^{-dk^2 m^2 delta_b}
  // own row passes (k_row4_fwd / k_row4_inv; nf % 4 == 0): Q = nf / 4 point transforms
  bool f4_rows = false;
  int32_t *f4_posQ = nullptr;
  double2 *f4_twQ = nullptr;
  alignas(8) char f4_stQ[256] = {};
};

struct VpTiles {          // sorted points binned into TS x TS tiles of a fine grid
  int TS = 32;
  int64_t ntx = 0, nty = 0;
  int64_t nsub = 0;       // spreading sub-problems
  int4 *sub = nullptr;    // (tile_x, tile_y, first batch, end batch)
};

// Grid description passed to kernels: point x sits at fractional cell (x - o) * inv_h of a periodic
// nfx x nfy grid whose rows are `row` doubles apart.
struct GridArgs {
  double *data;
  int64_t nfx, nfy, row;
  double ox, oy, h, inv_h;
};
inline GridArgs grid_args(const VpGrid &G) { return GridArgs{G.data, G.nf, G.nf, G.row, G.ox, G.oy, G.h, 1.0 / G.h}; }

// Points prepared for the atomic-free tile spreading kernel (vp_nufft.cu k_spread_nh): sorted by
// (tile, row-rank level, row) into batches of <= 32 points with pairwise distinct footprint rows.
struct VpSpreadSet {
  double *sx = nullptr, *sy = nullptr, *sw = nullptr;  // coords (in the grid's frame), weights
  int32_t *sperm = nullptr;                            // sorted -> user node index (f gather)
  int32_t *bstart = nullptr;                           // batch starts (n_batches + 1)
  int64_t n_batches = 0;
  VpTiles tiles;
  int det = 0;                 // deterministic mode: items sorted by tile colour, colour_off[c]..colour_off[c+1]
  int64_t color_off[5] = {};
  double *fs_out = nullptr;    // if set, the spread also writes f in this sorted order
  int strip = 0;               // 2: row-pair strips (k_spread_pair), 1: 32-column strips (k_spread_strip), both
                               // with sitems; 0: tile batches (tiles, bstart)
  int4 *sitems = nullptr;      // (strip_x, strip_y, first point, end point)
  int64_t n_sitems = 0;
};

// Level-band corrections for graded meshes: per-target level
// l(x) in 0..nlev, bands B_l (l = 1..l(x)) by box-local NUFFTs on one "virtual" grid of nbox boxes
// (box b = rows [b nfb, (b+1) nfb)), V_L evaluated with delta_{l(x)} = delta_1 / 4^{l(x)}.
struct VpBands {
  int nlev = 0;                   // finest level present (0 = no bands)
  int64_t nbox = 0, nfb = 0, rowb = 0, nmode = 0;
  int margin = 0, core = 0;       // fine cells
  double *grid = nullptr;         // nbox * nfb * rowb
  int32_t *box_level = nullptr;   // [nbox]
  double *lev_par = nullptr;      // [nlev + 1][4]: delta_l, delta_{l-1}, dk_l, scale_l
  double *deconv = nullptr;       // [nmode/2 + 1] grid-unit 1/Phi^2
  cufftHandle fwd = 0, inv = 0;
  bool has_plans = false;
  VpGrid fg;                      // fused-transform tables and spectra (fg.own_fft) instead of the cuFFT plans
  VpSpreadSet sp;
  int64_t n_lt = 0, n_ent = 0;    // targets with level >= 1; (target, level) entries
  int32_t *lt_t = nullptr;        // [n_lt] sorted target index
  int32_t *lt_off = nullptr;      // [n_lt + 1]
  double *ent_x = nullptr, *ent_y = nullptr;  // [n_ent] virtual-grid coordinates
  int64_t n_pairs = 0;            // (box, source) pairs spread
  int8_t *tlev = nullptr;         // [T] level per sorted target
  // staged interpolation of the entries (k_interp_local on the virtual grid): entries in (tile, bank) order
  double *e_x = nullptr, *e_y = nullptr;
  int32_t *e_perm = nullptr;      // staged order -> entry index
  int4 *e_items = nullptr;
  int64_t e_n_items = 0;
  double *ent_val = nullptr;      // [n_ent] band value per entry
  int64_t lev_count[16] = {};     // targets per level
};

// Boundary geometry of the local part V_L on the device (vp_boundary.cuh, vp_boundary.cu)
#define VP_CHUNK_MAXQ 32

struct VpBdryDev {
  int kind = VP_BDRY_NONE;
  int q = 0;            // CHUNKS: degree
  int64_t n = 0;        // POLYGON: vertices (after merging straight ones); CHUNKS: chunks
  double p[4] = {0, 0, 0, 0};
  const double *pts = nullptr;    // POLYGON [n][2] vertices; CHUNKS [n][q+1][2] nodes
  const double *coef = nullptr;   // CHUNKS [n][q+1][2] Legendre coefficients of gamma on [-1, 1]
  const double *snode = nullptr;  // CHUNKS [q+1] Gauss-Legendre points of [-1, 1] (node parameters)
  const int8_t *vkind = nullptr;  // POLYGON [n]: 1 convex right angle, 2 reflex right angle
  // uniform bins over the boundary's bounding box (+ reach): CHUNKS -> node ids (chunk * (q+1) + k),
  // POLYGON -> edge ids (edge i joins vertex i and i+1)
  double bx0 = 0, by0 = 0, bcell = 1;
  int64_t nbx = 0, nby = 0;
  const int32_t *bstart = nullptr, *bidx = nullptr;
  double reach = 0;    // 12 sqrt(delta_1) (the largest delta used)
  double gap = 0;      // CHUNKS: largest distance between consecutive nodes (incl. across chunk ends)
  double len_max = 0;  // CHUNKS: longest chunk (arc length)
  int *err = nullptr;  // device flag: set to 1 on an ambiguous closest point / unsupported local geometry
};

struct vp_plan_s {
  // sizes
  int64_t M = 0, N = 0, T = 0;
  int32_t p = 0;
  double tol = 0, eps = 0;
  vp_opts opts{};
  cudaStream_t stream = nullptr;       // the caller's stream (A): spread, NH chain, interpolation
  cudaStream_t s_fh = nullptr, s_loc = nullptr;  // forked streams: FH chain (B), local part (C)
  cudaEvent_t ev_fork = nullptr, ev_fh = nullptr, ev_loc = nullptr, ev_restr = nullptr;
  bool concurrent = true;              // fork/join eval (off while profiling: phases need serial order)
  // parameters
  double dx2 = 0, delta1 = 0, delta2 = 0, kmax_nh = 0, kmax_fh = 0, R = 0, S = 0, cx = 0, cy = 0;
  int w = 0;
  double beta = 0;
  VpGrid nh, fh;
  int fh_ratio = 1;         // h_FH = fh_ratio * h_NH
  int64_t fh_shift = 0;     // FH node i' sits on NH node fh_ratio * i' - fh_shift
  int tap_qh = 0;           // integer-ratio restriction taps w[q + QH], |q| <= QH (0: general tables)
  double tap_w[192] = {};
  VpHorner horner{};
  double horner_err = 0;
  // sources, sorted by (NH tile, row rank, row) into batches of <= 32 points with distinct rows
  VpSpreadSet sp;
  // graded-mesh level bands (a12)
  VpBands bands;
  VpBdryDev bdev;  // boundary geometry for V_L (plan-owned device copies; vp_build_boundary)
  // single-layer potential on the plan's grids (vp_layer.cu, vp_slp_prepare): boundary sources in strip order,
  // local stencils (chunk + q+1 weights) of the targets within 12 sqrt(delta_1) of the boundary
  bool slp_ready = false;
  VpSpreadSet bsp;
  double *slp_swt = nullptr;  // [q+1] Gauss-Legendre weights of [-1, 1]
  int64_t slp_n = 0;
  int32_t *slp_list = nullptr, *slp_chunk = nullptr;
  double *slp_w = nullptr;
  bool lay_common = false;  // slp_swt and the near list slp_list / slp_n (shared by S and D)
  // telescoped local parts (§4.1): J levels, NC chunk slots per near target, NP quadrature panels per chunk
  int lay_J = 3, lay_nc = 1, lay_np = 1;
  double *lay_tq = nullptr, *lay_tq1 = nullptr, *lay_gw = nullptr, *lay_lg = nullptr;
  double *lay_W = nullptr;  // [n (q+1)] boundary quadrature weights (set by vp_dlp_prepare)
  // double-layer potential (vp_dlp_prepare): dipole source sets W nu_1, W nu_2, local stencils, spectral derivative
  bool dlp_ready = false, dlp_has_plans = false;
  VpSpreadSet dsp1, dsp2;
  int32_t *dlp_chunk = nullptr;
  double *dlp_w = nullptr;
  double2 *dlp_spec[2] = {nullptr, nullptr};  // [NH, FH]: two half spectra each
  cufftHandle dlp_fwd[2] = {0, 0}, dlp_inv[2] = {0, 0};
  // FH <- NH restriction tables
  int32_t *r_lo = nullptr, *t_lo = nullptr;
  double *r_w = nullptr, *t_w = nullptr;
  int r_ntap = 0, t_ntap = 0;
  int64_t e_lo = 0, e_n = 0;
  double *scratch = nullptr;                           // n1 x e_n
  // targets, sorted by (TSI x TSI NH-grid tile, bank-slot rank) and cut into interpolation work items
  double *tx = nullptr, *ty = nullptr;
  int32_t *tperm = nullptr;  // sorted -> user target index (T < 2^31, checked in vp_plan)
  int TSI = 64;
  int4 *items = nullptr;     // (tile_x, tile_y, first target, end target)
  int64_t n_items = 0;
  // local part: V_L(t) = alpha_t * f(node_t) + sum_k omega_{t,k} f[idx_{t,k}]
  int K = 0, deg = 0, dmode = 0;
  int32_t *lidx = nullptr;     // [T][K] user node indices (sorted target order)
  double *lw = nullptr;        // [S][K] stencil weights
  double *lalpha = nullptr;    // [T]
  int32_t *lnode = nullptr;    // [T] user node index of the target (targets_are_nodes) or -1
  int64_t n_bdry = 0;
  int32_t *lptr = nullptr;     // [T] stencil slot of the target, -1 = TRIANGLE mode
  int64_t n_stencil = 0;
  int8_t *tri_ok = nullptr;    // [M] TRIANGLE mode usable
  double *tri_M = nullptr;     // [M][3] A^-1 A^-T (M11, M12, M22)
  double *tri_H = nullptr;     // [3][p][p] reference cubic-fit Hessian operators
  std::vector<double> tri_H_host;
  int trih_slot = -1;          // constant-bank slot of tri_H (p = 12), -1: shared-memory kernel
  double tri_c2 = 0;           // delta^2 / 2 (0 if series_order < 2)
  double *tri_vL = nullptr;    // [N] TRIANGLE-mode V_L per node (eval scratch; null outside TRIANGLE mode)
  double *st_vL = nullptr;     // [n_stencil] stencil part of V_L per stencil slot (eval scratch)
  double *fs = nullptr;        // [N] f in spreading order (eval scratch; stencil indices point into it)
  double *bgrid = nullptr;     // vp_eval_batch: (bcap - 1) extra NH grids
  double *fs_batch = nullptr;  // vp_eval_batch: [bcap][N] spreading-order copies of the fields (KNN stencils)
  int bcap = 1;
  // host-side eval staging (vp_eval_host)
  double *f_dev = nullptr, *out_dev = nullptr;
  // vp_eval_host_many: two device slots for f and out, copy streams and their events (allocated on first use)
  bool hm_ready = false;
  double *hm_f[2] = {nullptr, nullptr}, *hm_out[2] = {nullptr, nullptr};
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t hm_ev[7] = {};  // start, in[2], done[2], out[2]
  // profiling
  bool profiling = false;
  cudaEvent_t ev[12] = {};
  bool ev_init = false;
  double phase_ms[12] = {};
  int n_phase = 0;
  double plan_ms = 0;
  int64_t device_bytes = 0;
  std::vector<void *> allocs;
  int32_t n_kernels = 0, n_ffts = 0;
};

// device allocation tracked by the plan
template <typename T>
T *vp_alloc(vp_plan_s *P, size_t n) {
  void *p = nullptr;
  if (n == 0) n = 1;
  VP_CUDA(cudaMalloc(&p, n * sizeof(T)));
  P->allocs.push_back(p);
  P->device_bytes += (int64_t)(n * sizeof(T));
  return (T *)p;
}

// release one tracked allocation (nullptr accepted)
inline void vp_free(vp_plan_s *P, void *p) {
  if (!p) return;
  for (size_t i = 0; i < P->allocs.size(); i++)
    if (P->allocs[i] == p) {
      P->allocs.erase(P->allocs.begin() + i);
      cudaFree(p);
      return;
    }
}

// ---------------------------------------------------------------------------------------------
// launch helpers (defined in the .cu files)
void vp_launch_spread(vp_plan_s *P, const VpSpreadSet &S, const GridArgs &g, const double *f);
void vp_build_spread_order(vp_plan_s *P, VpSpreadSet &S, const double *xy, const double *w, const int32_t *node_of,
                           int64_t n, const GridArgs &g);
void vp_build_levels(vp_plan_s *P, const double *nodes, const double *weights);
void vp_launch_bands(vp_plan_s *P, const double *f, double *out);
double vp_solve_e1(double eps);
int64_t vp_next_smooth(int64_t n);
void vp_es_deconv_table(const vp_plan_s *P, double h, double L, int64_t nhalf, std::vector<double> &out);
void vp_upload_horner(int W, const VpHorner &h);
void vp_launch_restrict(vp_plan_s *P);
void vp_launch_prolong(vp_plan_s *P, int pass);
void vp_launch_tri_local(vp_plan_s *P, const double *f);
void vp_launch_multiply(vp_plan_s *P, VpGrid &G);
void vp_launch_interp_local(vp_plan_s *P, const double *f, double *out, bool local_kernels);
void vp_launch_interp_hist(vp_plan_s *P, double *out);  // history part only (no local part), out = u_H
void vp_slp_build(vp_plan_s *P);                         // vp_layer.cu
void vp_launch_slp_local(vp_plan_s *P, const double *sigma, double *out);
void vp_dlp_build(vp_plan_s *P);                         // vp_layer.cu
void vp_dlp_source_grids(vp_plan_s *P, const double *mu);
void vp_launch_dlp_local(vp_plan_s *P, const double *mu, double *out);
void vp_build_interp_order(vp_plan_s *P, const double *xy, int64_t n);
void vp_fft_setup(vp_plan_s *P, VpGrid &G);
void vp_fft_forward(vp_plan_s *P, VpGrid &G);
void vp_fft_columns(vp_plan_s *P, VpGrid &G);
void vp_fft_inverse(vp_plan_s *P, VpGrid &G);
bool vp_fft4_setup(vp_plan_s *P, VpGrid &G);
bool vp_fft4_rows_setup(vp_plan_s *P, VpGrid &G);
void vp_fft4_rows_fwd(vp_plan_s *P, VpGrid &G);
struct RowProlong;
void vp_fft4_rows_inv(vp_plan_s *P, VpGrid &G, const RowProlong *pr = nullptr);
bool vp_fft4_rows_prolong_ok(vp_plan_s *P);
void vp_fft4_rows_inv_prolong(vp_plan_s *P);  // NH inverse rows + prolongation x pass (after pass 1)
void vp_fft4_columns(vp_plan_s *P, VpGrid &G);
void vp_launch_spread_batch(vp_plan_s *P, const VpSpreadSet &S, const GridArgs &g, int K, const double *const *f,
                            double *const *grids, double *const *fs);
bool vp_fft_setup_bands(vp_plan_s *P);
void vp_fft_bands(vp_plan_s *P);
void vp_build_strip_order(vp_plan_s *P, VpSpreadSet &S, const double *xy, const double *weights,
                          const int32_t *node_of, int64_t n, const GridArgs &g);
void vp_build_interp_order_g(vp_plan_s *P, const double *xy, int64_t n, const GridArgs &g, double **otx,
                             double **oty, int32_t **otperm, int4 **oitems, int64_t *on_items);
void vp_remap_stencils(vp_plan_s *P);
void vp_build_local(vp_plan_s *P, const double *nodes_dev);
void vp_cubic_hessian_ops(const double *ref, int p, std::vector<double> &Hop);
int vp_acquire_trih_slot(const double *hop432);
int64_t vp_sort_points(vp_plan_s *P, const double *xy, int64_t n, double ox, double oy, double cell,
                       int64_t nbx, int64_t nby, double *xs, double *ys, int64_t *perm64, int32_t *perm32,
                       int64_t **bin_start_out);
