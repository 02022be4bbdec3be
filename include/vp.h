/*
 * vp.h -- C ABI of the B200-native volume-potential evaluator (libvp.so).
 *
 * Computes the 2D Poisson volume potential (§1, eqs. (volpotposgreen)/(GreenPoisson),
 * lines 55-68)
 *
 *     V[f](x) = \int_Omega -(1/2pi) log|x - x'| f(x') dx'
 *
 * from source values f at the nodes of a p-point quadrature rule on each of M triangles
 * (§2.2: "Omega* = U T_j ... p-point quadrature rule ... N = Mp"),
 * with the paper's heat-kernel splitting V = V_L + V_NH + V_FH (eqs. (heatdecomp),
 * (heatdecompdefs), lines 264-286):
 *   - V_NH + V_FH (the "history") via a NUFFT: type-1 spreading of f*w onto two uniform grids,
 *     FFT, multiplication by the split kernels' transforms, inverse FFT, type-2 interpolation
 *     (§3, Steps 1-4, lines 767-898);
 *   - V_L (the local part) from the asymptotic expansion at each target (§4,
 *     eq. (vplocO5) lines 1061-1087 with the sign reading of DESIGN.md, and the interior /
 *     on-boundary forms lines 1116-1127).
 *
 * All array arguments are DEVICE pointers (CUDA global memory, e.g. from torch tensors) unless
 * the function name ends in _host.  Layouts are C-contiguous, fp64.  No exception crosses the
 * ABI: every entry point returns a vp_status; vp_strerror() gives a static message.
 * Thread safety: distinct plans (also on distinct devices) may be used concurrently -- constant-bank tables are
 * per device and never overwritten with different contents; one plan must not be evaluated concurrently with
 * itself (it owns scratch grids).
 */
#ifndef VP_H_
#define VP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  VP_OK = 0,
  VP_ERR_ARG = -1,          /* null pointer, non-positive size, inconsistent option */
  VP_ERR_TOL = -2,          /* tol outside [1e-14, 1e-2] */
  VP_ERR_NONFINITE = -3,    /* NaN/Inf in nodes, weights, targets or f */
  VP_ERR_GEOMETRY = -4,     /* boundary descriptor invalid / targets outside it */
  VP_ERR_UNSUPPORTED = -5,  /* option combination not implemented */
  VP_ERR_OOM = -6,          /* device allocation failed or grid too large */
  VP_ERR_CUDA = -7,         /* CUDA runtime error */
  VP_ERR_CUFFT = -8         /* cuFFT error */
} vp_status;

/* Boundary of Omega, needed by the boundary-aware local part V_L (§4, eq. (vplocO5);
 * §2.2: boundary chunks and the closest point b).  A target within 12 sqrt(delta_1) of the boundary
 * gets the boundary form of V_L; others the interior series.
 *   NONE    no boundary terms (valid when f vanishes within 12 sqrt(delta_1) of the boundary).
 *   CHUNKS  a smooth closed curve, counter-clockwise (interior on the left), as n chunks of degree q = q_B in
 *           [2, 32] ("a polynomial of degree q_B ... at least q_B + 1 points on each
 *           segment"; reading R17: the q + 1 points of a chunk sample the curve at the Gauss-Legendre points of
 *           the chunk's parameter interval [-1, 1], in increasing order, and consecutive chunks share their end
 *           points).  pts = HOST array [n][q+1][2].  The closest point is the nearest node refined by Newton steps
 *           (lines 668-674); an ambiguous closest point within 12 sqrt(delta_1) of a target (medial axis) is
 *           VP_ERR_GEOMETRY; ends of consecutive chunks more than 1e-6 x chunk length apart, or a clockwise
 *           curve, is VP_ERR_GEOMETRY.
 *   POLYGON straight edges with right-angle corners (convex or reflex, any orientation; collinear vertices are
 *           merged), counter-clockwise, simple.  pts = HOST array [n][2].  Exact product-form V_L over the local
 *           half plane / quadrant / plane-minus-quadrant (R8; the paper is silent on corners).  A corner
 *           that is not a right angle is VP_ERR_UNSUPPORTED; a target within 12 sqrt(delta_1) of two edges that do
 *           not meet at a corner (a feature thinner than 24 sqrt(delta_1)) is VP_ERR_GEOMETRY.
 *   CIRCLE  analytic circle: p = (cx, cy, radius).
 *   RECT    analytic axis-aligned rectangle: p = (x0, y0, x1, y1) (all four sides and corners at once).
 * pts is read during vp_plan only (the plan keeps device copies). */
enum { VP_BDRY_NONE = 0, VP_BDRY_CIRCLE = 1, VP_BDRY_RECT = 2, VP_BDRY_POLYGON = 3, VP_BDRY_CHUNKS = 4 };
typedef struct {
  int32_t kind;       /* VP_BDRY_* */
  int32_t q;          /* CHUNKS: degree q_B (q + 1 nodes per chunk) */
  int64_t n;          /* POLYGON: vertices; CHUNKS: chunks */
  const double *pts;  /* HOST.  POLYGON [n][2]; CHUNKS [n][q+1][2] */
  double p[4];        /* CIRCLE: cx, cy, radius.   RECT: x0, y0, x1, y1 */
} vp_boundary;

/* How the Taylor jet of f at each target is estimated from nodal data (paper silent; DESIGN.md
 * reading R6).  KNN: least-squares fit over the K nearest nodes (stencil stored per target).
 * TRIANGLE: interior node targets of straight triangles with aspect <= tri_max_aspect use the
 * triangle's own p nodes (cubic fit, no per-target storage); all other targets use KNN.
 * AUTO: TRIANGLE when ref_nodes is given and N > 1e7, else KNN. */
enum { VP_DERIV_AUTO = 0, VP_DERIV_KNN = 1, VP_DERIV_TRIANGLE = 2 };
/* which parts of V to evaluate (tests) */
enum { VP_PART_HISTORY = 1, VP_PART_LOCAL = 2, VP_PART_ALL = 3 };

/* Options; a zero-initialised struct (or NULL) means defaults. */
typedef struct {
  double C;                  /* delta_1 = C * Dx^2, Dx^2 = sum(w)/N. 0 -> 3 */
  double delta2_over_delta1; /* 0 -> 32 */
  double delta1_override;    /* > 0: use this delta_1 directly */
  double eps_nufft;          /* NUFFT / truncation tolerance; 0 -> tol */
  int32_t series_order;      /* interior V_L terms n_L in sum_n delta^n Lap^{n-1} f / n!; 0 -> 3 */
  int32_t deriv_mode;        /* VP_DERIV_* */
  int32_t deriv_degree;      /* least-squares polynomial degree for KNN jets; 0 -> 6 (4 if N > 1e6) */
  int32_t deriv_k;           /* neighbours for KNN jets; 0 -> 2 * #monomials (degree >= 5), #monomials + 6 (degree 4) */
  int32_t parts;             /* VP_PART_*; 0 -> ALL */
  int32_t targets_are_nodes; /* 1: targets[t] == tri_nodes[t] for t < N = M p (T >= N; targets beyond N are
                                off-node points); enables the node fast path */
  vp_boundary boundary;
  void *cuda_stream;         /* cudaStream_t for vp_eval; NULL -> legacy default stream */
  /* HOST pointer [p][2] or NULL: reference-triangle coordinates (xi1, xi2) of the p-point rule on
   * (0,0),(1,0),(0,1).  Enables VP_DERIV_TRIANGLE: per-triangle cubic fit in reference coordinates
   * mapped by the triangle's affine Jacobian (straight, well-shaped triangles only; the rest use KNN). */
  const double *ref_nodes;
  double tri_max_aspect;     /* TRIANGLE mode aspect-ratio limit (sigma_max/sigma_min of the map); 0 -> 3 */
  /* Level-band corrections for graded meshes (reading R15; §4.1
   * telescoping "extends naturally to ... volume").  levels: -1 off, 0 auto (as many levels as the mesh
   * grading supports, <= 12), > 0 cap.  A target x gets level l(x) = the finest l such that every node y
   * within level_rho sqrt(delta_l) has delta_l >= level_cmin Dx_loc^2(y), delta_l = delta_1 / 4^l. */
  int32_t levels;
  double level_cmin;         /* 0 -> 1.5 */
  double level_rho;          /* 0 -> 4 */
  /* 1: bit-reproducible vp_eval.  The only order-dependent step of the default path is the fp64 atomic add of
   * spreading-tile halos into the grid; this mode launches the spreading once per tile colour (tx & 1, ty & 1)
   * with one work item per tile and plain read-add-write (slower on dense tiles). */
  int32_t deterministic;
  /* tuning: spread_tile 0 -> register strips (k_spread_strip), 8..64 -> shared-memory tile
   * batches of that side (k_spread_nh; always used in deterministic mode, tile side 32 when 0);
   * interp_tile: interpolation tile side (0 -> 64, 16..128) */
  int32_t spread_tile;
  int32_t interp_tile;
  /* transforms: 0 -> fused row/column FFT with the spectral multiply in the column pass (vp_fft.cu) for
   * grids with nf <= 6400, cuFFT D2Z + multiply + Z2D for 6400 < nf <= 10000, the four-step column pass above;
   * 1 -> cuFFT for every grid */
  int32_t fft_mode;
  /* register-strip spreading: 0 -> row-pair strips (k_spread_pair: 16 columns x 2 row phases
   * per warp) when w <= 12, else 32-column strips; 1 -> 32-column strips with column-disjoint packs of points per
   * step; 2 -> 32-column strips, one point per step (k_spread_strip) */
  int32_t spread_pack;
  /* grids above 10000^2 (four-step column pass): 0 -> own pruned row passes (nf % 4 == 0 and a whole row,
   * 2 x nf/4 complex values, in one CTA's shared memory: nf <= 28160), else cuFFT batched 1D row
   * transforms; 1 -> cuFFT batched 1D row transforms */
  int32_t fft_rows;
  /* vp_eval_batch with row-pair strips at w <= 10: 0 -> quadruples, then pairs, of fields share one spreading
   * pass (k_spread_pair4 / k_spread_pair2: footprint geometry, ES taps and shared-memory tap loads paid once per
   * four / two fields); 2 -> pairs only; 1 -> one k_spread_pair pass per field */
  int32_t batch_pair;
} vp_opts;

/* Plan parameters chosen by vp_plan (diagnostics; all derived from the rules in DESIGN.md). */
typedef struct {
  int64_t M, N, T;
  int32_t p, w_es;           /* quadrature points per triangle; ES kernel width */
  double beta_es;            /* ES kernel shape */
  double dx2, delta1, delta2;
  double kmax_nh, kmax_fh, L_nh, L_fh, R_trunc;
  int64_t nf_nh, nf_fh;      /* fine grid size per dimension (sigma = 2) */
  int64_t nmode_nh, nmode_fh;
  double x0, y0, S;          /* centre and side of the bounding square of nodes and targets */
  int32_t deriv_mode, deriv_degree, deriv_k;
  int64_t n_boundary_targets;
  double plan_ms;
  int64_t device_bytes;      /* device memory owned by the plan */
  int64_t n_stencil_targets; /* targets whose local part uses a stored KNN stencil */
  int64_t n_batches;         /* spreading work units: strip items (<= 2048 points) or tile batches (<= 32) */
  double horner_err;         /* max |Horner - ES| over the kernel taps */
  int32_t n_levels;          /* finest band level present (0: no level bands) */
  int64_t n_boxes;           /* band boxes (all levels) */
  int64_t n_level_targets;   /* targets with level >= 1 */
  int64_t n_band_pairs;      /* (box, source) pairs spread per eval */
  int64_t nf_band;           /* band box fine grid per dimension */
  int64_t level_targets[16]; /* targets per level */
  int32_t fft_path_nh, fft_path_fh; /* transforms of the NH / FH grid: 0 fused row/column kernels (nf <= 6400),
                                       1 cuFFT 2D D2Z + multiply + Z2D, 2 cuFFT row passes + four-step column pass,
                                       3 own pruned row passes + four-step column pass */
} vp_info;

typedef struct vp_plan_s *vp_handle;

/* Build a plan (§3 "Input" and Step 1, lines 782-821: nodes x[j] and smooth weights w[j] of a
 * p-point rule on M triangles, N = M p (§2.2), targets, tolerance).
 *   tri_nodes [M][p][2] fp64, x then y, grouped per triangle (device)
 *   weights   [M][p]    fp64, >= 0; zero allowed (degenerate triangles contribute nothing) (device)
 *   targets   [T][2]    fp64 (device); with opts->targets_are_nodes the first N targets must equal the nodes
 *   tol       in [1e-14, 1e-2]: relative accuracy goal for V (NUFFT eps = tol unless opts->eps_nufft)
 *   opts      NULL or zero-initialised for defaults (see vp_opts)
 *   out       receives the plan handle (NULL on failure)
 * The arrays are read during the call only: the plan copies and reorders what it keeps and owns all
 * device memory it allocates (released by vp_destroy).  Synchronises opts->cuda_stream.
 * Errors: VP_ERR_ARG (null pointer, M, p or T <= 0, sum of weights == 0, T < N with targets_are_nodes,
 * bad option), VP_ERR_TOL, VP_ERR_NONFINITE (NaN/Inf or negative weight in the inputs), VP_ERR_GEOMETRY
 * (invalid or ambiguous boundary, see vp_boundary), VP_ERR_UNSUPPORTED (N or T >= 2^31, TRIANGLE mode without ref_nodes,
 * a polygon corner that is not a right angle,
 * or a spreading tile row with more than 2^20 points), VP_ERR_OOM (a grid beyond the device),
 * VP_ERR_CUDA / VP_ERR_CUFFT (runtime failures; vp_last_error_detail says which call). */
vp_status vp_plan(const double *tri_nodes, const double *weights, int64_t M, int32_t p,
                  const double *targets, int64_t T, double tol, const vp_opts *opts, vp_handle *out);

/* Evaluate V = V_NH + V_FH + V_L (PAPER.md eq. (heatdecomp)) at the plan's targets.
 *   f   [M][p] fp64 source values at the nodes, same order as tri_nodes (device, read only)
 *   out [T]    fp64, fully overwritten, target order of vp_plan (device)
 * Asynchronous on the plan's stream (the caller synchronises); one plan must not be evaluated
 * concurrently with itself.  f is not checked for NaN/Inf here (that would need a host sync): a
 * non-finite f propagates to out; vp_check_finite tests f explicitly.
 * Errors: VP_ERR_ARG (null pointer), VP_ERR_CUDA / VP_ERR_CUFFT (launch failures). */
vp_status vp_eval(vp_handle plan, const double *f, double *out);

/* Same, with HOST buffers: copies f host->device, evaluates, copies out device->host, and
 * synchronises.  Pinned host memory is recommended. */
vp_status vp_eval_host(vp_handle plan, const double *f_host, double *out_host);

/* K fields from HOST memory, f_host[k] [M][p] -> out_host[k] [T] (k < K), with the transfers overlapped across
 * fields: the H2D copy of field k+1 and the D2H copy of field k-1 run on two plan-owned copy streams while field
 * k is evaluated (PCIe is full duplex), so the throughput is bound by the slowest of H2D, D2H and vp_eval instead
 * of their sum.  Pinned host memory is required for the overlap (pageable memory works, serialised).  The first
 * call allocates two device slots for f and out (2 x 8 (N + T) bytes, plan-owned) and the copy streams.  Work is
 * ordered after earlier work on the plan's stream; synchronous on return.  An output array may be passed for
 * several k (the D2H copies are ordered on one stream; it then holds the last of those fields).
 * Errors: VP_ERR_ARG (K < 1, null pointers), VP_ERR_OOM, VP_ERR_CUDA / VP_ERR_CUFFT. */
vp_status vp_eval_host_many(vp_handle plan, int32_t K, const double *const *f_host, double *const *out_host);

/* Evaluate K fields on the same plan ("batched multi-f vp_eval"; PAPER.md Steps 2-4,
 * lines 848-850, are linear in the strengths c_j = f_j w_j).
 *   K    number of fields, >= 1
 *   f    [K][M][p] fp64 source values (device, read only), field k at f + k M p
 *   out  [K][T]    fp64 (device), field k at out + k T, fully overwritten
 * The spreading of several fields shares one pass over the sorted nodes (geometry, ES weights and their
 * shared-memory loads are paid once per node): four, then two, fields per pass with row-pair strips at w <= 10
 * (the default; opts.batch_pair) and with 32-column strips; transforms, interpolation and the local part run per
 * field, each with vp_eval's schedule (fork/join streams on small grids, serial otherwise).  The first call with a
 * larger K than before synchronises the plan's stream, frees the previous extra buffers and allocates K-1 extra NH
 * grids (and K spreading-order copies of f for KNN stencils), owned by the plan.  Same stream and concurrency rules
 * as vp_eval.
 * Errors: VP_ERR_ARG (null pointer, K < 1), VP_ERR_OOM (extra grids beyond the device), VP_ERR_UNSUPPORTED
 * (deterministic mode or spread_tile > 0, which use the tile-batch spreading), VP_ERR_CUDA / VP_ERR_CUFFT. */
vp_status vp_eval_batch(vp_handle plan, int32_t K, const double *f, double *out);

/* Single-layer potential S[sigma](x_t) = int_Gamma -(1/2 pi) log|x_t - y| sigma(y) ds_y at the plan's targets, on
 * the plan's grids (§2.3, eq. sheatdecomp; local part Lemma slp, eq. slplocO5, lines
 * 955-987).  Requires opts.boundary of kind VP_BDRY_CHUNKS: the boundary quadrature nodes are the
 * chunks' q+1 Gauss-Legendre nodes, with weights w_k |gamma'(s_k)|.
 * vp_slp_prepare (once per plan, synchronous): sorts the boundary nodes into the spreading strips and builds a
 *   (q+1)-entry stencil of the local part S_L for every target within 12 sqrt(delta_1) of the boundary.
 * vp_eval_slp: sigma = DEVICE [n][q+1] densities at the chunk nodes (same layout as opts.boundary.pts), out =
 *   DEVICE [T] (fully overwritten), asynchronous on the plan's stream like vp_eval.  The history part reuses the
 *   plan's grids, so it must not run concurrently with vp_eval on the same plan.
 * Errors: VP_ERR_UNSUPPORTED (boundary not CHUNKS), VP_ERR_ARG (null pointers, vp_eval_slp before
 *   vp_slp_prepare), VP_ERR_CUDA / VP_ERR_CUFFT. */
/* Levels J (0..8, default 3) of the dyadic telescoping of the layer potentials' local parts (§4.1
 * "s:dyadicref", lines 1181-1269): S_L / D_L = asymptotic expansion at delta* = delta_1 / 4^J + the J difference
 * kernels integrated directly over the chunks within 12 sqrt(delta_1) of the target (panels of 16 Gauss-Legendre
 * points no longer than ~1.7 sqrt(delta*)).  J = 0: the expansion at delta_1 alone (truncation O(delta_1^{5/2})).
 * Must be called before the first vp_slp_prepare / vp_dlp_prepare.  Errors: VP_ERR_ARG (J out of range, called
 * after a prepare), VP_ERR_UNSUPPORTED at prepare time if a target has more than 64 chunks within reach. */
vp_status vp_layer_set_levels(vp_handle plan, int32_t J);
vp_status vp_slp_prepare(vp_handle plan);
vp_status vp_eval_slp(vp_handle plan, const double *sigma, double *out);

/* Double-layer potential D[mu](x_t) = int_Gamma d/dnu_y [-(1/2 pi) log|x_t - y|] mu(y) ds_y, nu the OUTWARD unit
 * normal, at the plan's targets on the plan's grids (eq. dheatdecomp; history
 * lemmas dnearkspace / dfarkspace, lines 522-553, with the -i k.nu multiplier of DESIGN.md reading R20; local
 * part Lemma dlp, eq. dlplocO5, in the outward frame of reading R21).  Jump relations: the
 * interior / exterior limits at b are D(b) -/+ mu(b)/2 (D(b) the direct value), as in the Dirichlet equation of
 * lines 1281-1287.  Same boundary requirement as S (VP_BDRY_CHUNKS).
 * vp_dlp_prepare (once per plan, synchronous): two dipole spreading sets (weights W nu_1, W nu_2), the (q+1)-entry
 *   D_L stencils of the targets within 12 sqrt(delta_1), and cuFFT plans plus two NH half spectra (owned by the
 *   plan; 2 x 16 nf_NH (nf_NH/2+1) bytes) for the spectral derivative.
 * vp_eval_dlp: mu = DEVICE [n][q+1] densities at the chunk nodes, out = DEVICE [T] (fully overwritten),
 *   asynchronous on the plan's stream; shares the plan's grids with vp_eval / vp_eval_slp (no concurrent calls).
 * Errors: as vp_slp_prepare / vp_eval_slp (VP_ERR_ARG for vp_eval_dlp before vp_dlp_prepare). */
vp_status vp_dlp_prepare(vp_handle plan);
vp_status vp_eval_dlp(vp_handle plan, const double *mu, double *out);

/* Boundary integral equations of the Poisson solve (§5 "s:bie", lines 1271-1330), solved
 * by restarted GMRES whose product is this library's GPU double-layer operator (the paper pairs GMRES with an FMM,
 * lines 1319-1324).  The plan's targets must be the boundary chunk nodes in the descriptor's order (T = n (q+1),
 * checked to 1e-12) and vp_dlp_prepare must have run.  kind:
 *   VP_BIE_DIRICHLET_INT  (-1/2 I + D) mu = rhs          (eq. dir_inteq: rhs = g - V[f]; u = V[f] + D[mu] inside)
 *   VP_BIE_DIRICHLET_EXT  (+1/2 I + D + int ds) mu = rhs  (eq. dir_repext: rhs = g - V[f] - A log|x - x0|;
 *                                                          u = V[f] + D[mu] + int mu ds + A log|x - x0| outside)
 *   VP_BIE_NEUMANN_INT    (+1/2 I + D) u = rhs            (lines 1310-1318: rhs = V[f] + S[g]; singular, the
 *                                                          solution is defined up to a constant)
 * rhs, x: DEVICE [T] (x is overwritten; the initial guess is 0).  tol: relative residual |b - A x| / |b|; maxit:
 * total Arnoldi steps; restart: Krylov dimension m (1..200; workspace (m+1) T doubles, allocated per call).
 * iters / resid (host, may be NULL): steps taken, final relative residual.  Synchronous.  Reaching maxit is not an
 * error (check resid).  Errors: VP_ERR_ARG (bad arguments, no vp_dlp_prepare, targets not the chunk nodes),
 * VP_ERR_CUDA / VP_ERR_CUFFT / VP_ERR_OOM. */
enum { VP_BIE_DIRICHLET_INT = 0, VP_BIE_DIRICHLET_EXT = 1, VP_BIE_NEUMANN_INT = 2 };
vp_status vp_bie_solve(vp_handle plan, int32_t kind, const double *rhs, double *x, double tol, int32_t maxit,
                       int32_t restart, int32_t *iters, double *resid);

/* Release all device memory and cuFFT plans owned by the plan.  NULL is accepted. */
vp_status vp_destroy(vp_handle plan);

const char *vp_strerror(vp_status s);

vp_status vp_get_info(vp_handle plan, vp_info *info);

/* Per-phase device times (ms) of the last vp_eval when profiling is on (vp_set_profiling).
 * names: "zero", "spread", "restrict", "fft_fwd", "multiply", "fft_inv", "prolong", "interp_local", "bands";
 * n_out <= 16. */
vp_status vp_set_profiling(vp_handle plan, int32_t on);
vp_status vp_get_phase_times(vp_handle plan, double *ms, int32_t *n_out, const char **names);

/* Number of kernels vp_eval launches (excluding cuFFT-internal kernels) and cuFFT executions. */
vp_status vp_eval_launch_count(vp_handle plan, int32_t *kernels, int32_t *fft_execs);

/* Check f [M][p] (device) for NaN/Inf: VP_OK or VP_ERR_NONFINITE.  Synchronises. */
vp_status vp_check_finite(vp_handle plan, const double *f);

/* Human-readable detail of the last CUDA / cuFFT failure on this thread. */
const char *vp_last_error_detail(void);

const char *vp_version(void);

/* sizeof(vp_opts), sizeof(vp_info), sizeof(vp_boundary) of this build.  A binding that mirrors the structs
 * (the ctypes classes of paper_2409_11998_b200/__init__.py) compares its own sizes with these when the library
 * is loaded and refuses to run on a mismatch.  out: 3 values. */
vp_status vp_struct_sizes(int64_t *out);

#ifdef __cplusplus
}
#endif
#endif /* VP_H_ */
