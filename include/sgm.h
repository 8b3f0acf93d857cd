/*
 * sgm.h -- C ABI of the B200-native explicit spline-geometric Maxwell step
 *          (arXiv 2302.04979, "second discretization scheme").
 *
 * What the library computes
 * -------------------------
 * State (reading Z8 in DESIGN.md): four fp64 coefficient vectors
 *   d in X~^2 (D, dual 2-form)      e in X^1_{h,0} (E, primal 1-form)    -- at t_n
 *   b in X^2_{h,0} (B, primal 2-form) h in X~^1 (H, dual 1-form)         -- at t_{n+1/2}
 * One leapfrog step (eqs. discrete2_ampere, _hodge_eps, _faraday, _hodge_mu):
 *   d <- d + dt (D~1 h - s_k j^)        D~1: integer dual curl
 *   e <- K1^{-1} M~2_{1/eps} d          K1: metric-free pairing, block diagonal with
 *                                        Kronecker blocks (eq. tensor_K)
 *   b <- b - dt D1 e                    D1: integer primal curl
 *   h <- K~1^{-1} M2_{1/mu} b           K~1 blocks: eq. tensor_Ktilde
 * The Kronecker inverses are applied mode by mode (eq. kroninverse, vec trick
 * P:L575-585) as batched banded LU sweeps of the 1D factors along x, y and z.
 *
 * Discretisation parameters: n_el[a] uniform elements per axis, open knots,
 * maximal smoothness, degree p >= 2 (primal p / p-1, dual p-1 / p-2); per axis
 *   a = n_el + p - 2 (trimmed S_p, S_{p-2}),  b = n_el + p - 1 (S_{p-1}).
 *
 * Memory layout: every form vector is its three components concatenated
 * in the order 1, 2, 3; each component is a C-order array [z][y][x] (x fastest).
 * Component extents (x, y, z):
 *   e, d :  (b,a,a) (a,b,a) (a,a,b)       N_e = N_d = 3 a^2 b  (per-axis a,b)
 *   b, h :  (a,b,b) (b,a,b) (b,b,a)       N_b = N_h = 3 a b^2
 * Quadrature-point arrays (materials, coordinates) are element-major:
 *   [ez][ey][ex][qz][qy][qx]  with Q = quad_points Gauss-Legendre points per axis per element.
 *
 * Conventions
 * -----------
 * - Every call returns sgm_status; no C++ exception crosses the ABI.  On a non-OK status
 *   sgm_last_error() returns a thread-local message.
 * - Device pointers are caller-owned, 8-byte-aligned fp64 buffers on the plan's device
 *   (e.g. torch.float64 CUDA tensors' data_ptr()).  `stream` is a cudaStream_t passed as void*
 *   (NULL = legacy default stream).  Calls marked async enqueue work on `stream` and return.
 * - Arguments are validated before any launch: on SGM_E_INVALID_ARG nothing was modified.
 * - The plan is immutable after create except through set_material / set_scheme (synchronous;
 *   must not overlap in-flight calls on the plan).  Concurrent calls on different streams with
 *   distinct workspaces are allowed (the plan-owned helper stream of the concurrent sweep pairs
 *   is fork/joined under a lock).
 * - Beyond the step: sgm_plan_set_scheme selects the paper's first scheme
 *   (mass-matrix Hodge stars); sgm_step_composed composes leapfrog sub-steps into
 *   higher-order symplectic steps; sgm_cfl estimates the stability limit; rational
 *   (NURBS) maps enter through sgm_plan_desc.geom_weights.
 * - There is no CPU fallback: a plan created with device < 0 answers queries (lengths,
 *   shapes, 1D tables, quadrature coordinates) but every compute call returns
 *   SGM_E_INVALID_ARG.
 */
#ifndef SGM_H
#define SGM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGM_PMIN 2
#define SGM_PMAX 4 /* degrees with compiled kernels */

typedef enum {
  SGM_OK = 0,
  SGM_E_INVALID_ARG = 1,       /* NULL/misaligned pointer, n_el < 1, dt non-finite, n_steps < 0,
                                  bad enum, too-small workspace, host-only plan */
  SGM_E_UNSUPPORTED = 2,       /* p < 2, p > SGM_PMAX, or extents beyond the kernel
                                  indexing limit: a form component above 2^31 - 2^20 elements,
                                  i.e. (n_x+p-1)(n_y+p-1)(n_z+p-1) (n ~ 1285 per axis for a cube).
                                  Lines longer than 392 (n_el + p - 1) are swept in overlapping
                                  windows of at most 392 rows */
  SGM_E_GEOMETRY = 3,          /* det DF <= 0 or non-finite at a quadrature point */
  SGM_E_MATERIAL = 4,          /* eps or mu <= 0 or non-finite at a quadrature point */
  SGM_E_SINGULAR = 5,          /* zero pivot or backward error > 1e-13 in a no-pivot 1D LU
                                  (reading Z14) */
  SGM_E_SOURCE_DIVERGENCE = 6, /* ||D~2 j^||_inf > 1e-12 ||j^||_inf */
  SGM_E_CUDA = 7,              /* CUDA runtime/launch failure; sticky for the plan */
  SGM_E_NOMEM = 8
} sgm_status;

typedef struct sgm_plan_t* sgm_plan; /* opaque */

typedef enum { SGM_FORM_E = 0, SGM_FORM_D = 1, SGM_FORM_B = 2, SGM_FORM_H = 3 } sgm_form;
/* K1 : X^1_{h,0} -> (X~^2)*   (rows dual 2-forms);  K~1 : X~^1 -> (X^2_{h,0})* */
typedef enum { SGM_K1 = 0, SGM_KT1 = 1 } sgm_pairing;
/* M~2_{1/eps} on X~^2, M2_{1/mu} on X^2_{h,0} */
typedef enum { SGM_MASS_EPS = 0, SGM_MASS_MU = 1 } sgm_mass;
/* D1 : X^1_{h,0} -> X^2_{h,0},  D~1 : X~^1 -> X~^2 */
typedef enum { SGM_CURL_PRIMAL = 0, SGM_CURL_DUAL = 1 } sgm_curl_kind;
typedef enum { SGM_EPS = 0, SGM_MU = 1 } sgm_material;
/* 1D matrices of one axis, for inspection (dense row-major L x L):
   Hat{G} (a x a) = int D''_k B_c, Hat{M} (b x b) = int B'_j D'_k;
   separable-Hodge Grams Gamma_B^{p-1} (b), Gamma_C^{p-2} (a), Gamma_B^{p} (a), Gamma_C^{p-1} (b). */
typedef enum {
  SGM_TAB_G = 0, SGM_TAB_M = 1, SGM_TAB_GAMMA_B1 = 2, SGM_TAB_GAMMA_C2 = 3,
  SGM_TAB_GAMMA_BP = 4, SGM_TAB_GAMMA_C1 = 5
} sgm_table;

typedef struct {
  int n_el[3];             /* elements per axis (x, y, z), >= 1 */
  int degree;              /* p, SGM_PMIN..SGM_PMAX */
  const double* geom_ctrl; /* host; NULL = identity map.  Control points of F in S_p(Xi)^3,
                              untrimmed B-splines, layout [(nz+p)][(ny+p)][(nx+p)][3].
                              Copied at create; caller keeps ownership. */
  int quad_points;         /* Q per axis per element for the geometry/material masses;
                              0 -> p+1 (reading Z13).  Allowed: p+1 .. 8 */
  int device;              /* CUDA ordinal; < 0 -> host-only plan (queries only) */
  const double* geom_weights; /* host; NULL = polynomial map.  Else positive weights, layout
                              [(nz+p)][(ny+p)][(nx+p)], of a rational (NURBS) map
                              F = sum w_i P_i N_i / sum w_i N_i with P_i = geom_ctrl (P:L136-137,
                              "a (rational) spline").  Copied at create; non-positive or non-finite
                              weights -> SGM_E_GEOMETRY. */
} sgm_plan_desc;

/* ---- plan lifetime and queries (synchronous) ------------------------------------------- */
sgm_status sgm_plan_create(const sgm_plan_desc* desc, sgm_plan* out);
sgm_status sgm_plan_destroy(sgm_plan plan);
sgm_status sgm_plan_len(sgm_plan plan, sgm_form form, size_t* n);           /* N_e, N_d, N_b, N_h */
sgm_status sgm_plan_shape(sgm_plan plan, sgm_form form, int comp, int xyz[3]); /* comp 0..2 */
sgm_status sgm_plan_qp_count(sgm_plan plan, size_t* n_qp);
/* Physical quadrature points F(x_q), host, element-major layout, 3 doubles per point. */
sgm_status sgm_plan_qp_coords(sgm_plan plan, double* host_xyz);
/* Dense 1D table of one axis into host_out (L*L doubles); *L receives the size. */
sgm_status sgm_plan_table(sgm_plan plan, sgm_table which, int axis, double* host_out, int* L);
/* Hodge classification: 1 = separable (Kronecker Grams, identity / axis-aligned affine F and
   constant material), 0 = general (weights at quadrature points). */
sgm_status sgm_plan_hodge_separable(sgm_plan plan, sgm_mass mass, int* separable);

/* Material eps (SGM_EPS) or mu (SGM_MU).  values == NULL -> constant c.  Otherwise values is a
   host array of the material at every quadrature point (element-major), > 0 and finite.
   Rebuilds the Hodge weights W = w_q (1/material) DF^T DF / det DF and uploads.
   Synchronous. */
sgm_status sgm_plan_set_material(sgm_plan plan, sgm_material which, const double* values, double c);

/* Workspace (device bytes) needed by sgm_step / kron_solve / pairing_apply / hodge_* /
   energy / gauss.  One workspace must not be shared by concurrent calls. */
sgm_status sgm_workspace_bytes(sgm_plan plan, size_t* bytes);

/* ---- the hot path (async on stream) ---------------------------------------------------- */
/* n_steps leapfrog steps in place.  j_hat: device, length N_d, a dual 2-form with D~2 j^ = 0
   (check once with sgm_check_source), NULL = no source.  j_amp: device, length n_steps,
   s_k multiplying j^ at step k (the paper's separable-in-time source); NULL -> 1.0.
   On exit d, e are at t_n + n_steps dt and b, h at t_{n+1/2} + n_steps dt.
   Launches: per step sgm_plan_kernels_per_step kernels with programmatic dependent launch
   (separable Hodge stars, reduced schedule: 7 -- an update and three sweeps for the eps half, an
   update and two sweeps for the mu half, independent sweeps concurrently on a plan-owned stream;
   SGM_OPT_FUSED: 4; see sgm_kernel_class).  On a non-default stream, with j_amp == NULL or n_steps == 1, the launch sequence of one
   step is captured into a CUDA graph on first use and replayed for later calls with identical
   arguments (pointers, dt; a replay reads the current value of j_amp[0]) -- the plan keeps one
   graph; set_material / set_scheme / set_options invalidate it; SGM_OPT_NO_GRAPH disables; a call
   on a stream that is being captured by the caller enqueues directly into the caller's capture.
   SGM_E_UNSUPPORTED after launch: no compiled kernel configuration fits the plan's line lengths
   (the state may be partially updated). */
sgm_status sgm_step(sgm_plan plan, double* d, double* e, double* b, double* h,
                    const double* j_hat, const double* j_amp, double dt, int n_steps,
                    void* workspace, size_t ws_bytes, void* stream);

/* Inhomogeneous Dirichlet data for E (sec. 3.5; the coaxial cable, P:L837-849;
   SURVEY 8(f) NEXT #2; reading Z29 in DESIGN.md).  E_h = E_{h,0} + E_{h,b} with the lifting
   E_{h,b}(t) = g(t) e^_b in X^1_h (boundary functions only) and data separable in space and time
   (P:L838): the boundary contributions are computed once by the caller and enter every step as
   scaled vectors ("multiplied by a known function of time at each time step"):
     (K1)_0 e = M~2 d - (K1)_b e_b        ->  e = K1^{-1} M~2_{1/eps} d - g_{n+1} w_e
     B_h in X^2_h, D1 : X^1_h -> X^2_h     ->  b_0 <- b_0 - dt (D1 e + g_{n+1} c_b)
                                               b_bnd = b_bnd(0) + beta_{n+1} u_b (implicit)
     M2 with columns in X^2_h              ->  h = K~1^{-1} M2_{1/mu} b_0 + q0 + beta_{n+1} q1
   with w_e = (K1)_0^{-1} (K1)_b e^_b (len N_e), c_b / u_b = the interior / boundary rows of D1 e^_b
   (c_b len N_b; the tangential curl on a face involves only that face's coefficients, so interior e
   never reaches b_bnd), q0 = K~1^{-1} M2_{0b} b_bnd(0), q1 = K~1^{-1} M2_{0b} u_b (len N_h), and per
   step k of the call g[k] = g(t_{n+1}), beta[k] = -dt sum_{m <= n+1} g(t_m) (device arrays of
   n_steps).  d, e, b, h are the interior (X^1_{h,0}, X^2_{h,0}) vectors of sgm_step.  NULL
   vectors are zero terms (g, beta required).  Scheme 2; the update is not fused (SGM_OPT_FUSED is
   ignored here); direct enqueue.  Other arguments and errors as sgm_step. */
typedef struct {
  const double* w_e;   /* device, N_e */
  const double* c_b;   /* device, N_b */
  const double* q0;    /* device, N_h */
  const double* q1;    /* device, N_h */
  const double* g;     /* device, n_steps */
  const double* beta;  /* device, n_steps */
} sgm_lifting;
sgm_status sgm_step_lifted(sgm_plan plan, double* d, double* e, double* b, double* h,
                           const double* j_hat, const double* j_amp, const sgm_lifting* lift,
                           double dt, int n_steps, void* workspace, size_t ws_bytes, void* stream);

/* The (e,h)-state variant of the step (reading Z30 in DESIGN.md): with
   e = K1^{-1} M~2_{1/eps} d and h = K~1^{-1} M2_{1/mu} b, one step of sgm_step is exactly
     e <- e + K1^{-1} M~2_{1/eps} (dt (D~1 h - s_k j^))      h <- h - K~1^{-1} M2_{1/mu} (dt D1 e)
   (the Petrov-Galerkin form in E_h, H_h), so d and b need not be stored: two state
   vectors instead of four.  e at t_n and h at t_{n+1/2} on entry, advanced by n_steps dt on exit;
   results equal sgm_step's e, h up to rounding.  Scheme 2 only (SGM_E_UNSUPPORTED otherwise); the
   energy of eq. P:L240 needs d, b (not available here).  Other arguments, graph replay and errors
   as sgm_step.  Async. */
sgm_status sgm_step_eh(sgm_plan plan, double* e, double* h, const double* j_hat, const double* j_amp,
                       double dt, int n_steps, void* workspace, size_t ws_bytes, void* stream);

/* Higher-order time integration by symmetric composition of leapfrog sub-steps (the paper's
   future work; reading Z25 in DESIGN.md).  Each of the n_steps steps
   applies the kick-drift-kick sub-steps S(w_0 dt) ... S(w_{n_w-1} dt), where S(tau) is
     b <- b - (tau/2) D1 e;  h <- K~1^{-1} M2 b;           (eq. discrete2_faraday / _hodge_mu)
     d <- d + tau (D~1 h - s j^);  e <- K1^{-1} M~2 d;      (eq. discrete2_ampere / _hodge_eps)
     b <- b - (tau/2) D1 e;  h <- K~1^{-1} M2 b.
   Adjacent half kicks are merged (n_steps*n_w + 1 kicks and n_steps*n_w drifts in total).
   Yoshida's 4th-order triple jump: n_w = 3, w = {x1, x0, x1}, x1 = 1/(2 - 2^(1/3)),
   x0 = -2^(1/3)/(2 - 2^(1/3)); n_w = 1, w = {1} is velocity Verlet.
   Unlike sgm_step, the state is SYNCHRONOUS: d, e, b, h at t_n on entry and at t_n + n_steps dt
   on exit.  weights: host [n_w], finite, 1 <= n_w <= SGM_MAX_STAGES.  j_amp: device
   [n_steps * n_w], s for drift i of step k at j_amp[k*n_w + i] (NULL -> 1).  Other arguments,
   aliasing rules and errors as sgm_step.  Async.  On a non-default stream, for n_steps <= 4, the
   call's launch sequence is captured into a CUDA graph on first use and replayed for later calls
   with identical arguments (pointers, weights, dt, n_steps); invalidated like sgm_step's graph. */
#define SGM_MAX_STAGES 16
sgm_status sgm_step_composed(sgm_plan plan, double* d, double* e, double* b, double* h,
                             const double* j_hat, const double* j_amp, const double* weights,
                             int n_w, double dt, int n_steps, void* workspace, size_t ws_bytes,
                             void* stream);
/* End-to-end variant on HOST buffers (pinned recommended): copies d,b,h (and j_hat, j_amp
   if given) host->device into plan-owned mirrors, runs sgm_step, copies d,e,b,h back and
   synchronises `stream`.  Synchronous.  The input e is not copied when n_steps >= 1: a step
   never reads it (the first half step recomputes e from d). */
sgm_status sgm_step_host(sgm_plan plan, double* d, double* e, double* b, double* h,
                         const double* j_hat, const double* j_amp, double dt, int n_steps,
                         void* stream);

/* x = K^{-1} rhs (transpose = 0) or K^{-T} rhs (transpose = 1), K in {K1, K~1}; mode-wise
   banded LU sweeps (eq. kroninverse).  rhs == x allowed.  Async. */
sgm_status sgm_kron_solve(sgm_plan plan, sgm_pairing which, int transpose, const double* rhs,
                          double* x, void* workspace, size_t ws_bytes, void* stream);
/* y = K x or K^T x (Kronecker banded mat-vecs).  x != y.  Async. */
sgm_status sgm_pairing_apply(sgm_plan plan, sgm_pairing which, int transpose, const double* x,
                             double* y, void* workspace, size_t ws_bytes, void* stream);
/* y = M x with M = M~2_{1/eps} (x, y in X~^2) or M2_{1/mu} (X^2_{h,0}).  x != y.  Async. */
sgm_status sgm_hodge_apply(sgm_plan plan, sgm_mass which, const double* x, double* y,
                           void* workspace, size_t ws_bytes, void* stream);
/* Discrete Hodge star of scheme 2: y = K1^{-1} M~2_{1/eps} x (EPS: d -> e) or
   y = K~1^{-1} M2_{1/mu} x (MU: b -> h) (eqs. discrete2_hodge_eps/_mu).  x != y.  Async. */
sgm_status sgm_hodge_star(sgm_plan plan, sgm_mass which, const double* x, double* y,
                          void* workspace, size_t ws_bytes, void* stream);
/* y = D1 x (PRIMAL: e-shaped -> b-shaped) or y = D~1 x (DUAL: h-shaped -> d-shaped).  Async. */
sgm_status sgm_curl(sgm_plan plan, sgm_curl_kind kind, const double* x, double* y, void* stream);
/* out_dev[0] = 1/2 (d^T K1 e + b^T K~1 h)  (eq. energy_matrix_wedge, with
   K~2 = K1^T, K2 = K~1^T).  Deterministic reduction.  Async. */
sgm_status sgm_energy(sgm_plan plan, const double* d, const double* e, const double* b,
                      const double* h, double* out_dev, void* workspace, size_t ws_bytes,
                      void* stream);
/* out_dev[0] = ||D~2 d||_inf, out_dev[1] = ||D2 b||_inf (Gauss laws).  Async. */
sgm_status sgm_gauss(sgm_plan plan, const double* d, const double* b, double* out_dev,
                     void* workspace, size_t ws_bytes, void* stream);
/* Checks ||D~2 j^||_inf <= 1e-12 ||j^||_inf.  Synchronous on stream. */
sgm_status sgm_check_source(sgm_plan plan, const double* j_hat, void* workspace,
                            size_t ws_bytes, void* stream);

/* Leapfrog stability limit (SURVEY 8(d) "Fixing dt reproducibly", K8; reading Z15 in DESIGN.md):
   n_iter power iterations on A = D~1 K~1^{-1} M2 D1 K1^{-1} M~2 (acting on dual 2-forms), which is
   self-adjoint and PSD in the M~2 inner product because K1^T D~1 = D1^T K~1.  With x
   normalised to unit 2-norm, each iteration computes e = K1^{-1} M~2 x, b = D1 e,
   h = K~1^{-1} M2 b (eqs. discrete2_hodge_*), the Rayleigh quotient
   lam = (b^T K~1 h) / (x^T K1 e), and x <- D~1 h / |D~1 h|_2.  The quotients increase
   monotonically towards lambda_max from below.
     x      in: start vector (device, len N_d; drawn by the caller), out: last normalised iterate
     e,b,h  device scratch of lengths N_e, N_b, N_h (the shapes of sgm_step's state); overwritten
     out_dev  device [2]: lam of the last iteration and dt_max = 2/sqrt(lam)
   All pointers distinct; n_iter >= 1.  Async (no host synchronisation). */
sgm_status sgm_cfl(sgm_plan plan, double* x, double* e, double* b, double* h, int n_iter,
                   double* out_dev, void* workspace, size_t ws_bytes, void* stream);

/* Select the discretization scheme of the Hodge stars used by sgm_step / sgm_step_composed /
   sgm_hodge_star / sgm_cfl: 2 (default) = the paper's second scheme, pairing
   solves e = K1^{-1} M~2_{1/eps} d, h = K~1^{-1} M2_{1/mu} b; 1 = the first scheme,
   mass solves M^1_eps e = K~2 d, M~^1_mu h = K2 b with K~2 = K1^T, K2 = K~1^T.
   Scheme 1 is built for every compiled degree (its eps star uses a p+1 table layout).  With the identity (axis-aligned affine)
   map and constant materials its 1-form masses are Kronecker products of 1D Grams, inverted mode by
   mode with the same sweeps (the own-axis factor of e and the other-axis factors of h are again
   exactly diagonal).  Otherwise (curved map or variable material) each star solves its 1-form mass
   by preconditioned conjugate gradients on the device: sum-factorised 1-form mass applies
   (weights w gamma DF^{-1} DF^{-T} det DF), the separable star with the mean material as
   preconditioner, no host synchronisation; the iteration count is calibrated per star when the
   weights are built (one solve with residual read-back, relative preconditioned residual 1e-14,
   plus 3).  The 1-form weights (and the calibration) are redone by
   sgm_plan_set_material while scheme 1 is selected. */
sgm_status sgm_plan_set_scheme(sgm_plan plan, int scheme);

/* Geometry input helpers (reading Z18: a map is represented in S_p(Xi)^3 by interpolation at the
   Greville points of the untrimmed basis).  Host-only, synchronous.
   sgm_geometry_greville: the n_el + p Greville abscissae of one axis into g_host.
   sgm_geometry_interpolate: control points (layout of sgm_plan_desc.geom_ctrl) whose spline
   interpolates the map values given at the tensor Greville grid, values_host laid out
   [(nz+p)][(ny+p)][(nx+p)][3] with x fastest (dense collocation LU per axis, mode by mode). */
sgm_status sgm_geometry_greville(int n_el, int degree, double* g_host);
sgm_status sgm_geometry_interpolate(const int n_el[3], int degree, const double* values_host,
                                    double* ctrl_host);

/* ---- schedule options (sgm_plan_set_options; all off = the production schedule) ----------
   They change which kernels run, never what is computed (results agree to rounding; the parity
   tests run every option).  Synchronous; invalidates the captured graphs. */
#define SGM_OPT_FULL_SCHEDULE 0x1u /* separable stars sweep every axis of every Kronecker factor (no
                                      diagonal-factor shortcut) */
#define SGM_OPT_EXACT_SPIKE 0x2u   /* untruncated SPIKE history/future scans (reading Z23 off) on
                                      lines of at most 392 rows (longer lines are windowed: always
                                      the truncated reach) */
#define SGM_OPT_SERIAL 0x4u        /* no concurrent sweep launches */
#define SGM_OPT_NO_GRAPH 0x8u      /* sgm_step / sgm_step_composed enqueue directly (no graph replay) */
#define SGM_OPT_FUSED 0x10u        /* separable scheme-2 stars: the Ampere / Faraday update fused into
                                      the first sweep launch of each half step (fsweep_kernel.cuh;
                                      4 launches per step instead of 7, 40 instead of 48 B per
                                      DOF-update; measured slower on B200 at 128^3, DESIGN.md s. 6) */
#define SGM_OPT_WIDE_TILES 0x20u   /* sweeps always use 64-line tiles (two lines per thread) where they
                                      fit; by default a launch with fewer lines than two such tiles
                                      per SM of its share uses 32-line tiles (latency bound sizes) */
#define SGM_OPT_OTF_GEOMETRY 0x40u /* general Hodge stars on a polynomial (non-rational) curved map,
                                      default quadrature: the brick kernel evaluates DF at the
                                      quadrature points from the map's control points (sum
                                      factorisation) and forms (w_q / material) / det DF * DF^T DF
                                      itself; the plan stores 1 double per quadrature point instead
                                      of 6.  Setting or
                                      clearing it rebuilds the weights from the stored material. */
sgm_status sgm_plan_set_options(sgm_plan plan, unsigned opts);
sgm_status sgm_plan_get_options(sgm_plan plan, unsigned* opts);

/* *on = 1 if separable Hodge stars use the reduced schedule (the diagonal 1D
   factors Hat M^{-1} Gamma_B^{p-1} = diag(1/s) and Hat M^{-T} Gamma_C^{p-1} = diag(s), verified at
   plan creation, replace their line sweeps by per-line scalings), 2 if in addition independent
   sweeps run concurrently on a plan-owned stream (default; SGM_OPT_SERIAL disables),
   3 with the fused update (SGM_OPT_FUSED), 0 if every axis is swept
   (SGM_OPT_FULL_SCHEDULE or a failed identity). */
sgm_status sgm_plan_reduced_schedule(sgm_plan plan, int* on);

/* Number of kernels one sgm_step step launches for this plan (for launch accounting). */
sgm_status sgm_plan_kernels_per_step(sgm_plan plan, int* n);

/* Per-kernel timing of sgm_step (CUDA events recorded on the launching stream around every
   kernel when enabled).  Kernel classes: */
typedef enum {
  /* Default (separable stars, reduced schedule): UPDATE, then
     EPS_Z = {0, 1 along z; 2 along y}, EPS_Y = {0 along y} and EPS_X = {1, 2 along x} (concurrent),
     UPDATE, MU_Z = {2 along z, 1 along y} and MU_X = {0 along x} (concurrent).
     SGM_OPT_FUSED: FUSED_EPS = Ampere update fused into {0, 1 along z; 2 along y} d -> t, then
     EPS_Y || EPS_X as above, FUSED_MU = Faraday update fused into {2 along z; 1 along y; 0 along x}.
     Full three-axis schedule: the z (or FUSED_*), y and x launches.  General Hodge: UPDATE,
     HODGE_GENERAL, SOLVE_Z, *_Y, *_X. */
  SGM_K_EPS_Z = 0,     /* eps half, first sweep launch (Gram mat-vec . K1 factor solve), d -> t */
  SGM_K_EPS_Y = 1,     /* eps half, y-line sweep */
  SGM_K_EPS_X = 2,     /* eps half, last sweep launch (writes e) */
  SGM_K_MU_Z = 3,      /* mu half, strided sweep (Gram mat-vec . K~1 factor solve), b -> h */
  SGM_K_MU_Y = 4,      /* mu half, y-line sweep (unmerged or full schedule only) */
  SGM_K_MU_X = 5,      /* mu half, x-line sweep (writes h) */
  SGM_K_UPDATE = 6,    /* Ampere / Faraday update d += dt (D~1 h - s j), b -= dt D1 e (both halves) */
  SGM_K_HODGE_GENERAL = 7, /* sum-factorised mass apply with quadrature weights (general Hodge) */
  SGM_K_SOLVE_Z = 8,   /* solve-only z sweep (general-Hodge path) */
  SGM_K_FUSED_EPS = 9, /* Ampere update fused into the first eps sweep launch */
  SGM_K_FUSED_MU = 10, /* Faraday update fused into the first mu sweep launch */
  SGM_K_CLASSES = 11
} sgm_kernel_class;
sgm_status sgm_plan_set_profiling(sgm_plan plan, int on);
/* Sums, per class, the event-timed milliseconds and launch counts recorded since the last call
   (synchronises on the recorded events), then clears the record.  ms/counts: SGM_K_CLASSES. */
sgm_status sgm_plan_profile(sgm_plan plan, double* ms, int* counts);
const char* sgm_last_error(void);
const char* sgm_version(void);

/* ---- verification build --------------------------------------------------------------------
   Only libsgm_checked.so (compiled with -DSGM_CHECKED, paper_2302_04979_b200/build.py
   checked=True) checks the producer/consumer and SPIKE-exchange protocols of the pipelined sweeps
   at run time (csrc/check.cuh: hand-off tags, release counts, slab poisoning, random delays) and
   counts violations in a library-wide device buffer.  sgm_check_read synchronises the device,
   writes the number of violations since the last reset to *count and the code of the first one
   to *first (0: none; 1 stage tag, 2 release count, 3 tails tag, 4 heads tag, 5 fused release
   count), and zeroes the counters when reset != 0.  count/first: host pointers (either may be
   NULL).  The product build returns SGM_E_UNSUPPORTED and writes nothing. */
sgm_status sgm_check_read(int reset, unsigned* count, unsigned* first);

#ifdef __cplusplus
}
#endif
#endif /* SGM_H */
