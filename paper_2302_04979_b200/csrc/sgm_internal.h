// Internal declarations of the sgm library (plan layout, table layout, kernel launchers).
// Not part of the C ABI (see include/sgm.h).
#pragma once

#include <cstddef>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sgm.h"
#include "tune.h"

namespace sgm {

// Univariate factors of one axis.
struct Axis {
  int n = 0;   // elements
  int a = 0;   // n + p - 2 : trimmed S_p and S_{p-2}(Xi'')
  int b = 0;   // n + p - 1 : S_{p-1}(Xi')
  // dense row-major 1D matrices
  std::vector<double> G;    // Hat{G}  a x a : int D''_k B_c
  std::vector<double> M;    // Hat{M}  b x b : int B'_j D'_k
  std::vector<double> GB1;  // Gamma_B^{p-1}  b x b
  std::vector<double> GC2;  // Gamma_C^{p-2}  a x a
  std::vector<double> GBp;  // Gamma_B^{p}    a x a
  std::vector<double> GC1;  // Gamma_C^{p-1}  b x b
  // Gauss points / weights of the Q-point rule, element by element
  std::vector<double> xq, wq;
};

// Device line-operator tables: per (axis, op), rows of RowLayout<P>::RS doubles (seg_sweep.cuh):
//   [ band(2P+1) | lo(P-1) | F(P-1) | dinv, upn(P-1) | B(P-1) ]  (groups padded to 16 bytes)
// band = banded mat-vec (mass or pairing factor); lo/upn/dinv = no-pivot banded LU
// (reading Z14); F/B = spikes of the partitioned (segmented) substitutions.
enum Op {
  OP_EPS_OWN = 0,  // band Gamma_B^{p-1} (b), LU(Hat M)
  OP_EPS_OTH = 1,  // band Gamma_C^{p-2} (a), LU(Hat G)
  OP_MU_OWN = 2,   // band Gamma_B^{p}   (a), LU(Hat G^T)
  OP_MU_OTH = 3,   // band Gamma_C^{p-1} (b), LU(Hat M^T)
  OP_APPLY_M = 4,  // band Hat M   (b)
  OP_APPLY_G = 5,  // band Hat G   (a)
  OP_APPLY_GT = 6, // band Hat G^T (a)
  OP_APPLY_MT = 7, // band Hat M^T (b)
  OP_S1_MU_OWN = 8,  // scheme 1, mu star own axis: band Hat G (a), LU(Gamma_C^{p-2})
  OP_COUNT = 9,
  OP_S1_EPS_OTH_W = 100  // scheme 1, eps star other axes: band Hat G^T (a), LU(Gamma_B^p) -- the
                         // LU has half-bandwidth p: stored in the "wide" tables (layout p + 1)
};

enum HodgeKind { HODGE_SEPARABLE = 0, HODGE_SCALAR = 1, HODGE_FULL = 2 };

struct MassData {
  HodgeKind kind = HODGE_SEPARABLE;
  double scale[3] = {1.0, 1.0, 1.0};   // per-component constant (separable / scalar kinds)
  double* W_dev = nullptr;             // SCALAR: 1 per qp; FULL: 6 per qp (xx,yy,zz,xy,xz,yz)
  bool const_material = true;
  double material_c = 1.0;             // constant material value (eps or mu)
  std::vector<double> values_host;     // the material at the quadrature points (variable case)
  bool otf = false;                    // FULL with on-the-fly DF: W_dev holds w_q / material (1 per qp)
};

// Arguments a captured sgm_step graph was recorded with (replayed only for identical calls).
struct GraphKey {
  const void *d, *e, *b, *h, *jhat, *jamp;
  double dt;
  int n_steps;
  const void* ws;
  bool operator==(const GraphKey& o) const {
    return d == o.d && e == o.e && b == o.b && h == o.h && jhat == o.jhat && jamp == o.jamp && dt == o.dt &&
           n_steps == o.n_steps && ws == o.ws;
  }
};

struct Plan {
  int p = 0;
  int Q = 0;
  int device = -1;
  int n[3] = {0, 0, 0};
  Axis ax[3];
  bool has_geom = false;
  std::vector<double> ctrl;           // (nz+p)(ny+p)(nx+p)*3
  std::vector<double> wts;            // rational map weights (nz+p)(ny+p)(nx+p); empty = polynomial
  bool affine_diag = true;            // DF constant diagonal
  double L_aff[3] = {1, 1, 1};        // diagonal of DF if affine_diag
  size_t n_qp = 0;
  MassData mass[2];                   // [SGM_MASS_EPS], [SGM_MASS_MU]
  MassData mass1[2];                  // scheme 1: 1-form masses M^1_eps, M~^1_mu (weights: material)
  double* pcg_buf = nullptr;          // scheme 1 with non-separable stars: 4 PCG vectors
  int pcg_iters_m[2] = {40, 40};      // PCG iterations per star (plan-time calibration)
  int pcg_fixed = 0;                  // SGM_PCG_ITERS: fixed count instead
  size_t pcg_n = 0;
  // device
  double* tables_dev = nullptr;       // [3][OP_COUNT][Lmax][RS] (seg_sweep.cuh row layout), then diag factors
  int Lmax = 0;                       // rows per table slot (max padded line length)
  int scheme = 2;                     // 2: pairing solves; 1: mass solves
  std::vector<double> wide_host;      // scheme-1 eps tables [3][Lmax][RowLayout<p+1>::RS] (p <= 3)
  double* wide_dev = nullptr;
  double* win_scratch = nullptr;      // one form component: input copy of in-place windowed sweeps (lines > kMaxLine)
  int wide_band_hw[3] = {}, wide_kh[3] = {}, wide_kf[3] = {};
  size_t diag_off = 0;                // offset (doubles) of the diagonal factors [3][2][Lmax]:
                                      // [axis][0] = 1/s (eps own axis), [axis][1] = s (mu other axes)
  bool diag_ok = true;                // reduced separable schedule usable (host_setup.cpp)
  int seg[3] = {0, 0, 0};             // register segment length per axis
  int rpad[3] = {0, 0, 0};            // padded line length per axis (multiple of seg)
  int band_hw[3][OP_COUNT] = {};      // actual half-bandwidth of each table's band part
  int spike_kh[3][OP_COUNT] = {};     // truncated-SPIKE reach (segments) of the history scan
  int spike_kf[3][OP_COUNT] = {};     // ... and of the future scan (host_setup.cpp spike_reach)
  double* basis_dev = nullptr;        // general Hodge: per-axis basis values at qp [n][Q][p+1]
  int* first_dev = nullptr;           // per-axis first local global index per element [n]
  size_t basis_off[3][4] = {};        // offsets (doubles) into basis_dev per axis and space
  int first0[3][4] = {};              // first index of element 0 per axis and space (first(e) = first0 + e)
  int basis_lo[3][4] = {}, basis_hi[3][4] = {};  // elements [lo, hi) whose table equals basis_mid bit for bit
  double basis_mid[3][4][25] = {};    // host copy of the middle element's table [Q][p+1] per axis and space
  size_t first_off[3][4] = {};        // offsets (ints) into first_dev per axis and space
  // on-the-fly geometry (SGM_OPT_OTF_GEOMETRY): control points [3][(nz+p)(ny+p)(nx+p)] then the
  // S_p value / derivative tables at the Gauss points [axis][s][n][Q][p+1]
  double* geo_dev = nullptr;
  size_t geo_ctrl_off[3] = {};
  size_t geo_tab_off[3][2] = {};
  // plan-owned mirrors for sgm_step_host
  double* mirror = nullptr;
  size_t mirror_bytes = 0;
  std::vector<double> tables_host;
  bool sticky_cuda_error = false;
  unsigned opts = 0;                  // SGM_OPT_* schedule options (sgm_plan_set_options)
  size_t hodge_scratch = 0;           // doubles of workspace for the deterministic general Hodge
  mutable int launch_fail = 0;             // a launcher found no compiled configuration (set while enqueuing)
  bool graph_enabled = true;          // SGM_GRAPH=0 disables the sgm_step graph cache
  // fork/join of independent sweep launches (reduced separable schedule): the second launch runs on
  // a plan-owned stream on its own share of the SMs; `fork_mu` serialises the enqueue of a fork/join
  bool fork_enabled = true;           // SGM_FORK=0 disables
  void* aux_stream = nullptr;         // cudaStream_t
  void* ev_fork = nullptr;            // cudaEvent_t (timing disabled)
  void* ev_join = nullptr;
  std::mutex fork_mu;
  void* graph_exec = nullptr;         // cudaGraphExec_t of the last captured sgm_step call
  GraphKey graph_key{};
  void* graph_exec_m = nullptr;       // the same arguments, kGraphChunk steps in one graph
  GraphKey graph_key_m{};
  void* graph_exec_e = nullptr;       // ... of the last captured sgm_step_eh call
  GraphKey graph_key_e{};
  void* graph_exec_c = nullptr;       // ... of the last captured sgm_step_composed call
  GraphKey graph_key_c{};
  std::vector<double> graph_w_c;      // its weights
  size_t N_e = 0, N_h = 0;
  // optional per-kernel event timing (sgm_plan_set_profiling)
  bool profiling = false;
  std::vector<void*> ev_pool;                        // cudaEvent_t
  struct ProfRec { int cls; void* a; void* b; };
  std::vector<ProfRec> prof;
};

// host setup (host_setup.cpp)
sgm_status build_axis(int p, int n, int Q, Axis& out, std::string& err);
sgm_status build_mass1(Plan& P, int which, std::vector<double>& W, std::string& err);
// on-the-fly geometry: whether the FULL 2-form weights of this plan may be evaluated in the brick
// kernel (option set, polynomial map, Q = p + 1, p = 2..4), and the host image of geo_dev
bool otf_geometry(const Plan& P);
void build_geo_buffer(const Plan& P, std::vector<double>& buf, size_t ctrl_off[3], size_t tab_off[3][2]);
std::vector<double> greville(int p, int n);
sgm_status interpolate_geometry(const int n_el[3], int p, const double* values, double* ctrl, std::string& err);
sgm_status banded_lu_nopivot(const std::vector<double>& A, int L, int m, std::vector<double>& LU,
                             std::string& err);
sgm_status build_tables(Plan& P, std::string& err);
sgm_status set_spike_reach(Plan& P, std::string& err);
int seg_for_line(int L);
sgm_status build_geometry(Plan& P, std::string& err);
void qp_coords(const Plan& P, double* xyz);
sgm_status build_mass(Plan& P, int which, const double* values, double c, std::vector<double>& W,
                      std::string& err);
void basis_values_1d(int p, int n, int Q, int space, std::vector<double>& vals, std::vector<int>& first);

// component extents helpers: form kind 0 = E-like (e, d), 1 = B-like (b, h)
inline void comp_shape(const Plan& P, int kind, int c, int xyz[3]) {
  for (int a = 0; a < 3; ++a) {
    bool own = (a == c);
    if (kind == 0) xyz[a] = own ? P.ax[a].b : P.ax[a].a;
    else xyz[a] = own ? P.ax[a].a : P.ax[a].b;
  }
}

void set_error(const std::string& s);

}  // namespace sgm
