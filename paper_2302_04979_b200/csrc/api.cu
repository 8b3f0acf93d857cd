// C ABI of the sgm library (include/sgm.h): plan management, argument validation and the
// launch schedules of the scheme-2 step and its building blocks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <new>
#include <string>

#include "check.cuh"
#include "kernels.cuh"
#include "sgm_internal.h"
#include "seg_sweep.cuh"

namespace sgm {

static thread_local std::string g_err;
void set_error(const std::string& s) { g_err = s; }

#ifdef SGM_CHECKED
// verification build (check.cuh): one zeroed [count, first code] violation buffer per device
unsigned* check_buffer() {
  static unsigned* bufs[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!bufs[dev]) {
    void* p = nullptr;
    if (cudaMalloc(&p, 2 * sizeof(unsigned)) != cudaSuccess) return nullptr;
    cudaMemset(p, 0, 2 * sizeof(unsigned));
    bufs[dev] = static_cast<unsigned*>(p);
  }
  return bufs[dev];
}
int check_inject() {
  const char* v = std::getenv("SGM_CHECK_INJECT");
  return v ? std::atoi(v) : 0;
}
#endif

#ifdef SGM_TUNING
// tuning build only: a per-launch timeline of one selected sweep launch (SGM_TRACE_LAUNCH = its
// ordinal among the sweep launches of the process), [cta][tile][event] globaltimer stamps
unsigned long long* g_trace_ptr = nullptr;
unsigned long long* trace_buffer() {
  static unsigned long long* buf = nullptr;
  static int count = 0;
  const char* v = std::getenv("SGM_TRACE_LAUNCH");
  if (!v) return nullptr;
  const int sel = std::atoi(v);
  if (count++ != sel) return nullptr;
  if (!buf) {
    if (cudaMalloc(&buf, kTraceLen * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
  }
  cudaMemset(buf, 0, kTraceLen * sizeof(unsigned long long));
  g_trace_ptr = buf;
  return buf;
}
#endif

namespace {

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = (cudaSetDevice(dev) == cudaSuccess);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

sgm_status fail(sgm_status s, const std::string& msg) {
  set_error(msg);
  return s;
}

// After enqueuing: a CUDA error is sticky for the plan; a launcher that found no compiled kernel
// configuration (P->launch_fail, e.g. shared memory of the pipelined sweeps at long lines) is
// reported as SGM_E_UNSUPPORTED (not sticky).
sgm_status cuda_check(Plan* P, const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (P) P->sticky_cuda_error = true;
    return fail(SGM_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  }
  if (P && P->launch_fail) {
    P->launch_fail = 0;
    return fail(SGM_E_UNSUPPORTED, std::string(where) +
                                       ": no compiled sweep configuration fits these line lengths (kernel not launched)");
  }
  return SGM_OK;
}

// Drop the captured graphs (their launches embed weights, tables, options)
void drop_graphs(Plan& P) {
  if (!(P.graph_exec || P.graph_exec_c || P.graph_exec_e || P.graph_exec_m) || P.device < 0) return;
  DeviceGuard g(P.device);
  if (P.graph_exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(P.graph_exec));
  if (P.graph_exec_c) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(P.graph_exec_c));
  if (P.graph_exec_e) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(P.graph_exec_e));
  if (P.graph_exec_m) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(P.graph_exec_m));
  P.graph_exec_m = nullptr;
  P.graph_exec = nullptr;
  P.graph_exec_c = nullptr;
  P.graph_exec_e = nullptr;
}

// the caller is capturing `st` into its own graph: enqueue directly (no nested capture)
bool stream_capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (st == nullptr) return false;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

inline bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7) == 0; }

size_t form_len(const Plan& P, int kind) {
  size_t n = 0;
  for (int c = 0; c < 3; ++c) {
    int e[3];
    comp_shape(P, kind, c, e);
    n += size_t(e[0]) * e[1] * e[2];
  }
  return n;
}

size_t comp_off(const Plan& P, int kind, int c) {
  size_t off = 0;
  for (int k = 0; k < c; ++k) {
    int e[3];
    comp_shape(P, kind, k, e);
    off += size_t(e[0]) * e[1] * e[2];
  }
  return off;
}

const double* table(const Plan& P, int axis, int op) {
  return P.tables_dev + (size_t(axis) * OP_COUNT + op) * P.Lmax * RowLayoutRT(P.p).RS;
}

struct WS {
  double* t;
  double* r;
  double* partials;
  double* scratch = nullptr;  // general Hodge output patches (or null)
  size_t scratch_cap = 0;
};

size_t ws_base(const Plan& P) {
  size_t nmax = std::max(P.N_e, P.N_h);
  return (2 * nmax + 4 * size_t(partial_blocks()) + 16) * sizeof(double);
}
// + the general Hodge's output-patch scratch (bitwise-reproducible accumulation, hodge.cu)
size_t ws_need(const Plan& P) { return ws_base(P) + P.hodge_scratch * sizeof(double); }

sgm_status ws_carve(const Plan& P, void* ws, size_t bytes, WS& w) {
  if (!ws || !aligned8(ws)) return fail(SGM_E_INVALID_ARG, "workspace is NULL or misaligned");
  if (bytes < ws_base(P)) return fail(SGM_E_INVALID_ARG, "workspace too small (see sgm_workspace_bytes)");
  size_t nmax = std::max(P.N_e, P.N_h);
  w.t = static_cast<double*>(ws);
  w.r = w.t + nmax;
  w.partials = w.r + nmax;
  // a workspace sized before set_material may lack the scratch: the general Hodge then accumulates
  // with atomics (correct, not bitwise reproducible)
  w.scratch = nullptr;
  w.scratch_cap = 0;
  if (P.hodge_scratch && bytes >= ws_need(P)) {
    w.scratch = reinterpret_cast<double*>(static_cast<char*>(ws) + ws_base(P));
    w.scratch_cap = P.hodge_scratch;
  }
  return SGM_OK;
}

void comps_of(const Plan& P, int kind, const double* base, double* out[3]) {
  for (int c = 0; c < 3; ++c) out[c] = const_cast<double*>(base) + comp_off(P, kind, c);
}

inline int own_or(int axis, int c, int own, int oth) { return axis == c ? own : oth; }

cudaEvent_t ev_get(Plan& P) {
  if (!P.ev_pool.empty()) {
    cudaEvent_t e = static_cast<cudaEvent_t>(P.ev_pool.back());
    P.ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Records CUDA events around one launch on its stream when profiling is enabled.
struct ProfScope {
  Plan& P;
  cudaStream_t st;
  int cls;
  cudaEvent_t a = nullptr;
  ProfScope(Plan& P_, int cls_, cudaStream_t st_) : P(P_), st(st_), cls(cls_) {
    if (P.profiling) {
      a = ev_get(P);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (P.profiling) {
      cudaEvent_t b = ev_get(P);
      cudaEventRecord(b, st);
      P.prof.push_back({cls, a, b});
    }
  }
};

// Affine terms of a Hodge star's last sweeps (sgm_step_lifted): out += sum_i c[i] * (*s[i] or 1) * w[i]
// (w[i]: whole-form base pointers; per-component offsets are added by the launchers)
struct Affine {
  const double* w[2];
  const double* s[2];
  double c[2];
};

// One axis pass over the 3 components of a form (kind 0: e/d shapes, 1: b/h shapes).
void sweep_pass(const Plan& P, int kind, int axis, double* const in[3], double* const out[3], int op_own,
                int op_oth, const double* scale, bool band, bool solve, cudaStream_t st, int reverse = 0,
                int accum = 0, const Affine* aff = nullptr) {
  SweepArgs a;
  std::memset(&a, 0, sizeof(a));
  a.ncomp = 3;
  a.axis = axis;
  a.band = band;
  a.solve = solve;
  a.tabs[0] = table(P, axis, op_own);
  a.tabs[1] = table(P, axis, op_oth);
  a.tab_rows = P.rpad[axis];
  a.band_hw = std::max(P.band_hw[axis][op_own], P.band_hw[axis][op_oth]);
  a.reverse = reverse;
  a.spike_kh = std::max(P.spike_kh[axis][op_own], P.spike_kh[axis][op_oth]);
  a.spike_kf = std::max(P.spike_kf[axis][op_own], P.spike_kf[axis][op_oth]);
  a.wscratch = P.win_scratch;
  for (int c = 0; c < 3; ++c) {
    comp_shape(P, kind, c, a.comp[c].ext);
    a.comp[c].in = in[c];
    a.comp[c].out = out[c];
    a.comp[c].tab = table(P, axis, own_or(axis, c, op_own, op_oth));
    a.comp[c].tslot = own_or(axis, c, 0, 1);
    a.comp[c].scale = scale ? scale[c] : 1.0;
    a.comp[c].accum = accum;
    if (aff)
      for (int t = 0; t < 2; ++t) {
        a.comp[c].aw[t] = aff->w[t] ? aff->w[t] + comp_off(P, kind, c) : nullptr;
        a.comp[c].as[t] = aff->s[t];
        a.comp[c].ac[t] = aff->c[t];
      }
  }
  a.wide = (P.opts & SGM_OPT_WIDE_TILES) ? 1 : 0;
  if (!launch_sweep(P.p, P.seg[axis], a, st)) P.launch_fail = 1;
}

// diagonal 1D factor of axis `axis`: kind 0 = 1/s (eps own axis), 1 = s (mu other axes)
const double* diag_factor(const Plan& P, int axis, int kind) {
  return P.tables_dev + P.diag_off + size_t(axis * 2 + kind) * P.Lmax;
}

// One axis pass over a subset of components (the reduced separable schedule).
struct PassComp {
  int axis;           // sweep axis of this component (a strided pass may mix y and z)
  int c;              // component
  const double* in;   // component arrays
  double* out;
  int op;             // line-operator table
  int dg[3];          // per axis: -1 = no diagonal, else the diag_factor kind applied along it
  double scale;
  int accum = 0;      // 1: out += scale * result ((e,h)-state increments)
  const Affine* aff = nullptr;  // affine store terms (last sweeps of a lifted star)
};

// Components of one launch share the line mode (x, or strided y/z) and the padded table rows and
// segment length of their axes (checked by the caller); at most two distinct tables.
struct Share {
  int k, n;  // k/n of the resident-CTA slots (0/0 = all)
};

void sweep_pass_list(const Plan& P, int kind, const PassComp* pc, int n, cudaStream_t st, int reverse,
                     Share sh = {0, 0}) {
  SweepArgs a;
  std::memset(&a, 0, sizeof(a));
  a.share_k = sh.k;
  a.share_n = sh.n;
  a.ncomp = n;
  a.axis = pc[0].axis;
  a.band = 1;
  a.solve = 1;
  // axes with the same element count have bitwise identical tables: use the first axis's copy so a
  // launch mixing such axes stages one table (shared memory decides whether two lines per thread fit)
  const bool wide = pc[0].op == OP_S1_EPS_OTH_W;  // scheme-1 eps tables: layout p + 1
  auto tab_of = [&](const PassComp& q) {
    const int ax = P.n[q.axis] == P.n[pc[0].axis] ? pc[0].axis : q.axis;
    return wide ? P.wide_dev + size_t(ax) * P.Lmax * RowLayoutRT(P.p + 1).RS : table(P, ax, q.op);
  };
  a.tabs[0] = tab_of(pc[0]);
  a.tabs[1] = nullptr;
  for (int i = 1; i < n; ++i) {
    const double* t = tab_of(pc[i]);
    if (t != a.tabs[0]) a.tabs[1] = t;
  }
  a.tab_rows = P.rpad[pc[0].axis];
  a.reverse = reverse;
  a.wscratch = P.win_scratch;
  for (int i = 0; i < n; ++i) {
    const PassComp& q = pc[i];
    const int axis = q.axis;
    // transverse coordinate slots: z-lines (x, y), y-lines (x, z), x-lines (y, z)
    const int t0 = (axis == 0) ? 1 : 0, t1 = (axis == 2) ? 1 : 2;
    a.band_hw = std::max(a.band_hw, wide ? P.wide_band_hw[axis] : P.band_hw[axis][q.op]);
    a.spike_kh = std::max(a.spike_kh, wide ? P.wide_kh[axis] : P.spike_kh[axis][q.op]);
    a.spike_kf = std::max(a.spike_kf, wide ? P.wide_kf[axis] : P.spike_kf[axis][q.op]);
    SweepComp& C = a.comp[i];
    comp_shape(P, kind, q.c, C.ext);
    C.in = const_cast<double*>(q.in);
    C.out = q.out;
    C.tab = tab_of(q);
    C.tslot = (a.tabs[1] && C.tab == a.tabs[1]) ? 1 : 0;
    C.axis = axis;
    C.scale = q.scale;
    C.accum = q.accum;
    if (q.aff)
      for (int t = 0; t < 2; ++t) {
        C.aw[t] = q.aff->w[t] ? q.aff->w[t] + comp_off(P, kind, q.c) : nullptr;
        C.as[t] = q.aff->s[t];
        C.ac[t] = q.aff->c[t];
      }
    C.dline[0] = q.dg[t0] >= 0 ? diag_factor(P, t0, q.dg[t0]) : nullptr;
    C.dline[1] = q.dg[t1] >= 0 ? diag_factor(P, t1, q.dg[t1]) : nullptr;
  }
  a.wide = (P.opts & SGM_OPT_WIDE_TILES) ? 1 : 0;
  if (!launch_sweep(wide ? P.p + 1 : P.p, P.seg[pc[0].axis], a, st)) P.launch_fail = 1;
}

// The line-operator table of a component: axes with the same element count have bitwise identical
// tables, so the lowest such axis's copy is used (fewer distinct tables per launch).
const double* dedup_table(const Plan& P, int axis, int op) {
  for (int a = 0; a < axis; ++a)
    if (P.n[a] == P.n[axis]) return table(P, a, op);
  return table(P, axis, op);
}

// Partition of a component list into launches: one segment length, one padded table length and at
// most two distinct tables per launch.  Returns the number of launches; grp[g][0..gn[g]) indices.
int group_passes(const Plan& P, const PassComp* pc, int n, int grp[3][3], int gn[3]) {
  bool used[3] = {false, false, false};
  int ng = 0;
  for (int i = 0; i < n; ++i) {
    if (used[i]) continue;
    int m = 0;
    const double* tabs[2] = {dedup_table(P, pc[i].axis, pc[i].op), nullptr};
    grp[ng][m++] = i;
    used[i] = true;
    for (int j = i + 1; j < n; ++j) {
      if (used[j] || P.seg[pc[j].axis] != P.seg[pc[i].axis] || P.rpad[pc[j].axis] != P.rpad[pc[i].axis]) continue;
      const double* t = dedup_table(P, pc[j].axis, pc[j].op);
      if (t != tabs[0] && t != tabs[1]) {
        if (tabs[1]) continue;
        tabs[1] = t;
      }
      grp[ng][m++] = j;
      used[j] = true;
    }
    gn[ng++] = m;
  }
  return ng;
}

// Fused update + first sweep (fsweep_kernel.cuh) over a list of components, each along its own
// axis, grouped into as few launches as possible (group_passes).  fuse = 1 / 2: the Ampere /
// Faraday update of each component's state (in[c]) from `pro` (the curl source, j^, s, dt).
// dry = true only checks that every group has a compiled configuration that fits (alignment,
// shared memory); returns false (nothing launched) otherwise.
bool fused_list(const Plan& P, int kind, const PassComp* pc, int n, cudaStream_t st, int reverse, int fuse,
                const PrologueArgs& pro, int cls, bool dry) {
  int grp[3][3], gn[3];
  const int ng = group_passes(P, pc, n, grp, gn);
  for (int g = 0; g < ng; ++g) {
    const int* idx = grp[g];
    const int m = gn[g];
    const int i = idx[0];
    const double* tabs[2] = {dedup_table(P, pc[i].axis, pc[i].op), nullptr};
    for (int k = 1; k < m; ++k) {
      const double* t = dedup_table(P, pc[idx[k]].axis, pc[idx[k]].op);
      if (t != tabs[0]) tabs[1] = t;
    }
    SweepArgs a;
    std::memset(&a, 0, sizeof(a));
    a.ncomp = m;
    a.axis = -1;
    a.band = 1;
    a.solve = 1;
    a.tabs[0] = tabs[0];
    a.tabs[1] = tabs[1];
    a.tab_rows = P.rpad[pc[i].axis];
    a.reverse = reverse;
    a.pro = pro;
    a.dry = dry ? 1 : 0;
    for (int k = 0; k < m; ++k) {
      const PassComp& q = pc[idx[k]];
      const int axis = q.axis;
      const int t0 = (axis == 0) ? 1 : 0, t1 = (axis == 2) ? 1 : 2;
      a.band_hw = std::max(a.band_hw, P.band_hw[axis][q.op]);
      a.spike_kh = std::max(a.spike_kh, P.spike_kh[axis][q.op]);
      a.spike_kf = std::max(a.spike_kf, P.spike_kf[axis][q.op]);
      SweepComp& C = a.comp[k];
      comp_shape(P, kind, q.c, C.ext);
      C.in = const_cast<double*>(q.in);
      C.out = q.out;
      C.tab = dedup_table(P, axis, q.op);
      C.tslot = (a.tabs[1] && C.tab == a.tabs[1]) ? 1 : 0;
      C.axis = axis;
      C.cidx = q.c;
      C.scale = q.scale;
      C.accum = q.accum;
      C.dline[0] = q.dg[t0] >= 0 ? diag_factor(P, t0, q.dg[t0]) : nullptr;
      C.dline[1] = q.dg[t1] >= 0 ? diag_factor(P, t1, q.dg[t1]) : nullptr;
    }
    if (dry) {
      if (!launch_fsweep(P.p, P.seg[pc[i].axis], fuse, a, st)) return false;
      continue;
    }
    ProfScope ps(const_cast<Plan&>(P), cls, st);
    if (!launch_fsweep(P.p, P.seg[pc[i].axis], fuse, a, st)) P.launch_fail = 1;
  }
  return true;
}

inline bool fused_sched(const Plan& P) { return (P.opts & SGM_OPT_FUSED) && P.scheme == 2; }
inline bool reduced_sched(const Plan& P) { return P.diag_ok && (P.scheme == 1 || !(P.opts & SGM_OPT_FULL_SCHEDULE)); }
inline bool fork_on(const Plan& P) { return P.fork_enabled && !(P.opts & SGM_OPT_SERIAL); }

// The mu star's z and y sweeps share one launch when their axes have equal table geometry.
bool mu_merged(const Plan& P) {
  return P.seg[1] == P.seg[2] && P.rpad[1] == P.rpad[2] && !tune_int("SGM_NOMERGE", 0);
}
// ... and so do the eps star's first z- and y-line sweeps
bool eps_merged(const Plan& P) { return mu_merged(P); }

// SM share of the strided side of a fork: proportional to the components each side sweeps, the
// strided side weighted 1.25 when its lines need so many segment warps that fewer than four
// producer warps fit the 16-warp CTA (measured at p = 3, 160^3: strided tiles ~25 % slower than x
// tiles; at p = 4 and such lengths both sides drop to one line per thread and the plain split wins)
// The x side is weighted 1.25 when its lines have even length (16-byte-aligned slab rows then give
// 4-way instead of 2-way bank conflicts in the consumers' line walks; measured at p = 2, 128^3:
// 145 -> 138 us per step), except at p = 4 where the strided side stays the slower one.
Share strided_share(const Plan& P, int axis, int n_strided, int n_x, bool x_even) {
  const int L = P.rpad[axis], nc = (L + P.seg[axis] - 1) / P.seg[axis];
  const double ws = n_strided * ((16 - nc) < 4 && P.p <= 3 ? 1.25 : 1.0);
  double wx = n_x * (x_even && P.p <= 3 ? 1.25 : 1.0);  // at p = 4 the strided side is the slower one
  // whole-tile bulk x passes hand their output tiles to the producer warp (sweep_kernel.cuh):
  // 15-20 % faster per tile than the line-by-line (L % 4 == 0) ones
  if (P.ax[0].a % 4 != 0) wx *= tune_int("SGM_XWM", 850) / 1000.0;
  const int k = int(1000.0 * ws / (ws + wx) + 0.5);
  return {k, 1000};
}

// Run f1 on `st` and f2 on the plan's auxiliary stream concurrently, both after everything
// already enqueued on `st`; `st` continues after both (event fork/join; captured into graphs).
template <class F1, class F2>
void fork_join(Plan& P, cudaStream_t st, F1&& f1, F2&& f2) {
  std::lock_guard<std::mutex> lk(P.fork_mu);
  cudaStream_t aux = static_cast<cudaStream_t>(P.aux_stream);
  cudaEvent_t fk = static_cast<cudaEvent_t>(P.ev_fork), jn = static_cast<cudaEvent_t>(P.ev_join);
  cudaEventRecord(fk, st);
  cudaStreamWaitEvent(aux, fk, 0);
  f1(st);
  f2(aux);
  cudaEventRecord(jn, aux);
  cudaStreamWaitEvent(st, jn, 0);
}

// Reduced separable Hodge star y = K^{-1} M x using the diagonal 1D factors (host_setup.cpp):
//   eps (kind 0): component c is swept (Gamma_C^{p-2}, LU Hat G) along the two axes != c and
//                 scaled by 1/s along axis c: z pass {0,1}, y pass {0 -> y, 2}, x pass {1,2 -> y};
//   mu  (kind 1): component c is swept (Gamma_B^{p}, LU Hat G^T) along axis c only and scaled by
//                 s along the other two: strided pass {2 along z, 1 along y} (or two passes), x pass {0}.
void hodge_star_reduced(Plan& P, int which, const double* x, double* y, double* t, cudaStream_t st,
                        const double* scale = nullptr, int accum = 0, const Affine* aff = nullptr) {
  const int kind = (which == SGM_MASS_EPS) ? 0 : 1;
  struct {
    const double* scale;
  } M{scale ? scale : P.mass[which].scale};
  double *X[3], *Y[3], *T[3];
  comps_of(P, kind, x, X);
  comps_of(P, kind, y, Y);
  comps_of(P, kind, t, T);
  const int kz = kind == 0 ? SGM_K_EPS_Z : SGM_K_MU_Z, ky = kind == 0 ? SGM_K_EPS_Y : SGM_K_MU_Y,
            kx = kind == 0 ? SGM_K_EPS_X : SGM_K_MU_X;
  if (kind == 0) {
    // scheme 2: Hat G^{-1} Gamma_C^{p-2}; scheme 1: Gamma_B^p^{-1} Hat G^T (own axis: diag(1/s) in both)
    const int op = P.scheme == 1 ? OP_S1_EPS_OTH_W : OP_EPS_OTH;
    if (fork_on(P) && eps_merged(P)) {
      // strided pass {0 along z, 1 along z, 2 along y}, then concurrently {0 along y} (strided,
      // 1/3 of the SMs) and {1, 2 along x} (2/3 of the SMs, plan-owned stream)
      PassComp a3[3] = {{2, 0, X[0], T[0], op, {-1, -1, -1}, 1.0},
                        {2, 1, X[1], T[1], op, {-1, -1, -1}, 1.0},
                        {1, 2, X[2], T[2], op, {-1, -1, -1}, 1.0}};
      PassComp b1[1] = {{1, 0, T[0], Y[0], op, {0, -1, -1}, M.scale[0], accum, aff}};
      PassComp c2[2] = {{0, 1, T[1], Y[1], op, {-1, 0, -1}, M.scale[1], accum, aff},
                        {0, 2, T[2], Y[2], op, {-1, -1, 0}, M.scale[2], accum, aff}};
      { ProfScope ps(P, kz, st); sweep_pass_list(P, 0, a3, 3, st, 1); }
      // x side: components 1, 2 of e/d, x-extent a (P.ax[0].a)
      const Share sb = strided_share(P, 1, 1, 2, (P.ax[0].a % 2) == 0), sc = {sb.n - sb.k, sb.n};
      fork_join(P, st, [&](cudaStream_t s1) { ProfScope ps(P, ky, s1); sweep_pass_list(P, 0, b1, 1, s1, 0, sb); },
                [&](cudaStream_t s2) { ProfScope ps(P, kx, s2); sweep_pass_list(P, 0, c2, 2, s2, 1, sc); });
      return;
    }
    PassComp z[2] = {{2, 0, X[0], T[0], op, {-1, -1, -1}, 1.0}, {2, 1, X[1], T[1], op, {-1, -1, -1}, 1.0}};
    PassComp yy[2] = {{1, 0, T[0], Y[0], op, {0, -1, -1}, M.scale[0], accum, aff}, {1, 2, X[2], T[2], op, {-1, -1, -1}, 1.0}};
    PassComp xx[2] = {{0, 1, T[1], Y[1], op, {-1, 0, -1}, M.scale[1], accum, aff},
                      {0, 2, T[2], Y[2], op, {-1, -1, 0}, M.scale[2], accum, aff}};
    { ProfScope ps(P, kz, st); sweep_pass_list(P, 0, z, 2, st, 1); }
    { ProfScope ps(P, ky, st); sweep_pass_list(P, 0, yy, 2, st, 0); }
    { ProfScope ps(P, kx, st); sweep_pass_list(P, 0, xx, 2, st, 1); }
  } else {
    // scheme 2: Hat G^{-T} Gamma_B^p; scheme 1: Gamma_C^{p-2}^{-1} Hat G (other axes: diag(s) in both)
    const int op = P.scheme == 1 ? OP_S1_MU_OWN : OP_MU_OWN;
    PassComp z[1] = {{2, 2, X[2], Y[2], op, {1, 1, -1}, M.scale[2], accum, aff}};
    PassComp yy[1] = {{1, 1, X[1], Y[1], op, {1, -1, 1}, M.scale[1], accum, aff}};
    PassComp xx[1] = {{0, 0, X[0], Y[0], op, {-1, 1, 1}, M.scale[0], accum, aff}};
    if (mu_merged(P)) {
      // z-lines of component 2 and y-lines of component 1 in one strided launch; the x-lines of
      // component 0 (independent) concurrently on the plan-owned stream when forking is enabled
      PassComp zy[2] = {z[0], yy[0]};
      if (fork_on(P)) {
        // x side: component 0 of b/h, x-extent a
        const Share sd = strided_share(P, 2, 2, 1, (P.ax[0].a % 2) == 0), se = {sd.n - sd.k, sd.n};
        fork_join(P, st, [&](cudaStream_t s1) { ProfScope ps(P, kz, s1); sweep_pass_list(P, 1, zy, 2, s1, 1, sd); },
                  [&](cudaStream_t s2) { ProfScope ps(P, kx, s2); sweep_pass_list(P, 1, xx, 1, s2, 1, se); });
        return;
      }
      { ProfScope ps(P, kz, st); sweep_pass_list(P, 1, zy, 2, st, 1); }
    } else {
      { ProfScope ps(P, kz, st); sweep_pass_list(P, 1, z, 1, st, 1); }
      { ProfScope ps(P, ky, st); sweep_pass_list(P, 1, yy, 1, st, 0); }
    }
    { ProfScope ps(P, kx, st); sweep_pass_list(P, 1, xx, 1, st, 1); }
  }
}

// Whether the fused kernel has a fitting configuration for this plan's half step `which` (shared
// memory and segments; pointers of a real call are checked again when it is enqueued).
PrologueArgs make_pro(const Plan& P, int src_kind, const double* src, const double* jhat, const double* s_ptr,
                      double dt);
bool fused_fits(const Plan& P, int which, bool with_source) {
  const int kind = which == SGM_MASS_EPS ? 0 : 1;
  alignas(16) static double dummy[2];
  PrologueArgs pro = make_pro(P, 1 - kind, dummy, nullptr, nullptr, 1.0);
  for (int c = 0; c < 3; ++c) pro.src[c] = dummy;
  if (kind == 0 && with_source) pro.jhat[0] = pro.jhat[1] = pro.jhat[2] = dummy;
  PassComp pc[3];
  const int own = kind == 0 ? OP_EPS_OWN : OP_MU_OWN, oth = kind == 0 ? OP_EPS_OTH : OP_MU_OTH;
  if (!reduced_sched(P)) {
    for (int c = 0; c < 3; ++c) pc[c] = {2, c, dummy, dummy, own_or(2, c, own, oth), {-1, -1, -1}, 1.0};
  } else if (kind == 0) {
    pc[0] = {2, 0, dummy, dummy, oth, {-1, -1, -1}, 1.0};
    pc[1] = {2, 1, dummy, dummy, oth, {-1, -1, -1}, 1.0};
    pc[2] = {1, 2, dummy, dummy, oth, {-1, -1, -1}, 1.0};
  } else {
    pc[0] = {2, 2, dummy, dummy, own, {-1, -1, -1}, 1.0};
    pc[1] = {1, 1, dummy, dummy, own, {-1, -1, -1}, 1.0};
    pc[2] = {0, 0, dummy, dummy, own, {-1, -1, -1}, 1.0};
  }
  return fused_list(P, kind, pc, 3, nullptr, 0, kind + 1, pro, 0, true);
}

// The fused separable half step (SGM_OPT_FUSED): the Ampere / Faraday update of the state x is
// fused into the first sweep launch of its Hodge star (fsweep_kernel.cuh, SURVEY 8(d) fused P1):
//   reduced eps: fused {0, 1 along z; 2 along y} x -> t, then {0 along y} || {1, 2 along x} t -> y
//                (pipelined sweeps, concurrent as in hodge_star_reduced);
//   reduced mu:  fused {2 along z; 1 along y; 0 along x} x -> y;
//   full:        fused z pass (all components) x -> t, then the y and x passes.
// Returns false (nothing enqueued) when the fused kernel has no fitting configuration.
// eh = true: the (e,h)-state step -- x is unused (the curl source in `pro` gives the increment) and
// the star's output is accumulated into y (y += dt S(curl)).
bool star_fused(Plan& P, int which, double* x, double* y, double* t, cudaStream_t st, const PrologueArgs& pro,
                bool eh = false) {
  const int kind = (which == SGM_MASS_EPS) ? 0 : 1;
  const int fuse = kind + 1 + (eh ? 2 : 0);
  const int acc = eh ? 1 : 0;
  const double* sc = P.mass[which].scale;
  double *X[3], *Y[3], *T[3];
  comps_of(P, kind, x, X);
  comps_of(P, kind, y, Y);
  comps_of(P, kind, t, T);
  const int cls = kind == 0 ? SGM_K_FUSED_EPS : SGM_K_FUSED_MU;
  if (!reduced_sched(P)) {
    const int own = kind == 0 ? OP_EPS_OWN : OP_MU_OWN, oth = kind == 0 ? OP_EPS_OTH : OP_MU_OTH;
    PassComp z3[3];
    for (int c = 0; c < 3; ++c) z3[c] = {2, c, X[c], T[c], own_or(2, c, own, oth), {-1, -1, -1}, 1.0};
    if (!fused_list(P, kind, z3, 3, st, 1, fuse, pro, cls, true)) return false;
    fused_list(P, kind, z3, 3, st, 1, fuse, pro, cls, false);
    const int ky = kind == 0 ? SGM_K_EPS_Y : SGM_K_MU_Y, kx = kind == 0 ? SGM_K_EPS_X : SGM_K_MU_X;
    { ProfScope ps(P, ky, st); sweep_pass(P, kind, 1, T, T, own, oth, nullptr, true, true, st, 0); }
    { ProfScope ps(P, kx, st); sweep_pass(P, kind, 0, T, Y, own, oth, sc, true, true, st, 1, acc); }
    return true;
  }
  if (kind == 0) {
    const int op = OP_EPS_OTH;
    PassComp a3[3] = {{2, 0, X[0], T[0], op, {-1, -1, -1}, 1.0},
                      {2, 1, X[1], T[1], op, {-1, -1, -1}, 1.0},
                      {1, 2, X[2], T[2], op, {-1, -1, -1}, 1.0}};
    if (!fused_list(P, 0, a3, 3, st, 1, fuse, pro, cls, true)) return false;
    fused_list(P, 0, a3, 3, st, 1, fuse, pro, cls, false);
    PassComp b1[1] = {{1, 0, T[0], Y[0], op, {0, -1, -1}, sc[0], acc}};
    PassComp c2[2] = {{0, 1, T[1], Y[1], op, {-1, 0, -1}, sc[1], acc}, {0, 2, T[2], Y[2], op, {-1, -1, 0}, sc[2], acc}};
    if (fork_on(P)) {
      const Share sb = strided_share(P, 1, 1, 2, (P.ax[0].a % 2) == 0), sc2 = {sb.n - sb.k, sb.n};
      fork_join(P, st, [&](cudaStream_t s1) { ProfScope ps(P, SGM_K_EPS_Y, s1); sweep_pass_list(P, 0, b1, 1, s1, 0, sb); },
                [&](cudaStream_t s2) { ProfScope ps(P, SGM_K_EPS_X, s2); sweep_pass_list(P, 0, c2, 2, s2, 1, sc2); });
    } else {
      { ProfScope ps(P, SGM_K_EPS_Y, st); sweep_pass_list(P, 0, b1, 1, st, 0); }
      { ProfScope ps(P, SGM_K_EPS_X, st); sweep_pass_list(P, 0, c2, 2, st, 1); }
    }
    return true;
  }
  const int op = OP_MU_OWN;
  PassComp m3[3] = {{2, 2, X[2], Y[2], op, {1, 1, -1}, sc[2], acc},
                    {1, 1, X[1], Y[1], op, {1, -1, 1}, sc[1], acc},
                    {0, 0, X[0], Y[0], op, {-1, 1, 1}, sc[0], acc}};
  if (!fused_list(P, 1, m3, 3, st, 1, fuse, pro, cls, true)) return false;
  fused_list(P, 1, m3, 3, st, 1, fuse, pro, cls, false);
  return true;
}

// y = (A_z (x) A_y (x) A_x) x per component with 3 sweeps x -> t -> t -> y (x == y allowed).
// Axis order z, y, x: the Kronecker factors commute; the strided axes go first so
// a fused Ampere/Faraday update (first pass) reads its curl stencil coalesced.
void kron_pass3(const Plan& P, int kind, const double* x, double* y, double* t, int op_own, int op_oth,
                const double* scale, bool band, bool solve, cudaStream_t st) {
  double *X[3], *T[3], *Y[3];
  comps_of(P, kind, x, X);
  comps_of(P, kind, t, T);
  comps_of(P, kind, y, Y);
  sweep_pass(P, kind, 2, X, T, op_own, op_oth, nullptr, band, solve, st);
  sweep_pass(P, kind, 1, T, T, op_own, op_oth, nullptr, band, solve, st);
  sweep_pass(P, kind, 0, T, Y, op_own, op_oth, scale, band, solve, st);
}

PrologueArgs make_pro(const Plan& P, int src_kind, const double* src, const double* jhat, const double* s_ptr,
                      double dt) {
  PrologueArgs pa;
  std::memset(&pa, 0, sizeof(pa));
  double* S[3];
  comps_of(P, src_kind, src, S);
  for (int c = 0; c < 3; ++c) {
    pa.src[c] = S[c];
    comp_shape(P, src_kind, c, pa.sext[c]);
  }
  if (jhat) {  // the source of the updated state: j^ (Ampere, e-shaped) or c_b (Faraday, b-shaped)
    double* J[3];
    comps_of(P, 1 - src_kind, jhat, J);
    for (int c = 0; c < 3; ++c) pa.jhat[c] = J[c];
  }
  pa.s_ptr = s_ptr;
  pa.dt = dt;
  return pa;
}

// form1 = false: the 2-form masses of scheme 2 (eps: dual 2-forms, mu: primal 2-forms);
// form1 = true:  the 1-form masses of scheme 1 (eps: primal 1-forms of e, mu: dual 1-forms of h)
void hodge_args(const Plan& P, int which, const double* x, double* y, HodgeArgs& h, bool form1 = false,
                const WS* w = nullptr) {
  std::memset(&h, 0, sizeof(h));
  if (w) {
    h.scratch = w->scratch;
    h.scratch_cap = w->scratch_cap;
  }
  int kind = (which == SGM_MASS_EPS) ? 0 : 1;
  const MassData& MD = form1 ? P.mass1[which] : P.mass[which];
  double *X[3], *Y[3];
  comps_of(P, kind, x, X);
  comps_of(P, kind, y, Y);
  for (int c = 0; c < 3; ++c) {
    h.x[c] = X[c];
    h.y[c] = Y[c];
    comp_shape(P, kind, c, h.ext[c]);
    h.scale[c] = MD.scale[c];
  }
  h.W = MD.W_dev;
  h.full = (MD.kind == HODGE_FULL) ? 1 : 0;
  if (!form1 && MD.otf) {
    h.otf = 1;
    h.geo_tab = P.geo_dev;
    for (int r = 0; r < 3; ++r) h.geo_ctrl[r] = P.geo_dev + P.geo_ctrl_off[r];
    for (int a = 0; a < 3; ++a)
      for (int sv = 0; sv < 2; ++sv) h.geo_tab_off[a][sv] = int(P.geo_tab_off[a][sv]);
  }
  // own/other univariate spaces (space ids of basis_values_1d: Sp 0, Sp1 1, Dp1 2, Dp2 3):
  //   dual 2-forms own Dp1, other Dp2; primal 2-forms own Sp, other Sp1   (sec. 4.1)
  //   primal 1-forms own Sp1, other Sp;  dual 1-forms own Dp2, other Dp1
  int own, oth;
  if (!form1) {
    own = (which == SGM_MASS_EPS) ? 2 : 0;
    oth = (which == SGM_MASS_EPS) ? 3 : 1;
  } else {
    own = (which == SGM_MASS_EPS) ? 1 : 3;
    oth = (which == SGM_MASS_EPS) ? 0 : 2;
  }
  h.basis = P.basis_dev;
  h.first = P.first_dev;
  for (int a = 0; a < 3; ++a) {
    h.basis_off[a][0] = int(P.basis_off[a][own]);
    h.basis_off[a][1] = int(P.basis_off[a][oth]);
    h.first_off[a][0] = int(P.first_off[a][own]);
    h.first_off[a][1] = int(P.first_off[a][oth]);
    h.first0[a][0] = P.first0[a][own];
    h.first0[a][1] = P.first0[a][oth];
    h.nel[a] = P.n[a];
    std::copy_n(P.basis_mid[a][own], 25, h.uni[0][a]);
    std::copy_n(P.basis_mid[a][oth], 25, h.uni[1][a]);
    h.uni_lo[a][0] = P.basis_lo[a][own];
    h.uni_hi[a][0] = P.basis_hi[a][own];
    h.uni_lo[a][1] = P.basis_lo[a][oth];
    h.uni_hi[a][1] = P.basis_hi[a][oth];
  }
  h.Q = P.Q;
  h.dual = (which == SGM_MASS_EPS) ? 1 : 0;
  h.form = form1 ? (which == SGM_MASS_EPS ? 2 : 3) : h.dual;
}

// y = M x for one 2-form mass (separable: Kronecker of 1D Grams; else sum factorisation)
void mass_apply(const Plan& P, int which, const double* x, double* y, double* t, cudaStream_t st,
                const WS* w = nullptr) {
  int kind = (which == SGM_MASS_EPS) ? 0 : 1;
  const MassData& M = P.mass[which];
  if (M.kind == HODGE_SEPARABLE) {
    int own = (which == SGM_MASS_EPS) ? OP_EPS_OWN : OP_MU_OWN;
    int oth = (which == SGM_MASS_EPS) ? OP_EPS_OTH : OP_MU_OTH;
    kron_pass3(P, kind, x, y, t, own, oth, M.scale, true, false, st);
    return;
  }
  HodgeArgs h;
  hodge_args(P, which, x, y, h, false, w);
  launch_hodge_general(P.p, h, st);
}

// y = M^1 x for one scheme-1 1-form mass (sum factorisation with the 1-form weights)
void mass1_apply(const Plan& P, int which, const double* x, double* y, cudaStream_t st, const WS* w = nullptr) {
  HodgeArgs h;
  hodge_args(P, which, x, y, h, true, w);
  launch_hodge_general(P.p, h, st);
}

// Scheme 1 with a non-separable 1-form mass (curved map or variable material): the Hodge star
// M^1 y = K^T x (K = K1 for eps, K~1 for mu) by preconditioned conjugate gradients,
// entirely on the device (scalars stay in device memory, a fixed iteration count).  Preconditioner:
// the separable scheme-1 star with the mean material, P^{-1} v = S1(K^{-T} v) where
// S1 = M^1_sep^{-1} K^T is the reduced sweep schedule, so P = M^1_sep (Kronecker Grams).
void pcg_star(Plan& P, int which, const double* x, double* y, const WS& w, cudaStream_t st,
              std::vector<double>* trace = nullptr) {
  const int kind = (which == SGM_MASS_EPS) ? 0 : 1;
  const size_t N = form_len(P, kind);
  double* res = P.pcg_buf;
  double* z = res + P.pcg_n;
  double* pv = z + P.pcg_n;
  double* q = pv + P.pcg_n;
  double* scal = w.partials + 4 * partial_blocks();  // [0..3]: rz (two slots), pq
  // transposed pairing apply and solve tables: K1^T = Hat M^T (own) x Hat G^T (other);
  // K~1^T = Hat G (own) x Hat M (other)
  const int app_own = kind == 0 ? OP_APPLY_MT : OP_APPLY_G, app_oth = kind == 0 ? OP_APPLY_GT : OP_APPLY_M;
  const int sol_own = kind == 0 ? OP_MU_OTH : OP_EPS_OTH, sol_oth = kind == 0 ? OP_MU_OWN : OP_EPS_OWN;
  const double gbar = P.mass1[which].material_c;  // the material's mean (upload_mass1)
  const double psc[3] = {1.0 / gbar, 1.0 / gbar, 1.0 / gbar};
  auto precond = [&](const double* v, double* out) {
    kron_pass3(P, kind, v, out, w.t, sol_own, sol_oth, nullptr, false, true, st);  // K^{-T} v
    hodge_star_reduced(P, which, out, out, w.t, st, psc);                          // S1 (in place)
  };
  kron_pass3(P, kind, x, res, w.t, app_own, app_oth, nullptr, true, false, st);  // r = K^T x
  cudaMemsetAsync(y, 0, N * sizeof(double), st);
  precond(res, z);
  cudaMemcpyAsync(pv, z, N * sizeof(double), cudaMemcpyDeviceToDevice, st);
  int a = 0;
  launch_dot_partials(res, z, N, w.partials, 0, st);
  launch_finalize_sum(w.partials, 1, 1.0, scal + a, st);
  // calibration (plan time): record r.z after every iteration (host synchronisation)
  auto record = [&](const double* dev_scalar) {
    double v = 0.0;
    cudaMemcpyAsync(&v, dev_scalar, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    trace->push_back(v);
  };
  if (trace) record(scal + a);
  const int iters = trace ? 200 : (P.pcg_fixed > 0 ? P.pcg_fixed : P.pcg_iters_m[which]);
  for (int k = 0; k < iters; ++k) {
    mass1_apply(P, which, pv, q, st, &w);
    launch_dot_partials(pv, q, N, w.partials, 0, st);
    launch_finalize_sum(w.partials, 1, 1.0, scal + 2, st);
    launch_axpy_ratio(y, pv, N, scal + a, scal + 2, 1.0, st);
    launch_axpy_ratio(res, q, N, scal + a, scal + 2, -1.0, st);
    precond(res, z);
    launch_dot_partials(res, z, N, w.partials, 0, st);
    launch_finalize_sum(w.partials, 1, 1.0, scal + (1 - a), st);
    launch_xpby_ratio(pv, z, N, scal + (1 - a), scal + a, st);
    a = 1 - a;
    if (trace) {
      record(scal + a);
      if (!(trace->back() > 1e-28 * trace->front())) break;  // preconditioned residual 1e-14 relative
    }
  }
}

// Plan-time choice of the PCG iteration count of each non-separable scheme-1 star: solve once for a
// deterministic right-hand side with the residual read back after every iteration; the count that
// reaches a relative preconditioned residual of 1e-14, plus 3, is used from then on.
sgm_status calibrate_pcg(Plan& P) {
  std::vector<double> xh(std::max(P.N_e, P.N_h));
  uint64_t st64 = 0x9e3779b97f4a7c15ULL;
  for (double& v : xh) {  // splitmix64 uniforms in (-1, 1): any RHS exciting all modes will do
    st64 += 0x9e3779b97f4a7c15ULL;
    uint64_t z = st64;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    v = double(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
  double *x = nullptr, *y = nullptr;
  void* ws = nullptr;
  const size_t n = xh.size(), wb = ws_need(P);
  if (cudaMalloc(&x, n * 8) != cudaSuccess || cudaMalloc(&y, n * 8) != cudaSuccess || cudaMalloc(&ws, wb) != cudaSuccess) {
    cudaFree(x);
    cudaFree(y);
    cudaFree(ws);
    return fail(SGM_E_NOMEM, "cudaMalloc failed for the PCG calibration");
  }
  cudaMemcpy(x, xh.data(), n * 8, cudaMemcpyHostToDevice);
  WS w;
  ws_carve(P, ws, wb, w);
  for (int m = 0; m < 2; ++m) {
    if (P.mass1[m].kind == HODGE_SEPARABLE) continue;
    std::vector<double> tr;
    pcg_star(P, m, x, y, w, nullptr, &tr);
    P.pcg_iters_m[m] = std::min(200, std::max(5, int(tr.size()) - 1 + 3));
  }
  cudaFree(x);
  cudaFree(y);
  cudaFree(ws);
  return cuda_check(&P, "calibrate_pcg");
}

sgm_status ensure_pcg(Plan& P) {
  const size_t n = std::max(P.N_e, P.N_h);
  if (P.pcg_buf && P.pcg_n >= n) return SGM_OK;
  if (P.pcg_buf) cudaFree(P.pcg_buf);
  P.pcg_buf = nullptr;
  if (cudaMalloc(&P.pcg_buf, 4 * n * sizeof(double)) != cudaSuccess) return fail(SGM_E_NOMEM, "cudaMalloc failed for PCG");
  P.pcg_n = n;
  return SGM_OK;
}

// build and upload the scheme-1 1-form weights of both masses (host-only plans: classification)
sgm_status upload_mass1(Plan& P) {
  if (P.device < 0) {
    for (int m = 0; m < 2; ++m) {
      P.mass1[m].const_material = P.mass[m].const_material;
      P.mass1[m].kind = P.mass[m].kind;
    }
    return SGM_OK;
  }
  for (int m = 0; m < 2; ++m) {
    std::vector<double> W;
    std::string err;
    sgm_status st = build_mass1(P, m, W, err);
    if (st != SGM_OK) return fail(st, err);
    MassData& M = P.mass1[m];
    if (!M.const_material) {  // preconditioner material: the mean over the quadrature points
      double s = 0.0;
      for (double v : P.mass[m].values_host) s += v;
      M.material_c = s / double(P.mass[m].values_host.size());
    }
    if (M.W_dev) cudaFree(M.W_dev);
    M.W_dev = nullptr;
    if (!W.empty() && P.device >= 0) {
      if (hodge_uses_brick(P.p, P.Q)) hodge_brick_relayout(P.Q, P.n, int(W.size() / P.n_qp), W);
      if (cudaMalloc(&M.W_dev, W.size() * sizeof(double)) != cudaSuccess)
        return fail(SGM_E_NOMEM, "cudaMalloc failed for scheme-1 weights");
      cudaMemcpy(M.W_dev, W.data(), W.size() * sizeof(double), cudaMemcpyHostToDevice);
    }
  }
  if (P.device >= 0) {
    for (int m = 0; m < 2; ++m)
      if (P.mass1[m].kind != HODGE_SEPARABLE) {
        sgm_status st = ensure_pcg(P);
        if (st != SGM_OK) return st;
        return calibrate_pcg(P);
      }
  }
  return SGM_OK;
}

sgm_status upload_basis(Plan& P) {
  std::vector<double> vals_all;
  std::vector<int> first_all;
  for (int a = 0; a < 3; ++a)
    for (int s = 0; s < 4; ++s) {
      std::vector<double> v;
      std::vector<int> f;
      basis_values_1d(P.p, P.n[a], P.Q, s, v, f);
      P.basis_off[a][s] = vals_all.size();
      if (P.Q * (P.p + 1) <= 25) {
        const size_t tl = size_t(P.Q) * (P.p + 1);
        const int mid = P.n[a] / 2;
        std::copy_n(v.begin() + mid * tl, tl, P.basis_mid[a][s]);
        auto same = [&](int e) { return std::equal(v.begin() + e * tl, v.begin() + (e + 1) * tl, v.begin() + mid * tl); };
        int lo = mid, hi = mid + 1;
        while (lo > 0 && same(lo - 1)) --lo;
        while (hi < P.n[a] && same(hi)) ++hi;
        P.basis_lo[a][s] = lo;
        P.basis_hi[a][s] = hi;
      }
      P.first_off[a][s] = first_all.size();
      P.first0[a][s] = f[0];
      for (int e = 0; e < P.n[a]; ++e)
        if (f[e] != f[0] + e) return fail(SGM_E_UNSUPPORTED, "first-index table is not affine");
      vals_all.insert(vals_all.end(), v.begin(), v.end());
      first_all.insert(first_all.end(), f.begin(), f.end());
    }
  if (cudaMalloc(&P.basis_dev, vals_all.size() * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&P.first_dev, first_all.size() * sizeof(int)) != cudaSuccess)
    return fail(SGM_E_NOMEM, "cudaMalloc failed for basis tables");
  cudaMemcpy(P.basis_dev, vals_all.data(), vals_all.size() * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(P.first_dev, first_all.data(), first_all.size() * sizeof(int), cudaMemcpyHostToDevice);
  return cuda_check(&P, "upload_basis");
}

// workspace doubles of the general Hodge's deterministic accumulation (the largest of the non-separable
// masses: scheme-2 2-forms, and with scheme 1 its 1-forms); device plans only
void update_scratch_need(Plan& P) {
  size_t need = 0;
  if (P.device >= 0) {
    for (int m = 0; m < 2; ++m) {
      if (P.mass[m].kind != HODGE_SEPARABLE)
        need = std::max(need, hodge_scratch_doubles(P.p, P.Q, m == SGM_MASS_EPS ? 1 : 0,
                                                    P.mass[m].kind == HODGE_FULL ? 1 : 0, P.n));
      if (P.scheme == 1 && P.mass1[m].kind != HODGE_SEPARABLE)
        need = std::max(need, hodge_scratch_doubles(P.p, P.Q, m == SGM_MASS_EPS ? 2 : 3,
                                                    P.mass1[m].kind == HODGE_FULL ? 1 : 0, P.n));
    }
  }
  P.hodge_scratch = need;
}

sgm_status set_material_impl(Plan& P, int which, const double* values, double c) {
  std::vector<double> W;
  std::string err;
  // host-only plans classify but do not build weights
  if (P.device < 0) {
    if (values) {
      for (size_t i = 0; i < P.n_qp; ++i)
        if (!(values[i] > 0.0) || !std::isfinite(values[i]))
          return fail(SGM_E_MATERIAL, "material must be positive and finite at every quadrature point");
    } else if (!(c > 0.0) || !std::isfinite(c)) {
      return fail(SGM_E_MATERIAL, "material constant must be positive and finite");
    }
    MassData& M = P.mass[which];
    M.const_material = (values == nullptr);
    M.kind = P.affine_diag ? (values ? HODGE_SCALAR : HODGE_SEPARABLE) : HODGE_FULL;
    return SGM_OK;
  }
  sgm_status st = build_mass(P, which, values, c, W, err);
  if (st != SGM_OK) return fail(st, err);
  MassData& M = P.mass[which];
  if (M.W_dev) {
    cudaFree(M.W_dev);
    M.W_dev = nullptr;
  }
  if (!W.empty()) {
    // the brick kernel's HBM layout (one contiguous chunk per brick and element layer)
    if (hodge_uses_brick(P.p, P.Q)) hodge_brick_relayout(P.Q, P.n, int(W.size() / P.n_qp), W);
    if (cudaMalloc(&M.W_dev, W.size() * sizeof(double)) != cudaSuccess)
      return fail(SGM_E_NOMEM, "cudaMalloc failed for Hodge weights");
    cudaMemcpy(M.W_dev, W.data(), W.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  if (M.otf && !P.geo_dev) {
    // on-the-fly geometry: the map's control points and S_p tables (once per plan)
    std::vector<double> buf;
    build_geo_buffer(P, buf, P.geo_ctrl_off, P.geo_tab_off);
    if (cudaMalloc(&P.geo_dev, buf.size() * sizeof(double)) != cudaSuccess)
      return fail(SGM_E_NOMEM, "cudaMalloc failed for the map tables");
    cudaMemcpy(P.geo_dev, buf.data(), buf.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  update_scratch_need(P);
  return cuda_check(&P, "set_material");
}

sgm_status check_plan(sgm_plan plan, bool need_device) {
  if (!plan) return fail(SGM_E_INVALID_ARG, "plan is NULL");
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (need_device && P->device < 0) return fail(SGM_E_INVALID_ARG, "host-only plan cannot run device calls");
  if (P->sticky_cuda_error) return fail(SGM_E_CUDA, "plan has a sticky CUDA error");
  return SGM_OK;
}

inline Plan* PL(sgm_plan p) { return reinterpret_cast<Plan*>(p); }

// one half step on device pointers (SURVEY 8(a) a1-a3 for half 0, a4-a6 for half 1):
//   half 0 (eps, kind 0): d <- d + tau (D~1 h - s j); e <- K1^{-1} M~2_{1/eps} d
//   half 1 (mu,  kind 1): b <- b - tau D1 e;          h <- K~1^{-1} M2_{1/mu} b
// lift (sgm_step_lifted, step k of the call): the lifted star and Faraday terms of the time-separable
// inhomogeneous Dirichlet data (reading Z29):
//   e <- S_eps d - g_k w_e;   b <- b - tau (D1 e + g_k c_b);   h <- S_mu b + q0 + beta_k q1
void half_step(Plan& P, int half, double* d, double* e, double* b, double* h, const double* jhat,
               const double* s_ptr, double tau, const WS& w, cudaStream_t st, const sgm_lifting* lift = nullptr,
               int k = 0) {
  double *D[3], *E[3], *B[3], *H[3], *T[3], *Rr[3];
  comps_of(P, 0, d, D);
  comps_of(P, 0, e, E);
  comps_of(P, 1, b, B);
  comps_of(P, 1, h, H);
  const int kind = half;
  const int mass = half == 0 ? SGM_MASS_EPS : SGM_MASS_MU;
  const int pro = half == 0 ? PRO_AMPERE : PRO_FARADAY;
  const int own = half == 0 ? OP_EPS_OWN : OP_MU_OWN, oth = half == 0 ? OP_EPS_OTH : OP_MU_OTH;
  const int kx = half == 0 ? SGM_K_EPS_Z : SGM_K_MU_Z;
  const int ky = half == 0 ? SGM_K_EPS_Y : SGM_K_MU_Y, kz = half == 0 ? SGM_K_EPS_X : SGM_K_MU_X;
  double** state = half == 0 ? D : B;
  double** outv = half == 0 ? E : H;
  PrologueArgs pa = half == 0 ? make_pro(P, 1, h, jhat, s_ptr, tau)
                               : make_pro(P, 0, e, lift ? lift->c_b : nullptr, lift ? lift->g + k : nullptr, tau);
  const MassData& M = P.mass[mass];
  comps_of(P, kind, w.t, T);
  Affine af{};
  const Affine* aff = nullptr;
  if (lift && half == 0 && lift->w_e) {
    af = Affine{{lift->w_e, nullptr}, {lift->g + k, nullptr}, {-1.0, 0.0}};
    aff = &af;
  } else if (lift && half == 1 && (lift->q0 || lift->q1)) {
    af = Affine{{lift->q0, lift->q1}, {nullptr, lift->beta + k}, {1.0, 1.0}};
    aff = &af;
  }
  // fused schedule (SGM_OPT_FUSED): the update runs inside the first sweep launch of the half step
  // (falls back to the separate update kernel when the fused kernel has no fitting configuration)
  if (!lift && M.kind == HODGE_SEPARABLE && fused_sched(P) && star_fused(P, mass, state[0], outv[0], w.t, st, pa))
    return;
  SweepArgs a;
  std::memset(&a, 0, sizeof(a));
  a.ncomp = 3;
  for (int c = 0; c < 3; ++c) {
    comp_shape(P, kind, c, a.comp[c].ext);
    a.comp[c].in = state[c];
  }
  a.pro = pa;
  { ProfScope ps(P, SGM_K_UPDATE, st); launch_update(pro, a, st); }
  if (P.scheme == 1 && P.mass1[mass].kind != HODGE_SEPARABLE) {
    { ProfScope ps(P, SGM_K_HODGE_GENERAL, st); pcg_star(P, mass, state[0], outv[0], w, st); }
  } else if (M.kind == HODGE_SEPARABLE && reduced_sched(P)) {
    hodge_star_reduced(P, mass, state[0], outv[0], w.t, st, nullptr, 0, aff);
  } else if (M.kind == HODGE_SEPARABLE) {
    // streaming update kernel, then the three mass . solve sweeps (z, y, x); snake order: update
    // forward, z backward, y forward, x backward (each kernel starts on the tiles its predecessor
    // wrote last)
    { ProfScope ps(P, kx, st); sweep_pass(P, kind, 2, state, T, own, oth, nullptr, true, true, st, 1); }
    { ProfScope ps(P, ky, st); sweep_pass(P, kind, 1, T, T, own, oth, nullptr, true, true, st, 0); }
    { ProfScope ps(P, kz, st); sweep_pass(P, kind, 0, T, outv, own, oth, M.scale, true, true, st, 1, 0, aff); }
  } else {
    { ProfScope ps(P, SGM_K_HODGE_GENERAL, st); mass_apply(P, mass, state[0], w.r, w.t, st, &w); }
    comps_of(P, kind, w.r, Rr);
    { ProfScope ps(P, SGM_K_SOLVE_Z, st); sweep_pass(P, kind, 2, Rr, T, own, oth, nullptr, false, true, st); }
    { ProfScope ps(P, ky, st); sweep_pass(P, kind, 1, T, T, own, oth, nullptr, false, true, st); }
    { ProfScope ps(P, kz, st); sweep_pass(P, kind, 0, T, outv, own, oth, nullptr, false, true, st, 0, 0, aff); }
  }
}

// One half step of the (e,h)-state variant (reading Z30): with e = K1^{-1} M~2 d
// and h = K~1^{-1} M2 b the four-vector step is, exactly,
//   half 0: e <- e + K1^{-1} M~2_{1/eps} (tau (D~1 h - s j^))      (eqs. discrete2_ampere + hodge_eps)
//   half 1: h <- h - K~1^{-1} M2_{1/mu} (tau D1 e)                  (eqs. discrete2_faraday + hodge_mu)
// (the Petrov-Galerkin form in E_h, H_h), so d and b are never stored.  The increment's
// curl is the update kernel in increment mode (or fused into the first sweep with SGM_OPT_FUSED) and
// the star's last sweeps accumulate into e / h.
void half_step_eh(Plan& P, int half, double* e, double* h, const double* jhat, const double* s_ptr, double tau,
                  const WS& w, cudaStream_t st) {
  const int kind = half;
  const int mass = half == 0 ? SGM_MASS_EPS : SGM_MASS_MU;
  const int own = half == 0 ? OP_EPS_OWN : OP_MU_OWN, oth = half == 0 ? OP_EPS_OTH : OP_MU_OTH;
  const int ky = half == 0 ? SGM_K_EPS_Y : SGM_K_MU_Y, kx = half == 0 ? SGM_K_EPS_X : SGM_K_MU_X;
  double* out = half == 0 ? e : h;
  PrologueArgs pa = half == 0 ? make_pro(P, 1, h, jhat, s_ptr, tau) : make_pro(P, 0, e, nullptr, nullptr, tau);
  const MassData& M = P.mass[mass];
  if (M.kind == HODGE_SEPARABLE && fused_sched(P) && star_fused(P, mass, nullptr, out, w.t, st, pa, true)) return;
  // the increment r = tau (D~1 h - s j^) or -tau D1 e into the workspace
  double* r = M.kind == HODGE_SEPARABLE ? w.r : w.t;
  SweepArgs a;
  std::memset(&a, 0, sizeof(a));
  a.ncomp = 3;
  double* R[3];
  comps_of(P, kind, r, R);
  for (int c = 0; c < 3; ++c) {
    comp_shape(P, kind, c, a.comp[c].ext);
    a.comp[c].in = R[c];
  }
  a.pro = pa;
  { ProfScope ps(P, SGM_K_UPDATE, st); launch_update(half == 0 ? PRO_AMPERE_INC : PRO_FARADAY_INC, a, st); }
  double *T[3], *O[3], *Rr[3];
  comps_of(P, kind, w.t, T);
  comps_of(P, kind, out, O);
  if (M.kind == HODGE_SEPARABLE && reduced_sched(P)) {
    hodge_star_reduced(P, mass, r, out, w.t, st, nullptr, 1);
  } else if (M.kind == HODGE_SEPARABLE) {
    { ProfScope ps(P, half == 0 ? SGM_K_EPS_Z : SGM_K_MU_Z, st); sweep_pass(P, kind, 2, R, T, own, oth, nullptr, true, true, st, 1); }
    { ProfScope ps(P, ky, st); sweep_pass(P, kind, 1, T, T, own, oth, nullptr, true, true, st, 0); }
    { ProfScope ps(P, kx, st); sweep_pass(P, kind, 0, T, O, own, oth, M.scale, true, true, st, 1, 1); }
  } else {
    { ProfScope ps(P, SGM_K_HODGE_GENERAL, st); mass_apply(P, mass, w.t, w.r, nullptr, st, &w); }
    comps_of(P, kind, w.r, Rr);
    { ProfScope ps(P, SGM_K_SOLVE_Z, st); sweep_pass(P, kind, 2, Rr, T, own, oth, nullptr, false, true, st); }
    { ProfScope ps(P, ky, st); sweep_pass(P, kind, 1, T, T, own, oth, nullptr, false, true, st); }
    { ProfScope ps(P, kx, st); sweep_pass(P, kind, 0, T, O, own, oth, nullptr, false, true, st, 0, 1); }
  }
}

// one leapfrog step (eqs. discrete2_*)
void step_once(Plan& P, double* d, double* e, double* b, double* h, const double* jhat, const double* s_ptr,
               double dt, const WS& w, cudaStream_t st) {
  half_step(P, 0, d, e, b, h, jhat, s_ptr, dt, w, st);
  half_step(P, 1, d, e, b, h, jhat, s_ptr, dt, w, st);
}

}  // namespace
}  // namespace sgm

using namespace sgm;

extern "C" {

const char* sgm_last_error(void) { return g_err.c_str(); }
#ifdef SGM_CHECKED
const char* sgm_version(void) { return "sgm 0.1 (sm_100a, fp64, checked)"; }
#else
const char* sgm_version(void) { return "sgm 0.1 (sm_100a, fp64)"; }
#endif

#ifdef SGM_TUNING
// tuning build only (not part of sgm.h): copy the traced launch's timeline to the host
extern "C" int sgm_tune_trace(unsigned long long* host, size_t n) {
  unsigned long long* d = sgm::g_trace_ptr;
  if (!d) return 1;
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  if (n > sgm::kTraceLen) n = sgm::kTraceLen;
  return cudaMemcpy(host, d, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 3;
}
#endif

sgm_status sgm_check_read(int reset, unsigned* count, unsigned* first) {
#ifdef SGM_CHECKED
  unsigned h[2] = {0u, 0u};
  unsigned* d = sgm::check_buffer();
  if (!d) return fail(SGM_E_CUDA, "sgm_check_read: no violation buffer");
  if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(SGM_E_CUDA, "sgm_check_read: device error");
  if (reset && cudaMemset(d, 0, sizeof(h)) != cudaSuccess) return fail(SGM_E_CUDA, "sgm_check_read: reset failed");
  if (count) *count = h[0];
  if (first) *first = h[1];
  return SGM_OK;
#else
  (void)reset;
  (void)count;
  (void)first;
  return fail(SGM_E_UNSUPPORTED, "sgm_check_read: not a verification build (libsgm_checked.so)");
#endif
}

sgm_status sgm_plan_create(const sgm_plan_desc* desc, sgm_plan* out) {
  if (!desc || !out) return fail(SGM_E_INVALID_ARG, "desc/out is NULL");
  *out = nullptr;
  const int p = desc->degree;
  for (int a = 0; a < 3; ++a)
    if (desc->n_el[a] < 1) return fail(SGM_E_INVALID_ARG, "n_el must be >= 1");
  if (p < SGM_PMIN || p > SGM_PMAX) return fail(SGM_E_UNSUPPORTED, "degree outside the compiled range 2..4");
  int Q = desc->quad_points == 0 ? p + 1 : desc->quad_points;
  if (Q < p + 1 || Q > 8) return fail(SGM_E_INVALID_ARG, "quad_points must be 0 or in [p+1, 8]");
  // lines longer than kMaxLine are swept in overlapping windows (launch_sweep); the kernels index
  // the elements of one component with 32-bit integers
  if (long(desc->n_el[0] + p - 1) * (desc->n_el[1] + p - 1) * (desc->n_el[2] + p - 1) > kMaxCompElems)
    return fail(SGM_E_UNSUPPORTED, "a form component above 2^31 - 2^20 elements (32-bit indices)");
  Plan* P = new (std::nothrow) Plan();
  if (!P) return fail(SGM_E_NOMEM, "out of host memory");
  P->p = p;
  P->Q = Q;
  P->device = desc->device;
  P->graph_enabled = tune_int("SGM_GRAPH", 1) != 0;
  std::string err;
  for (int a = 0; a < 3; ++a) {
    P->n[a] = desc->n_el[a];
    build_axis(p, P->n[a], Q, P->ax[a], err);
  }
  P->N_e = form_len(*P, 0);
  P->N_h = form_len(*P, 1);
  if (desc->geom_ctrl) {
    P->has_geom = true;
    size_t nc = size_t(P->n[0] + p) * (P->n[1] + p) * (P->n[2] + p) * 3;
    P->ctrl.assign(desc->geom_ctrl, desc->geom_ctrl + nc);
    if (desc->geom_weights) {
      P->wts.assign(desc->geom_weights, desc->geom_weights + nc / 3);
      for (double w : P->wts)
        if (!(w > 0.0) || !std::isfinite(w)) {
          delete P;
          return fail(SGM_E_GEOMETRY, "rational map weights must be positive and finite");
        }
    }
  }
  sgm_status st = build_tables(*P, err);
  if (st == SGM_OK) st = build_geometry(*P, err);
#ifdef SGM_CHECKED
  if (st == SGM_OK) {  // allocate the violation buffer now: the launchers may run under stream capture
    DeviceGuard dg(P->device);
    if (!check_buffer()) st = SGM_E_CUDA;
  }
#endif
  if (st != SGM_OK) {
    delete P;
    return fail(st, err);
  }
  if (P->device >= 0) {
    DeviceGuard g(P->device);
    if (!g.ok) {
      delete P;
      return fail(SGM_E_CUDA, "cudaSetDevice failed");
    }
    size_t tb = P->tables_host.size() * sizeof(double);
    if (cudaMalloc(&P->tables_dev, tb) != cudaSuccess) {
      delete P;
      return fail(SGM_E_NOMEM, "cudaMalloc failed for tables");
    }
    cudaMemcpy(P->tables_dev, P->tables_host.data(), tb, cudaMemcpyHostToDevice);
    if (!P->wide_host.empty()) {
      const size_t wb = P->wide_host.size() * sizeof(double);
      if (cudaMalloc(&P->wide_dev, wb) != cudaSuccess) {
        delete P;
        return fail(SGM_E_NOMEM, "cudaMalloc failed for tables");
      }
      cudaMemcpy(P->wide_dev, P->wide_host.data(), wb, cudaMemcpyHostToDevice);
    }
    if (std::max({P->ax[0].b, P->ax[1].b, P->ax[2].b}) > kMaxLine) {
      // lines swept in windows: in-place sweeps read their input from a copy (launch_sweep)
      const size_t cb = size_t(P->ax[0].b) * P->ax[1].b * P->ax[2].b * sizeof(double);
      if (cudaMalloc(&P->win_scratch, cb) != cudaSuccess) {
        cudaFree(P->tables_dev);
        cudaFree(P->wide_dev);
        delete P;
        return fail(SGM_E_NOMEM, "cudaMalloc failed for the window scratch");
      }
    }
    {
      cudaStream_t aux;
      cudaEvent_t e1, e2;
      cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&e1, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
      P->aux_stream = aux;
      P->ev_fork = e1;
      P->ev_join = e2;
      P->fork_enabled = tune_int("SGM_FORK", 1) != 0;
      if (const int it = tune_int("SGM_PCG_ITERS", 0)) P->pcg_fixed = std::max(1, it);
    }
    st = upload_basis(*P);
    if (st != SGM_OK) {
      sgm_plan_destroy(reinterpret_cast<sgm_plan>(P));
      return st;
    }
  }
  for (int m = 0; m < 2; ++m) {
    DeviceGuard g(P->device >= 0 ? P->device : 0);
    st = set_material_impl(*P, m, nullptr, 1.0);
    if (st != SGM_OK) {
      std::string e2 = g_err;
      sgm_plan_destroy(reinterpret_cast<sgm_plan>(P));
      return fail(st, e2);
    }
  }
  *out = reinterpret_cast<sgm_plan>(P);
  return SGM_OK;
}

sgm_status sgm_plan_destroy(sgm_plan plan) {
  if (!plan) return SGM_OK;
  Plan* P = PL(plan);
  if (P->device >= 0) {
    DeviceGuard g(P->device);
    if (P->graph_exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(P->graph_exec));
    if (P->graph_exec_m) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(P->graph_exec_m));
    if (P->graph_exec_c) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(P->graph_exec_c));
    if (P->graph_exec_e) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(P->graph_exec_e));
    cudaFree(P->tables_dev);
    cudaFree(P->wide_dev);
    cudaFree(P->win_scratch);
    cudaFree(P->basis_dev);
    cudaFree(P->first_dev);
    for (int m = 0; m < 2; ++m) cudaFree(P->mass[m].W_dev);
    cudaFree(P->geo_dev);
    for (int m = 0; m < 2; ++m) cudaFree(P->mass1[m].W_dev);
    cudaFree(P->pcg_buf);
    cudaFree(P->mirror);
    for (auto& r : P->prof) {
      cudaEventDestroy(static_cast<cudaEvent_t>(r.a));
      cudaEventDestroy(static_cast<cudaEvent_t>(r.b));
    }
    for (void* e : P->ev_pool) cudaEventDestroy(static_cast<cudaEvent_t>(e));
    if (P->aux_stream) cudaStreamDestroy(static_cast<cudaStream_t>(P->aux_stream));
    if (P->ev_fork) cudaEventDestroy(static_cast<cudaEvent_t>(P->ev_fork));
    if (P->ev_join) cudaEventDestroy(static_cast<cudaEvent_t>(P->ev_join));
  }
  delete P;
  return SGM_OK;
}

sgm_status sgm_plan_len(sgm_plan plan, sgm_form form, size_t* n) {
  if (!plan || !n) return fail(SGM_E_INVALID_ARG, "NULL argument");
  switch (form) {
    case SGM_FORM_E: case SGM_FORM_D: *n = PL(plan)->N_e; return SGM_OK;
    case SGM_FORM_B: case SGM_FORM_H: *n = PL(plan)->N_h; return SGM_OK;
  }
  return fail(SGM_E_INVALID_ARG, "bad form");
}

sgm_status sgm_plan_shape(sgm_plan plan, sgm_form form, int comp, int xyz[3]) {
  if (!plan || !xyz || comp < 0 || comp > 2) return fail(SGM_E_INVALID_ARG, "bad argument");
  if (form < SGM_FORM_E || form > SGM_FORM_H) return fail(SGM_E_INVALID_ARG, "bad form");
  int kind = (form == SGM_FORM_E || form == SGM_FORM_D) ? 0 : 1;
  comp_shape(*PL(plan), kind, comp, xyz);
  return SGM_OK;
}

sgm_status sgm_plan_qp_count(sgm_plan plan, size_t* n_qp) {
  if (!plan || !n_qp) return fail(SGM_E_INVALID_ARG, "NULL argument");
  *n_qp = PL(plan)->n_qp;
  return SGM_OK;
}

sgm_status sgm_plan_qp_coords(sgm_plan plan, double* host_xyz) {
  if (!plan || !host_xyz) return fail(SGM_E_INVALID_ARG, "NULL argument");
  qp_coords(*PL(plan), host_xyz);
  return SGM_OK;
}

sgm_status sgm_plan_table(sgm_plan plan, sgm_table which, int axis, double* host_out, int* L) {
  if (!plan || !L || axis < 0 || axis > 2) return fail(SGM_E_INVALID_ARG, "bad argument");
  const Axis& X = PL(plan)->ax[axis];
  const std::vector<double>* src = nullptr;
  int n = 0;
  switch (which) {
    case SGM_TAB_G: src = &X.G; n = X.a; break;
    case SGM_TAB_M: src = &X.M; n = X.b; break;
    case SGM_TAB_GAMMA_B1: src = &X.GB1; n = X.b; break;
    case SGM_TAB_GAMMA_C2: src = &X.GC2; n = X.a; break;
    case SGM_TAB_GAMMA_BP: src = &X.GBp; n = X.a; break;
    case SGM_TAB_GAMMA_C1: src = &X.GC1; n = X.b; break;
    default: return fail(SGM_E_INVALID_ARG, "bad table");
  }
  *L = n;
  if (host_out) std::memcpy(host_out, src->data(), src->size() * sizeof(double));
  return SGM_OK;
}

sgm_status sgm_plan_hodge_separable(sgm_plan plan, sgm_mass mass, int* separable) {
  if (!plan || !separable || (mass != SGM_MASS_EPS && mass != SGM_MASS_MU))
    return fail(SGM_E_INVALID_ARG, "bad argument");
  *separable = PL(plan)->mass[mass].kind == HODGE_SEPARABLE ? 1 : 0;
  return SGM_OK;
}

sgm_status sgm_plan_set_scheme(sgm_plan plan, int scheme) {
  if (!plan) return fail(SGM_E_INVALID_ARG, "plan is NULL");
  Plan* P = PL(plan);
  if (scheme != 1 && scheme != 2) return fail(SGM_E_INVALID_ARG, "scheme must be 1 or 2");
  if (scheme == 1 && P->wide_host.empty()) return fail(SGM_E_UNSUPPORTED, "scheme 1 tables missing");
  if (scheme == 1 && !P->diag_ok) return fail(SGM_E_UNSUPPORTED, "scheme 1 needs the reduced separable schedule");
  if (scheme == P->scheme) return SGM_OK;  // nothing to rebuild (the graphs stay valid)
  drop_graphs(*P);                          // captured launches embed the scheme's weights and tables
  if (scheme == 1) {
    DeviceGuard g(P->device >= 0 ? P->device : 0);
    sgm_status st = upload_mass1(*P);
    if (st != SGM_OK) return st;
  }
  P->scheme = scheme;
  update_scratch_need(*P);
  return SGM_OK;
}

sgm_status sgm_geometry_greville(int n_el, int degree, double* g_host) {
  if (!g_host || n_el < 1) return fail(SGM_E_INVALID_ARG, "NULL output or n_el < 1");
  if (degree < SGM_PMIN || degree > SGM_PMAX) return fail(SGM_E_UNSUPPORTED, "degree outside the compiled range");
  const std::vector<double> g = greville(degree, n_el);
  std::copy(g.begin(), g.end(), g_host);
  return SGM_OK;
}

sgm_status sgm_geometry_interpolate(const int n_el[3], int degree, const double* values_host, double* ctrl_host) {
  if (!n_el || !values_host || !ctrl_host) return fail(SGM_E_INVALID_ARG, "NULL argument");
  if (n_el[0] < 1 || n_el[1] < 1 || n_el[2] < 1) return fail(SGM_E_INVALID_ARG, "n_el < 1");
  if (degree < SGM_PMIN || degree > SGM_PMAX) return fail(SGM_E_UNSUPPORTED, "degree outside the compiled range");
  std::string err;
  const sgm_status st = interpolate_geometry(n_el, degree, values_host, ctrl_host, err);
  return st == SGM_OK ? st : fail(st, err);
}

sgm_status sgm_plan_reduced_schedule(sgm_plan plan, int* on) {
  if (!plan || !on) return fail(SGM_E_INVALID_ARG, "NULL argument");
  const Plan& P = *PL(plan);
  *on = reduced_sched(P) ? (fused_sched(P) ? 3 : (fork_on(P) && eps_merged(P) ? 2 : 1)) : 0;
  return SGM_OK;
}

sgm_status sgm_plan_set_options(sgm_plan plan, unsigned opts) {
  if (!plan) return fail(SGM_E_INVALID_ARG, "plan is NULL");
  const unsigned all = SGM_OPT_FULL_SCHEDULE | SGM_OPT_EXACT_SPIKE | SGM_OPT_SERIAL | SGM_OPT_NO_GRAPH | SGM_OPT_FUSED |
                       SGM_OPT_WIDE_TILES | SGM_OPT_OTF_GEOMETRY;
  if (opts & ~all) return fail(SGM_E_INVALID_ARG, "unknown option bits");
  Plan* P = PL(plan);
  if (P->device >= 0) {
    DeviceGuard g(P->device);
    cudaDeviceSynchronize();
  }
  drop_graphs(*P);
  const bool spike_changed = ((P->opts ^ opts) & SGM_OPT_EXACT_SPIKE) != 0;
  const bool otf_changed = ((P->opts ^ opts) & SGM_OPT_OTF_GEOMETRY) != 0;
  P->opts = opts;
  if (otf_changed && P->device >= 0) {
    // rebuild the general 2-form weights in the other representation from the stored material
    DeviceGuard g(P->device);
    for (int m = 0; m < 2; ++m) {
      if (P->mass[m].kind != HODGE_FULL) continue;
      const std::vector<double> v = P->mass[m].values_host;
      const sgm_status st = set_material_impl(*P, m, v.empty() ? nullptr : v.data(), P->mass[m].material_c);
      if (st != SGM_OK) return st;
    }
  }
  if (spike_changed) {
    std::string err;
    const sgm_status st = set_spike_reach(*P, err);
    if (st != SGM_OK) return fail(st, err);
  }
  return SGM_OK;
}

sgm_status sgm_plan_get_options(sgm_plan plan, unsigned* opts) {
  if (!plan || !opts) return fail(SGM_E_INVALID_ARG, "NULL argument");
  *opts = PL(plan)->opts;
  return SGM_OK;
}

sgm_status sgm_plan_set_material(sgm_plan plan, sgm_material which, const double* values, double c) {
  if (plan) drop_graphs(*PL(plan));  // captured launches embed the old weights
  sgm_status s = check_plan(plan, false);
  if (s != SGM_OK) return s;
  if (which != SGM_EPS && which != SGM_MU) return fail(SGM_E_INVALID_ARG, "bad material");
  Plan* P = PL(plan);
  if (P->device >= 0) {
    DeviceGuard g(P->device);
    cudaDeviceSynchronize();
    s = set_material_impl(*P, which, values, c);
  } else {
    s = set_material_impl(*P, which, values, c);
  }
  if (s == SGM_OK && P->scheme == 1) {
    DeviceGuard g(P->device >= 0 ? P->device : 0);
    s = upload_mass1(*P);
  }
  if (P->device >= 0) {
    DeviceGuard g(P->device);
    update_scratch_need(*P);
  }
  drop_graphs(*P);
  return s;
}

sgm_status sgm_workspace_bytes(sgm_plan plan, size_t* bytes) {
  if (!plan || !bytes) return fail(SGM_E_INVALID_ARG, "NULL argument");
  *bytes = ws_need(*PL(plan));
  return SGM_OK;
}

sgm_status sgm_plan_kernels_per_step(sgm_plan plan, int* n) {
  if (!plan || !n) return fail(SGM_E_INVALID_ARG, "NULL argument");
  const Plan& P = *PL(plan);
  auto groups = [&](std::initializer_list<std::pair<int, int>> axop) {
    PassComp pc[3];
    int m = 0;
    for (const auto& q : axop) {
      pc[m] = {q.first, m, nullptr, nullptr, q.second, {-1, -1, -1}, 1.0};
      ++m;
    }
    int grp[3][3], gn[3];
    return group_passes(P, pc, m, grp, gn);
  };
  int k = 0;
  for (int m = 0; m < 2; ++m) {
    const int own = m == 0 ? OP_EPS_OWN : OP_MU_OWN, oth = m == 0 ? OP_EPS_OTH : OP_MU_OTH;
    auto axis_groups = [&](int ax) {
      return groups({{ax, own_or(ax, 0, own, oth)}, {ax, own_or(ax, 1, own, oth)}, {ax, own_or(ax, 2, own, oth)}});
    };
    const bool sep = P.mass[m].kind == HODGE_SEPARABLE;
    if (sep && fused_sched(P) && fused_fits(P, m, false)) {
      if (!reduced_sched(P)) k += axis_groups(2) + 2;
      else if (m == 0) k += groups({{2, oth}, {2, oth}, {1, oth}}) + 2;
      else k += groups({{2, own}, {1, own}, {0, own}});
      continue;
    }
    k += 1;  // the update kernel
    if (P.scheme == 1 && P.mass1[m].kind != HODGE_SEPARABLE) k += 4;  // (PCG: counted as one star)
    else if (sep && reduced_sched(P)) k += (m == SGM_MASS_MU && mu_merged(P)) ? 2 : 3;
    else if (sep) k += 3;
    else k += 4;
  }
  *n = k;
  return SGM_OK;
}

// steps per graph of long sgm_step calls, and the largest plan (N_e + N_h) that uses them
constexpr int kGraphChunk = 8;
constexpr double kGraphChunkDofs = 20e6;

sgm_status sgm_step(sgm_plan plan, double* d, double* e, double* b, double* h, const double* j_hat,
                    const double* j_amp, double dt, int n_steps, void* workspace, size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!d || !e || !b || !h || !aligned8(d) || !aligned8(e) || !aligned8(b) || !aligned8(h))
    return fail(SGM_E_INVALID_ARG, "state pointers must be non-NULL and 8-byte aligned");
  if ((j_hat && !aligned8(j_hat)) || (j_amp && !aligned8(j_amp))) return fail(SGM_E_INVALID_ARG, "misaligned source");
  if (!std::isfinite(dt)) return fail(SGM_E_INVALID_ARG, "dt must be finite");
  if (n_steps < 0) return fail(SGM_E_INVALID_ARG, "n_steps < 0");
  if (d == e || d == b || d == h || e == b || e == h || b == h) return fail(SGM_E_INVALID_ARG, "state vectors alias");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n_steps == 0) return SGM_OK;
  // CUDA graph: the launch sequence of ONE step is captured once per argument set and replayed
  // n_steps times (removes the per-kernel host enqueue cost, which dominates on small meshes).
  // Used when every step has identical arguments (no per-step source amplitudes), not on the
  // legacy default stream (capture is not allowed there) and not while profiling records events.
  // With per-step amplitudes the captured step reads s from j_amp[0]: replayable for n_steps == 1
  // (a caller that refreshes the same device scalar every step, as a simulation loop does).
  const bool use_graph = !P->profiling && stream != nullptr && P->graph_enabled && !(P->opts & SGM_OPT_NO_GRAPH) &&
                         (j_amp == nullptr || n_steps == 1) && !stream_capturing(st);
  if (use_graph) {
    // (re)capture `steps` consecutive steps with these arguments into *exec (key: arguments + steps)
    auto capture = [&](void*& exec_slot, GraphKey& key_slot, int steps) -> sgm_status {
      const GraphKey key{d, e, b, h, j_hat, j_amp, dt, steps, workspace};
      if (exec_slot && key_slot == key) return SGM_OK;
      if (exec_slot) {
        cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec_slot));
        exec_slot = nullptr;
      }
      cudaGraph_t graph = nullptr;
      if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
        return cuda_check(P, "sgm_step: begin capture");
      P->launch_fail = 0;
      for (int k = 0; k < steps; ++k) step_once(*P, d, e, b, h, j_hat, j_amp, dt, w, st);
      if (cudaStreamEndCapture(st, &graph) != cudaSuccess) return cuda_check(P, "sgm_step: end capture");
      if (P->launch_fail) {  // incomplete step: do not keep (or run) it
        cudaGraphDestroy(graph);
        return cuda_check(P, "sgm_step");
      }
      cudaGraphExec_t exec = nullptr;
      const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) return cuda_check(P, "sgm_step: graph instantiate");
      // upload now: otherwise the first launch of the graph pays it (the chunk graph may first
      // run in a later call)
      if (cudaGraphUpload(exec, st) != cudaSuccess) return cuda_check(P, "sgm_step: graph upload");
      exec_slot = exec;
      key_slot = key;
      return SGM_OK;
    };
    // Calls without per-step amplitudes also get a graph of kGraphChunk steps, captured together
    // with the one-step graph at the first call with these arguments (so a later long call pays
    // no capture): inside one graph the kernels of consecutive steps chain by programmatic
    // dependent launch as well, where a graph boundary waits for the previous graph to finish
    // (C2 32^3: 21.1 -> 18.2 us per step; 64^3 .. 144^3: 1.4 - 5 % per step).  Long calls replay the
    // chunk graph, the remainder the one-step graph.  Measured slower from 160^3 on (p = 2, 3:
    // +10 - 18 %), so plans above kGraphChunkDofs DOFs keep one-step graphs.
    const bool small = double(P->N_e) + double(P->N_h) <= kGraphChunkDofs;
    const int chunk = (j_amp == nullptr && small) ? tune_int("SGM_GRAPH_CHUNK", kGraphChunk) : 1;
    if ((s = capture(P->graph_exec, P->graph_key, 1)) != SGM_OK) return s;
    if (chunk > 1 && (s = capture(P->graph_exec_m, P->graph_key_m, chunk)) != SGM_OK) return s;
    int left = n_steps;
    if (chunk > 1)
      for (; left >= chunk; left -= chunk) cudaGraphLaunch(static_cast<cudaGraphExec_t>(P->graph_exec_m), st);
    for (int k = 0; k < left; ++k) cudaGraphLaunch(static_cast<cudaGraphExec_t>(P->graph_exec), st);
    return cuda_check(P, "sgm_step (graph)");
  }
  for (int k = 0; k < n_steps; ++k) step_once(*P, d, e, b, h, j_hat, j_amp ? j_amp + k : nullptr, dt, w, st);
  return cuda_check(P, "sgm_step");
}

sgm_status sgm_step_lifted(sgm_plan plan, double* d, double* e, double* b, double* h, const double* j_hat,
                           const double* j_amp, const sgm_lifting* lift, double dt, int n_steps, void* workspace,
                           size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!lift || !lift->g || !lift->beta) return fail(SGM_E_INVALID_ARG, "lifting descriptor with g and beta required");
  const double* v[6] = {lift->w_e, lift->c_b, lift->q0, lift->q1, lift->g, lift->beta};
  for (const double* x : v)
    if (x && !aligned8(x)) return fail(SGM_E_INVALID_ARG, "misaligned lifting vector");
  if (!d || !e || !b || !h || !aligned8(d) || !aligned8(e) || !aligned8(b) || !aligned8(h))
    return fail(SGM_E_INVALID_ARG, "state pointers must be non-NULL and 8-byte aligned");
  if ((j_hat && !aligned8(j_hat)) || (j_amp && !aligned8(j_amp))) return fail(SGM_E_INVALID_ARG, "misaligned source");
  if (!std::isfinite(dt)) return fail(SGM_E_INVALID_ARG, "dt must be finite");
  if (n_steps < 0) return fail(SGM_E_INVALID_ARG, "n_steps < 0");
  if (d == e || d == b || d == h || e == b || e == h || b == h) return fail(SGM_E_INVALID_ARG, "state vectors alias");
  if (P->scheme != 2) return fail(SGM_E_UNSUPPORTED, "the lifted step is built for the second scheme");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int k = 0; k < n_steps; ++k) {
    const double* sp = j_amp ? j_amp + k : nullptr;
    half_step(*P, 0, d, e, b, h, j_hat, sp, dt, w, st, lift, k);
    half_step(*P, 1, d, e, b, h, j_hat, sp, dt, w, st, lift, k);
  }
  return cuda_check(P, "sgm_step_lifted");
}

sgm_status sgm_step_eh(sgm_plan plan, double* e, double* h, const double* j_hat, const double* j_amp, double dt,
                       int n_steps, void* workspace, size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!e || !h || !aligned8(e) || !aligned8(h)) return fail(SGM_E_INVALID_ARG, "state pointers must be non-NULL and 8-byte aligned");
  if ((j_hat && !aligned8(j_hat)) || (j_amp && !aligned8(j_amp))) return fail(SGM_E_INVALID_ARG, "misaligned source");
  if (!std::isfinite(dt)) return fail(SGM_E_INVALID_ARG, "dt must be finite");
  if (n_steps < 0) return fail(SGM_E_INVALID_ARG, "n_steps < 0");
  if (e == h) return fail(SGM_E_INVALID_ARG, "state vectors alias");
  if (P->scheme != 2) return fail(SGM_E_UNSUPPORTED, "the (e,h)-state step is built for the second scheme");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n_steps == 0) return SGM_OK;
  // one step captured into a CUDA graph and replayed, as sgm_step
  const bool use_graph = !P->profiling && stream != nullptr && P->graph_enabled && !(P->opts & SGM_OPT_NO_GRAPH) &&
                         (j_amp == nullptr || n_steps == 1) && !stream_capturing(st);
  if (use_graph) {
    const GraphKey key{nullptr, e, nullptr, h, j_hat, j_amp, dt, 1, workspace};
    if (!(P->graph_exec_e && P->graph_key_e == key)) {
      if (P->graph_exec_e) {
        cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(P->graph_exec_e));
        P->graph_exec_e = nullptr;
      }
      cudaGraph_t graph = nullptr;
      if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
        return cuda_check(P, "sgm_step_eh: begin capture");
      P->launch_fail = 0;
      half_step_eh(*P, 0, e, h, j_hat, j_amp, dt, w, st);
      half_step_eh(*P, 1, e, h, j_hat, j_amp, dt, w, st);
      if (cudaStreamEndCapture(st, &graph) != cudaSuccess) return cuda_check(P, "sgm_step_eh: end capture");
      if (P->launch_fail) {
        cudaGraphDestroy(graph);
        return cuda_check(P, "sgm_step_eh");
      }
      cudaGraphExec_t exec = nullptr;
      const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) return cuda_check(P, "sgm_step_eh: graph instantiate");
      P->graph_exec_e = exec;
      P->graph_key_e = key;
    }
    for (int k = 0; k < n_steps; ++k) cudaGraphLaunch(static_cast<cudaGraphExec_t>(P->graph_exec_e), st);
    return cuda_check(P, "sgm_step_eh (graph)");
  }
  for (int k = 0; k < n_steps; ++k) {
    const double* sp = j_amp ? j_amp + k : nullptr;
    half_step_eh(*P, 0, e, h, j_hat, sp, dt, w, st);
    half_step_eh(*P, 1, e, h, j_hat, sp, dt, w, st);
  }
  return cuda_check(P, "sgm_step_eh");
}

sgm_status sgm_step_composed(sgm_plan plan, double* d, double* e, double* b, double* h, const double* j_hat,
                             const double* j_amp, const double* weights, int n_w, double dt, int n_steps,
                             void* workspace, size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!d || !e || !b || !h || !aligned8(d) || !aligned8(e) || !aligned8(b) || !aligned8(h))
    return fail(SGM_E_INVALID_ARG, "state pointers must be non-NULL and 8-byte aligned");
  if ((j_hat && !aligned8(j_hat)) || (j_amp && !aligned8(j_amp))) return fail(SGM_E_INVALID_ARG, "misaligned source");
  if (d == e || d == b || d == h || e == b || e == h || b == h) return fail(SGM_E_INVALID_ARG, "state vectors alias");
  if (!weights || n_w < 1 || n_w > SGM_MAX_STAGES) return fail(SGM_E_INVALID_ARG, "need 1 <= n_w <= SGM_MAX_STAGES weights");
  for (int i = 0; i < n_w; ++i)
    if (!std::isfinite(weights[i])) return fail(SGM_E_INVALID_ARG, "weights must be finite");
  if (!std::isfinite(dt)) return fail(SGM_E_INVALID_ARG, "dt must be finite");
  if (n_steps < 0) return fail(SGM_E_INVALID_ARG, "n_steps < 0");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n_steps == 0) return SGM_OK;
  // kick-drift-kick sub-steps S(w_i dt) in sequence; adjacent half kicks of b are merged
  // (b -= a D1 e; b -= c D1 e with the same e is b -= (a + c) D1 e)
  auto enqueue = [&]() {
    const double* W = weights;
    half_step(*P, 1, d, e, b, h, nullptr, nullptr, 0.5 * W[0] * dt, w, st);
    for (int k = 0; k < n_steps; ++k)
      for (int i = 0; i < n_w; ++i) {
        const double* s_ptr = j_amp ? j_amp + size_t(k) * n_w + i : nullptr;
        half_step(*P, 0, d, e, b, h, j_hat, s_ptr, W[i] * dt, w, st);
        double kick;
        if (i + 1 < n_w) kick = 0.5 * (W[i] + W[i + 1]);
        else if (k + 1 < n_steps) kick = 0.5 * (W[i] + W[0]);
        else kick = 0.5 * W[i];
        half_step(*P, 1, d, e, b, h, nullptr, nullptr, kick * dt, w, st);
      }
  };
  // the whole call's launch sequence is captured once per argument set and replayed (non-default
  // stream, not profiling, at most 4 composed steps per call so the graph stays small)
  if (!P->profiling && stream != nullptr && P->graph_enabled && !(P->opts & SGM_OPT_NO_GRAPH) && n_steps <= 4 &&
      !stream_capturing(st)) {
    const GraphKey key{d, e, b, h, j_hat, j_amp, dt, n_steps, workspace};
    const std::vector<double> wv(weights, weights + n_w);
    if (!(P->graph_exec_c && P->graph_key_c == key && P->graph_w_c == wv)) {
      if (P->graph_exec_c) {
        cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(P->graph_exec_c));
        P->graph_exec_c = nullptr;
      }
      cudaGraph_t graph = nullptr;
      if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
        return cuda_check(P, "sgm_step_composed: begin capture");
      P->launch_fail = 0;
      enqueue();
      if (cudaStreamEndCapture(st, &graph) != cudaSuccess) return cuda_check(P, "sgm_step_composed: end capture");
      if (P->launch_fail) {  // incomplete: do not keep (or run) it
        cudaGraphDestroy(graph);
        return cuda_check(P, "sgm_step_composed");
      }
      cudaGraphExec_t exec = nullptr;
      const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) return cuda_check(P, "sgm_step_composed: graph instantiate");
      P->graph_exec_c = exec;
      P->graph_key_c = key;
      P->graph_w_c = wv;
    }
    cudaGraphLaunch(static_cast<cudaGraphExec_t>(P->graph_exec_c), st);
    return cuda_check(P, "sgm_step_composed (graph)");
  }
  enqueue();
  return cuda_check(P, "sgm_step_composed");
}

sgm_status sgm_step_host(sgm_plan plan, double* d, double* e, double* b, double* h, const double* j_hat,
                         const double* j_amp, double dt, int n_steps, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!d || !e || !b || !h) return fail(SGM_E_INVALID_ARG, "NULL state");
  if (n_steps < 0) return fail(SGM_E_INVALID_ARG, "n_steps < 0");
  DeviceGuard g(P->device);
  size_t ne = P->N_e, nh = P->N_h;
  size_t wsb = ws_need(*P);
  size_t need = (2 * ne + 2 * nh + ne + size_t(std::max(n_steps, 1))) * sizeof(double) + wsb + 64;
  if (P->mirror_bytes < need) {
    cudaFree(P->mirror);
    P->mirror = nullptr;
    P->mirror_bytes = 0;
    if (cudaMalloc(&P->mirror, need) != cudaSuccess) return fail(SGM_E_NOMEM, "cudaMalloc failed for mirrors");
    P->mirror_bytes = need;
  }
  double* md = P->mirror;
  double* me = md + ne;
  double* mb = me + ne;
  double* mh = mb + nh;
  double* mj = mh + nh;
  double* ma = mj + ne;
  void* ws = ma + std::max(n_steps, 1);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaMemcpyAsync(md, d, ne * sizeof(double), cudaMemcpyHostToDevice, st);
  // e is not read by a step (the first half step recomputes it from d: K1 e = M~2 d, or the
  // scheme-1 star from a zero start), so it is uploaded only when no step runs
  if (n_steps == 0) cudaMemcpyAsync(me, e, ne * sizeof(double), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(mb, b, nh * sizeof(double), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(mh, h, nh * sizeof(double), cudaMemcpyHostToDevice, st);
  if (j_hat) cudaMemcpyAsync(mj, j_hat, ne * sizeof(double), cudaMemcpyHostToDevice, st);
  if (j_amp) cudaMemcpyAsync(ma, j_amp, size_t(n_steps) * sizeof(double), cudaMemcpyHostToDevice, st);
  s = sgm_step(plan, md, me, mb, mh, j_hat ? mj : nullptr, j_amp ? ma : nullptr, dt, n_steps, ws, wsb, stream);
  if (s != SGM_OK) return s;
  cudaMemcpyAsync(d, md, ne * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(e, me, ne * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(b, mb, nh * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(h, mh, nh * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check(P, "sgm_step_host");
  return cuda_check(P, "sgm_step_host");
}

sgm_status sgm_kron_solve(sgm_plan plan, sgm_pairing which, int transpose, const double* rhs, double* x,
                          void* workspace, size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!rhs || !x || !aligned8(rhs) || !aligned8(x)) return fail(SGM_E_INVALID_ARG, "bad vector pointers");
  if (which != SGM_K1 && which != SGM_KT1) return fail(SGM_E_INVALID_ARG, "bad pairing");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  // LU tables: K1 own Hat M, other Hat G; K1^T own M^T, other G^T;
  //            K~1 own G^T, other M^T;   K~1^T own G, other M   (eqs. tensor_K, tensor_Ktilde)
  int kind = (which == SGM_K1) ? 0 : 1;
  int own, oth;
  if (which == SGM_K1) { own = transpose ? OP_MU_OTH : OP_EPS_OWN; oth = transpose ? OP_MU_OWN : OP_EPS_OTH; }
  else { own = transpose ? OP_EPS_OTH : OP_MU_OWN; oth = transpose ? OP_EPS_OWN : OP_MU_OTH; }
  kron_pass3(*P, kind, rhs, x, w.t, own, oth, nullptr, false, true, static_cast<cudaStream_t>(stream));
  return cuda_check(P, "sgm_kron_solve");
}

sgm_status sgm_pairing_apply(sgm_plan plan, sgm_pairing which, int transpose, const double* x, double* y,
                             void* workspace, size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!x || !y || x == y || !aligned8(x) || !aligned8(y)) return fail(SGM_E_INVALID_ARG, "bad vector pointers");
  if (which != SGM_K1 && which != SGM_KT1) return fail(SGM_E_INVALID_ARG, "bad pairing");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  int kind = (which == SGM_K1) ? 0 : 1;
  int own, oth;
  if (which == SGM_K1) { own = transpose ? OP_APPLY_MT : OP_APPLY_M; oth = transpose ? OP_APPLY_GT : OP_APPLY_G; }
  else { own = transpose ? OP_APPLY_G : OP_APPLY_GT; oth = transpose ? OP_APPLY_M : OP_APPLY_MT; }
  kron_pass3(*P, kind, x, y, w.t, own, oth, nullptr, true, false, static_cast<cudaStream_t>(stream));
  return cuda_check(P, "sgm_pairing_apply");
}

sgm_status sgm_hodge_apply(sgm_plan plan, sgm_mass which, const double* x, double* y, void* workspace,
                           size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!x || !y || x == y || !aligned8(x) || !aligned8(y)) return fail(SGM_E_INVALID_ARG, "bad vector pointers");
  if (which != SGM_MASS_EPS && which != SGM_MASS_MU) return fail(SGM_E_INVALID_ARG, "bad mass");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  mass_apply(*P, which, x, y, w.t, static_cast<cudaStream_t>(stream), &w);
  return cuda_check(P, "sgm_hodge_apply");
}

// y = K^{-1} M x for one Hodge star (eqs. discrete2_hodge_eps / _mu)
void hodge_star_impl(const Plan& P, int which, const double* x, double* y, const WS& w, cudaStream_t st) {
  int kind = (which == SGM_MASS_EPS) ? 0 : 1;
  int own = (which == SGM_MASS_EPS) ? OP_EPS_OWN : OP_MU_OWN;
  int oth = (which == SGM_MASS_EPS) ? OP_EPS_OTH : OP_MU_OTH;
  const MassData& M = P.mass[which];
  if (P.scheme == 1 && P.mass1[which].kind != HODGE_SEPARABLE) {
    pcg_star(const_cast<Plan&>(P), which, x, y, w, st);
  } else if (M.kind == HODGE_SEPARABLE && reduced_sched(P)) {
    hodge_star_reduced(const_cast<Plan&>(P), which, x, y, w.t, st);
  } else if (M.kind == HODGE_SEPARABLE) {
    kron_pass3(P, kind, x, y, w.t, own, oth, M.scale, true, true, st);
  } else {
    mass_apply(P, which, x, w.r, w.t, st, &w);
    kron_pass3(P, kind, w.r, y, w.t, own, oth, nullptr, false, true, st);
  }
}

void curl_impl(const Plan& P, int kind, const double* x, double* y, cudaStream_t st) {
  int skind = (kind == SGM_CURL_PRIMAL) ? 0 : 1;  // primal: e -> b ; dual: h -> d
  int dkind = 1 - skind;
  double *S[3], *Dd[3];
  comps_of(P, skind, x, S);
  comps_of(P, dkind, y, Dd);
  int se[3][3], de[3][3];
  for (int c = 0; c < 3; ++c) {
    comp_shape(P, skind, c, se[c]);
    comp_shape(P, dkind, c, de[c]);
  }
  const double* Sc[3] = {S[0], S[1], S[2]};
  launch_curl(kind == SGM_CURL_DUAL ? 1 : 0, Sc, se, Dd, de, st);
}

sgm_status sgm_hodge_star(sgm_plan plan, sgm_mass which, const double* x, double* y, void* workspace,
                          size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!x || !y || x == y || !aligned8(x) || !aligned8(y)) return fail(SGM_E_INVALID_ARG, "bad vector pointers");
  if (which != SGM_MASS_EPS && which != SGM_MASS_MU) return fail(SGM_E_INVALID_ARG, "bad mass");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  hodge_star_impl(*P, which, x, y, w, static_cast<cudaStream_t>(stream));
  return cuda_check(P, "sgm_hodge_star");
}

sgm_status sgm_curl(sgm_plan plan, sgm_curl_kind kind, const double* x, double* y, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!x || !y || x == y || !aligned8(x) || !aligned8(y)) return fail(SGM_E_INVALID_ARG, "bad vector pointers");
  if (kind != SGM_CURL_PRIMAL && kind != SGM_CURL_DUAL) return fail(SGM_E_INVALID_ARG, "bad curl kind");
  DeviceGuard g(P->device);
  curl_impl(*P, kind, x, y, static_cast<cudaStream_t>(stream));
  return cuda_check(P, "sgm_curl");
}

sgm_status sgm_energy(sgm_plan plan, const double* d, const double* e, const double* b, const double* h,
                      double* out_dev, void* workspace, size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!d || !e || !b || !h || !out_dev) return fail(SGM_E_INVALID_ARG, "NULL argument");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // K1 e and K~1 h by banded Kronecker mat-vecs, then d.(K1 e) + b.(K~1 h)
  kron_pass3(*P, 0, e, w.r, w.t, OP_APPLY_M, OP_APPLY_G, nullptr, true, false, st);
  launch_dot_partials(d, w.r, P->N_e, w.partials, 0, st);
  kron_pass3(*P, 1, h, w.r, w.t, OP_APPLY_GT, OP_APPLY_MT, nullptr, true, false, st);
  launch_dot_partials(b, w.r, P->N_h, w.partials, 1, st);
  launch_finalize_sum(w.partials, 2, 0.5, out_dev, st);
  return cuda_check(P, "sgm_energy");
}

sgm_status sgm_gauss(sgm_plan plan, const double* d, const double* b, double* out_dev, void* workspace,
                     size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!d || !b || !out_dev) return fail(SGM_E_INVALID_ARG, "NULL argument");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *Dd[3], *Bb[3];
  comps_of(*P, 0, d, Dd);
  comps_of(*P, 1, b, Bb);
  int de[3][3], be[3][3];
  for (int c = 0; c < 3; ++c) {
    comp_shape(*P, 0, c, de[c]);
    comp_shape(*P, 1, c, be[c]);
  }
  const double* Dc[3] = {Dd[0], Dd[1], Dd[2]};
  const double* Bc[3] = {Bb[0], Bb[1], Bb[2]};
  launch_div_max(1, Dc, de, w.partials, 0, st);
  launch_div_max(0, Bc, be, w.partials, 1, st);
  launch_finalize_max(w.partials, 1, 2, out_dev, st);
  return cuda_check(P, "sgm_gauss");
}

sgm_status sgm_check_source(sgm_plan plan, const double* j_hat, void* workspace, size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  if (!j_hat) return fail(SGM_E_INVALID_ARG, "NULL source");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* J[3];
  comps_of(*P, 0, j_hat, J);
  int je[3][3];
  for (int c = 0; c < 3; ++c) comp_shape(*P, 0, c, je[c]);
  const double* Jc[3] = {J[0], J[1], J[2]};
  launch_div_max(1, Jc, je, w.partials, 0, st);
  launch_absmax(j_hat, P->N_e, w.partials, 1, st);
  double* out = w.partials + 2 * partial_blocks();
  launch_finalize_max(w.partials, 1, 2, out, st);
  double hv[2] = {0, 0};
  cudaMemcpyAsync(hv, out, 2 * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check(P, "sgm_check_source");
  if (hv[0] > 1e-12 * hv[1])
    return fail(SGM_E_SOURCE_DIVERGENCE, "||D~2 j||_inf = " + std::to_string(hv[0]) + " exceeds 1e-12 ||j||_inf");
  return cuda_check(P, "sgm_check_source");
}

sgm_status sgm_cfl(sgm_plan plan, double* x, double* e, double* b, double* h, int n_iter, double* out_dev,
                   void* workspace, size_t ws_bytes, void* stream) {
  sgm_status s = check_plan(plan, true);
  if (s != SGM_OK) return s;
  Plan* P = PL(plan);
  const double* v[5] = {x, e, b, h, out_dev};
  for (int i = 0; i < 5; ++i) {
    if (!v[i] || !aligned8(v[i])) return fail(SGM_E_INVALID_ARG, "NULL or misaligned pointer");
    for (int j = 0; j < i; ++j)
      if (v[i] == v[j]) return fail(SGM_E_INVALID_ARG, "x, e, b, h, out_dev must be distinct");
  }
  if (n_iter < 1) return fail(SGM_E_INVALID_ARG, "n_iter must be >= 1");
  WS w;
  if ((s = ws_carve(*P, workspace, ws_bytes, w)) != SGM_OK) return s;
  DeviceGuard g(P->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // x <- x0 / |x0|, then per iteration (oracle workloads.cfl_power):
  //   e = K1^{-1} M~2 x, b = D1 e, h = K~1^{-1} M2 b, lam = (b.K~1 h)/(x.K1 e), x = D~1 h / |D~1 h|
  // partial slots: 0 = b.K~1 h, 1 = x.K1 e, 2 = |x|^2.
  launch_dot_partials(x, x, P->N_e, w.partials, 2, st);
  launch_normalize(x, P->N_e, w.partials, 2, st);
  for (int k = 0; k < n_iter; ++k) {
    hodge_star_impl(*P, SGM_MASS_EPS, x, e, w, st);
    curl_impl(*P, SGM_CURL_PRIMAL, e, b, st);
    hodge_star_impl(*P, SGM_MASS_MU, b, h, w, st);
    kron_pass3(*P, 0, e, w.r, w.t, OP_APPLY_M, OP_APPLY_G, nullptr, true, false, st);
    launch_dot_partials(x, w.r, P->N_e, w.partials, 1, st);
    kron_pass3(*P, 1, h, w.r, w.t, OP_APPLY_GT, OP_APPLY_MT, nullptr, true, false, st);
    launch_dot_partials(b, w.r, P->N_h, w.partials, 0, st);
    curl_impl(*P, SGM_CURL_DUAL, h, x, st);
    launch_dot_partials(x, x, P->N_e, w.partials, 2, st);
    launch_normalize(x, P->N_e, w.partials, 2, st);
  }
  launch_rayleigh(w.partials, out_dev, st);
  return cuda_check(P, "sgm_cfl");
}

sgm_status sgm_plan_set_profiling(sgm_plan plan, int on) {
  if (!plan) return fail(SGM_E_INVALID_ARG, "plan is NULL");
  PL(plan)->profiling = (on != 0);
  return SGM_OK;
}

sgm_status sgm_plan_profile(sgm_plan plan, double* ms, int* counts) {
  if (!plan || !ms || !counts) return fail(SGM_E_INVALID_ARG, "NULL argument");
  Plan* P = PL(plan);
  for (int k = 0; k < SGM_K_CLASSES; ++k) {
    ms[k] = 0.0;
    counts[k] = 0;
  }
  if (P->device < 0) return SGM_OK;
  DeviceGuard g(P->device);
  for (auto& r : P->prof) {
    cudaEvent_t a = static_cast<cudaEvent_t>(r.a), b = static_cast<cudaEvent_t>(r.b);
    cudaEventSynchronize(b);
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    if (r.cls >= 0 && r.cls < SGM_K_CLASSES) {
      ms[r.cls] += t;
      counts[r.cls] += 1;
    }
    P->ev_pool.push_back(r.a);
    P->ev_pool.push_back(r.b);
  }
  P->prof.clear();
  return cuda_check(P, "sgm_plan_profile");
}

}  // extern "C"
