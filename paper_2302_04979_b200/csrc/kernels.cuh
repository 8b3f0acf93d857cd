// Kernel parameter blocks and launcher declarations (sm_100a only).
#pragma once
#include <vector>
#include <cuda_runtime.h>

#include <cstdint>

namespace sgm {

constexpr int kMaxLine = 392;  // <= 14 segments of <= 28 rows: the longest line one sweep CTA holds
                               // (longer lines are swept in overlapping windows, launch_sweep)
constexpr long kMaxCompElems = (1L << 31) - (1L << 20);  // 32-bit element indices within a component

// One component handled by a line sweep along `axis` (or by the update kernel: `in` = state).
struct SweepComp {
  double* in;         // input component array [z][y][x] (the state, for the update kernel)
  double* out;        // output component array (may equal in)
  const double* tab;  // line-operator table (seg_sweep.cuh rows), global memory
  int tslot;          // which of SweepArgs::tabs this component uses (staged in shared memory)
  int ext[3];         // component extents (x, y, z)
  double scale;       // multiplies the stored result
  // optional per-line diagonal factors: the stored line is also multiplied by dline[0][t0] and
  // dline[1][t1], (t0, t1) its transverse coordinates: (x, y) for z-lines, (x, z) for y-lines,
  // (y, z) for x-lines (the diagonal 1D factors of the reduced separable schedule, api.cu)
  const double* dline[2];
  int axis;           // strided passes: this component's sweep axis (1 or 2); 0 = SweepArgs::axis
  int cidx;           // component index 0..2 of the form (fused update: which curl component)
  int accum;          // 1: out += scale * result (the (e,h)-state increments), 0: out = scale * result
  // affine store terms (time-separable boundary data, sgm_step_lifted): out += sum_i ac[i] *
  // (as[i] ? *as[i] : 1) * aw[i][same index]; aw[i] = null: no term
  const double* aw[2];
  const double* as[2];
  double ac[2];
  // window of a long line (launch_sweep): the sweep solves rows [win0, win0 + wlen) of every line
  // and stores window rows [slo, shi); wlen = 0: the whole line
  int win0, wlen, slo, shi;
};

// Element-wise state update of a half step (launch_update):
//   AMPERE : in[c] += dt * ((D~1 src)_c - s * jhat[c])   (eq. discrete2_ampere)
//   FARADAY: in[c] -= dt * (D1 src)_c                    (eq. discrete2_faraday)
//   AMPERE_INC / FARADAY_INC: the increments alone, in[c] = dt ((D~1 src)_c - s jhat[c]) and
//   in[c] = -dt (D1 src)_c (the (e,h)-state step, sgm_step_eh; in[c] is a workspace array)
enum Prologue { PRO_NONE = 0, PRO_AMPERE = 1, PRO_FARADAY = 2, PRO_AMPERE_INC = 3, PRO_FARADAY_INC = 4 };

struct PrologueArgs {
  const double* src[3];  // h components (AMPERE) or e components (FARADAY)
  int sext[3][3];        // their extents
  const double* jhat[3]; // AMPERE source components or null
  const double* s_ptr;   // device pointer to the amplitude s_k, or null (-> 1)
  double dt;
};

struct SweepArgs {
  SweepComp comp[3];
  int ncomp;
  int axis;       // 0 = x (contiguous lines), 1 = y, 2 = z
  int band;       // apply the banded mat-vec (mass / pairing factor)
  int solve;      // apply the banded LU solve
  const double* tabs[2];  // the (at most two) distinct line-operator tables of this pass
  int tab_rows;           // rows per table (padded line length of this axis)
  int band_hw;            // half-bandwidth of the banded mat-vec of this pass (<= P)
  int spike_kh, spike_kf; // truncated-SPIKE reach of the history / future scans (segments)
  int reverse;            // process the work items last-to-first ("snake" order across kernels:
                          // a kernel starts on what its predecessor wrote last, still in L2)
  PrologueArgs pro;       // update kernel only
  int share_k, share_n;   // sweeps: use share_k/share_n of the resident-CTA slots (0/0 = all)
  int dry;                // fused sweeps: only check that a configuration fits (launch nothing)
  int wide;               // SGM_OPT_WIDE_TILES: 64-line tiles even for launches with few lines
  double* wscratch;       // windowed sweeps (lines > kMaxLine) in place: a component-sized buffer the
                          // input is copied to first (overlapping windows read rows others store)
};

// General (non-separable) Hodge apply y = M x by sum factorisation per element.
struct HodgeArgs {
  const double* x[3];
  double* y[3];
  int ext[3][3];
  const double* W;       // SCALAR: 1/qp ; FULL: 6/qp
  int full;              // 0 scalar, 1 full
  double scale[3];
  const double* basis;   // per-axis basis tables (see api.cu)
  int basis_off[3][2];   // [axis][own/other] offsets (doubles) of [n][Q][p+1] value blocks
  const int* first;      // per-axis first-index tables
  int first_off[3][2];
  int first0[3][2];      // first index of element 0 (the tables are affine: first(e) = first0 + e)
  int nel[3];
  int Q;
  double* scratch;       // brick kernel: per-item output patches (deterministic two-pass
  size_t scratch_cap;    // accumulation, hodge.cu); null or too small -> fp64 atomics (y += ...)
  // brick kernel: the element table [Q][p+1] shared by the interior elements of the uniform mesh,
  // [role own/other][axis] (read as constant-bank operands on bricks / layers of interior elements),
  // and per [axis][role] the range [uni_lo, uni_hi) of elements whose table equals it bit for bit
  double uni[2][3][25];
  int uni_lo[3][2], uni_hi[3][2];
  int dual;              // 1: dual 2-forms (M~2_{1/eps}), 0: primal 2-forms (M2_{1/mu})
  int form;              // brick kernel form type: 0 primal 2-form, 1 dual 2-form, 2 primal 1-form
                         // (M^1_eps, scheme 1), 3 dual 1-form (M~^1_mu, scheme 1)
  // on-the-fly geometry (SGM_OPT_OTF_GEOMETRY, polynomial maps, 2-form brick kernel): W holds
  // w_q / material per point; DF is evaluated from the map's control points
  int otf;
  const double* geo_ctrl[3];  // control point coordinate r, [(z * (ny+p) + y) * (nx+p) + x]
  const double* geo_tab;      // S_p values (s = 0) / derivatives (s = 1) at the Gauss points [n][Q][p+1]
  int geo_tab_off[3][2];      // [axis][s] offsets (doubles) into geo_tab
};

// pipelined (producer/consumer) sweeps; false: no compiled configuration fits, nothing launched
bool launch_sweep(int p, int seg, const SweepArgs& a, cudaStream_t st);
bool launch_sweep_p2(int seg, const SweepArgs& a, cudaStream_t st);  // sweep_p2.cu
bool launch_sweep_p3(int seg, const SweepArgs& a, cudaStream_t st);  // sweep_p3.cu
bool launch_sweep_p4(int seg, const SweepArgs& a, cudaStream_t st);  // sweep_p4.cu
bool launch_sweep_p5(int seg, const SweepArgs& a, cudaStream_t st);  // sweep_p5.cu (scheme-1 layout at p = 4)
// fused update + first sweep (fsweep_kernel.cuh); fuse: 1 Ampere update, 2 Faraday update (the
// curl source, j^, s and dt in a.pro; every component carries its own axis and cidx).  Returns
// false when no compiled configuration fits (shared memory, alignment); nothing launched then.
bool launch_fsweep(int p, int seg, int fuse, const SweepArgs& a, cudaStream_t st);
bool launch_fsweep_p2(int seg, int fuse, const SweepArgs& a, cudaStream_t st);
bool launch_fsweep_p3(int seg, int fuse, const SweepArgs& a, cudaStream_t st);
bool launch_fsweep_p4(int seg, int fuse, const SweepArgs& a, cudaStream_t st);
void launch_update(int pro, const SweepArgs& a, cudaStream_t st);
void launch_curl(int kind, const double* const src[3], const int sext[3][3], double* const dst[3],
                 const int dext[3][3], cudaStream_t st);
void launch_hodge_general(int p, const HodgeArgs& a, cudaStream_t st);
// doubles of scratch the deterministic brick Hodge needs for this plan geometry (current device)
size_t hodge_scratch_doubles(int p, int Q, int form, int full, const int nel[3]);
// the brick kernel serves the plan (default rule Q = p + 1, p = 2..4): its weights live in HBM in the
// brick layout (hodge_brick_relayout converts the element-major host vector in place)
bool hodge_uses_brick(int p, int Q);
void hodge_brick_relayout(int Q, const int nel[3], int nw, std::vector<double>& W);
void launch_dot_partials(const double* x, const double* y, size_t n, double* partials, int slot, cudaStream_t st);
void launch_finalize_sum(const double* partials, int nslots, double scale, double* out, cudaStream_t st);
void launch_div_max(int kind, const double* const src[3], const int sext[3][3], double* partials,
                    int slot, cudaStream_t st);
void launch_absmax(const double* x, size_t n, double* partials, int slot, cudaStream_t st);
void launch_finalize_max(const double* partials, int nslots_each, int ngroups, double* out, cudaStream_t st);
void launch_normalize(double* x, size_t n, const double* partials, int slot, cudaStream_t st);
void launch_rayleigh(const double* partials, double* out, cudaStream_t st);
void launch_axpy_ratio(double* x, const double* p, size_t n, const double* num, const double* den, double sign,
                       cudaStream_t st);
void launch_xpby_ratio(double* p, const double* z, size_t n, const double* num, const double* den, cudaStream_t st);
int partial_blocks();

}  // namespace sgm
