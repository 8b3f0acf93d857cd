// sm_100a kernels of the scheme-2 leapfrog step (arXiv 2302.04979) and their launchers.
//
// * Line sweeps (sweep_kernel.cuh): the Kronecker factors applied mode by mode (eq. kroninverse
//   P:L571 with the vec trick P:L575-585): per line, a banded 1D mat-vec (separable Hodge Gram or
//   pairing factor) and a partitioned no-pivot banded LU solve, in persistent warp-specialised CTAs.
// * Ampere / Faraday updates (integer +-1 curls, eqs. discrete2_ampere / _faraday):
//   a streaming element-wise kernel.
// * General Hodge (curved F or variable material, hodge_brick.cuh): element-wise sum
//   factorisation with the quadrature weights W streamed from HBM.
// * Curls, divergences (Gauss laws) and deterministic two-pass reductions (energy).
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels.cuh"
#include "seg_sweep.cuh"
#include "launch_util.cuh"
#include "pipe_sweep.cuh"

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <utility>

namespace sgm {

namespace {

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 296;  // 2 x 148 SMs

// ---- integer-incidence curls (SURVEY 8.0 stencils) ---------------------------------
// dual   (dv)_j = v_{j+1} - v_j           (free ends)
// primal (du)_j = u_j - u_{j-1}, u_{-1} = u_a = 0   (trimmed, PEC)
__device__ __forceinline__ double dterm_dual(const double* __restrict__ s, const int* e, int ax, int x, int y, int z) {
  long idx = x + long(e[0]) * (y + long(e[1]) * z);
  long st = (ax == 0) ? 1 : (ax == 1 ? long(e[0]) : long(e[0]) * e[1]);
  return __ldg(s + idx + st) - __ldg(s + idx);
}
__device__ __forceinline__ double dterm_primal(const double* __restrict__ s, const int* e, int ax, int x, int y, int z) {
  int pa = (ax == 0) ? x : (ax == 1 ? y : z);
  long idx = x + long(e[0]) * (y + long(e[1]) * z);
  long st = (ax == 0) ? 1 : (ax == 1 ? long(e[0]) : long(e[0]) * e[1]);
  double v = 0.0;
  if (pa < e[ax]) v = __ldg(s + idx);
  if (pa >= 1) v -= __ldg(s + idx - st);
  return v;
}
// component c of curl: d_{a1} src_{c1} - d_{a2} src_{c2}, (a1,c1) = (c+1, c+2), (a2,c2) = (c+2, c+1)
template <bool DUAL>
__device__ __forceinline__ double curl_comp(const double* const* src, const int (*sext)[3], int c, int x, int y, int z) {
  int a1 = (c + 1) % 3, c1 = (c + 2) % 3, a2 = (c + 2) % 3, c2 = (c + 1) % 3;
  if (DUAL) return dterm_dual(src[c1], sext[c1], a1, x, y, z) - dterm_dual(src[c2], sext[c2], a2, x, y, z);
  return dterm_primal(src[c1], sext[c1], a1, x, y, z) - dterm_primal(src[c2], sext[c2], a2, x, y, z);
}


// ---- element-wise Ampere / Faraday update (eqs. discrete2_ampere / _faraday) ----
//   AMPERE : d_c <- d_c + dt ((D~1 h)_c - s j_c)     dual   (dv)_k = v_{k+1} - v_k
//   FARADAY: b_c <- b_c - dt (D1 e)_c                primal (du)_k = u_k - u_{k-1}, u_{-1} = u_a = 0
// Streaming kernel: consecutive threads take consecutive elements of a component (coalesced),
// each thread U elements 256 apart with all loads issued before use.  A thread decomposes its
// first element into (x, y, z) once and advances the coordinates by 256 elements with carries
// (no per-element division); the differentiated axes are compile-time per component.
struct UpdTerm {
  const double* src;
  int X, Y;   // src extents x, y
  int ext_a;  // src extent along the differentiated axis
  int da;     // src index offset of one step along that axis
};
struct UpdComp {
  double* state;
  const double* jhat;
  int X, Y, N;          // component extents x, y and size
  unsigned mX, mY;      // floor((2^32-1)/X), floor((2^32-1)/Y)
  int sx, sy, sz;       // 256 elements = sz planes + sy rows + sx columns
  int chunk0;           // first chunk (256*U elements) of this component
  UpdTerm t[2];         // (D x)_c = d_{a1} x_{c1} - d_{a2} x_{c2}, a1 = c+1, a2 = c+2 (mod 3)
};
struct UpdArgs {
  UpdComp c[3];
  const double* s_ptr;
  double dt;
  int nchunks;
  int reverse;  // walk the chunks last-to-first
};

__device__ __forceinline__ unsigned fdiv(unsigned n, unsigned d, unsigned m, unsigned& r) {
  unsigned q = __umulhi(n, m);
  r = n - q * d;
  if (r >= d) { ++q; r -= d; }
  return q;
}

template <int PRO, int U, int CC, bool FULL>
__device__ __forceinline__ void update_chunk(const UpdArgs& A, const UpdComp& C, int e0) {
  constexpr bool DUAL = (PRO == PRO_AMPERE || PRO == PRO_AMPERE_INC);
  constexpr bool INC = (PRO == PRO_AMPERE_INC || PRO == PRO_FARADAY_INC);
  constexpr int AX[2] = {(CC + 1) % 3, (CC + 2) % 3};  // differentiated axis of each term
  // parameters into registers once (unpredicated)
  const double* __restrict__ src[2] = {C.t[0].src, C.t[1].src};
  const int TX[2] = {C.t[0].X, C.t[1].X}, TY[2] = {C.t[0].Y, C.t[1].Y};
  const int da[2] = {C.t[0].da, C.t[1].da}, ea[2] = {C.t[0].ext_a, C.t[1].ext_a};
  const int X = C.X, Y = C.Y, N = C.N, sx = C.sx, sy = C.sy, sz = C.sz;
  double* __restrict__ state = C.state;
  const double* __restrict__ jhat = C.jhat;
  int x, y, z;
  {
    unsigned r, q, yy;
    q = fdiv(unsigned(min(e0, N - 1)), unsigned(X), C.mX, r);
    z = int(fdiv(q, unsigned(Y), C.mY, yy));
    x = int(r);
    y = int(yy);
  }
  double vh[U][2], vl[U][2], old[U], jv[U];
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int e = e0 + 256 * k;
    const bool in = FULL || e < N;
    const int p3[3] = {x, y, z};
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const double* ps = src[t] + (x + TX[t] * (y + TY[t] * z));
      const int pa = p3[AX[t]];
      if (DUAL) {
        vh[k][t] = in ? __ldg(ps + da[t]) : 0.0;
        vl[k][t] = in ? __ldg(ps) : 0.0;
      } else {
        vh[k][t] = (in && pa < ea[t]) ? __ldg(ps) : 0.0;
        vl[k][t] = (in && pa >= 1) ? __ldg(ps - da[t]) : 0.0;
      }
    }
    old[k] = (in && !INC) ? state[e] : 0.0;
    jv[k] = (jhat && in) ? __ldg(jhat + e) : 0.0;
    // advance (x, y, z) by 256 elements
    x += sx;
    const int cx = x >= X;
    x -= cx ? X : 0;
    y += sy + cx;
    const int cy = y >= Y;
    y -= cy ? Y : 0;
    z += sz + cy;
  }
  const double dt = A.dt;
  const double sdt = jhat ? dt * (A.s_ptr ? __ldg(A.s_ptr) : 1.0) : 0.0;
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const double cu = (vh[k][0] - vl[k][0]) - (vh[k][1] - vl[k][1]);
    const double val = DUAL ? fma(-sdt, jv[k], fma(dt, cu, old[k])) : fma(-sdt, jv[k], fma(-dt, cu, old[k]));
    if (FULL || e0 + 256 * k < N) state[e0 + 256 * k] = val;
  }
}

template <int PRO, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) update_kernel(const __grid_constant__ UpdArgs A) {
  pipe::griddep_launch_dependents();
  pipe::griddep_wait();
  for (int ch0 = blockIdx.x; ch0 < A.nchunks; ch0 += gridDim.x) {
    const int ch = A.reverse ? A.nchunks - 1 - ch0 : ch0;
    const int c = (ch >= A.c[2].chunk0) ? 2 : (ch >= A.c[1].chunk0 ? 1 : 0);
    const UpdComp& C = A.c[c];
    const int base = (ch - C.chunk0) * (256 * U);
    const int e0 = base + threadIdx.x;
    const bool full = base + 256 * U <= C.N;  // interior chunk: no bounds checks
    if (full) {
      if (c == 0) update_chunk<PRO, U, 0, true>(A, C, e0);
      else if (c == 1) update_chunk<PRO, U, 1, true>(A, C, e0);
      else update_chunk<PRO, U, 2, true>(A, C, e0);
    } else {
      if (c == 0) update_chunk<PRO, U, 0, false>(A, C, e0);
      else if (c == 1) update_chunk<PRO, U, 1, false>(A, C, e0);
      else update_chunk<PRO, U, 2, false>(A, C, e0);
    }
  }
}

template <bool DUAL>
__global__ void curl_kernel(const double* s0, const double* s1, const double* s2, int3 e0, int3 e1, int3 e2,
                            double* d0, double* d1, double* d2, int3 f0, int3 f1, int3 f2) {
  const int c = blockIdx.y;
  const double* src[3] = {s0, s1, s2};
  const int sext[3][3] = {{e0.x, e0.y, e0.z}, {e1.x, e1.y, e1.z}, {e2.x, e2.y, e2.z}};
  int3 f = (c == 0) ? f0 : (c == 1 ? f1 : f2);
  double* dst = (c == 0) ? d0 : (c == 1 ? d1 : d2);
  const long N = long(f.x) * f.y * f.z;
  for (long idx = long(blockIdx.x) * blockDim.x + threadIdx.x; idx < N; idx += long(gridDim.x) * blockDim.x) {
    int x = int(idx % f.x);
    long r = idx / f.x;
    int y = int(r % f.y), z = int(r / f.y);
    dst[idx] = curl_comp<DUAL>(src, sext, c, x, y, z);
  }
}

// ---- deterministic reductions ------------------------------------------------------------
__device__ __forceinline__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  double r = sh[0];
  __syncthreads();
  return r;
}
__device__ __forceinline__ double block_max(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  double r = sh[0];
  __syncthreads();
  return r;
}

__global__ void dot_partials_kernel(const double* __restrict__ x, const double* __restrict__ y, size_t n,
                                    double* partials, int slot) {
  __shared__ double sh[kRedThreads];
  double acc = 0.0;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    acc = fma(x[i], y[i], acc);
  double s = block_sum(acc, sh);
  if (threadIdx.x == 0) partials[size_t(slot) * gridDim.x + blockIdx.x] = s;
}

__global__ void finalize_sum_kernel(const double* partials, int n, double scale, double* out) {
  __shared__ double sh[kRedThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partials[i];
  double s = block_sum(acc, sh);
  if (threadIdx.x == 0) out[0] = scale * s;
}

// x <- x / sqrt(sum of the partials in `slot`); every block re-reduces the (few) partials in the
// same order, so all blocks use the identical norm (deterministic).
__global__ void normalize_kernel(double* __restrict__ x, size_t n, const double* __restrict__ partials, int slot) {
  __shared__ double sh[kRedThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < kRedBlocks; i += blockDim.x) acc += partials[size_t(slot) * kRedBlocks + i];
  const double nrm = sqrt(block_sum(acc, sh));
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    x[i] = x[i] / nrm;
}

// PCG vector updates with device-resident scalars (no host synchronisation):
//   x += sign * (num / den) * p        and        p = z + (num / den) * p
__global__ void axpy_ratio_kernel(double* __restrict__ x, const double* __restrict__ p, size_t n,
                                  const double* num, const double* den, double sign) {
  // a zero denominator means a zero search direction (converged, or a zero right-hand side):
  // the step is zero, not NaN
  const double dn = __ldg(den);
  const double a = dn != 0.0 ? sign * (__ldg(num) / dn) : 0.0;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    x[i] = fma(a, p[i], x[i]);
}
__global__ void xpby_ratio_kernel(double* __restrict__ p, const double* __restrict__ z, size_t n,
                                  const double* num, const double* den) {
  const double dn = __ldg(den);
  const double b = dn != 0.0 ? __ldg(num) / dn : 0.0;  // r.z = 0: restart from z
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    p[i] = fma(b, p[i], z[i]);
}

// out[0] = lambda = (sum slot 0) / (sum slot 1), out[1] = 2 / sqrt(lambda)  (CFL Rayleigh quotient)
__global__ void rayleigh_kernel(const double* __restrict__ partials, double* out) {
  __shared__ double sh[kRedThreads];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < kRedBlocks; i += blockDim.x) {
    a += partials[i];
    b += partials[kRedBlocks + i];
  }
  const double num = block_sum(a, sh);
  const double den = block_sum(b, sh);
  if (threadIdx.x == 0) {
    out[0] = num / den;
    out[1] = 2.0 / sqrt(num / den);
  }
}

template <bool DUAL>
__global__ void div_max_kernel(const double* s0, const double* s1, const double* s2, int3 e0, int3 e1, int3 e2, int3 f,
                               double* partials, int slot) {
  __shared__ double sh[kRedThreads];
  const double* src[3] = {s0, s1, s2};
  const int sext[3][3] = {{e0.x, e0.y, e0.z}, {e1.x, e1.y, e1.z}, {e2.x, e2.y, e2.z}};
  const long N = long(f.x) * f.y * f.z;
  double m = 0.0;
  for (long idx = long(blockIdx.x) * blockDim.x + threadIdx.x; idx < N; idx += long(gridDim.x) * blockDim.x) {
    int x = int(idx % f.x);
    long r = idx / f.x;
    int y = int(r % f.y), z = int(r / f.y);
    double v = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c)
      v += DUAL ? dterm_dual(src[c], sext[c], c, x, y, z) : dterm_primal(src[c], sext[c], c, x, y, z);
    m = fmax(m, fabs(v));
  }
  double r = block_max(m, sh);
  if (threadIdx.x == 0) partials[size_t(slot) * gridDim.x + blockIdx.x] = r;
}

__global__ void absmax_kernel(const double* __restrict__ x, size_t n, double* partials, int slot) {
  __shared__ double sh[kRedThreads];
  double m = 0.0;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    m = fmax(m, fabs(x[i]));
  double r = block_max(m, sh);
  if (threadIdx.x == 0) partials[size_t(slot) * gridDim.x + blockIdx.x] = r;
}

__global__ void finalize_max_kernel(const double* partials, int n_each, int ngroups, double* out) {
  __shared__ double sh[kRedThreads];
  for (int g = 0; g < ngroups; ++g) {
    double m = 0.0;
    for (int i = threadIdx.x; i < n_each; i += blockDim.x) m = fmax(m, partials[size_t(g) * n_each + i]);
    double r = block_max(m, sh);
    if (threadIdx.x == 0) out[g] = r;
  }
}

}  // namespace

int partial_blocks() { return kRedBlocks; }

namespace {
bool launch_sweep_one(int p, int seg, const SweepArgs& a, cudaStream_t st) {
  switch (p) {
    case 2: return launch_sweep_p2(seg, a, st);
    case 3: return launch_sweep_p3(seg, a, st);
    case 4: return launch_sweep_p4(seg, a, st);
    case 5: return launch_sweep_p5(seg, a, st);
    default: return false;
  }
}

// Line length of component c of a sweep launch (its own axis, or the launch's)
int comp_line(const SweepArgs& a, int c) {
  const SweepComp& C = a.comp[c];
  const int ax = (a.axis != 0 && C.axis > 0) ? C.axis : a.axis;
  return C.ext[ax];
}

// Lines longer than one CTA holds (kMaxLine = 14 segments) are swept in overlapping windows of at
// most 14 segments, one launch per component and window.  A window starts on a segment boundary,
// so its rows of the line-operator table (band, LU, spikes: all defined per row and per segment)
// are the full line's; it runs the same truncated-SPIKE solve (reading Z23) with zero history
// before its first segment and zero future after its last.  Segment s of the window then has the
// full line's history once s > kh (the scan reaches back kh segments, and the first segment's
// band mat-vec lacks the rows before the window), and the full line's future once s < S_w - 1 - kf
// (the last segment lacks the rows after the window): the window stores only those segments, plus
// the true line start / end in the first / last window.  Consecutive windows overlap by kh + kf + 2
// segments.  Without a solve (band mat-vec only) one segment of margin on each side suffices.
bool launch_sweep_windows(int p, int seg, const SweepArgs& a, cudaStream_t st) {
  const int maxs = kMaxLine / seg;  // segments per window
  const int kh = a.solve ? a.spike_kh + 1 : 1, kf = a.solve ? a.spike_kf + 1 : 1;
  if (maxs - kh - kf < 1) return false;
  const int RS = RowLayoutRT(p).RS;
  for (int c = 0; c < a.ncomp; ++c) {
    SweepComp C = a.comp[c];
    if (C.in == C.out && !a.dry) {
      // in place: the windows overlap, so every window reads the input from a copy
      if (!a.wscratch) return false;
      const size_t bytes = size_t(C.ext[0]) * C.ext[1] * C.ext[2] * sizeof(double);
      if (cudaMemcpyAsync(a.wscratch, C.in, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return false;
      C.in = a.wscratch;
    }
    const int L = comp_line(a, c);
    const int S = (L + seg - 1) / seg;
    const int ax = (a.axis != 0 && C.axis > 0) ? C.axis : a.axis;
    for (int o = 0;;) {  // o: first segment of the window
      const int sw = std::min(maxs, S - o);
      SweepArgs w = a;
      w.ncomp = 1;
      w.comp[0] = C;
      w.comp[0].tslot = 0;
      w.comp[0].axis = ax;
      w.comp[0].win0 = o * seg;
      w.comp[0].wlen = std::min(L - o * seg, sw * seg);
      const bool last = o + sw >= S;
      w.comp[0].slo = o == 0 ? 0 : kh * seg;
      w.comp[0].shi = last ? w.comp[0].wlen : (sw - kf) * seg;
      w.tabs[0] = C.tab + size_t(o) * seg * RS;
      w.tabs[1] = nullptr;
      w.tab_rows = sw * seg;
      if (!launch_sweep_one(p, seg, w, st)) return false;
      if (last) break;
      o += sw - kf - kh;  // the next window stores from where this one stops
    }
  }
  return true;
}
}  // namespace

bool launch_sweep(int p, int seg, const SweepArgs& a, cudaStream_t st) {
  for (int c = 0; c < a.ncomp; ++c)
    if (comp_line(a, c) > kMaxLine) return launch_sweep_windows(p, seg, a, st);
  switch (p) {
    case 2: return launch_sweep_p2(seg, a, st);
    case 3: return launch_sweep_p3(seg, a, st);
    case 4: return launch_sweep_p4(seg, a, st);
    case 5: return launch_sweep_p5(seg, a, st);
    default: return false;
  }
}

bool launch_fsweep(int p, int seg, int fuse, const SweepArgs& a, cudaStream_t st) {
  switch (p) {
    case 2: return launch_fsweep_p2(seg, fuse, a, st);
    case 3: return launch_fsweep_p3(seg, fuse, a, st);
    case 4: return launch_fsweep_p4(seg, fuse, a, st);
    default: return false;
  }
}

void launch_update(int pro, const SweepArgs& a, cudaStream_t st) {
  UpdArgs U;
  std::memset(&U, 0, sizeof(U));
  const int minb = tune_int("SGM_UPD_MINB", 1);
  int UU = tune_int("SGM_UPD_U", 4);
  if (!((UU == 4 && minb == 1) || (UU == 8 && minb == 1) || (UU == 4 && minb == 4) || (UU == 8 && minb == 2) ||
        (UU == 2 && minb == 4)))
    UU = 4;
  const int CH = 256 * UU;
  int chunk = 0;
  for (int c = 0; c < 3; ++c) {
    UpdComp& C = U.c[c];
    C.state = a.comp[c].in;
    C.jhat = a.pro.jhat[c];  // Ampere: j^; Faraday: the lifting's interior curl c_b (sgm_step_lifted)
    C.X = a.comp[c].ext[0];
    C.Y = a.comp[c].ext[1];
    C.N = a.comp[c].ext[0] * a.comp[c].ext[1] * a.comp[c].ext[2];
    C.mX = 0xffffffffu / unsigned(C.X);
    C.mY = 0xffffffffu / unsigned(C.Y);
    C.sx = 256 % C.X;
    C.sy = (256 / C.X) % C.Y;
    C.sz = 256 / (C.X * C.Y);
    C.chunk0 = chunk;
    chunk += (C.N + CH - 1) / CH;
    const int a1 = (c + 1) % 3, c1 = (c + 2) % 3, a2 = (c + 2) % 3, c2 = (c + 1) % 3;
    const int aa[2] = {a1, a2}, cc[2] = {c1, c2};
    for (int t = 0; t < 2; ++t) {
      C.t[t].src = a.pro.src[cc[t]];
      C.t[t].X = a.pro.sext[cc[t]][0];
      C.t[t].Y = a.pro.sext[cc[t]][1];
      C.t[t].ext_a = a.pro.sext[cc[t]][aa[t]];
      C.t[t].da = aa[t] == 0 ? 1 : (aa[t] == 1 ? C.t[t].X : C.t[t].X * C.t[t].Y);
    }
  }
  U.nchunks = chunk;
  U.reverse = tune_int("SGM_SNAKE", 1) ? a.reverse : 0;
  U.s_ptr = a.pro.s_ptr;
  U.dt = a.pro.dt;
  // grid: exactly the resident CTAs (a grid-stride loop over equal chunks: no partial last wave;
  // measured 35 us vs 37 us for 8 CTAs per SM at 128^3 p=3); SGM_UPD_GRID = CTAs per SM override
  auto launch = [&](auto kern) {
    int per_sm = tune_int("SGM_UPD_GRID", 0);
    if (per_sm <= 0) {
      static thread_local std::map<const void*, int> occ;  // per kernel instance (per host thread)
      int& o = occ[reinterpret_cast<const void*>(kern)];
      if (o == 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, 256, 0);
      per_sm = o > 0 ? o : 1;
    }
    int grid = per_sm * sm_count();
    if (grid > chunk) grid = chunk;
    launch_pdl(kern, unsigned(grid), 256u, 0, st, U);
  };
  // U elements per thread (all loads issued before use); MINB: minimum resident blocks per SM
#define SGM_UPD(UV, MB)                                                         \
  if (UU == UV && minb == MB) {                                                 \
    if (pro == PRO_AMPERE) launch(update_kernel<PRO_AMPERE, UV, MB>);           \
    else if (pro == PRO_FARADAY) launch(update_kernel<PRO_FARADAY, UV, MB>);    \
    else if (pro == PRO_AMPERE_INC) launch(update_kernel<PRO_AMPERE_INC, 4, 1>); \
    else launch(update_kernel<PRO_FARADAY_INC, 4, 1>);                          \
    return;                                                                     \
  }
  SGM_UPD(4, 1) SGM_UPD(8, 1) SGM_UPD(4, 4) SGM_UPD(8, 2) SGM_UPD(2, 4)
#undef SGM_UPD
  if (pro == PRO_AMPERE) launch(update_kernel<PRO_AMPERE, 4, 1>);
  else if (pro == PRO_FARADAY) launch(update_kernel<PRO_FARADAY, 4, 1>);
  else if (pro == PRO_AMPERE_INC) launch(update_kernel<PRO_AMPERE_INC, 4, 1>);
  else launch(update_kernel<PRO_FARADAY_INC, 4, 1>);
}

void launch_curl(int kind, const double* const src[3], const int sext[3][3], double* const dst[3],
                 const int dext[3][3], cudaStream_t st) {
  int3 e[3], f[3];
  for (int c = 0; c < 3; ++c) {
    e[c] = make_int3(sext[c][0], sext[c][1], sext[c][2]);
    f[c] = make_int3(dext[c][0], dext[c][1], dext[c][2]);
  }
  dim3 grid(2 * 148, 3);
  if (kind == 1)
    curl_kernel<true><<<grid, 256, 0, st>>>(src[0], src[1], src[2], e[0], e[1], e[2], dst[0], dst[1], dst[2], f[0], f[1], f[2]);
  else
    curl_kernel<false><<<grid, 256, 0, st>>>(src[0], src[1], src[2], e[0], e[1], e[2], dst[0], dst[1], dst[2], f[0], f[1], f[2]);
}

void launch_dot_partials(const double* x, const double* y, size_t n, double* partials, int slot, cudaStream_t st) {
  dot_partials_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(x, y, n, partials, slot);
}

void launch_finalize_sum(const double* partials, int nslots, double scale, double* out, cudaStream_t st) {
  finalize_sum_kernel<<<1, kRedThreads, 0, st>>>(partials, nslots * kRedBlocks, scale, out);
}

void launch_div_max(int kind, const double* const src[3], const int sext[3][3], double* partials, int slot,
                    cudaStream_t st) {
  int3 e[3];
  for (int c = 0; c < 3; ++c) e[c] = make_int3(sext[c][0], sext[c][1], sext[c][2]);
  // output (3-form) extents: dual -> own axis shrinks by one; primal -> grows by one
  int3 f;
  if (kind == 1) f = make_int3(sext[0][0] - 1, sext[1][1] - 1, sext[2][2] - 1);
  else f = make_int3(sext[0][0] + 1, sext[1][1] + 1, sext[2][2] + 1);
  if (kind == 1)
    div_max_kernel<true><<<kRedBlocks, kRedThreads, 0, st>>>(src[0], src[1], src[2], e[0], e[1], e[2], f, partials, slot);
  else
    div_max_kernel<false><<<kRedBlocks, kRedThreads, 0, st>>>(src[0], src[1], src[2], e[0], e[1], e[2], f, partials, slot);
}

void launch_absmax(const double* x, size_t n, double* partials, int slot, cudaStream_t st) {
  absmax_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(x, n, partials, slot);
}

void launch_normalize(double* x, size_t n, const double* partials, int slot, cudaStream_t st) {
  normalize_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(x, n, partials, slot);
}

void launch_axpy_ratio(double* x, const double* p, size_t n, const double* num, const double* den, double sign,
                       cudaStream_t st) {
  axpy_ratio_kernel<<<4 * kRedBlocks, kRedThreads, 0, st>>>(x, p, n, num, den, sign);
}

void launch_xpby_ratio(double* p, const double* z, size_t n, const double* num, const double* den, cudaStream_t st) {
  xpby_ratio_kernel<<<4 * kRedBlocks, kRedThreads, 0, st>>>(p, z, n, num, den);
}

void launch_rayleigh(const double* partials, double* out, cudaStream_t st) {
  rayleigh_kernel<<<1, kRedThreads, 0, st>>>(partials, out);
}

void launch_finalize_max(const double* partials, int nslots_each, int ngroups, double* out, cudaStream_t st) {
  finalize_max_kernel<<<1, kRedThreads, 0, st>>>(partials, nslots_each * kRedBlocks, ngroups, out);
}

}  // namespace sgm
