// sm_100a kernels of the scheme-2 leapfrog step (arXiv 2302.04979).
//
// * Line sweeps (Kronecker factors applied mode by mode, eq. kroninverse P:L571 with the vec
//   trick P:L575-585): a CTA stages `nl` whole lines of one component in shared memory
//   (cp.async, no register staging), each thread then walks one line: an optional banded
//   mat-vec (separable Hodge Gram or pairing factor) fused with the forward substitution of a
//   no-pivot banded LU, then the backward substitution, in place in shared memory; the result
//   is stored coalesced.  x-lines are contiguous and use an odd smem pitch (conflict-free
//   line walks); y/z lines are strided and are staged element-major so that the 32 lanes of
//   a warp touch 32 consecutive x.
// * The Ampere / Faraday updates (integer +-1 curls, eqs. discrete2_ampere / _faraday,
//   P:L201) are fused into the load of the first (x) sweep of each half step.
// * General Hodge (curved F or variable material): per-element sum factorisation with the
//   quadrature weights W streamed from HBM, accumulated with fp64 atomics.
// * Deterministic two-pass reductions for the energy and Gauss residuals.
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels.cuh"
#include "seg_sweep.cuh"
#include "sweep_kernel.cuh"

#include <cstdint>
#include <cstdlib>
#include <cstring>

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

template <int PRO>
__device__ __forceinline__ double update_value(const PrologueArgs& P, int c, const double* state, long idx, int x, int y,
                                               int z) {
  if (PRO == PRO_AMPERE) {
    double cu = curl_comp<true>(P.src, P.sext, c, x, y, z);
    if (P.jhat[c]) {
      double s = P.s_ptr ? __ldg(P.s_ptr) : 1.0;
      cu -= s * __ldg(P.jhat[c] + idx);
    }
    return state[idx] + P.dt * cu;                    // d + dt (D~1 h - s j)
  } else {
    double cu = curl_comp<false>(P.src, P.sext, c, x, y, z);
    return state[idx] - P.dt * cu;                    // b - dt D1 e
  }
}

// element-wise update (general-Hodge path): same arithmetic as the fused prologue
template <int PRO>
__global__ void update_kernel(const __grid_constant__ SweepArgs A) {
  const int c = blockIdx.y;
  const SweepComp& C = A.comp[c];
  const int X = C.ext[0], Y = C.ext[1], Z = C.ext[2];
  const long N = long(X) * Y * Z;
  for (long idx = long(blockIdx.x) * blockDim.x + threadIdx.x; idx < N; idx += long(gridDim.x) * blockDim.x) {
    int x = int(idx % X);
    long r = idx / X;
    int y = int(r % Y), z = int(r / Y);
    C.in[idx] = update_value<PRO>(A.pro, c, C.in, idx, x, y, z);
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

// ---- general Hodge: one CTA per element, Q^3 threads, sum factorisation ------------------
// y_c[i] += sum_q phi_{c,i}(x_q) sum_c' W_{cc'}(q) sum_j phi_{c',j}(x_q) x_{c'}[j]
template <int P>
__global__ void hodge_general_kernel(const __grid_constant__ HodgeArgs A) {
  constexpr int NL = P + 1;
  const int Q = A.Q;
  const int nx = A.nel[0], ny = A.nel[1];
  const long e = blockIdx.x;
  const int ex = int(e % nx), ey = int((e / nx) % ny), ez = int(e / (long(nx) * ny));
  const int t = threadIdx.x, nt = blockDim.x;
  const int M = (NL > Q ? NL : Q);
  extern __shared__ double sm[];
  double* U = sm;                   // [3][M^3]
  double* V = sm + 3 * M * M * M;   // [3][M^3]
  const int MM = M * M * M;
  // basis pointers per comp per axis
  const double* B[3][3];
  int f[3][3];
  for (int c = 0; c < 3; ++c)
    for (int a = 0; a < 3; ++a) {
      int role = (a == c) ? 0 : 1;
      int el = (a == 0) ? ex : (a == 1 ? ey : ez);
      B[c][a] = A.basis + A.basis_off[a][role] + size_t(el) * Q * NL;
      f[c][a] = A.first[A.first_off[a][role] + el];
    }
  // load local coefficient boxes U0[c][k][j][i]
  for (int idx = t; idx < 3 * NL * NL * NL; idx += nt) {
    int c = idx / (NL * NL * NL), r = idx % (NL * NL * NL);
    int i = r % NL, j = (r / NL) % NL, k = r / (NL * NL);
    int gi = f[c][0] + i, gj = f[c][1] + j, gk = f[c][2] + k;
    double v = 0.0;
    if (gi >= 0 && gi < A.ext[c][0] && gj >= 0 && gj < A.ext[c][1] && gk >= 0 && gk < A.ext[c][2])
      v = __ldg(A.x[c] + gi + long(A.ext[c][0]) * (gj + long(A.ext[c][1]) * gk));
    U[c * MM + (k * NL + j) * NL + i] = v;
  }
  __syncthreads();
  // x: V[c][k][j][qx] = sum_i Bx[qx][i] U[c][k][j][i]
  for (int idx = t; idx < 3 * NL * NL * Q; idx += nt) {
    int c = idx / (NL * NL * Q), r = idx % (NL * NL * Q);
    int qx = r % Q, jk = r / Q;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NL; ++i) s = fma(__ldg(B[c][0] + qx * NL + i), U[c * MM + jk * NL + i], s);
    V[c * MM + jk * Q + qx] = s;
  }
  __syncthreads();
  // y: U[c][k][qy][qx] = sum_j By[qy][j] V[c][k][j][qx]
  for (int idx = t; idx < 3 * NL * Q * Q; idx += nt) {
    int c = idx / (NL * Q * Q), r = idx % (NL * Q * Q);
    int qx = r % Q, qy = (r / Q) % Q, k = r / (Q * Q);
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NL; ++j) s = fma(__ldg(B[c][1] + qy * NL + j), V[c * MM + (k * NL + j) * Q + qx], s);
    U[c * MM + (k * Q + qy) * Q + qx] = s;
  }
  __syncthreads();
  // z + weights: one thread per quadrature point
  const long qbase = e * long(Q) * Q * Q;
  for (int q = t; q < Q * Q * Q; q += nt) {
    int qx = q % Q, qy = (q / Q) % Q, qz = q / (Q * Q);
    double u[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < NL; ++k) s = fma(__ldg(B[c][2] + qz * NL + k), U[c * MM + (k * Q + qy) * Q + qx], s);
      u[c] = s;
    }
    double v[3];
    if (A.full) {
      const double* w = A.W + (qbase + q) * 6;
      double wxx = __ldg(w), wyy = __ldg(w + 1), wzz = __ldg(w + 2), wxy = __ldg(w + 3), wxz = __ldg(w + 4),
             wyz = __ldg(w + 5);
      v[0] = wxx * u[0] + wxy * u[1] + wxz * u[2];
      v[1] = wxy * u[0] + wyy * u[1] + wyz * u[2];
      v[2] = wxz * u[0] + wyz * u[1] + wzz * u[2];
    } else {
      double w = __ldg(A.W + qbase + q);
      v[0] = A.scale[0] * w * u[0];
      v[1] = A.scale[1] * w * u[1];
      v[2] = A.scale[2] * w * u[2];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) V[c * MM + q] = v[c];
  }
  __syncthreads();
  // test z: U[c][k][qy][qx] = sum_qz Bz[qz][k] V[c][qz][qy][qx]
  for (int idx = t; idx < 3 * NL * Q * Q; idx += nt) {
    int c = idx / (NL * Q * Q), r = idx % (NL * Q * Q);
    int qx = r % Q, qy = (r / Q) % Q, k = r / (Q * Q);
    double s = 0.0;
    for (int qz = 0; qz < Q; ++qz) s = fma(__ldg(B[c][2] + qz * NL + k), V[c * MM + (qz * Q + qy) * Q + qx], s);
    U[c * MM + (k * Q + qy) * Q + qx] = s;
  }
  __syncthreads();
  // test y: V[c][k][j][qx] = sum_qy By[qy][j] U[c][k][qy][qx]
  for (int idx = t; idx < 3 * NL * NL * Q; idx += nt) {
    int c = idx / (NL * NL * Q), r = idx % (NL * NL * Q);
    int qx = r % Q, j = (r / Q) % NL, k = r / (Q * NL);
    double s = 0.0;
    for (int qy = 0; qy < Q; ++qy) s = fma(__ldg(B[c][1] + qy * NL + j), U[c * MM + (k * Q + qy) * Q + qx], s);
    V[c * MM + (k * NL + j) * Q + qx] = s;
  }
  __syncthreads();
  // test x + scatter-add
  for (int idx = t; idx < 3 * NL * NL * NL; idx += nt) {
    int c = idx / (NL * NL * NL), r = idx % (NL * NL * NL);
    int i = r % NL, j = (r / NL) % NL, k = r / (NL * NL);
    int gi = f[c][0] + i, gj = f[c][1] + j, gk = f[c][2] + k;
    if (gi < 0 || gi >= A.ext[c][0] || gj < 0 || gj >= A.ext[c][1] || gk < 0 || gk >= A.ext[c][2]) continue;
    double s = 0.0;
    for (int qx = 0; qx < Q; ++qx) s = fma(__ldg(B[c][0] + qx * NL + i), V[c * MM + (k * NL + j) * Q + qx], s);
    atomicAdd(A.y[c] + gi + long(A.ext[c][0]) * (gj + long(A.ext[c][1]) * gk), s);
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return s ? atoi(s) : dflt;
}

template <int P, int SEG, int LPT, int MODE, int OPS>
bool launch_sweep_t(const SweepArgs& a, cudaStream_t st) {
  using sweep::Cfg;
  Cfg cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  constexpr int TW = 32 * LPT;
  int Lmax = 0;
  for (int c = 0; c < 3; ++c) {
    if (c >= a.ncomp) continue;
    const SweepComp& C = a.comp[c];
    sweep::CompGeom& g = cfg.g[c];
    const int X = C.ext[0], Y = C.ext[1], Z = C.ext[2];
    g.L = C.ext[a.axis];
    g.magic = 0xffffffffu / unsigned(X);
    g.nlines = X * Y * Z / g.L;
    g.X = X;
    g.rowlen = X;
    g.gs = (a.axis == 0) ? 1 : (a.axis == 1 ? X : X * Y);
    g.os = (a.axis == 1) ? X * Y : X;  // transverse index l / X: z (y pass) or y (z pass)
    cfg.tiles[c] = (g.nlines + TW - 1) / TW;
    cfg.nitems += cfg.tiles[c];
    Lmax = g.L > Lmax ? g.L : Lmax;
  }
  cfg.NC = (Lmax + SEG - 1) / SEG;
  cfg.rows = cfg.NC * SEG + P;
  // x axis: a tile of whole lines is one contiguous range -> one bulk copy in and one out (TMA
  // engine), if the component bases are 16-byte aligned and the component has an even size.
  // (Strided tiles are many small row runs: measured slower on the bulk engine than cp.async.)
  bool bulk = (MODE == 3) && env_int("SGM_BULK", 1) != 0;
  for (int c = 0; c < a.ncomp && bulk; ++c) {
    const SweepComp& C = a.comp[c];
    if ((reinterpret_cast<uintptr_t>(C.in) & 15) || (reinterpret_cast<uintptr_t>(C.out) & 15)) bulk = false;
    if ((long(C.ext[0]) * C.ext[1] * C.ext[2]) & 1) bulk = false;
  }
  cfg.bulk = bulk ? 1 : 0;
  if (bulk) cfg.NP = 1;
  else cfg.NP = (MODE == 1 || MODE == 2) ? env_int("SGM_NP_UPD", 16 - cfg.NC) : env_int("SGM_NP", MODE == 3 ? 4 : 2);
  if (cfg.NP < 1) cfg.NP = 1;
  if (cfg.NC + cfg.NP > 16) cfg.NP = 16 - cfg.NC;
  if (cfg.NP < 1) return false;
  if (MODE == 3) {
    cfg.pitch = bulk ? Lmax : (cfg.rows | 1);  // bulk: whole-tile copy, pitch = line length
    cfg.W = 0;
    cfg.slab = TW * cfg.pitch + cfg.rows + 2;
  } else {
    cfg.pitch = 0;
    cfg.W = TW;
    cfg.slab = cfg.W * cfg.rows;
  }
  cfg.slab = (cfg.slab + 1) & ~1;  // keep every slab 16-byte aligned
  cfg.ntabs = (a.tabs[1] != nullptr && a.tabs[1] != a.tabs[0]) ? 2 : 1;
  cfg.tab_dbl = a.tab_rows * RowLayout<P>::RS;
  cfg.dbg = env_int("SGM_PIPE_DBG", 0);
  if (MODE == 1 || MODE == 2) {
    for (int c = 0; c < 3; ++c) {
      // (D x)_c = d_{a1} x_{c1} - d_{a2} x_{c2}, (a1, c1) = (c+1, c+2), (a2, c2) = (c+2, c+1)
      const int a1 = (c + 1) % 3, c1 = (c + 2) % 3, a2 = (c + 2) % 3, c2 = (c + 1) % 3;
      const int aa[2] = {a1, a2}, cc[2] = {c1, c2};
      for (int t = 0; t < 2; ++t) {
        auto& T = cfg.term[c][t];
        T.src = a.pro.src[cc[t]];
        T.X = a.pro.sext[cc[t]][0];
        T.Y = a.pro.sext[cc[t]][1];
        T.a = aa[t];
        T.ext_a = a.pro.sext[cc[t]][aa[t]];
        T.sign = t == 0 ? 1 : -1;
      }
    }
  }
  constexpr int M = P - 1;
  const size_t smem = (size_t(cfg.ntabs) * cfg.tab_dbl + size_t(2) * cfg.slab + size_t(2) * cfg.NC * M * TW + 2) *
                      sizeof(double);
  if (smem > 227 * 1024) return false;
  const int NT = (cfg.NC + cfg.NP) * 32;
  static int attr_done = 0;
  if (!attr_done) {
    cudaFuncSetAttribute(sweep::sweep_kernel<P, SEG, LPT, MODE, OPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    attr_done = 1;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep::sweep_kernel<P, SEG, LPT, MODE, OPS>, NT, smem);
  if (per_sm < 1) per_sm = 1;
  const int cap = env_int("SGM_CTAS_PER_SM", 0);
  if (cap > 0 && cap < per_sm) per_sm = cap;
  long grid = long(per_sm) * sm_count();
  if (grid > cfg.nitems) grid = cfg.nitems;
  if (grid < 1) grid = 1;
  sweep::sweep_kernel<P, SEG, LPT, MODE, OPS><<<unsigned(grid), NT, smem, st>>>(a, cfg);
  return true;
}

template <int P, int SEG, int MODE, int OPS>
void launch_sweep_m(const SweepArgs& a, cudaStream_t st) {
  // two lines per thread when the register budget allows (SEG <= 17) and the slabs fit
  if constexpr (SEG <= 17) {
    if (env_int("SGM_LPT", 2) == 2 && launch_sweep_t<P, SEG, 2, MODE, OPS>(a, st)) return;
  }
  launch_sweep_t<P, SEG, 1, MODE, OPS>(a, st);
}

template <int P, int SEG, int MODE>
void launch_sweep_o(const SweepArgs& a, cudaStream_t st) {
  if (a.band && a.solve) launch_sweep_m<P, SEG, MODE, 3>(a, st);
  else if (a.solve) launch_sweep_m<P, SEG, MODE, 2>(a, st);
  else launch_sweep_m<P, SEG, MODE, 1>(a, st);
}

template <int P, int SEG>
void launch_sweep_s(const SweepArgs& a, cudaStream_t st) {
  if (a.axis == 0) launch_sweep_o<P, SEG, 3>(a, st);
  else if (a.pro_kind == PRO_AMPERE) launch_sweep_m<P, SEG, 1, 3>(a, st);
  else if (a.pro_kind == PRO_FARADAY) launch_sweep_m<P, SEG, 2, 3>(a, st);
  else launch_sweep_o<P, SEG, 0>(a, st);
}

template <int P>
void launch_sweep_p(int seg, const SweepArgs& a, cudaStream_t st) {
  switch (seg) {
    case 12: launch_sweep_s<P, 12>(a, st); break;
    case 17: launch_sweep_s<P, 17>(a, st); break;
    case 22: launch_sweep_s<P, 22>(a, st); break;
    default: launch_sweep_s<P, 28>(a, st); break;
  }
}

}  // namespace

int partial_blocks() { return kRedBlocks; }

void launch_sweep(int p, int seg, const SweepArgs& a, cudaStream_t st) {
  switch (p) {
    case 2: launch_sweep_p<2>(seg, a, st); break;
    case 3: launch_sweep_p<3>(seg, a, st); break;
    case 4: launch_sweep_p<4>(seg, a, st); break;
    default: break;
  }
}

void launch_update(int pro, const SweepArgs& a, cudaStream_t st) {
  dim3 grid(4 * 148, a.ncomp);
  if (pro == PRO_AMPERE) update_kernel<PRO_AMPERE><<<grid, 256, 0, st>>>(a);
  else update_kernel<PRO_FARADAY><<<grid, 256, 0, st>>>(a);
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

void launch_hodge_general(int p, const HodgeArgs& a, cudaStream_t st) {
  long nel = long(a.nel[0]) * a.nel[1] * a.nel[2];
  int Q = a.Q;
  int M = (p + 1 > Q) ? p + 1 : Q;
  size_t smem = size_t(6) * M * M * M * sizeof(double);
  int threads = Q * Q * Q;
  if (threads < 32) threads = 32;
  switch (p) {
    case 2: hodge_general_kernel<2><<<unsigned(nel), threads, smem, st>>>(a); break;
    case 3: hodge_general_kernel<3><<<unsigned(nel), threads, smem, st>>>(a); break;
    case 4: hodge_general_kernel<4><<<unsigned(nel), threads, smem, st>>>(a); break;
    default: break;
  }
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

void launch_finalize_max(const double* partials, int nslots_each, int ngroups, double* out, cudaStream_t st) {
  finalize_max_kernel<<<1, kRedThreads, 0, st>>>(partials, nslots_each * kRedBlocks, ngroups, out);
}

}  // namespace sgm
