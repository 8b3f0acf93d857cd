// General (non-separable) Hodge launchers: brick-tiled sum factorisation (hodge_brick.cuh) and a
// generic CTA-per-element kernel for quadrature rules other than p+1 points.
#include <cuda_runtime.h>

#include <algorithm>

#include <type_traits>

#include "hodge_brick.cuh"
#include <vector>

#include "kernels.cuh"
#include "launch_util.cuh"

namespace sgm {
namespace {

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
  extern __shared__ __align__(16) double sm[];
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

// Work decomposition of the brick kernel: bricks of E x E elements in (x, y) times z chunks.
template <int P, int Q, int DUAL, bool FULL, bool OTF = false>
void brick_plan(const int nel[3], int& zchunk, long& items, long& slots, size_t& smem) {
  constexpr int E = 4;
  using L = brick::Layout<P, Q, DUAL, E>;
  smem = size_t(L::template total<FULL, OTF>()) * sizeof(double);
  static unsigned long long attr = 0;  // per device
  if (first_on_device(attr))
    cudaFuncSetAttribute(brick::hodge_brick_kernel<P, Q, DUAL, FULL, E, OTF>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, brick::hodge_brick_kernel<P, Q, DUAL, FULL, E, OTF>, brick::brick_threads(P),
                                                smem);
  if (per_sm < 1) per_sm = 1;
  slots = long(per_sm) * sm_count();
  const long bricks = long((nel[0] + E - 1) / E) * ((nel[1] + E - 1) / E);
  // z chunks per brick: the count that minimises rounds x (layers per chunk + the per-item cost of
  // about two layers: tables, window fill, the extra flushed layers), rounds = items over resident
  // CTAs rounded up; chunks of at least 4 layers
  long best = -1;
  for (long bzn = 1; bzn <= std::max(1, nel[2] / 4); ++bzn) {
    const long zc = (nel[2] + bzn - 1) / bzn;
    const long its = bricks * ((nel[2] + zc - 1) / zc);
    const long cost = ((its + slots - 1) / slots) * (zc + 2);
    if (best < 0 || cost < best) best = cost, zchunk = int(zc);
  }
  if (const int zc = tune_int("SGM_HODGE_ZCHUNK", 0)) zchunk = zc;
  items = bricks * ((nel[2] + zchunk - 1) / zchunk);
}

// y = M x.  With a large enough scratch (the plan's, sized by hodge_scratch_doubles): every work item
// writes its output patches to the scratch and hodge_gather_kernel sums them in a fixed order --
// bitwise reproducible.  Otherwise fp64 atomics into a zeroed y.
template <int P, int Q, int DUAL, bool FULL, bool OTF = false>
void launch_hodge_brick(const HodgeArgs& a, cudaStream_t st) {
  constexpr int E = 4;
  int zchunk = 0;
  long items = 0, slots = 0;
  size_t smem = 0;
  brick_plan<P, Q, DUAL, FULL, OTF>(a.nel, zchunk, items, slots, smem);
  const long grid = items < slots ? items : slots;
  const size_t need = size_t(items) * brick::item_stride<P, Q, DUAL, E>(zchunk);
  HodgeArgs b = a;
  if (!a.scratch || a.scratch_cap < need) {
    b.scratch = nullptr;
    for (int c = 0; c < 3; ++c)
      cudaMemsetAsync(a.y[c], 0, size_t(a.ext[c][0]) * a.ext[c][1] * a.ext[c][2] * sizeof(double), st);
  }
  brick::hodge_brick_kernel<P, Q, DUAL, FULL, E, OTF><<<unsigned(grid), brick::brick_threads(P), smem, st>>>(b, zchunk);
  if (b.scratch) brick::hodge_gather_kernel<P, Q, DUAL, E><<<unsigned(4 * sm_count()), 256, 0, st>>>(b, zchunk);
}

template <int P, int Q, int DUAL>
size_t scratch_of(int full, const int nel[3]) {
  int zchunk = 0;
  long items = 0, slots = 0;
  size_t smem = 0;
  size_t need = 0;
  if (full) {
    brick_plan<P, Q, DUAL, true>(nel, zchunk, items, slots, smem);
    need = size_t(items) * brick::item_stride<P, Q, DUAL, 4>(zchunk);
    if (DUAL <= 1) {
      // the on-the-fly-geometry kernel (its occupancy, hence z chunks, may differ)
      brick_plan<P, Q, DUAL, true, DUAL <= 1>(nel, zchunk, items, slots, smem);
      need = std::max(need, size_t(items) * brick::item_stride<P, Q, DUAL, 4>(zchunk));
    }
  } else {
    brick_plan<P, Q, DUAL, false>(nel, zchunk, items, slots, smem);
    need = size_t(items) * brick::item_stride<P, Q, DUAL, 4>(zchunk);
  }
  return need;
}

template <int P, int Q>
void launch_hodge2(const HodgeArgs& a, cudaStream_t st) {
  if (a.form >= 2) {
    // 1-form masses (scheme 1): brick kernel only
    if (a.form == 2) {
      if (a.full) launch_hodge_brick<P, Q, 2, true>(a, st);
      else launch_hodge_brick<P, Q, 2, false>(a, st);
    } else {
      if (a.full) launch_hodge_brick<P, Q, 3, true>(a, st);
      else launch_hodge_brick<P, Q, 3, false>(a, st);
    }
    return;
  }
  if (a.dual) {
    if (a.full && a.otf) launch_hodge_brick<P, Q, 1, true, true>(a, st);
    else if (a.full) launch_hodge_brick<P, Q, 1, true>(a, st);
    else launch_hodge_brick<P, Q, 1, false>(a, st);
  } else {
    if (a.full && a.otf) launch_hodge_brick<P, Q, 0, true, true>(a, st);
    else if (a.full) launch_hodge_brick<P, Q, 0, true>(a, st);
    else launch_hodge_brick<P, Q, 0, false>(a, st);
  }
}

}  // namespace

bool hodge_uses_brick(int p, int Q) { return Q == p + 1 && p >= 2 && p <= 4; }

// Element-major weights W[e][point][nw] (e = ex + nx (ey + ny ez), point = (qz Q + qy) Q + qx) ->
// the brick kernel's HBM layout: per element layer ez and brick (by, bx) one chunk of nw planes of
// NU = Q * EQ * (EQ + 1) slots (slot of a point: brick::uidx); pad slots and elements past the mesh
// edge are zero.
void hodge_brick_relayout(int Q, const int nel[3], int nw, std::vector<double>& W) {
  constexpr int E = 4;
  const int EQ = E * Q, RS = EQ + 1;
  const size_t NU = size_t(Q) * EQ * RS;
  const int nx = nel[0], ny = nel[1], nz = nel[2];
  const int bxn = (nx + E - 1) / E, byn = (ny + E - 1) / E;
  std::vector<double> out(size_t(nz) * byn * bxn * nw * NU, 0.0);
  const size_t QQQ = size_t(Q) * Q * Q;
#pragma omp parallel for collapse(2) schedule(static)
  for (int ez = 0; ez < nz; ++ez)
    for (int ey = 0; ey < ny; ++ey)
      for (int ex = 0; ex < nx; ++ex) {
        const size_t e = size_t(ex) + size_t(nx) * (size_t(ey) + size_t(ny) * ez);
        const size_t chunk = (size_t(ez) * byn + ey / E) * bxn + ex / E;
        double* dst = out.data() + chunk * nw * NU;
        const double* src = W.data() + e * QQQ * nw;
        const int exl = ex % E, eyl = ey % E;
        for (int qz = 0; qz < Q; ++qz)
          for (int qy = 0; qy < Q; ++qy)
            for (int qx = 0; qx < Q; ++qx) {
              const size_t slot = (size_t(qz) * EQ + eyl * Q + qy) * RS + exl * Q + qx;
              const size_t pt = (size_t(qz) * Q + qy) * Q + qx;
              for (int k = 0; k < nw; ++k) dst[k * NU + slot] = src[pt * nw + k];
            }
      }
  W.swap(out);
}

size_t hodge_scratch_doubles(int p, int Q, int form, int full, const int nel[3]) {
  if (Q != p + 1) return 0;  // the generic kernel accumulates with atomics
  auto pick = [&](auto pq) -> size_t {
    constexpr int PP = decltype(pq)::value;
    switch (form) {
      case 0: return scratch_of<PP, PP + 1, 0>(full, nel);
      case 1: return scratch_of<PP, PP + 1, 1>(full, nel);
      case 2: return scratch_of<PP, PP + 1, 2>(full, nel);
      default: return scratch_of<PP, PP + 1, 3>(full, nel);
    }
  };
  switch (p) {
    case 2: return pick(std::integral_constant<int, 2>{});
    case 3: return pick(std::integral_constant<int, 3>{});
    case 4: return pick(std::integral_constant<int, 4>{});
    default: return 0;
  }
}

void launch_hodge_general(int p, const HodgeArgs& a, cudaStream_t st) {
  // brick sum-factorisation kernel (hodge_brick.cuh) for the default rule Q = p + 1; the generic
  // CTA-per-element kernel for larger rules (quad_points > p + 1)
  if (a.Q == p + 1) {
    switch (p) {
      case 2: launch_hodge2<2, 3>(a, st); return;
      case 3: launch_hodge2<3, 4>(a, st); return;
      case 4: launch_hodge2<4, 5>(a, st); return;
      default: break;
    }
  }
  for (int c = 0; c < 3; ++c)
    cudaMemsetAsync(a.y[c], 0, size_t(a.ext[c][0]) * a.ext[c][1] * a.ext[c][2] * sizeof(double), st);
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

}  // namespace sgm
