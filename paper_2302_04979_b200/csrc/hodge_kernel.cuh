// General (non-separable) 2-form Hodge apply y = M x (P:L360 M~2_{1/eps}, P:L366 M2_{1/mu}) by
// element-wise sum factorisation (sm_100a, fp64).
//
// On element e the 2-form mass is  y_c += sum_{c'} V_c^T W_{cc'} V_{c'} x_{c'}  where V_c is the
// tensor product of the 1D element bases at the Q Gauss points per axis (component c uses the
// "own" space along axis c and the "other" space along the two other axes) and
// W holds, per quadrature point, w_q / material * DF^T DF / det DF (FULL, 6 symmetric entries) or
// w_q / material with a per-component constant (SCALAR; identity / axis-aligned affine map).
// The exact local box of each component is used (dual 2-forms: p functions along the own axis,
// p-1 along the others; primal: p+1 and p).
//
// One warp walks a z-pencil of elements (ex, ey, 0..nz-1).  Consecutive elements share all but one
// coefficient layer along z, so the coefficient boxes shift by one layer per element (the new layer
// is prefetched into registers while the previous element is computed) and the output boxes are
// accumulated in shared memory; after each element the lowest output layer is complete and is
// flushed with fp64 atomics (only neighbouring pencils share it).  Interpolation: lane (qx, qy)
// computes its z-column of quadrature values; testing: lanes take the roles (qx, jy) and (jx, jy)
// so every reduction over quadrature points is a per-lane loop over shared memory.  W is streamed
// from HBM coalesced (element-major [e][qz][qy][qx]).
#pragma once

#include "kernels.cuh"

namespace sgm {
namespace hodge {

template <int P, bool DUAL, int C, int AX>
__host__ __device__ constexpr int nloc() {
  return (C == AX) ? (DUAL ? P : P + 1) : (DUAL ? P - 1 : P);
}
template <int P, bool DUAL>
__host__ __device__ constexpr int max_box() {
  return DUAL ? P * (P - 1) * (P - 1) : (P + 1) * P * P;
}

struct ElemBasis {
  const double* v[3];  // this component's 1D element basis per axis: [Q][P+1]
  int first[3];        // global index of local function 0 per axis
};

template <int P, bool DUAL, int C>
__device__ __forceinline__ ElemBasis elem_basis(const HodgeArgs& A, int ex, int ey, int ez) {
  constexpr int NL = P + 1;
  ElemBasis B;
  const int el[3] = {ex, ey, ez};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int role = (a == C) ? 0 : 1;
    B.v[a] = A.basis + A.basis_off[a][role] + size_t(el[a]) * A.Q * NL;
    B.first[a] = __ldg(A.first + A.first_off[a][role] + el[a]);
  }
  return B;
}


template <int P, bool DUAL, int C>
struct Box {
  static constexpr int NX = nloc<P, DUAL, C, 0>(), NY = nloc<P, DUAL, C, 1>(), NZ = nloc<P, DUAL, C, 2>();
  static constexpr int LAYER = NX * NY, SIZE = LAYER * NZ;
};

// load coefficient layer jz (global z index gz) of component C into X (zero outside the component)
template <int P, bool DUAL, int C>
__device__ __forceinline__ void load_layer(const ElemBasis& B, const double* __restrict__ xg, const int* ext, int gz,
                                           double* Xl, int lane) {
  using BX = Box<P, DUAL, C>;
  for (int o = lane; o < BX::LAYER; o += 32) {
    const int jx = o % BX::NX, jy = o / BX::NX;
    const int gx = B.first[0] + jx, gy = B.first[1] + jy;
    double val = 0.0;
    if (gx >= 0 && gx < ext[0] && gy >= 0 && gy < ext[1] && gz >= 0 && gz < ext[2])
      val = __ldg(xg + gx + long(ext[0]) * (gy + long(ext[1]) * gz));
    Xl[o] = val;
  }
}

// one value of coefficient layer gz of component C for lane `lane` (< LAYER), zero outside
template <int P, bool DUAL, int C>
__device__ __forceinline__ double fetch_layer_elem(const ElemBasis& B, const double* __restrict__ xg, const int* ext,
                                                   int gz, int lane) {
  using BX = Box<P, DUAL, C>;
  if (lane >= BX::LAYER) return 0.0;
  const int jx = lane % BX::NX, jy = lane / BX::NX;
  const int gx = B.first[0] + jx, gy = B.first[1] + jy;
  if (gx >= 0 && gx < ext[0] && gy >= 0 && gy < ext[1] && gz >= 0 && gz < ext[2])
    return __ldg(xg + gx + long(ext[0]) * (gy + long(ext[1]) * gz));
  return 0.0;
}

// flush output layer 0 (global z index gz) of component C with atomics, shift the box down a layer
template <int P, bool DUAL, int C>
__device__ __forceinline__ void flush_shift(const ElemBasis& B, double* __restrict__ yg, const int* ext, int gz,
                                            double* Y, double* X, int lane, bool shift_x) {
  using BX = Box<P, DUAL, C>;
  for (int o = lane; o < BX::LAYER; o += 32) {
    const int jx = o % BX::NX, jy = o / BX::NX;
    const int gx = B.first[0] + jx, gy = B.first[1] + jy;
    if (gx >= 0 && gx < ext[0] && gy >= 0 && gy < ext[1] && gz >= 0 && gz < ext[2])
      atomicAdd(yg + gx + long(ext[0]) * (gy + long(ext[1]) * gz), Y[o]);
  }
  __syncwarp();
  for (int o = lane; o < BX::SIZE - BX::LAYER; o += 32) {
    Y[o] = Y[o + BX::LAYER];
    if (shift_x) X[o] = X[o + BX::LAYER];
  }
  __syncwarp();
  for (int o = lane; o < BX::LAYER; o += 32) Y[BX::SIZE - BX::LAYER + o] = 0.0;
  __syncwarp();
}


// ---- interpolation / testing of one component (lane roles above); the pencil's x and y bases
// live in shared memory for the whole pencil, the element's z bases are staged per element.
template <int P, int Q, bool DUAL, int C>
__device__ __forceinline__ void interp_pencil(const double* X, const double* Vx, const double* Vy, const double* Vz,
                                          int lane, double (&u)[Q]) {
  using BX = Box<P, DUAL, C>;
  constexpr int NX = BX::NX, NY = BX::NY, NZ = BX::NZ, NL = P + 1;
  if (lane < Q * Q) {
    const int qx = lane % Q, qy = lane / Q;
    double vx[NX], vy[NY];
#pragma unroll
    for (int j = 0; j < NX; ++j) vx[j] = Vx[qx * NL + j];
#pragma unroll
    for (int j = 0; j < NY; ++j) vy[j] = Vy[qy * NL + j];
    double b[NZ];
#pragma unroll
    for (int jz = 0; jz < NZ; ++jz) {
      double acc = 0.0;
#pragma unroll
      for (int jy = 0; jy < NY; ++jy) {
        double t = 0.0;
#pragma unroll
        for (int jx = 0; jx < NX; ++jx) t = fma(vx[jx], X[(jz * NY + jy) * NX + jx], t);
        acc = fma(vy[jy], t, acc);
      }
      b[jz] = acc;
    }
#pragma unroll
    for (int qz = 0; qz < Q; ++qz) {
      double s = 0.0;
#pragma unroll
      for (int jz = 0; jz < NZ; ++jz) s = fma(Vz[qz * NL + jz], b[jz], s);
      u[qz] = s;
    }
  }
}

template <int P, int Q, bool DUAL, int C>
__device__ __forceinline__ void test_pencil(double* Y, const double* Vx, const double* Vy, const double* Vz, double* Cb,
                                        double* Tb, int lane, const double (&v)[Q]) {
  using BX = Box<P, DUAL, C>;
  constexpr int NX = BX::NX, NY = BX::NY, NZ = BX::NZ, NL = P + 1;
  // (qx, qy): C[jz][qy][qx] = sum_qz Vz[qz][jz] v[qz]
  if (lane < Q * Q) {
#pragma unroll
    for (int jz = 0; jz < NZ; ++jz) {
      double s = 0.0;
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) s = fma(Vz[qz * NL + jz], v[qz], s);
      Cb[jz * Q * Q + lane] = s;
    }
  }
  __syncwarp();
  // (qx, jy): T[jz][jy][qx] = sum_qy Vy[qy][jy] C[jz][qy][qx]
  if (lane < Q * NY) {
    const int qx = lane % Q, jy = lane / Q;
    double vyc[Q];
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) vyc[qy] = Vy[qy * NL + jy];
#pragma unroll
    for (int jz = 0; jz < NZ; ++jz) {
      double s = 0.0;
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) s = fma(vyc[qy], Cb[(jz * Q + qy) * Q + qx], s);
      Tb[(jz * NY + jy) * Q + qx] = s;
    }
  }
  __syncwarp();
  // (jx, jy): Y[jz][jy][jx] += sum_qx Vx[qx][jx] T[jz][jy][qx]
  if (lane < NX * NY) {
    const int jx = lane % NX, jy = lane / NX;
    double vxc[Q];
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) vxc[qx] = Vx[qx * NL + jx];
#pragma unroll
    for (int jz = 0; jz < NZ; ++jz) {
      double s = 0.0;
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) s = fma(vxc[qx], Tb[(jz * NY + jy) * Q + qx], s);
      Y[(jz * NY + jy) * NX + jx] += s;
    }
  }
  __syncwarp();
}

template <int P, int Q, bool DUAL, bool FULL>
__global__ void __launch_bounds__(256, 2) hodge_pencil_kernel(const __grid_constant__ HodgeArgs A) {
  constexpr int QQQ = Q * Q * Q, NL = P + 1;
  constexpr int XB = max_box<P, DUAL>();
  constexpr int VB = Q * NL;                 // one 1D element basis [Q][NL]
  constexpr int CB = (P + 1) * Q * Q;        // >= NZ*Q*Q
  constexpr int TB = (P + 1) * (P + 1) * Q;  // >= NZ*NY*Q
  constexpr int WSZ = 6 * XB + 9 * VB + CB + TB;
  static_assert(Q * Q <= 32, "lane (qx, qy) roles need Q*Q <= 32");
  extern __shared__ double smp[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* base = smp + wib * WSZ;
  double* X[3] = {base, base + XB, base + 2 * XB};
  double* Y[3] = {base + 3 * XB, base + 4 * XB, base + 5 * XB};
  double* Vb = base + 6 * XB;  // [comp][axis x, y, z][Q][NL]
  double* Cb = Vb + 9 * VB;
  double* Tb = Cb + CB;
  const int nx = A.nel[0], ny = A.nel[1], nz = A.nel[2];
  const long npen = long(nx) * ny;
  const long wstride = long(gridDim.x) * (blockDim.x >> 5);
  for (long pen = long(blockIdx.x) * (blockDim.x >> 5) + wib; pen < npen; pen += wstride) {
    const int ex = int(pen % nx), ey = int(pen / nx);
    ElemBasis B0 = elem_basis<P, DUAL, 0>(A, ex, ey, 0);
    ElemBasis B1 = elem_basis<P, DUAL, 1>(A, ex, ey, 0);
    ElemBasis B2 = elem_basis<P, DUAL, 2>(A, ex, ey, 0);
    // the pencil's x and y bases per component
    const ElemBasis* BB[3] = {&B0, &B1, &B2};
    for (int o = lane; o < 3 * 2 * VB; o += 32) {
      const int c = o / (2 * VB), r = o % (2 * VB), a = r / VB, i = r % VB;
      Vb[(c * 3 + a) * VB + i] = __ldg(BB[c]->v[a] + i);
    }
    for (int o = lane; o < 3 * XB; o += 32) Y[0][o] = 0.0;  // Y[0..2] are contiguous
    __syncwarp();
    for (int jz = 0; jz + 1 < Box<P, DUAL, 0>::NZ; ++jz)
      load_layer<P, DUAL, 0>(B0, A.x[0], A.ext[0], B0.first[2] + jz, X[0] + jz * Box<P, DUAL, 0>::LAYER, lane);
    for (int jz = 0; jz + 1 < Box<P, DUAL, 1>::NZ; ++jz)
      load_layer<P, DUAL, 1>(B1, A.x[1], A.ext[1], B1.first[2] + jz, X[1] + jz * Box<P, DUAL, 1>::LAYER, lane);
    for (int jz = 0; jz + 1 < Box<P, DUAL, 2>::NZ; ++jz)
      load_layer<P, DUAL, 2>(B2, A.x[2], A.ext[2], B2.first[2] + jz, X[2] + jz * Box<P, DUAL, 2>::LAYER, lane);
    // software pipeline: element ez+1's new coefficient layer and z bases are loaded into registers
    // while element ez is computed (one value per lane per component: LAYER <= 32)
    static_assert(Box<P, DUAL, 0>::LAYER <= 32 && Box<P, DUAL, 1>::LAYER <= 32 && Box<P, DUAL, 2>::LAYER <= 32, "");
    constexpr int RV = (3 * VB + 31) / 32;
    double pfx[3], pfv[RV];
    auto prefetch = [&](int ez1) {
      const ElemBasis N0 = elem_basis<P, DUAL, 0>(A, ex, ey, ez1);
      const ElemBasis N1 = elem_basis<P, DUAL, 1>(A, ex, ey, ez1);
      const ElemBasis N2 = elem_basis<P, DUAL, 2>(A, ex, ey, ez1);
      pfx[0] = fetch_layer_elem<P, DUAL, 0>(N0, A.x[0], A.ext[0], N0.first[2] + Box<P, DUAL, 0>::NZ - 1, lane);
      pfx[1] = fetch_layer_elem<P, DUAL, 1>(N1, A.x[1], A.ext[1], N1.first[2] + Box<P, DUAL, 1>::NZ - 1, lane);
      pfx[2] = fetch_layer_elem<P, DUAL, 2>(N2, A.x[2], A.ext[2], N2.first[2] + Box<P, DUAL, 2>::NZ - 1, lane);
#pragma unroll
      for (int r = 0; r < RV; ++r) {
        const int o = lane + 32 * r;
        const int c = o / VB;
        const double* vz = (c == 0) ? N0.v[2] : (c == 1 ? N1.v[2] : N2.v[2]);
        pfv[r] = (o < 3 * VB) ? __ldg(vz + (o % VB)) : 0.0;
      }
    };
    prefetch(0);
    for (int ez = 0; ez < nz; ++ez) {
      const long e = ex + long(nx) * (ey + long(ny) * ez);
      B0 = elem_basis<P, DUAL, 0>(A, ex, ey, ez);
      B1 = elem_basis<P, DUAL, 1>(A, ex, ey, ez);
      B2 = elem_basis<P, DUAL, 2>(A, ex, ey, ez);
      // store the prefetched top layers and z bases of this element
      if (lane < Box<P, DUAL, 0>::LAYER) X[0][(Box<P, DUAL, 0>::NZ - 1) * Box<P, DUAL, 0>::LAYER + lane] = pfx[0];
      if (lane < Box<P, DUAL, 1>::LAYER) X[1][(Box<P, DUAL, 1>::NZ - 1) * Box<P, DUAL, 1>::LAYER + lane] = pfx[1];
      if (lane < Box<P, DUAL, 2>::LAYER) X[2][(Box<P, DUAL, 2>::NZ - 1) * Box<P, DUAL, 2>::LAYER + lane] = pfx[2];
#pragma unroll
      for (int r = 0; r < RV; ++r) {
        const int o = lane + 32 * r;
        if (o < 3 * VB) Vb[((o / VB) * 3 + 2) * VB + (o % VB)] = pfv[r];
      }
      if (ez + 1 < nz) prefetch(ez + 1);
      __syncwarp();
      double u0[Q], u1[Q], u2[Q];
      interp_pencil<P, Q, DUAL, 0>(X[0], Vb + 0 * VB, Vb + 1 * VB, Vb + 2 * VB, lane, u0);
      interp_pencil<P, Q, DUAL, 1>(X[1], Vb + 3 * VB, Vb + 4 * VB, Vb + 5 * VB, lane, u1);
      interp_pencil<P, Q, DUAL, 2>(X[2], Vb + 6 * VB, Vb + 7 * VB, Vb + 8 * VB, lane, u2);
      double v0[Q], v1[Q], v2[Q];
      if (lane < Q * Q) {
        if (FULL) {
          const double* w = A.W + (e * QQQ + lane) * 6;
#pragma unroll
          for (int qz = 0; qz < Q; ++qz) {
            const double* wq = w + qz * Q * Q * 6;
            const double wxx = __ldg(wq), wyy = __ldg(wq + 1), wzz = __ldg(wq + 2), wxy = __ldg(wq + 3),
                         wxz = __ldg(wq + 4), wyz = __ldg(wq + 5);
            v0[qz] = wxx * u0[qz] + wxy * u1[qz] + wxz * u2[qz];
            v1[qz] = wxy * u0[qz] + wyy * u1[qz] + wyz * u2[qz];
            v2[qz] = wxz * u0[qz] + wyz * u1[qz] + wzz * u2[qz];
          }
        } else {
          const double* w = A.W + e * QQQ + lane;
#pragma unroll
          for (int qz = 0; qz < Q; ++qz) {
            const double wq = __ldg(w + qz * Q * Q);
            v0[qz] = A.scale[0] * wq * u0[qz];
            v1[qz] = A.scale[1] * wq * u1[qz];
            v2[qz] = A.scale[2] * wq * u2[qz];
          }
        }
      }
      test_pencil<P, Q, DUAL, 0>(Y[0], Vb + 0 * VB, Vb + 1 * VB, Vb + 2 * VB, Cb, Tb, lane, v0);
      test_pencil<P, Q, DUAL, 1>(Y[1], Vb + 3 * VB, Vb + 4 * VB, Vb + 5 * VB, Cb, Tb, lane, v1);
      test_pencil<P, Q, DUAL, 2>(Y[2], Vb + 6 * VB, Vb + 7 * VB, Vb + 8 * VB, Cb, Tb, lane, v2);
      flush_shift<P, DUAL, 0>(B0, A.y[0], A.ext[0], B0.first[2], Y[0], X[0], lane, true);
      flush_shift<P, DUAL, 1>(B1, A.y[1], A.ext[1], B1.first[2], Y[1], X[1], lane, true);
      flush_shift<P, DUAL, 2>(B2, A.y[2], A.ext[2], B2.first[2], Y[2], X[2], lane, true);
    }
    ElemBasis L0 = elem_basis<P, DUAL, 0>(A, ex, ey, nz - 1);
    ElemBasis L1 = elem_basis<P, DUAL, 1>(A, ex, ey, nz - 1);
    ElemBasis L2 = elem_basis<P, DUAL, 2>(A, ex, ey, nz - 1);
    for (int jz = 1; jz < Box<P, DUAL, 0>::NZ; ++jz)
      flush_shift<P, DUAL, 0>(L0, A.y[0], A.ext[0], L0.first[2] + jz, Y[0], X[0], lane, false);
    for (int jz = 1; jz < Box<P, DUAL, 1>::NZ; ++jz)
      flush_shift<P, DUAL, 1>(L1, A.y[1], A.ext[1], L1.first[2] + jz, Y[1], X[1], lane, false);
    for (int jz = 1; jz < Box<P, DUAL, 2>::NZ; ++jz)
      flush_shift<P, DUAL, 2>(L2, A.y[2], A.ext[2], L2.first[2] + jz, Y[2], X[2], lane, false);
  }
}

}  // namespace hodge
}  // namespace sgm
