// General (non-separable) 2-form Hodge apply y += M x by brick-tiled sum factorisation
// (sm_100a, fp64); the operator of P:L360 (M~2_{1/eps}) and P:L366 (M2_{1/mu}):
// on element e,  y_c += V_c^T W_{cc'} V_{c'} x_{c'},  V_c the tensor product of the 1D element
// bases at the Q Gauss points per axis, W = w_q / material * DF^T DF / det DF (FULL) or
// w_q / material times a per-component constant (SCALAR).
//
// A CTA owns a brick of E x E elements in (x, y) and walks a range of element layers in z.  The
// brick's coefficients of each component form a patch of PX x PY functions (consecutive elements
// share all but one function per axis: PX = E - 1 + NX); along z a window of NZ coefficient layers
// slides by one layer per element, and the output window accumulates in shared memory, its lowest
// layer complete after each element and written to the work item's patch in the scratch
// (hodge_gather_kernel sums the patches in a fixed order: bitwise reproducible; without a scratch
// the layer is flushed with fp64 atomics).  Both windows are circular (layer jz in slot
// (base + jz) % NZ), so nothing is copied.  Per element layer: [y interpolation | z testing and
// flush of the previous layer] -> [x interpolation, scalar W fused] -> ([3 x 3 W multiply]) ->
// [x testing] -> [y testing | load and z interpolation of the next layer], a block barrier between
// the intervals.  Every 1D contraction is a small register-blocked loop (one thread produces a
// row of outputs from a row of inputs); on bricks / layers of interior elements the basis values
// are kernel parameters (constant-bank FMA operands), else shared-memory broadcasts.  W of a layer
// arrives by one bulk copy (TMA engine) from its brick-layout chunk in HBM.  Shared-memory strides
// are padded so that the consecutive tasks of a stage fall on distinct bank pairs.
#pragma once

#include "kernels.cuh"
#include "pipe_sweep.cuh"

#ifndef SGM_BRICK_NT4
#define SGM_BRICK_NT4 256
#endif

namespace sgm {
namespace brick {

// Local functions per element of component C along axis AX.  DUAL is the form type:
//   0 primal 2-form (own S_p: p+1, other S_{p-1} CS: p)   1 dual 2-form (own S_{p-1}: p, other S_{p-2}: p-1)
//   2 primal 1-form (own S_{p-1} CS: p, other S_p: p+1)   3 dual 1-form (own S_{p-2}: p-1, other S_{p-1}: p)
template <int P, int DUAL, int C, int AX>
__host__ __device__ constexpr int nloc() {
  return DUAL == 0 ? (C == AX ? P + 1 : P)
       : DUAL == 1 ? (C == AX ? P : P - 1)
       : DUAL == 2 ? (C == AX ? P : P + 1)
                   : (C == AX ? P - 1 : P);
}

// Shared-memory strides are padded against bank conflicts (fp64: 16 eight-byte bank pairs): a
// stage whose consecutive tasks t walk a buffer with stride s is conflict-free when s is odd, and a
// stage whose tasks are (plane, px) pairs when the plane stride is congruent to PX modulo 16.
__host__ __device__ constexpr int pad_to(int n, int r) { return n + (((r - n) % 16) + 16) % 16; }

template <int P, int Q, int DUAL, int E, int C>
struct Geo {
  static constexpr int NX = nloc<P, DUAL, C, 0>(), NY = nloc<P, DUAL, C, 1>(), NZ = nloc<P, DUAL, C, 2>();
  static constexpr int PX = E - 1 + NX, PY = E - 1 + NY;
  static constexpr int EQ = E * Q;
  static constexpr int WIN = NZ * PY * PX;   // coefficient / output window
  static constexpr int LAYP = pad_to(PY * PX, PX);  // plane stride of Z1
  static constexpr int PXP = PX | 1;                 // row stride of Z2
  // plane stride of Z2: padded for the y stages' (plane, px) tasks; at p = 4 the pad buys little
  // (simulated 9.1 % against 8.5 % excess wavefronts) and costs the x stages' tasks a division to
  // split their row index (qz, Y), so the planes are contiguous there and a row sits at row * PXP
  static constexpr int Z2P = P >= 4 ? EQ * PXP : pad_to(EQ * PXP, PX);
  __device__ static __forceinline__ int z2row(int row) {
    return Z2P == EQ * PXP ? row * PXP : (row / EQ) * Z2P + (row % EQ) * PXP;
  }
  static constexpr int RSU = EQ + 1;                 // row stride of U (EQ = E * Q is even)
  static constexpr int Z1 = Q * LAYP;        // after the z stage: [qz][py][px]
  static constexpr int Z2 = Q * Z2P;         // after the y stage: [qz][Y][px]
  static constexpr int U = Q * EQ * RSU;     // quadrature values: [qz][Y][X]
  // Z1 (next layer's z interpolation) and T1 (this layer's y testing) are live from the y-testing
  // interval to the next y-interpolation interval, when U is dead: they alias U
  static constexpr int TOT = 2 * WIN + Z2 + U;
  static_assert(2 * Z1 <= U, "Z1 and T1 alias U");
};

template <int P, int Q, int DUAL, int E>
struct Layout {
  using G0 = Geo<P, Q, DUAL, E, 0>;
  using G1 = Geo<P, Q, DUAL, E, 1>;
  using G2 = Geo<P, Q, DUAL, E, 2>;
  static constexpr int NL = P + 1;
  static constexpr int VXY = E * Q * NL;  // brick basis table of one axis and role: [e][q][k]
  static constexpr int VZ = Q * NL;       // one element's z basis of one role
  // per component: Xw, Yw, Z1, Z2, U; then tables [role][axis x, y] and [role] z
  static constexpr int OFF1 = G0::TOT, OFF2 = OFF1 + G1::TOT, TAB = OFF2 + G2::TOT;
  // W of one element layer (one bulk copy per layer: 16-byte aligned, hence the even offset)
  static constexpr int WB = (TAB + 2 * 2 * VXY + 2 * VZ + 1) & ~1;
  static constexpr int NU = G0::U;  // quadrature-point slots of one component (all components: the same)
  // on-the-fly geometry (OTF): the staged W is w_q / material (1 per point); after it the map's
  // partial sums A[r][s][qz][py][px] (z contracted, s = value / derivative), B[r][m][qz][Y][px]
  // (z and y contracted, m = (val,val), (val,der), (der,val)) and the brick's x / y map tables
  // [axis][s][e][q][k] (S_p values / derivatives at the Gauss points)
  static constexpr int PM = E + P;  // map control points of the brick per axis (S_p, E elements)
  static constexpr int MA = 3 * 2 * Q * PM * PM, MB = 3 * 3 * Q * E * Q * PM, MT = 2 * 2 * E * Q * NL;
  template <bool FULL, bool OTF = false>
  __host__ __device__ static constexpr int wdoubles() { return NU * (FULL && !OTF ? 6 : 1); }
  template <bool FULL, bool OTF = false>
  __host__ __device__ static constexpr int total() { return WB + wdoubles<FULL, OTF>() + (OTF ? MA + MB + MT : 0); }
};

struct Brick {
  int ex0, ey0, nex, ney;  // first element and number of live elements of the brick
  int ez0, ez1;            // element layers [ez0, ez1)
};

// quadrature values are stored brick-wide, U[qz][Y = ey*Q + qy][X = ex*Q + qx] with rows padded to
// E*Q + 1 doubles: the x stages' tasks (qz, Y) then walk U with an odd stride (no bank conflicts);
// W uses the same slots, in HBM as well: per brick and element layer one contiguous chunk of NW
// planes (entry k of a point in plane k at the point's U slot; pad slots and elements past the
// mesh edge hold zeros), so a layer's W is staged by a single bulk copy (host: hodge_brick_relayout)
template <int Q, int E>
__device__ __forceinline__ int uidx(int qz, int Yq, int ex, int qx) {
  return (qz * (E * Q) + Yq) * (E * Q + 1) + ex * Q + qx;
}

// per-component pointers into shared memory
template <int P, int Q, int DUAL, int E, int C>
struct CompSm {
  using G = Geo<P, Q, DUAL, E, C>;
  double *Xw, *Yw, *Z1, *T1, *Z2, *U;
  const double *Vx, *Vy, *Vz;  // role-selected basis tables
  // window slot of layer 0 (circular: layer jz lives in slot (base + jz) % NZ); the coefficient
  // window runs one element layer ahead of the output window, hence two bases
  int xbase = 0, ybase = 0;
  __device__ __forceinline__ int slotx(int jz) const {
    const int s = xbase + jz;
    return s >= G::NZ ? s - G::NZ : s;
  }
  __device__ __forceinline__ int sloty(int jz) const {
    const int s = ybase + jz;
    return s >= G::NZ ? s - G::NZ : s;
  }
  // view of component C2's buffers for the x stages, whose code depends on the component only
  // through NX and the x role: components 1 and 2 share one instantiation (less code, and warps
  // whose tasks span both components do not diverge)
  template <int C2>
  __device__ __forceinline__ explicit CompSm(const CompSm<P, Q, DUAL, E, C2>& o)
      : Xw(o.Xw), Yw(o.Yw), Z1(o.Z1), T1(o.T1), Z2(o.Z2), U(o.U), Vx(o.Vx), Vy(o.Vy), Vz(o.Vz) {
    static_assert(Geo<P, Q, DUAL, E, C2>::NX == G::NX && (C == 0) == (C2 == 0), "x-stage compatible components");
  }
  __device__ CompSm(double* sm) {
    using L = Layout<P, Q, DUAL, E>;
    double* b = sm + (C == 0 ? 0 : (C == 1 ? L::OFF1 : L::OFF2));
    Xw = b;
    Yw = Xw + G::WIN;
    Z2 = Yw + G::WIN;
    U = Z2 + G::Z2;
    Z1 = U;
    T1 = U + G::Z1;
    const double* tab = sm + L::TAB;
    // role 0 = own (axis == C), 1 = other
    Vx = tab + ((C == 0 ? 0 : 1) * 2 + 0) * L::VXY;
    Vy = tab + ((C == 1 ? 0 : 1) * 2 + 1) * L::VXY;
    Vz = tab + 4 * L::VXY + (C == 2 ? 0 : 1) * L::VZ;
  }
};

// first global function index of element e along `axis` for `role`
// (uniform open knots: first(e) = first(0) + e, checked when the tables are uploaded, so the index
// is arithmetic on a kernel parameter instead of a table load)
__device__ __forceinline__ int first_of(const HodgeArgs& A, int axis, int role, int e) {
  return A.first0[axis][role] + e;
}

// load coefficient layer jz (global z index gz) of component C's patch into the window
template <int P, int Q, int DUAL, int E, int C>
__device__ __forceinline__ void load_layer(const HodgeArgs& A, const CompSm<P, Q, DUAL, E, C>& S, int gx0, int gy0,
                                           int gz, int jz) {
  using G = Geo<P, Q, DUAL, E, C>;
  const int* ext = A.ext[C];
  const double* __restrict__ x = A.x[C];
  for (int o = threadIdx.x; o < G::PY * G::PX; o += blockDim.x) {
    const int px = o % G::PX, py = o / G::PX;
    const int gx = gx0 + px, gy = gy0 + py;
    double v = 0.0;
    if (gx >= 0 && gx < ext[0] && gy >= 0 && gy < ext[1] && gz >= 0 && gz < ext[2])
      v = __ldg(x + gx + long(ext[0]) * (gy + long(ext[1]) * gz));
    S.Xw[jz * G::PY * G::PX + o] = v;
  }
}

// atomically add the output window slot `sl` (global z index gz) of component C's patch to y and
// clear the slot for reuse as the top layer
// scr: this item's patch layers of component C in the scratch (layer rel = gz - first z of the
// item), or null -> fp64 atomics into y
template <int P, int Q, int DUAL, int E, int C>
__device__ __forceinline__ void flush_layer(const HodgeArgs& A, const CompSm<P, Q, DUAL, E, C>& S, int gx0, int gy0,
                                            int gz, int sl, double* scr, int rel, double sc) {
  using G = Geo<P, Q, DUAL, E, C>;
  constexpr int LAY = G::PY * G::PX;
  const int* ext = A.ext[C];
  double* __restrict__ y = A.y[C];
  for (int o = threadIdx.x; o < LAY; o += blockDim.x) {
    const int px = o % G::PX, py = o / G::PX;
    const int gx = gx0 + px, gy = gy0 + py;
    if (gx >= 0 && gx < ext[0] && gy >= 0 && gy < ext[1] && gz >= 0 && gz < ext[2]) {
      if (scr) scr[rel * LAY + o] = sc * S.Yw[sl * LAY + o];
      else atomicAdd(y + gx + long(ext[0]) * (gy + long(ext[1]) * gz), sc * S.Yw[sl * LAY + o]);
    }
    S.Yw[sl * LAY + o] = 0.0;
  }
}

// ---- interpolation stages of component C (tasks numbered from 0; `t` is this thread's task) ----
// z: Z1[qz][py][px] = sum_jz Vz[qz][jz] Xw[jz][py][px]          (tasks: py, px)
template <int P, int Q, int DUAL, int E, int C>
__device__ __forceinline__ void interp_z(const CompSm<P, Q, DUAL, E, C>& S, int t) {
  using G = Geo<P, Q, DUAL, E, C>;
  constexpr int NL = P + 1, LAY = G::PY * G::PX;
  if (t >= LAY) return;
  double xv[G::NZ];
#pragma unroll
  for (int jz = 0; jz < G::NZ; ++jz) xv[jz] = S.Xw[S.slotx(jz) * LAY + t];
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double s = 0.0;
#pragma unroll
    for (int jz = 0; jz < G::NZ; ++jz) s = fma(S.Vz[qz * NL + jz], xv[jz], s);
    S.Z1[qz * G::LAYP + t] = s;
  }
}

// y: Z2[qz][ey*Q+qy][px] = sum_jy Vy[ey][qy][jy] Z1[qz][ey+jy][px]   (tasks: qz, px)
// UNI: every element of the brick has the same 1D basis table along this axis (interior
// elements of a uniform mesh): the Q x N coefficients live in registers for the whole task.
// UNI: the interior table of the axis and role comes from the kernel parameters (HodgeArgs::uni),
// so the FMAs take the coefficients as constant-bank operands: no loads and no registers.
template <int Q, int N, int NL, bool UNI, int ROLE, int AXIS>
struct Coef {
  const HodgeArgs& A;
  __device__ __forceinline__ Coef(const HodgeArgs& a) : A(a) {}
  __device__ __forceinline__ double operator()(const double* V, int e, int q, int j) const {
    return UNI ? A.uni[ROLE][AXIS][q * NL + j] : V[(e * Q + q) * NL + j];
  }
};

// (tasks: half, qz, px -- each half of the brick's elements along y is a separate task)
template <int P, int Q, int DUAL, int E, int C, bool UNI>
__device__ __forceinline__ void interp_y(const HodgeArgs& A, const CompSm<P, Q, DUAL, E, C>& S, int t) {
  using G = Geo<P, Q, DUAL, E, C>;
  constexpr int NL = P + 1, EH = E / 2;
  if (t >= 2 * Q * G::PX) return;
  const int hf = t / (Q * G::PX);
  t -= hf * Q * G::PX;
  const int px = t % G::PX, qz = t / G::PX;
  const Coef<Q, G::NY, NL, UNI, (C == 1 ? 0 : 1), 1> V(A);
  double zv[EH - 1 + G::NY];
#pragma unroll
  for (int py = 0; py < EH - 1 + G::NY; ++py) zv[py] = S.Z1[qz * G::LAYP + (hf * EH + py) * G::PX + px];
#pragma unroll
  for (int el = 0; el < EH; ++el)
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) {
      double s = 0.0;
#pragma unroll
      for (int jy = 0; jy < G::NY; ++jy) s = fma(V(S.Vy, hf * EH + el, qy, jy), zv[el + jy], s);
      S.Z2[qz * G::Z2P + ((hf * EH + el) * Q + qy) * G::PXP + px] = s;
    }
}

// x: U[qz][Y][ex*Q+qx] = sum_jx Vx[ex][qx][jx] Z2[qz][Y][ex+jx]    (tasks: qz, Y)
template <int P, int Q, int DUAL, int E, int C, bool UNI>
__device__ __forceinline__ void interp_x(const HodgeArgs& A, const CompSm<P, Q, DUAL, E, C>& S, int t, const double* Wm = nullptr,
                                         int nex = E, int ney = E) {
  // (tasks: half, qz, Y -- each half of the brick's elements along x is a separate task).  With Wm
  // (scalar W, staged in the U slots) the quadrature multiply u *= w is fused here; the
  // per-component constant of the scalar Hodge is applied when an output layer is flushed.
  using G = Geo<P, Q, DUAL, E, C>;
  constexpr int NL = P + 1, EH = E / 2;
  if (t >= 2 * Q * G::EQ) return;
  const int hf = t >= Q * G::EQ ? 1 : 0;
  t -= hf * Q * G::EQ;  // the row (qz, Y)
  const Coef<Q, G::NX, NL, UNI, (C == 0 ? 0 : 1), 0> V(A);
  double zv[EH - 1 + G::NX];
  const double* zr = S.Z2 + G::z2row(t) + hf * EH;
#pragma unroll
  for (int px = 0; px < EH - 1 + G::NX; ++px) zv[px] = zr[px];
#pragma unroll
  for (int el = 0; el < EH; ++el)
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      double s = 0.0;
#pragma unroll
      for (int jx = 0; jx < G::NX; ++jx) s = fma(V(S.Vx, hf * EH + el, qx, jx), zv[el + jx], s);
      const int ui = t * G::RSU + (hf * EH + el) * Q + qx;  // uidx(qz, Y, ex, qx), row = qz * EQ + Y
      // (W is zero at the slots of elements past the mesh edge, where s is finite: zero tables)
      if (Wm) s *= Wm[ui];
      S.U[ui] = s;
    }
}

// ---- testing stages (transposes of the above) ----
// x: Z2[qz][Y][px] = sum_{ex,qx} Vx[ex][qx][px-ex] U[qz][Y][ex*Q+qx]   (tasks: qz, Y)
template <int P, int Q, int DUAL, int E, int C, bool UNI>
__device__ __forceinline__ void test_x(const HodgeArgs& A, const CompSm<P, Q, DUAL, E, C>& S, int t) {
  using G = Geo<P, Q, DUAL, E, C>;
  constexpr int NL = P + 1;
  if (t >= Q * G::EQ) return;
  const Coef<Q, G::NX, NL, UNI, (C == 0 ? 0 : 1), 0> V(A);
  double acc[G::PX];
#pragma unroll
  for (int px = 0; px < G::PX; ++px) acc[px] = 0.0;
#pragma unroll
  for (int ex = 0; ex < E; ++ex)
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      const double u = S.U[t * G::RSU + ex * Q + qx];  // uidx(qz, Y, ex, qx), row t = qz * EQ + Y
#pragma unroll
      for (int jx = 0; jx < G::NX; ++jx) acc[ex + jx] = fma(V(S.Vx, ex, qx, jx), u, acc[ex + jx]);
    }
  double* zo = S.Z2 + G::z2row(t);
#pragma unroll
  for (int px = 0; px < G::PX; ++px) zo[px] = acc[px];
}

// y: T1[qz][py][px] = sum_{ey,qy} Vy[ey][qy][py-ey] Z2[qz][ey*Q+qy][px]   (tasks: qz, px)
template <int P, int Q, int DUAL, int E, int C, bool UNI>
__device__ __forceinline__ void test_y(const HodgeArgs& A, const CompSm<P, Q, DUAL, E, C>& S, int t) {
  using G = Geo<P, Q, DUAL, E, C>;
  constexpr int NL = P + 1;
  if (t >= Q * G::PX) return;
  const Coef<Q, G::NY, NL, UNI, (C == 1 ? 0 : 1), 1> V(A);
  const int px = t % G::PX, qz = t / G::PX;
  double acc[G::PY];
#pragma unroll
  for (int py = 0; py < G::PY; ++py) acc[py] = 0.0;
#pragma unroll
  for (int ey = 0; ey < E; ++ey)
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) {
      const double z = S.Z2[qz * G::Z2P + (ey * Q + qy) * G::PXP + px];
#pragma unroll
      for (int jy = 0; jy < G::NY; ++jy) acc[ey + jy] = fma(V(S.Vy, ey, qy, jy), z, acc[ey + jy]);
    }
#pragma unroll
  for (int py = 0; py < G::PY; ++py) S.T1[qz * G::LAYP + py * G::PX + px] = acc[py];
}

// The (py, px) columns of component C.  The same thread owns a column in both functions, which run
// in different barrier intervals next to the y stages (whose tasks leave threads idle):
// column_test (with the next layer's y interpolation): test along z of element layer ez,
//   Yw[jz][py][px] += sum_qz Vz[qz][jz] T1[qz][py][px], and flush of the completed output slot
//   (scratch or atomics to y; slot cleared).  vz: the z basis (global, [Q][NL]) of layer ez; UNIZ:
//   the layer is interior along z (its table is the parameter copy A.uni[role][2]).
template <int P, int Q, int DUAL, int E, int C, bool UNIZ>
__device__ __forceinline__ void column_test(const HodgeArgs& A, const CompSm<P, Q, DUAL, E, C>& S, int t, int gx0,
                                            int gy0, int gz_flush, const double* __restrict__ vz, double* scr,
                                            int rel, double sc) {
  using G = Geo<P, Q, DUAL, E, C>;
  constexpr int NL = P + 1, LAY = G::PY * G::PX;
  if (t >= LAY) return;
  const int px = t % G::PX, py = t / G::PX;
  const int gx = gx0 + px, gy = gy0 + py;
  const int* ext = A.ext[C];
  const bool inxy = gx >= 0 && gx < ext[0] && gy >= 0 && gy < ext[1];
  double zv[Q];
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) zv[qz] = S.T1[qz * G::LAYP + t];
#pragma unroll
  for (int jz = 0; jz < G::NZ; ++jz) {
    const int sl = S.sloty(jz);
    double acc = S.Yw[sl * LAY + t];
#pragma unroll
    for (int qz = 0; qz < Q; ++qz)
      acc = fma(UNIZ ? A.uni[C == 2 ? 0 : 1][2][qz * NL + jz] : __ldg(vz + qz * NL + jz), zv[qz], acc);
    if (jz == 0) {
      if (inxy && gz_flush >= 0 && gz_flush < ext[2]) {
        if (scr) scr[rel * LAY + t] = sc * acc;
        else atomicAdd(A.y[C] + gx + long(ext[0]) * (gy + long(ext[1]) * gz_flush), sc * acc);
      }
      S.Yw[sl * LAY + t] = 0.0;
    } else {
      S.Yw[sl * LAY + t] = acc;
    }
  }
}

// column_next (with the current layer's y testing): the top coefficient layer of the next element
// layer (global z index gz_load) into the freed window slot and the next layer's z interpolation,
// Z1[qz][py][px] = sum_jz Vz[qz][jz] Xw[jz][py][px].  vz: the z basis of the next layer.
template <int P, int Q, int DUAL, int E, int C, bool UNIZ>
__device__ __forceinline__ void column_next(const HodgeArgs& A, const CompSm<P, Q, DUAL, E, C>& S, int t, int gx0,
                                            int gy0, int gz_load, const double* __restrict__ vz) {
  using G = Geo<P, Q, DUAL, E, C>;
  constexpr int NL = P + 1, LAY = G::PY * G::PX;
  if (t >= LAY) return;
  const int px = t % G::PX, py = t / G::PX;
  const int gx = gx0 + px, gy = gy0 + py;
  const int* ext = A.ext[C];
  const bool inxy = gx >= 0 && gx < ext[0] && gy >= 0 && gy < ext[1];
  double v = 0.0;
  if (inxy && gz_load >= 0 && gz_load < ext[2]) v = __ldg(A.x[C] + gx + long(ext[0]) * (gy + long(ext[1]) * gz_load));
  S.Xw[S.slotx(0) * LAY + t] = v;
  double xv[G::NZ];
#pragma unroll
  for (int jz = 0; jz < G::NZ; ++jz) xv[jz] = (jz + 1 < G::NZ) ? S.Xw[S.slotx(jz + 1) * LAY + t] : v;
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    double s = 0.0;
#pragma unroll
    for (int jz = 0; jz < G::NZ; ++jz)
      s = fma(UNIZ ? A.uni[C == 2 ? 0 : 1][2][qz * NL + jz] : __ldg(vz + qz * NL + jz), xv[jz], s);
    S.Z1[qz * G::LAYP + t] = s;
  }
}

// run stage F for the three components, tasks of component c offset so that all threads work
#define SGM_BRICK_STAGE3(F, N0, N1, N2)                                     \
  {                                                                         \
    for (int t = threadIdx.x; t < (N0) + (N1) + (N2); t += NT) {           \
      if (t < (N0)) F<P, Q, DUAL, E, 0>(S0, t);                             \
      else if (t < (N0) + (N1)) F<P, Q, DUAL, E, 1>(S1, t - (N0));          \
      else F<P, Q, DUAL, E, 2>(S2, t - (N0) - (N1));                        \
    }                                                                       \
    __syncthreads();                                                        \
  }
// the same with the per-axis uniform-basis flags (own role of component c along the axis when
// the axis is c's own, else the other role)
#define SGM_BRICK_TASKS3U(F, AXIS, N0, N1, N2)                                                       \
  {                                                                                                  \
    const bool u0 = uni[(AXIS == 0 ? 0 : 1) * 2 + AXIS], u1 = uni[(AXIS == 1 ? 0 : 1) * 2 + AXIS],  \
               u2 = uni[1 * 2 + AXIS];                                                               \
    for (int t = threadIdx.x; t < (N0) + (N1) + (N2); t += NT) {                                    \
      if (t < (N0)) {                                                                                \
        if (u0) F<P, Q, DUAL, E, 0, true>(A, S0, t); else F<P, Q, DUAL, E, 0, false>(A, S0, t);            \
      } else if (t < (N0) + (N1)) {                                                                  \
        if (u1) F<P, Q, DUAL, E, 1, true>(A, S1, t - (N0)); else F<P, Q, DUAL, E, 1, false>(A, S1, t - (N0)); \
      } else {                                                                                       \
        if (u2) F<P, Q, DUAL, E, 2, true>(A, S2, t - (N0) - (N1));                                      \
        else F<P, Q, DUAL, E, 2, false>(A, S2, t - (N0) - (N1));                                        \
      }                                                                                              \
    }                                                                                                \
  }
#define SGM_BRICK_STAGE3U(F, AXIS, N0, N1, N2) \
  SGM_BRICK_TASKS3U(F, AXIS, N0, N1, N2)       \
  __syncthreads();

// doubles of one work item's output patches in the scratch (all three components, zchunk + NZ - 1
// layers each)
template <int P, int Q, int DUAL, int E>
__host__ __device__ constexpr size_t item_stride(int zchunk) {
  using G0 = Geo<P, Q, DUAL, E, 0>;
  using G1 = Geo<P, Q, DUAL, E, 1>;
  using G2 = Geo<P, Q, DUAL, E, 2>;
  return size_t(zchunk + G0::NZ - 1) * G0::PY * G0::PX + size_t(zchunk + G1::NZ - 1) * G1::PY * G1::PX +
         size_t(zchunk + G2::NZ - 1) * G2::PY * G2::PX;
}

// Second pass of the deterministic accumulation: y_c[g] = sum over the work items whose patches
// contain g (at most 2 bricks per axis x 2 z chunks), in the fixed order (chunk, brick y, brick x).
// One thread per output entry; the brick / chunk candidates of an index are the two around
// g / E (patch origins are the first functions of the bricks' first elements).
template <int P, int Q, int DUAL, int E, int C>
__device__ __forceinline__ double gather_one(const HodgeArgs& A, int zchunk, int gx, int gy, int gz) {
  using G = Geo<P, Q, DUAL, E, C>;
  const int nx = A.nel[0], ny = A.nel[1], nz = A.nel[2];
  const int bxn = (nx + E - 1) / E, byn = (ny + E - 1) / E, bzn = (nz + zchunk - 1) / zchunk;
  const int rx = C == 0 ? 0 : 1, ry = C == 1 ? 0 : 1, rz = C == 2 ? 0 : 1;
  const size_t stride = item_stride<P, Q, DUAL, E>(zchunk);
  const size_t coff = C == 0 ? 0
                    : (C == 1 ? size_t(zchunk + Geo<P, Q, DUAL, E, 0>::NZ - 1) * Geo<P, Q, DUAL, E, 0>::PY * Geo<P, Q, DUAL, E, 0>::PX
                              : size_t(zchunk + Geo<P, Q, DUAL, E, 0>::NZ - 1) * Geo<P, Q, DUAL, E, 0>::PY * Geo<P, Q, DUAL, E, 0>::PX +
                                size_t(zchunk + Geo<P, Q, DUAL, E, 1>::NZ - 1) * Geo<P, Q, DUAL, E, 1>::PY * Geo<P, Q, DUAL, E, 1>::PX);
  // the (at most two) bricks per axis and chunks along z containing the index, with the index's
  // position in their patches, found once (patch origins are monotone in the brick index)
  int bxs[2], pxs[2], nbx = 0;
  for (int bx = max(0, gx / E - 2); bx <= min(bxn - 1, gx / E + 1) && nbx < 2; ++bx) {
    const int px = gx - first_of(A, 0, rx, bx * E);
    if (px >= 0 && px < G::PX) bxs[nbx] = bx, pxs[nbx++] = px;
  }
  int bys[2], pys[2], nby = 0;
  for (int by = max(0, gy / E - 2); by <= min(byn - 1, gy / E + 1) && nby < 2; ++by) {
    const int py = gy - first_of(A, 1, ry, by * E);
    if (py >= 0 && py < G::PY) bys[nby] = by, pys[nby++] = py;
  }
  double s = 0.0;
  for (int iz = max(0, gz / zchunk - 2); iz <= min(bzn - 1, gz / zchunk + 1); ++iz) {
    const int ez0 = iz * zchunk, ez1 = min(nz, ez0 + zchunk);
    const int rel = gz - first_of(A, 2, rz, ez0);
    if (rel < 0 || gz > first_of(A, 2, rz, ez1 - 1) + G::NZ - 1) continue;
    for (int j = 0; j < nby; ++j)
      for (int i = 0; i < nbx; ++i) {
        const long item = (long(iz) * byn + bys[j]) * bxn + bxs[i];
        s += __ldg(A.scratch + item * stride + coff + (size_t(rel) * G::PY + pys[j]) * G::PX + pxs[i]);
      }
  }
  return s;
}

template <int P, int Q, int DUAL, int E>
__global__ void __launch_bounds__(256) hodge_gather_kernel(const __grid_constant__ HodgeArgs A, int zchunk) {
  const long n0 = long(A.ext[0][0]) * A.ext[0][1] * A.ext[0][2];
  const long n1 = long(A.ext[1][0]) * A.ext[1][1] * A.ext[1][2];
  const long n2 = long(A.ext[2][0]) * A.ext[2][1] * A.ext[2][2];
  for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < n0 + n1 + n2; i += long(gridDim.x) * blockDim.x) {
    const int c = i < n0 ? 0 : (i < n0 + n1 ? 1 : 2);
    const long k = i - (c == 0 ? 0 : (c == 1 ? n0 : n0 + n1));
    // (a component has fewer than 2^31 entries: 32-bit divisions)
    const unsigned X = unsigned(A.ext[c][0]), Y = unsigned(A.ext[c][1]), ku = unsigned(k), row = ku / X;
    const int gx = int(ku - row * X), gz = int(row / Y), gy = int(row - unsigned(gz) * Y);
    double v;
    if (c == 0) v = gather_one<P, Q, DUAL, E, 0>(A, zchunk, gx, gy, gz);
    else if (c == 1) v = gather_one<P, Q, DUAL, E, 1>(A, zchunk, gx, gy, gz);
    else v = gather_one<P, Q, DUAL, E, 2>(A, zchunk, gx, gy, gz);
    A.y[c][k] = v;
  }
}

// threads per CTA.  At p = 4 the x stages have 300 (testing) and 600 (interpolation) tasks: one and
// two rounds of 320 threads instead of two and three of 256, but 320 threads leave 96 registers per
// thread (spills) and measured slower (C4 apply 1.12 -> 1.19 ms), so SGM_BRICK_NT4 stays 256
__host__ __device__ constexpr int brick_threads(int p) { return p == 4 ? SGM_BRICK_NT4 : 256; }

template <int P, int Q, int DUAL, bool FULL, int E, bool OTF>
__global__ void __launch_bounds__(brick_threads(P), 2) hodge_brick_kernel(const __grid_constant__ HodgeArgs A, int zchunk) {
  static_assert(!OTF || FULL, "on-the-fly geometry: general maps only");
  using L = Layout<P, Q, DUAL, E>;
  using G0 = Geo<P, Q, DUAL, E, 0>;
  using G1 = Geo<P, Q, DUAL, E, 1>;
  using G2 = Geo<P, Q, DUAL, E, 2>;
  constexpr int NL = P + 1, EQ = E * Q, NT = brick_threads(P);
  extern __shared__ __align__(16) double sm[];
  __shared__ unsigned long long wbar;  // completion of the staged W (one phase per element layer)
  unsigned wphase = 0;
  if (threadIdx.x == 0) pipe::mbar_init(&wbar, 1);
  pipe::fence_proxy_async_smem();
  __syncthreads();
  CompSm<P, Q, DUAL, E, 0> S0(sm);
  CompSm<P, Q, DUAL, E, 1> S1(sm);
  CompSm<P, Q, DUAL, E, 2> S2(sm);
  const CompSm<P, Q, DUAL, E, 1> S2x(S2);  // component 2 through component 1's x-stage code
  double* tab = sm + L::TAB;
  double* Wsm = sm + L::WB;
  // OTF: map partial sums and the brick's x / y map tables (see Layout)
  double* MAs = Wsm + L::template wdoubles<FULL, OTF>();
  double* MBs = MAs + (OTF ? L::MA : 0);
  double* MTs = MBs + (OTF ? L::MB : 0);
  constexpr int PM = L::PM;
  const int nx = A.nel[0], ny = A.nel[1], nz = A.nel[2];
  const int bx = (nx + E - 1) / E, by = (ny + E - 1) / E, bzn = (nz + zchunk - 1) / zchunk;
  const long items = long(bx) * by * bzn;
  for (long it = blockIdx.x; it < items; it += gridDim.x) {
    Brick B;
    {
      const int ib = int(it % (long(bx) * by)), iz = int(it / (long(bx) * by));
      B.ex0 = (ib % bx) * E;
      B.ey0 = (ib / bx) * E;
      B.nex = min(E, nx - B.ex0);
      B.ney = min(E, ny - B.ey0);
      B.ez0 = iz * zchunk;
      B.ez1 = min(nz, B.ez0 + zchunk);
    }
    // brick x / y basis tables [role][axis][e][q][k] (elements past the mesh edge: zeros)
    for (int o = threadIdx.x; o < 2 * 2 * L::VXY; o += NT) {
      const int role = o / (2 * L::VXY), r = o % (2 * L::VXY), axis = r / L::VXY, i = r % L::VXY;
      const int e = i / (Q * NL), rem = i % (Q * NL);
      const int eg = (axis == 0 ? B.ex0 : B.ey0) + e;
      const int ng = axis == 0 ? nx : ny;
      tab[o] = (eg < ng) ? __ldg(A.basis + A.basis_off[axis][role] + size_t(eg) * Q * NL + rem) : 0.0;
    }
    if (OTF) {
      // map tables of the brick's x / y elements [axis][s][e][q][k] (zeros past the mesh edge)
      for (int o = threadIdx.x; o < L::MT; o += NT) {
        const int axis = o / (2 * E * Q * NL), r = o % (2 * E * Q * NL), sv = r / (E * Q * NL), i = r % (E * Q * NL);
        const int e = i / (Q * NL), rem = i % (Q * NL);
        const int eg = (axis == 0 ? B.ex0 : B.ey0) + e;
        const int ng = axis == 0 ? nx : ny;
        MTs[o] = (eg < ng) ? __ldg(A.geo_tab + A.geo_tab_off[axis][sv] + size_t(eg) * Q * NL + rem) : 0.0;
      }
    }
    __syncthreads();
    // uni[role*2 + axis]: the brick is full and all its elements lie in the axis' interior range, whose
    // element tables equal the parameter copy A.uni bit for bit (ranges found on the host)
    bool uni[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int ax = r % 2, role = r / 2, e0 = ax == 0 ? B.ex0 : B.ey0;
      uni[r] = (ax == 0 ? B.nex : B.ney) == E && e0 >= A.uni_lo[ax][role] && e0 + E <= A.uni_hi[ax][role];
    }
    auto uniz = [&](int c, int ez) {
      const int role = c == 2 ? 0 : 1;
      // (the parameter-bank column variants pay at p <= 3: C3 0.1255 -> 0.1235 ms per apply; at p = 4
      // their extra code costs more than the loads they save: C4 1.129 -> 1.156 ms)
      return P <= 3 && ez >= A.uni_lo[2][role] && ez < A.uni_hi[2][role];
    };
    // deterministic accumulation: this item's output patches go to the scratch (summed in a fixed
    // order by hodge_gather_kernel); layer rel of component c at scr_c + rel * PY_c * PX_c
    double *scr0 = nullptr, *scr1 = nullptr, *scr2 = nullptr;
    if (A.scratch) {
      double* b = A.scratch + size_t(it) * item_stride<P, Q, DUAL, E>(zchunk);
      scr0 = b;
      scr1 = scr0 + size_t(zchunk + G0::NZ - 1) * G0::PY * G0::PX;
      scr2 = scr1 + size_t(zchunk + G1::NZ - 1) * G1::PY * G1::PX;
    }
    const int fx[3] = {first_of(A, 0, 0, B.ex0), first_of(A, 0, 1, B.ex0), 0};  // own / other
    const int fy[3] = {first_of(A, 1, 0, B.ey0), first_of(A, 1, 1, B.ey0), 0};
    // patch origins per component: own role along its own axis
    const int gx0[3] = {fx[0], fx[1], fx[1]}, gy0[3] = {fy[1], fy[0], fy[1]};
    auto zfirst = [&](int c, int ez) { return first_of(A, 2, c == 2 ? 0 : 1, ez); };
    // zero output windows, load the NZ coefficient layers and z bases of the first element layer
    S0.xbase = S1.xbase = S2.xbase = 0;
    S0.ybase = S1.ybase = S2.ybase = 0;
    for (int o = threadIdx.x; o < G0::WIN; o += NT) S0.Yw[o] = 0.0;
    for (int o = threadIdx.x; o < G1::WIN; o += NT) S1.Yw[o] = 0.0;
    for (int o = threadIdx.x; o < G2::WIN; o += NT) S2.Yw[o] = 0.0;
    for (int jz = 0; jz < G0::NZ; ++jz) load_layer<P, Q, DUAL, E, 0>(A, S0, gx0[0], gy0[0], zfirst(0, B.ez0) + jz, jz);
    for (int jz = 0; jz < G1::NZ; ++jz) load_layer<P, Q, DUAL, E, 1>(A, S1, gx0[1], gy0[1], zfirst(1, B.ez0) + jz, jz);
    for (int jz = 0; jz < G2::NZ; ++jz) load_layer<P, Q, DUAL, E, 2>(A, S2, gx0[2], gy0[2], zfirst(2, B.ez0) + jz, jz);
    auto load_vz = [&](int ez) {
      for (int o = threadIdx.x; o < 2 * L::VZ; o += NT) {
        const int role = o / L::VZ;
        tab[4 * L::VXY + o] = __ldg(A.basis + A.basis_off[2][role] + size_t(ez) * Q * NL + (o % L::VZ));
      }
    };
    load_vz(B.ez0);
    // W of element layer ez -> Wsm: one bulk copy (TMA engine) of the brick's chunk, completion on
    // wbar.  Called after the block barrier that follows the last read of the previous layer's W.
    auto stage_w = [&](int ez) {
      constexpr unsigned bytes = unsigned(L::template wdoubles<FULL, OTF>()) * 8u;
      if (threadIdx.x == 0) {
        const long chunk = (long(ez) * by + B.ey0 / E) * bx + B.ex0 / E;
        pipe::fence_proxy_async_smem();
        pipe::mbar_arrive_expect_tx(&wbar, bytes);
        pipe::bulk_g2s(Wsm, A.W + chunk * (bytes / 8u), bytes, &wbar);
      }
    };
    stage_w(B.ez0);
    __syncthreads();
    SGM_BRICK_STAGE3(interp_z, G0::PY * G0::PX, G1::PY * G1::PX, G2::PY * G2::PX)
    auto vzp = [&](int c, int ez) {
      return A.basis + A.basis_off[2][c == 2 ? 0 : 1] + size_t(ez) * Q * NL;
    };
    // output scale: the scalar Hodge's per-component constant (the full W carries everything)
    const double osc[3] = {FULL ? 1.0 : A.scale[0], FULL ? 1.0 : A.scale[1], FULL ? 1.0 : A.scale[2]};
    // the columns' tasks start at thread `shift` (after the y stage's tasks of the same interval)
    constexpr int NC0 = G0::PY * G0::PX, NC1 = G1::PY * G1::PX, NC2 = G2::PY * G2::PX;
    auto columns_test = [&](int ezl, int shift) {
      for (int t = (threadIdx.x + NT - shift % NT) % NT; t < NC0 + NC1 + NC2; t += NT) {
#define SGM_COLT(C, S, T, SCR)                                                                              \
  if (uniz(C, ezl))                                                                                          \
    column_test<P, Q, DUAL, E, C, true>(A, S, T, gx0[C], gy0[C], zfirst(C, ezl), vzp(C, ezl), SCR,           \
                                        zfirst(C, ezl) - zfirst(C, B.ez0), osc[C]);                          \
  else                                                                                                       \
    column_test<P, Q, DUAL, E, C, false>(A, S, T, gx0[C], gy0[C], zfirst(C, ezl), vzp(C, ezl), SCR,          \
                                         zfirst(C, ezl) - zfirst(C, B.ez0), osc[C]);
        if (t < NC0) {
          SGM_COLT(0, S0, t, scr0)
        } else if (t < NC0 + NC1) {
          SGM_COLT(1, S1, t - NC0, scr1)
        } else {
          SGM_COLT(2, S2, t - NC0 - NC1, scr2)
        }
#undef SGM_COLT
      }
      S0.ybase = S0.sloty(1);
      S1.ybase = S1.sloty(1);
      S2.ybase = S2.sloty(1);
    };
    auto columns_next = [&](int ezn, int shift) {
      for (int t = (threadIdx.x + NT - shift % NT) % NT; t < NC0 + NC1 + NC2; t += NT) {
#define SGM_COLN(C, S, T, NZC)                                                                             \
  if (uniz(C, ezn))                                                                                         \
    column_next<P, Q, DUAL, E, C, true>(A, S, T, gx0[C], gy0[C], zfirst(C, ezn) + NZC - 1, vzp(C, ezn));   \
  else                                                                                                      \
    column_next<P, Q, DUAL, E, C, false>(A, S, T, gx0[C], gy0[C], zfirst(C, ezn) + NZC - 1, vzp(C, ezn));
        if (t < NC0) {
          SGM_COLN(0, S0, t, G0::NZ)
        } else if (t < NC0 + NC1) {
          SGM_COLN(1, S1, t - NC0, G1::NZ)
        } else {
          SGM_COLN(2, S2, t - NC0 - NC1, G2::NZ)
        }
#undef SGM_COLN
      }
      S0.xbase = S0.slotx(1);
      S1.xbase = S1.slotx(1);
      S2.xbase = S2.slotx(1);
    };
    for (int ez = B.ez0; ez < B.ez1; ++ez) {
      if (OTF) {
        // map, z: A[r][s][qz][py][px] = sum_k Tz_s[qz][k] ctrl_r[ez + k][ey0 + py][ex0 + px]
        // (S_p: element e's functions are e .. e + p; control points past the grid edge: zero)
        const int NXm = nx + P, NYm = ny + P;
        const double* tz0 = A.geo_tab + A.geo_tab_off[2][0] + size_t(ez) * Q * NL;
        const double* tz1 = A.geo_tab + A.geo_tab_off[2][1] + size_t(ez) * Q * NL;
        for (int t = threadIdx.x; t < 3 * PM * PM; t += NT) {
          const int r = t / (PM * PM), o = t - r * PM * PM, py = o / PM, px = o - py * PM;
          const int gx = B.ex0 + px, gy = B.ey0 + py;
          double c[NL];
#pragma unroll
          for (int k = 0; k < NL; ++k)
            c[k] = (gx < NXm && gy < NYm) ? __ldg(A.geo_ctrl[r] + (size_t(ez + k) * NYm + gy) * NXm + gx) : 0.0;
#pragma unroll
          for (int qz = 0; qz < Q; ++qz) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int k = 0; k < NL; ++k) {
              s0 = fma(__ldg(tz0 + qz * NL + k), c[k], s0);
              s1 = fma(__ldg(tz1 + qz * NL + k), c[k], s1);
            }
            MAs[((r * 2 + 0) * Q + qz) * PM * PM + o] = s0;
            MAs[((r * 2 + 1) * Q + qz) * PM * PM + o] = s1;
          }
        }
      }
      // y interpolation of this layer; on the threads it leaves idle, the previous layer's z testing
      // and flush (T1 of the previous layer is not written again before this layer's y testing)
      SGM_BRICK_TASKS3U(interp_y, 1, 2 * Q * G0::PX, 2 * Q * G1::PX, 2 * Q * G2::PX)
      if (ez > B.ez0) columns_test(ez - 1, 2 * Q * (G0::PX + G1::PX + G2::PX));
      // W of this layer (staged by cp.async since the previous layer) must be in shared memory
      // before the x interpolation (scalar W is multiplied there) or the quadrature stage (full W)
      pipe::mbar_wait(&wbar, wphase);
      wphase ^= 1u;
      __syncthreads();
      {
        const bool u0 = uni[0 * 2 + 0], u1 = uni[1 * 2 + 0];  // (components 1 and 2: the other role along x)
        const double* Wm = FULL ? nullptr : Wsm;
        for (int t = threadIdx.x; t < 3 * 2 * Q * EQ; t += NT) {
          const int c = t < 2 * Q * EQ ? 0 : (t < 4 * Q * EQ ? 1 : 2), tt = t - c * (2 * Q * EQ);
          if (c == 0) {
            if (u0) interp_x<P, Q, DUAL, E, 0, true>(A, S0, tt, Wm, B.nex, B.ney);
            else interp_x<P, Q, DUAL, E, 0, false>(A, S0, tt, Wm, B.nex, B.ney);
          } else {
            const CompSm<P, Q, DUAL, E, 1> Sx = c == 1 ? S1 : S2x;
            if (u1) interp_x<P, Q, DUAL, E, 1, true>(A, Sx, tt, Wm, B.nex, B.ney);
            else interp_x<P, Q, DUAL, E, 1, false>(A, Sx, tt, Wm, B.nex, B.ney);
          }
        }
        if (OTF) {
          // map, y: B[r][m][qz][ey*Q+qy][px] = sum_j Ty_sy[ey][qy][j] A[r][sz][qz][ey + j][px],
          // m = 0: (sz, sy) = (val, val), 1: (val, der), 2: (der, val)
          for (int t = threadIdx.x; t < 9 * Q * PM; t += NT) {
            const int rm = t / (Q * PM), o = t - rm * Q * PM, qz = o / PM, px = o - qz * PM;
            const int r = rm / 3, m = rm - r * 3, sz = m == 2 ? 1 : 0, sy = m == 1 ? 1 : 0;
            const double* a = MAs + ((r * 2 + sz) * Q + qz) * PM * PM + px;
            const double* ty = MTs + (1 * 2 + sy) * E * Q * NL;
            double zv[PM];
#pragma unroll
            for (int py = 0; py < PM; ++py) zv[py] = a[py * PM];
            double* b = MBs + (rm * Q + qz) * EQ * PM + px;
#pragma unroll
            for (int ey = 0; ey < E; ++ey)
#pragma unroll
              for (int qy = 0; qy < Q; ++qy) {
                double v = 0.0;
#pragma unroll
                for (int j = 0; j < NL; ++j) v = fma(ty[(ey * Q + qy) * NL + j], zv[ey + j], v);
                b[(ey * Q + qy) * PM] = v;
              }
          }
        }
        __syncthreads();
      }
      if (FULL) {
        // quadrature points: v_c = sum_c' W_cc' u_c' (the 3 x 3 W couples the components)
        {
          // consecutive threads take consecutive points (U slots but for the pad slot of each row)
          for (int pt = threadIdx.x; pt < Q * EQ * EQ; pt += NT) {
            const int X = pt % EQ, row = pt / EQ, Yq = row % EQ;
            const int i = row * (EQ + 1) + X;  // the point's U slot
            const int ex = X / Q, ey = Yq / Q;
            const bool live = ex < B.nex && ey < B.ney;
            const double u0 = S0.U[i], u1 = S1.U[i], u2 = S2.U[i];
            double wxx, wyy, wzz, wxy, wxz, wyz;
            if (OTF) {
              // DF at the point from the map's partial sums, then the 2-form pull-back weights
              // W = (w_q / material) / det DF * DF^T DF, as the host builds them
              wxx = wyy = wzz = wxy = wxz = wyz = 0.0;
              if (live) {
                const int qzp = row / EQ, qy = Yq - ey * Q, qx = X - ex * Q;
                const double* tv = MTs + (0 * 2 + 0) * E * Q * NL + (ex * Q + qx) * NL;  // x values
                const double* td = MTs + (0 * 2 + 1) * E * Q * NL + (ex * Q + qx) * NL;  // x derivatives
                double D[9];
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                  for (int m = 0; m < 3; ++m) {
                    const double* b = MBs + ((r * 3 + m) * Q + qzp) * EQ * PM + (ey * Q + qy) * PM + ex;
                    const double* tx = m == 0 ? td : tv;
                    double v = 0.0;
#pragma unroll
                    for (int k = 0; k < NL; ++k) v = fma(tx[k], b[k], v);
                    D[r * 3 + (m == 0 ? 0 : (m == 1 ? 1 : 2))] = v;  // dF_r / dx^_j
                  }
                const double det = D[0] * (D[4] * D[8] - D[5] * D[7]) - D[1] * (D[3] * D[8] - D[5] * D[6]) +
                                   D[2] * (D[3] * D[7] - D[4] * D[6]);
                const double g = Wsm[i] / det;
                auto mm = [&](int a, int c) { return D[0 * 3 + a] * D[0 * 3 + c] + D[1 * 3 + a] * D[1 * 3 + c] + D[2 * 3 + a] * D[2 * 3 + c]; };
                wxx = g * mm(0, 0);
                wyy = g * mm(1, 1);
                wzz = g * mm(2, 2);
                wxy = g * mm(0, 1);
                wxz = g * mm(0, 2);
                wyz = g * mm(1, 2);
              }
            } else {
              // (zero at the slots of elements past the mesh edge)
              const double* w = Wsm + i;
              wxx = w[0 * L::NU];
              wyy = w[1 * L::NU];
              wzz = w[2 * L::NU];
              wxy = w[3 * L::NU];
              wxz = w[4 * L::NU];
              wyz = w[5 * L::NU];
            }
            S0.U[i] = wxx * u0 + wxy * u1 + wxz * u2;
            S1.U[i] = wxy * u0 + wyy * u1 + wyz * u2;
            S2.U[i] = wxz * u0 + wyz * u1 + wzz * u2;
          }
        }
        __syncthreads();
      }
      if (ez + 1 < B.ez1) stage_w(ez + 1);
      {
        const bool u0 = uni[0 * 2 + 0], u1 = uni[1 * 2 + 0];
        for (int t = threadIdx.x; t < 3 * Q * EQ; t += NT) {
          if (t < Q * EQ) {
            if (u0) test_x<P, Q, DUAL, E, 0, true>(A, S0, t);
            else test_x<P, Q, DUAL, E, 0, false>(A, S0, t);
          } else {
            const bool second = t >= 2 * Q * EQ;
            const CompSm<P, Q, DUAL, E, 1> Sx = second ? S2x : S1;
            const int tt = t - (second ? 2 : 1) * Q * EQ;
            if (u1) test_x<P, Q, DUAL, E, 1, true>(A, Sx, tt);
            else test_x<P, Q, DUAL, E, 1, false>(A, Sx, tt);
          }
        }
        __syncthreads();
      }
      // y testing of this layer; on the threads it leaves idle, the next layer's top coefficient
      // layer and z interpolation (Z1 was last read by this layer's y interpolation)
      SGM_BRICK_TASKS3U(test_y, 1, Q * G0::PX, Q * G1::PX, Q * G2::PX)
      if (ez + 1 < B.ez1) columns_next(ez + 1, Q * (G0::PX + G1::PX + G2::PX));
      __syncthreads();
    }
    // z testing and flush of the last element layer (columns and flush_layer map threads differently)
    columns_test(B.ez1 - 1, 0);
    __syncthreads();
    // the remaining NZ-1 output layers of the last element layer (layer jz now sits in slot jz-1)
    for (int jz = 1; jz < G0::NZ; ++jz)
      flush_layer<P, Q, DUAL, E, 0>(A, S0, gx0[0], gy0[0], zfirst(0, B.ez1 - 1) + jz, S0.sloty(jz - 1), scr0,
                                    zfirst(0, B.ez1 - 1) + jz - zfirst(0, B.ez0), osc[0]);
    for (int jz = 1; jz < G1::NZ; ++jz)
      flush_layer<P, Q, DUAL, E, 1>(A, S1, gx0[1], gy0[1], zfirst(1, B.ez1 - 1) + jz, S1.sloty(jz - 1), scr1,
                                    zfirst(1, B.ez1 - 1) + jz - zfirst(1, B.ez0), osc[1]);
    for (int jz = 1; jz < G2::NZ; ++jz)
      flush_layer<P, Q, DUAL, E, 2>(A, S2, gx0[2], gy0[2], zfirst(2, B.ez1 - 1) + jz, S2.sloty(jz - 1), scr2,
                                    zfirst(2, B.ez1 - 1) + jz - zfirst(2, B.ez0), osc[2]);
    __syncthreads();
  }
}

#undef SGM_BRICK_STAGE3
#undef SGM_BRICK_STAGE3U

}  // namespace brick
}  // namespace sgm
