// Register-segment line sweeps with a partitioned (SPIKE-type) banded LU solve.
//
// One CTA owns 32 lines of one component along one axis; warp s owns segment s (rows
// [s*SEG, s*SEG+SEG)) of all 32 lines, lane j owns line j.  The SEG values of a line segment live
// in registers.  Per segment:
//   1. load (strided axes: straight from global, the 32 lanes touch 32 consecutive x;
//      x axis: through a shared-memory slab so global traffic stays coalesced), with the
//      Ampere/Faraday update fused into the load when this is the first pass of a half step;
//   2. banded mat-vec y = A x (separable Hodge Gram or pairing factor), halo of P values;
//   3. forward substitution with zero history (local), exchange the m = P-1 tail values through
//      shared memory, rebuild the true history from the "spike" table F, correct;
//   4. backward substitution with zero future (local), exchange heads, correct with spikes B;
//   5. scale and store.
// The result equals the sequential no-pivot LU solve up to rounding (SPIKE is exact algebra).
//
// Table row r (RS = 6P-2 doubles): [band(2P+1) | lo(m) | upn(m) | dinv | F(m) | B(m)] with
// band[q+P] = A[r][r+q], lo[k-1] = L_{r,r-k}, upn[k-1] = U_{r,r+k}/U_rr, dinv = 1/U_rr,
// F[j-1] = d z_r / d z_{r0-j} (segment start r0), B[j-1] = d u_r / d u_{r1+j} (segment end r1).
#pragma once

#include "kernels.cuh"

namespace sgm {

template <int P>
struct RowLayout {
  static constexpr int M = P - 1;
  static constexpr int RS = 6 * P - 2;
  static constexpr int BAND = 0;
  static constexpr int LO = 2 * P + 1;
  static constexpr int UP = 2 * P + 1 + M;
  static constexpr int DINV = 2 * P + 1 + 2 * M;
  static constexpr int F = 2 * P + 2 + 2 * M;
  static constexpr int B = 2 * P + 2 + 3 * M;
};

}  // namespace sgm
