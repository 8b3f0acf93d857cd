// Line-operator table layout of the partitioned (SPIKE-type) banded sweeps.
//
// One 1D line operator (one axis, one of the ops of sgm_internal.h) is a table of rows; row r
// holds everything the sweep needs at line element r, grouped by the phase that reads it and
// padded so every group starts on a 16-byte boundary (double2 loads from shared memory):
//   BAND [2P+2] : band[q+P] = B[r][r+q], q = -P..P   (banded mat-vec: Hodge Gram or pairing factor)
//   LO   [LW]   : lo[k-1] = L_{r,r-k}, k = 1..M      (no-pivot banded LU of A, unit lower part)
//   F    [LW]   : F[j-1] = d z_r / d z_{r0-j}        (forward spike, segment start r0)
//   UP   [UW]   : dinv = 1/U_rr, then upn[k-1] = U_{r,r+k}/U_rr, k = 1..M
//   B    [LW]   : B[j-1] = d u_r / d u_{r1+j}        (backward spike, segment end r1)
// M = P-1 (half-bandwidth of the pairing factors), LW = M rounded up to even, UW = M+1 rounded
// up to even.  Segments are SEG rows long; spikes are exact (SPIKE is exact algebra), so the
// partitioned solve equals the sequential substitution up to rounding.
#pragma once

namespace sgm {

#if defined(__CUDACC__)
#define SGM_HD __host__ __device__
#else
#define SGM_HD
#endif

template <int P>
struct RowLayout {
  static constexpr int M = P - 1;
  static constexpr int LW = (M + 1) & ~1;
  static constexpr int UW = (M + 2) & ~1;
  static constexpr int BAND = 0;
  static constexpr int LO = 2 * P + 2;
  static constexpr int F = LO + LW;
  static constexpr int UP = F + LW;       // dinv at UP, upn[k-1] at UP + k
  static constexpr int B = UP + UW;
  static constexpr int RS = B + LW;
};

// runtime mirror for host code
struct RowLayoutRT {
  int M, LW, UW, BAND, LO, F, UP, B, RS;
  SGM_HD explicit RowLayoutRT(int P) {
    M = P - 1;
    LW = (M + 1) & ~1;
    UW = (M + 2) & ~1;
    BAND = 0;
    LO = 2 * P + 2;
    F = LO + LW;
    UP = F + LW;
    B = UP + UW;
    RS = B + LW;
  }
};

}  // namespace sgm
