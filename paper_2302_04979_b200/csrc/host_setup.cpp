// Host-side plan setup: knots, Gauss rules, univariate bases, 1D pairing/Gram matrices,
// no-pivot banded LU, geometry Jacobians and Hodge weights.  (Table 1 "setup" rows,
// O(p^3 n) 1D assembly, O(p^2 n) factorisation; mass weights O(n^3 p^3).)
// Nothing here runs per time step.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"
#include "sgm_internal.h"
#include "seg_sweep.cuh"

namespace sgm {

namespace {

// p-open uniform knot vector with n elements: p+1 zeros, k/n, p+1 ones.
std::vector<double> open_knots(int p, int n) {
  std::vector<double> U;
  for (int i = 0; i <= p; ++i) U.push_back(0.0);
  for (int k = 1; k < n; ++k) U.push_back(double(k) / n);
  for (int i = 0; i <= p; ++i) U.push_back(1.0);
  return U;
}

// Values of the q+1 B-splines of degree q that are non-zero on knot span s at x
// (the standard triangular recurrence of de Boor / Cox).
void basis_funs(const double* U, int s, double x, int q, double* N) {
  double left[16], right[16];
  N[0] = 1.0;
  for (int j = 1; j <= q; ++j) {
    left[j] = x - U[s + 1 - j];
    right[j] = U[s + j] - x;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      double temp = N[r] / (right[r + 1] + left[j - r]);
      N[r] = saved + right[r + 1] * temp;
      saved = left[j - r] * temp;
    }
    N[j] = saved;
  }
}

// First derivatives of the q+1 degree-q B-splines non-zero on span s at x.
void basis_ders(const double* U, int s, double x, int q, double* dN) {
  if (q == 0) { dN[0] = 0.0; return; }
  double Nm[16];
  basis_funs(U, s, x, q - 1, Nm);  // B_{s-q+1 .. s, q-1}
  for (int k = 0; k <= q; ++k) {
    int i = s - q + k;
    double v = 0.0;
    // B_{i,q-1} is Nm[k-1] when i in [s-q+1, s]
    if (k >= 1) {
      double den = U[i + q] - U[i];
      if (den > 0) v += q / den * Nm[k - 1];
    }
    if (k <= q - 1) {
      double den = U[i + q + 1] - U[i + 1];
      if (den > 0) v -= q / den * Nm[k];
    }
    dN[k] = v;
  }
}

// Gauss-Legendre nodes/weights on [-1,1] by Newton iteration on P_Q.
void gauss_legendre(int Q, std::vector<double>& x, std::vector<double>& w) {
  x.assign(Q, 0.0);
  w.assign(Q, 0.0);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < Q; ++i) {
    double z = std::cos(pi * (i + 0.75) / (Q + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int k = 1; k <= Q; ++k) {
        double p2 = p1;
        p1 = p0;
        p0 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p2) / k;
      }
      dp = Q * (z * p0 - p1) / (z * z - 1.0);
      double dz = p0 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    // recompute derivative at the converged node
    double p0 = 1.0, p1 = 0.0;
    for (int k = 1; k <= Q; ++k) {
      double p2 = p1;
      p1 = p0;
      p0 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p2) / k;
    }
    dp = Q * (z * p0 - p1) / (z * z - 1.0);
    x[Q - 1 - i] = z;   // ascending
    w[Q - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

}  // namespace

// Per-element local values of one univariate space at the Q Gauss points of each element.
// space: 0 = Sp (primal S_p B-splines, trimmed), 1 = Sp1 (primal S_{p-1}(Xi') CS),
//        2 = Dp1 (dual S_{p-1}(Xi') B-splines), 3 = Dp2 (dual S_{p-2}(Xi'') CS).
// vals[(e*Q + q)*(p+1) + k] is the value of local function k (global index first[e] + k)
// on element e; local functions beyond the space's degree+1 have value 0.  For Sp, the
// global index is the trimmed index (may be -1 or a for the removed end functions: value 0).
void basis_values_1d(int p, int n, int Q, int space, std::vector<double>& vals, std::vector<int>& first) {
  std::vector<double> U = open_knots(p, n);
  std::vector<double> gx, gw;
  gauss_legendre(Q, gx, gw);
  const int nl = p + 1;
  vals.assign(size_t(n) * Q * nl, 0.0);
  first.assign(n, 0);
  const double* U0 = U.data();
  const double* U1 = U.data() + 1;  // Xi'
  const double* U2 = U.data() + 2;  // Xi''
  const int a = n + p - 2;
  for (int e = 0; e < n; ++e) {
    double xa = double(e) / n, xb = double(e + 1) / n;
    for (int q = 0; q < Q; ++q) {
      double x = xa + (gx[q] + 1.0) * 0.5 * (xb - xa);
      double N[16];
      double* out = &vals[(size_t(e) * Q + q) * nl];
      if (space == 0) {
        basis_funs(U0, p + e, x, p, N);  // globals e .. e+p of S_p
        first[e] = e - 1;                 // trimmed index
        for (int k = 0; k <= p; ++k) {
          int t = e - 1 + k;
          out[k] = (t >= 0 && t < a) ? N[k] : 0.0;
        }
      } else if (space == 1 || space == 2) {
        basis_funs(U1, p - 1 + e, x, p - 1, N);  // globals e .. e+p-1
        first[e] = e;
        for (int k = 0; k < p; ++k) {
          int i = e + k;
          double sc = (space == 1) ? p / (U1[i + p] - U1[i]) : 1.0;  // CS scale (reading Z2)
          out[k] = N[k] * sc;
        }
      } else {
        basis_funs(U2, p - 2 + e, x, p - 2, N);  // globals e .. e+p-2
        first[e] = e;
        for (int k = 0; k < p - 1; ++k) {
          int i = e + k;
          double sc = (p - 1) / (U2[i + p - 1] - U2[i]);
          out[k] = N[k] * sc;
        }
      }
    }
  }
  // Elements whose functions see only uniform knots have the same local table in exact arithmetic;
  // the evaluation above differs between them by rounding only (about n * 1e-16 relative).  Such an
  // element takes its predecessor's table bit for bit, so that kernels can hold one element table
  // in registers for all interior elements (the brick kernel's uniform-basis path).
  const size_t tl = size_t(Q) * nl;
  for (int e = 1; e < n; ++e) {
    if (first[e] - first[e - 1] != 1) continue;
    const double* prev = &vals[size_t(e - 1) * tl];
    double* cur = &vals[size_t(e) * tl];
    bool same = true;
    for (size_t i = 0; i < tl && same; ++i)
      same = std::fabs(cur[i] - prev[i]) <= 1e-11 * std::max(std::fabs(prev[i]), std::fabs(cur[i]));
    if (same) std::copy(prev, prev + tl, cur);
  }
}

namespace {

int space_dim(int space, int p, int n) { return (space == 0 || space == 3) ? n + p - 2 : n + p - 1; }

// Dense Gram of two univariate spaces with the exact (p+1)-point rule per element.
std::vector<double> gram(int p, int n, int row_space, int col_space) {
  const int Qe = p + 1;  // exact for degree <= 2p+1 (Gamma_B^p has degree 2p)
  std::vector<double> gx, gw;
  gauss_legendre(Qe, gx, gw);
  std::vector<double> vr, vc;
  std::vector<int> fr, fc;
  basis_values_1d(p, n, Qe, row_space, vr, fr);
  basis_values_1d(p, n, Qe, col_space, vc, fc);
  int R = space_dim(row_space, p, n), C = space_dim(col_space, p, n);
  std::vector<double> A(size_t(R) * C, 0.0);
  const int nl = p + 1;
  for (int e = 0; e < n; ++e) {
    double h = 1.0 / n;
    for (int q = 0; q < Qe; ++q) {
      double w = gw[q] * 0.5 * h;
      const double* r = &vr[(size_t(e) * Qe + q) * nl];
      const double* c = &vc[(size_t(e) * Qe + q) * nl];
      for (int i = 0; i < nl; ++i) {
        int gi = fr[e] + i;
        if (gi < 0 || gi >= R || r[i] == 0.0) continue;
        for (int j = 0; j < nl; ++j) {
          int gj = fc[e] + j;
          if (gj < 0 || gj >= C || c[j] == 0.0) continue;
          A[size_t(gi) * C + gj] += w * r[i] * c[j];
        }
      }
    }
  }
  return A;
}

}  // namespace

sgm_status build_axis(int p, int n, int Q, Axis& out, std::string& err) {
  (void)err;
  out.n = n;
  out.a = n + p - 2;
  out.b = n + p - 1;
  out.G = gram(p, n, 3, 0);    // rows D'' (dual S_{p-2} CS), cols trimmed S_p
  out.M = gram(p, n, 2, 1);    // rows B' (dual S_{p-1}), cols D' (primal S_{p-1} CS)
  out.GB1 = gram(p, n, 2, 2);
  out.GC2 = gram(p, n, 3, 3);
  out.GBp = gram(p, n, 0, 0);
  out.GC1 = gram(p, n, 1, 1);
  std::vector<double> gx, gw;
  gauss_legendre(Q, gx, gw);
  out.xq.resize(size_t(n) * Q);
  out.wq.resize(size_t(n) * Q);
  for (int e = 0; e < n; ++e)
    for (int q = 0; q < Q; ++q) {
      double h = 1.0 / n;
      out.xq[e * Q + q] = e * h + (gx[q] + 1.0) * 0.5 * h;
      out.wq[e * Q + q] = gw[q] * 0.5 * h;
    }
  return SGM_OK;
}

// In-place no-pivot LU of a banded matrix (half-bandwidth m on both sides), stored dense.
// Reading Z14: B-spline pairing matrices are totally positive compositions, so elimination
// without pivoting exists and is stable; we still check pivots and the backward error.
sgm_status banded_lu_nopivot(const std::vector<double>& A, int L, int m, std::vector<double>& LU,
                             std::string& err) {
  double amax = 0.0;
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < L; ++j) {
      double v = A[size_t(i) * L + j];
      amax = std::max(amax, std::fabs(v));
      if (std::abs(i - j) > m && v != 0.0) {
        err = "1D matrix is not banded with half-bandwidth p-1";
        return SGM_E_SINGULAR;
      }
    }
  LU = A;
  for (int k = 0; k < L; ++k) {
    double piv = LU[size_t(k) * L + k];
    if (!(std::fabs(piv) > 1e-14 * amax)) {
      err = "zero pivot in no-pivot banded LU";
      return SGM_E_SINGULAR;
    }
    for (int i = k + 1; i <= std::min(L - 1, k + m); ++i) {
      double l = LU[size_t(i) * L + k] / piv;
      LU[size_t(i) * L + k] = l;
      for (int j = k + 1; j <= std::min(L - 1, k + m); ++j) LU[size_t(i) * L + j] -= l * LU[size_t(k) * L + j];
    }
  }
  // backward error ||L U - A||_max / ||A||_max
  double be = 0.0;
  for (int i = 0; i < L; ++i)
    for (int j = std::max(0, i - m); j <= std::min(L - 1, i + m); ++j) {
      double s = 0.0;
      for (int k = std::max(0, std::max(i, j) - m); k <= std::min(i, j); ++k) {
        double l = (k == i) ? 1.0 : LU[size_t(i) * L + k];
        double u = LU[size_t(k) * L + j];
        if (k <= i && k <= j) s += l * u;
      }
      be = std::max(be, std::fabs(s - A[size_t(i) * L + j]));
    }
  if (be > 1e-13 * amax) {
    err = "no-pivot banded LU backward error above 1e-13";
    return SGM_E_SINGULAR;
  }
  return SGM_OK;
}

namespace {

std::vector<double> transpose(const std::vector<double>& A, int L) {
  std::vector<double> T(A.size());
  for (int i = 0; i < L; ++i)
    for (int j = 0; j < L; ++j) T[size_t(j) * L + i] = A[size_t(i) * L + j];
  return T;
}

// Fill one line-operator table (layout: seg_sweep.cuh): Rpad rows of RowLayout<P>::RS doubles
//   [band(2P+1) | lo(m) | F(m) | dinv, upn(m) | B(m)],  m = P-1, groups padded to 16 bytes.
// Rows >= L are identity padding.  F/B are the spike tables of the partitioned solve for
// segments of SEG rows: F[j-1] of row r = d z_r / d z_{r0-j}, B[j-1] = d u_r / d u_{r1+j}.
sgm_status fill_table(double* T, int P, int L, int Rpad, int SEG, const std::vector<double>* band,
                      const std::vector<double>* lu_src, std::string& err) {
  const RowLayoutRT RL(P);
  const int m = RL.M, RS = RL.RS;
  const int LO = RL.LO, UP = RL.UP, DI = RL.UP, FF = RL.F, BB = RL.B;  // DI: dinv sits at UP
  for (int i = 0; i < Rpad; ++i) {
    double* row = T + size_t(i) * RS;
    for (int k = 0; k < RS; ++k) row[k] = 0.0;
    row[DI] = 1.0;
    if (i >= L) continue;
    if (band) {
      for (int k = -P; k <= P; ++k) {
        int j = i + k;
        if (j >= 0 && j < L) row[k + P] = (*band)[size_t(i) * L + j];
      }
      for (int j = 0; j < L; ++j)  // entries outside the stored band must vanish exactly
        if (std::abs(j - i) > P && (*band)[size_t(i) * L + j] != 0.0) {
          err = "1D band matrix wider than the compiled band";
          return SGM_E_UNSUPPORTED;
        }
    } else {
      row[P] = 1.0;
    }
  }
  if (!lu_src) return SGM_OK;
  std::vector<double> LU;
  sgm_status st = banded_lu_nopivot(*lu_src, L, m, LU, err);
  if (st != SGM_OK) return st;
  for (int i = 0; i < L; ++i) {
    double* row = T + size_t(i) * RS;
    double uii = LU[size_t(i) * L + i];
    for (int k = 1; k <= m; ++k) {
      if (i - k >= 0) row[LO + k - 1] = LU[size_t(i) * L + (i - k)];
      if (i + k < L) row[UP + k] = LU[size_t(i) * L + (i + k)] / uii;
    }
    row[DI] = 1.0 / uii;
  }
  // spikes: response of the zero-history local recurrences to unit histories
  const int S = Rpad / SEG;
  std::vector<double> z(SEG + m);
  for (int s = 0; s < S; ++s) {
    const int r0 = s * SEG;
    for (int j = 1; j <= m; ++j) {
      // forward: z_{r0-q} = delta_{qj}; z_r = -sum_k lo_{r,k} z_{r-k}
      for (int q = 1; q <= m; ++q) z[m - q] = (q == j) ? 1.0 : 0.0;   // z[m-q] <-> row r0-q
      for (int r = r0; r < r0 + SEG; ++r) {
        const double* row = T + size_t(r) * RS;
        double acc = 0.0;
        for (int k = 1; k <= m; ++k) acc -= row[LO + k - 1] * z[m + (r - r0) - k];
        z[m + (r - r0)] = acc;
        T[size_t(r) * RS + FF + j - 1] = acc;
      }
      // backward: u_{r1+q} = delta_{qj}; u_r = -sum_k upn_{r,k} u_{r+k}
      const int r1 = r0 + SEG - 1;
      std::vector<double> u(SEG + m, 0.0);  // u[(r - r0)] for r in segment, u[SEG + q - 1] <-> r1+q
      for (int q = 1; q <= m; ++q) u[SEG + q - 1] = (q == j) ? 1.0 : 0.0;
      for (int r = r1; r >= r0; --r) {
        const double* row = T + size_t(r) * RS;
        double acc = 0.0;
        for (int k = 1; k <= m; ++k) acc -= row[UP + k] * u[(r - r0) + k];
        u[r - r0] = acc;
        T[size_t(r) * RS + BB + j - 1] = acc;
      }
    }
  }
  return SGM_OK;
}

// Largest |q| with a nonzero band coefficient in any row (the table's band half-width).
int table_band_hw(const double* T, int P, int L) {
  const RowLayoutRT RL(P);
  int hw = 0;
  for (int i = 0; i < L; ++i)
    for (int q = -P; q <= P; ++q)
      if (T[size_t(i) * RL.RS + RL.BAND + q + P] != 0.0) hw = std::max(hw, std::abs(q));
  return hw;
}

// Truncated SPIKE reach (reading Z23 in DESIGN.md): the true history of segment s is
//   hist_s = tail_{s-1} + Fm_{s-1} hist_{s-1},   Fm_t[jj][q] = F[t*SEG + SEG - jj][q]
// so starting the scan K segments back with a zero history leaves the error
// (Fm_{s-1} ... Fm_{s-K}) hist_{s-K}.  The spikes of the B-spline pairing factors decay
// geometrically; K is the smallest reach with every such product below 1e-17 in the infinity
// norm (likewise for the backward spikes Bm_t[jj][q] = B[t*SEG + jj - 1][q]).  K >= S means no
// truncation.
void spike_reach(const double* T, int P, int L, int SEG, int& kh, int& kf) {
  const RowLayoutRT RL(P);
  const int m = RL.M, RS = RL.RS;
  const int S = (L + SEG - 1) / SEG;
  auto mat = [&](int t, bool fwd, std::vector<double>& A) {
    A.assign(size_t(m) * m, 0.0);
    for (int jj = 1; jj <= m; ++jj)
      for (int q = 1; q <= m; ++q) {
        const int row = fwd ? t * SEG + SEG - jj : t * SEG + jj - 1;
        A[size_t(jj - 1) * m + (q - 1)] = T[size_t(row) * RS + (fwd ? RL.F : RL.B) + q - 1];
      }
  };
  auto reach = [&](bool fwd) {
    std::vector<double> A, Pm, Q;
    for (int K = 1; K < S; ++K) {
      double worst = 0.0;
      for (int s = 0; s < S; ++s) {
        // fwd: Fm_{s-1} ... Fm_{s-K} (exact when s - K <= 0); bwd: Bm_{s+1} ... Bm_{s+K} (exact when s + K >= S - 1)
        if (fwd ? (s - K <= 0) : (s + K >= S - 1)) continue;
        Pm.assign(size_t(m) * m, 0.0);
        for (int i = 0; i < m; ++i) Pm[size_t(i) * m + i] = 1.0;
        for (int i = 1; i <= K; ++i) {
          mat(fwd ? s - i : s + i, fwd, A);
          Q.assign(size_t(m) * m, 0.0);
          for (int x = 0; x < m; ++x)
            for (int y = 0; y < m; ++y)
              for (int z = 0; z < m; ++z) Q[size_t(x) * m + y] += Pm[size_t(x) * m + z] * A[size_t(z) * m + y];
          Pm = Q;
        }
        double nrm = 0.0;
        for (int x = 0; x < m; ++x) {
          double r = 0.0;
          for (int y = 0; y < m; ++y) r += std::fabs(Pm[size_t(x) * m + y]);
          nrm = std::max(nrm, r);
        }
        worst = std::max(worst, nrm);
      }
      if (worst <= 1e-17) return K;
    }
    return S;
  };
  kh = reach(true);
  kf = reach(false);
}

}  // namespace

int seg_for_line(int L) {
  // segment length of the partitioned line solve: one consumer warp per segment, at most 14
  // segments (16 warps per CTA with the producers); shortest segment that fits (more warps, fewer
  // registers).  Override in a tuning build: SGM_SEG.
  if (const int v = tune_int("SGM_SEG", 0)) {
    if ((v == 12 || v == 17 || v == 28) && (L + v - 1) / v <= 14) return v;
  }
  const int cands[3] = {12, 17, 28};
  for (int c : cands)
    if ((L + c - 1) / c <= 14) return c;
  return 28;
}

// Truncated-SPIKE reaches of every table (reading Z23), or the exact untruncated scans with
// SGM_OPT_EXACT_SPIKE.  Also the band half-widths.  Recomputed by sgm_plan_set_options.
sgm_status set_spike_reach(Plan& P, std::string& err) {
  (void)err;
  const bool noskip = (P.opts & SGM_OPT_EXACT_SPIKE) != 0;
  const int p = P.p, RS = RowLayoutRT(p).RS;
  const int Rmax = P.Lmax;
  for (int a = 0; a < 3; ++a) {
    const Axis& X = P.ax[a];
    const int SEG = P.seg[a];
    auto T = [&](int op) { return P.tables_host.data() + (size_t(a) * OP_COUNT + op) * Rmax * RS; };
    if (!P.wide_host.empty()) {
      const int RSw = RowLayoutRT(p + 1).RS;
      const double* Tw = P.wide_host.data() + size_t(a) * Rmax * RSw;
      if (noskip && X.a <= kMaxLine) P.wide_kh[a] = P.wide_kf[a] = (X.a + SEG - 1) / SEG;
      else spike_reach(Tw, p + 1, X.a, SEG, P.wide_kh[a], P.wide_kf[a]);
    }
    const int Ls[OP_COUNT] = {X.b, X.a, X.a, X.b, X.b, X.a, X.a, X.b, X.a};
    for (int op = 0; op < OP_COUNT; ++op) {
      const int S = (Ls[op] + SEG - 1) / SEG;
      P.band_hw[a][op] = table_band_hw(T(op), p, Ls[op]);
      // (lines above kMaxLine run in windows, launch_sweep: always the truncated reach)
      if ((noskip && Ls[op] <= kMaxLine) || (op >= OP_APPLY_M && op <= OP_APPLY_MT)) {
        P.spike_kh[a][op] = P.spike_kf[a][op] = S;
      } else {
        spike_reach(T(op), p, Ls[op], SEG, P.spike_kh[a][op], P.spike_kf[a][op]);
      }
      if (tune_int("SGM_DEBUG_PLAN", 0))
        fprintf(stderr, "sgm plan: axis %d op %d L %d SEG %d S %d band_hw %d spike reach hist %d fut %d\n", a, op,
                Ls[op], SEG, S, P.band_hw[a][op], P.spike_kh[a][op], P.spike_kf[a][op]);
    }
  }
  return SGM_OK;
}

sgm_status build_tables(Plan& P, std::string& err) {
  P.diag_ok = true;
  const int p = P.p, RS = RowLayoutRT(p).RS;
  int Rmax = 0;
  for (int a = 0; a < 3; ++a) {
    P.seg[a] = seg_for_line(P.ax[a].b);
    P.rpad[a] = ((P.ax[a].b + P.seg[a] - 1) / P.seg[a]) * P.seg[a];
    Rmax = std::max(Rmax, P.rpad[a]);
  }
  P.Lmax = Rmax;  // rows per table slot
  P.diag_off = size_t(3) * OP_COUNT * Rmax * RS;
  P.tables_host.assign(P.diag_off + size_t(3) * 2 * Rmax, 0.0);
  for (int a = 0; a < 3; ++a) {
    const Axis& X = P.ax[a];
    const int R = P.rpad[a], SEG = P.seg[a];
    std::vector<double> GT = transpose(X.G, X.a), MT = transpose(X.M, X.b);
    auto T = [&](int op) { return P.tables_host.data() + (size_t(a) * OP_COUNT + op) * Rmax * RS; };
    sgm_status st;
    if ((st = fill_table(T(OP_EPS_OWN), p, X.b, R, SEG, &X.GB1, &X.M, err)) != SGM_OK) return st;
    if ((st = fill_table(T(OP_EPS_OTH), p, X.a, R, SEG, &X.GC2, &X.G, err)) != SGM_OK) return st;
    if ((st = fill_table(T(OP_MU_OWN), p, X.a, R, SEG, &X.GBp, &GT, err)) != SGM_OK) return st;
    if ((st = fill_table(T(OP_MU_OTH), p, X.b, R, SEG, &X.GC1, &MT, err)) != SGM_OK) return st;
    if ((st = fill_table(T(OP_APPLY_M), p, X.b, R, SEG, &X.M, nullptr, err)) != SGM_OK) return st;
    if ((st = fill_table(T(OP_APPLY_G), p, X.a, R, SEG, &X.G, nullptr, err)) != SGM_OK) return st;
    if ((st = fill_table(T(OP_APPLY_GT), p, X.a, R, SEG, &GT, nullptr, err)) != SGM_OK) return st;
    if ((st = fill_table(T(OP_APPLY_MT), p, X.b, R, SEG, &MT, nullptr, err)) != SGM_OK) return st;
    // scheme 1: h_c own factor Gamma_C^{p-2}^{-1} Hat G; e_c other factor
    // Gamma_B^p^{-1} Hat G^T, whose LU has half-bandwidth p -> wide layout p + 1
    if ((st = fill_table(T(OP_S1_MU_OWN), p, X.a, R, SEG, &X.G, &X.GC2, err)) != SGM_OK) return st;
    if (p <= 4) {
      const int RSw = RowLayoutRT(p + 1).RS;
      if (P.wide_host.empty()) P.wide_host.assign(size_t(3) * Rmax * RSw, 0.0);
      double* Tw = P.wide_host.data() + size_t(a) * Rmax * RSw;
      if ((st = fill_table(Tw, p + 1, X.a, R, SEG, &GT, &X.GBp, err)) != SGM_OK) return st;
      P.wide_band_hw[a] = table_band_hw(Tw, p + 1, X.a);
    }
    // Diagonal 1D factors ("reduced separable schedule"): with the CS normalisation
    // D'_k = s_k B'_k, Hat M = Gamma_B^{p-1} diag(s) and Gamma_C^{p-1} =
    // diag(s) Gamma_B^{p-1} diag(s), so the own-axis factor of the eps Hodge star,
    // Hat M^{-1} Gamma_B^{p-1} = diag(1/s), and the other-axis factor of the mu Hodge star,
    // Hat M^{-T} Gamma_C^{p-1} = diag(s), are diagonal.  Checked here; the schedule falls back to
    // full sweeps on every axis if an identity fails (SGM_OPT_FULL_SCHEDULE forces them).
    {
      const int L = X.b;
      double* dg_eps = P.tables_host.data() + P.diag_off + size_t(a * 2 + 0) * Rmax;
      double* dg_mu = P.tables_host.data() + P.diag_off + size_t(a * 2 + 1) * Rmax;
      double mM = 0.0, mC = 0.0, eM = 0.0, eC = 0.0;
      std::vector<double> sk(L);
      for (int k = 0; k < L; ++k) sk[k] = X.M[size_t(k) * L + k] / X.GB1[size_t(k) * L + k];
      for (int i = 0; i < L; ++i)
        for (int j = 0; j < L; ++j) {
          const double m = X.M[size_t(i) * L + j], c = X.GC1[size_t(i) * L + j], g = X.GB1[size_t(i) * L + j];
          mM = std::max(mM, std::fabs(m));
          mC = std::max(mC, std::fabs(c));
          eM = std::max(eM, std::fabs(m - g * sk[j]));
          eC = std::max(eC, std::fabs(c - sk[i] * g * sk[j]));
        }
      const bool ok = std::isfinite(eM) && std::isfinite(eC) && eM <= 1e-13 * mM && eC <= 1e-13 * mC;
      if (!ok) P.diag_ok = false;
      for (int k = 0; k < L; ++k) {
        dg_eps[k] = 1.0 / sk[k];
        dg_mu[k] = sk[k];
      }
      if (tune_int("SGM_DEBUG_PLAN", 0))
        fprintf(stderr, "sgm plan: axis %d diagonal factors: |M - G diag(s)| %.3g, |Gc - diag(s) G diag(s)| %.3g\n", a,
                eM / mM, eC / mC);
    }
  }
  return set_spike_reach(P, err);
}

// ---- geometry -------------------------------------------------------------------------------

namespace {

// Evaluate F and DF at every quadrature point of elements [ez] (element-major order) from the
// spline control points.  DF[9] row-major: DF[i*3+j] = dF_i / dx^_j.
struct GeoEval {
  const Plan& P;
  std::vector<double> v[3], d[3];  // per-axis S_p (untrimmed) values/derivs at qp: [n][Q][p+1]
  explicit GeoEval(const Plan& P_) : P(P_) {
    const int p = P.p, Q = P.Q;
    std::vector<double> gx, gw;
    gauss_legendre(Q, gx, gw);
    for (int a = 0; a < 3; ++a) {
      int n = P.n[a];
      std::vector<double> U = open_knots(p, n);
      v[a].assign(size_t(n) * Q * (p + 1), 0.0);
      d[a].assign(size_t(n) * Q * (p + 1), 0.0);
      for (int e = 0; e < n; ++e)
        for (int q = 0; q < Q; ++q) {
          double x = (e + (gx[q] + 1.0) * 0.5) / n;
          basis_funs(U.data(), p + e, x, p, &v[a][(size_t(e) * Q + q) * (p + 1)]);
          basis_ders(U.data(), p + e, x, p, &d[a][(size_t(e) * Q + q) * (p + 1)]);
        }
    }
  }
  // element (ex,ey,ez), point (qx,qy,qz)
  void eval(int ex, int ey, int ez, int qx, int qy, int qz, double* F, double* DF) const {
    const int p = P.p, Q = P.Q, nl = p + 1;
    const int NX = P.n[0] + p, NY = P.n[1] + p;
    const double* vx = &v[0][(size_t(ex) * Q + qx) * nl];
    const double* vy = &v[1][(size_t(ey) * Q + qy) * nl];
    const double* vz = &v[2][(size_t(ez) * Q + qz) * nl];
    const double* dx = &d[0][(size_t(ex) * Q + qx) * nl];
    const double* dy = &d[1][(size_t(ey) * Q + qy) * nl];
    const double* dz = &d[2][(size_t(ez) * Q + qz) * nl];
    for (int i = 0; i < 3; ++i) F[i] = 0.0;
    for (int i = 0; i < 9; ++i) DF[i] = 0.0;
    const bool rat = !P.wts.empty();
    double W = 0.0, dW[3] = {0.0, 0.0, 0.0};  // rational map: denominator sum w N and its gradient
    for (int k = 0; k < nl; ++k)
      for (int j = 0; j < nl; ++j)
        for (int i = 0; i < nl; ++i) {
          const size_t id = (size_t(ez + k) * NY + (ey + j)) * NX + (ex + i);
          const double* c = &P.ctrl[id * 3];
          const double wt = rat ? P.wts[id] : 1.0;
          double w0 = wt * vx[i] * vy[j] * vz[k];
          double wx = wt * dx[i] * vy[j] * vz[k];
          double wy = wt * vx[i] * dy[j] * vz[k];
          double wz = wt * vx[i] * vy[j] * dz[k];
          for (int r = 0; r < 3; ++r) {
            F[r] += c[r] * w0;
            DF[r * 3 + 0] += c[r] * wx;
            DF[r * 3 + 1] += c[r] * wy;
            DF[r * 3 + 2] += c[r] * wz;
          }
          W += w0;
          dW[0] += wx;
          dW[1] += wy;
          dW[2] += wz;
        }
    if (rat) {
      // F = N / W,  dF_r/dx^_j = (dN_r/dx^_j - F_r dW/dx^_j) / W   (quotient rule)
      for (int r = 0; r < 3; ++r) F[r] /= W;
      for (int r = 0; r < 3; ++r)
        for (int j = 0; j < 3; ++j) DF[r * 3 + j] = (DF[r * 3 + j] - F[r] * dW[j]) / W;
    }
  }
};

inline double det3(const double* A) {
  return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
         A[2] * (A[3] * A[7] - A[4] * A[6]);
}

template <class Fn>
void for_each_qp(const Plan& P, Fn fn) {
  const int Q = P.Q;
  const int nx = P.n[0], ny = P.n[1], nz = P.n[2];
#pragma omp parallel for schedule(static)
  for (int ez = 0; ez < nz; ++ez)
    for (int ey = 0; ey < ny; ++ey)
      for (int ex = 0; ex < nx; ++ex)
        for (int qz = 0; qz < Q; ++qz)
          for (int qy = 0; qy < Q; ++qy)
            for (int qx = 0; qx < Q; ++qx) {
              size_t idx = ((((size_t(ez) * ny + ey) * nx + ex) * Q + qz) * Q + qy) * Q + qx;
              fn(idx, ex, ey, ez, qx, qy, qz);
            }
}

}  // namespace

sgm_status build_geometry(Plan& P, std::string& err) {
  P.n_qp = size_t(P.n[0]) * P.n[1] * P.n[2] * P.Q * P.Q * P.Q;
  if (!P.has_geom) {
    P.affine_diag = true;
    P.L_aff[0] = P.L_aff[1] = P.L_aff[2] = 1.0;
    return SGM_OK;
  }
  GeoEval G(P);
  // reference DF at the first point for the affine-diagonal test
  double F0[3], D0[9];
  G.eval(0, 0, 0, 0, 0, 0, F0, D0);
  int bad = 0, nonaff = 0;
  const double scale = std::fabs(D0[0]) + std::fabs(D0[4]) + std::fabs(D0[8]);
  for_each_qp(P, [&](size_t, int ex, int ey, int ez, int qx, int qy, int qz) {
    double F[3], D[9];
    G.eval(ex, ey, ez, qx, qy, qz, F, D);
    double dt = det3(D);
    if (!(dt > 0.0) || !std::isfinite(dt)) {
#pragma omp atomic
      bad++;
    }
    bool aff = true;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double ref = (i == j) ? D0[i * 3 + j] : 0.0;
        if (std::fabs(D[i * 3 + j] - ref) > 1e-13 * scale) aff = false;
      }
    if (!aff) {
#pragma omp atomic
      nonaff++;
    }
  });
  if (bad) {
    err = "det DF <= 0 or non-finite at " + std::to_string(bad) + " quadrature points";
    return SGM_E_GEOMETRY;
  }
  P.affine_diag = (nonaff == 0);
  if (P.affine_diag) {
    P.L_aff[0] = D0[0];
    P.L_aff[1] = D0[4];
    P.L_aff[2] = D0[8];
  }
  return SGM_OK;
}

void qp_coords(const Plan& P, double* xyz) {
  if (!P.has_geom) {
    for_each_qp(P, [&](size_t idx, int ex, int ey, int ez, int qx, int qy, int qz) {
      xyz[idx * 3 + 0] = P.ax[0].xq[ex * P.Q + qx];
      xyz[idx * 3 + 1] = P.ax[1].xq[ey * P.Q + qy];
      xyz[idx * 3 + 2] = P.ax[2].xq[ez * P.Q + qz];
    });
    return;
  }
  GeoEval G(P);
  for_each_qp(P, [&](size_t idx, int ex, int ey, int ez, int qx, int qy, int qz) {
    double F[3], D[9];
    G.eval(ex, ey, ez, qx, qy, qz, F, D);
    xyz[idx * 3 + 0] = F[0];
    xyz[idx * 3 + 1] = F[1];
    xyz[idx * 3 + 2] = F[2];
  });
}

// Hodge weights for one material (the 2-form Piola pull-back gives
// int gamma eta.omega dx = int gamma eta^ (DF^T DF / det DF) omega^ dx^):
//   SEPARABLE: constant material, affine-diagonal F -> per-component scale only
//   SCALAR   : variable material, affine-diagonal F -> W(q) = w_q / material(q), scale_c
//   FULL     : general F -> W6(q) = w_q / material(q) * (DF^T DF)/det (xx,yy,zz,xy,xz,yz)
sgm_status build_mass(Plan& P, int which, const double* values, double c, std::vector<double>& W,
                      std::string& err) {
  MassData& M = P.mass[which];
  W.clear();
  if (!values) {
    if (!(c > 0.0) || !std::isfinite(c)) {
      err = "material constant must be positive and finite";
      return SGM_E_MATERIAL;
    }
  } else {
    size_t badm = 0;
#pragma omp parallel for reduction(+ : badm)
    for (long long i = 0; i < (long long)P.n_qp; ++i)
      if (!(values[i] > 0.0) || !std::isfinite(values[i])) badm++;
    if (badm) {
      err = "material must be positive and finite at every quadrature point";
      return SGM_E_MATERIAL;
    }
  }
  M.const_material = (values == nullptr);
  M.material_c = c;
  if (values) M.values_host.assign(values, values + P.n_qp);
  else M.values_host.clear();
  const double Lx = P.L_aff[0], Ly = P.L_aff[1], Lz = P.L_aff[2];
  const double detL = Lx * Ly * Lz;
  if (P.affine_diag) {
    double s[3] = {Lx * Lx / detL, Ly * Ly / detL, Lz * Lz / detL};
    if (M.const_material) {
      M.kind = HODGE_SEPARABLE;
      for (int k = 0; k < 3; ++k) M.scale[k] = s[k] / c;
      return SGM_OK;
    }
    M.kind = HODGE_SCALAR;
    for (int k = 0; k < 3; ++k) M.scale[k] = s[k];
    W.resize(P.n_qp);
    for_each_qp(P, [&](size_t idx, int ex, int ey, int ez, int qx, int qy, int qz) {
      double w = P.ax[0].wq[ex * P.Q + qx] * P.ax[1].wq[ey * P.Q + qy] * P.ax[2].wq[ez * P.Q + qz];
      W[idx] = w / values[idx];
    });
    return SGM_OK;
  }
  M.kind = HODGE_FULL;
  for (int k = 0; k < 3; ++k) M.scale[k] = 1.0;
  M.otf = otf_geometry(P);
  if (M.otf) {
    // on-the-fly DF: only the scalar factor w_q / material per point (the brick kernel forms
    // (w_q / material) / det DF * DF^T DF from the map, hodge_brick.cuh)
    W.resize(P.n_qp);
    for_each_qp(P, [&](size_t idx, int ex, int ey, int ez, int qx, int qy, int qz) {
      double w = P.ax[0].wq[ex * P.Q + qx] * P.ax[1].wq[ey * P.Q + qy] * P.ax[2].wq[ez * P.Q + qz];
      W[idx] = w / (values ? values[idx] : c);
    });
    return SGM_OK;
  }
  W.resize(P.n_qp * 6);
  GeoEval G(P);
  for_each_qp(P, [&](size_t idx, int ex, int ey, int ez, int qx, int qy, int qz) {
    double F[3], D[9];
    G.eval(ex, ey, ez, qx, qy, qz, F, D);
    double dt = det3(D);
    double w = P.ax[0].wq[ex * P.Q + qx] * P.ax[1].wq[ey * P.Q + qy] * P.ax[2].wq[ez * P.Q + qz];
    double g = w / (values ? values[idx] : c) / dt;
    // (DF^T DF)_{ij} = sum_r DF[r][i] DF[r][j]
    auto m = [&](int i, int j) { return D[0 * 3 + i] * D[0 * 3 + j] + D[1 * 3 + i] * D[1 * 3 + j] + D[2 * 3 + i] * D[2 * 3 + j]; };
    double* o = &W[idx * 6];
    o[0] = g * m(0, 0);
    o[1] = g * m(1, 1);
    o[2] = g * m(2, 2);
    o[3] = g * m(0, 1);
    o[4] = g * m(0, 2);
    o[5] = g * m(1, 2);
  });
  return SGM_OK;
}

bool otf_geometry(const Plan& P) {
  return (P.opts & SGM_OPT_OTF_GEOMETRY) && !P.affine_diag && P.wts.empty() && P.Q == P.p + 1 && P.p >= 2 &&
         P.p <= 4;
}

void build_geo_buffer(const Plan& P, std::vector<double>& buf, size_t ctrl_off[3], size_t tab_off[3][2]) {
  const size_t N0 = size_t(P.n[0] + P.p) * (P.n[1] + P.p) * (P.n[2] + P.p);
  GeoEval G(P);
  size_t tot = 3 * N0;
  for (int a = 0; a < 3; ++a) tot += G.v[a].size() + G.d[a].size();
  buf.assign(tot, 0.0);
  for (int r = 0; r < 3; ++r) {
    ctrl_off[r] = size_t(r) * N0;
    for (size_t i = 0; i < N0; ++i) buf[ctrl_off[r] + i] = P.ctrl[i * 3 + r];
  }
  size_t o = 3 * N0;
  for (int a = 0; a < 3; ++a) {
    tab_off[a][0] = o;
    std::copy(G.v[a].begin(), G.v[a].end(), buf.begin() + o);
    o += G.v[a].size();
    tab_off[a][1] = o;
    std::copy(G.d[a].begin(), G.d[a].end(), buf.begin() + o);
    o += G.d[a].size();
  }
}

// Scheme 1: weights of the 1-form masses M^1_eps (which = EPS, primal 1-forms) and
// M~^1_mu (which = MU, dual 1-forms) from the material stored by build_mass:
//   W = w_q gamma(q) DF^{-1} DF^{-T} det DF  (1-form pull-back; FULL, 6 symmetric entries), or for
//   an axis-aligned affine map w_q gamma(q) with the per-component scale prod(L) / L_c^2 (SCALAR),
//   or nothing for a constant material on such a map (SEPARABLE: Kronecker Grams).
sgm_status build_mass1(Plan& P, int which, std::vector<double>& W, std::string& err) {
  const MassData& M2 = P.mass[which];
  MassData& M = P.mass1[which];
  W.clear();
  M.const_material = M2.const_material;
  M.material_c = M2.material_c;
  const double* values = M2.const_material ? nullptr : M2.values_host.data();
  const double c = M2.material_c;
  if (!M2.const_material && M2.values_host.size() != P.n_qp) {
    err = "scheme 1: material values missing";
    return SGM_E_MATERIAL;
  }
  const double Lx = P.L_aff[0], Ly = P.L_aff[1], Lz = P.L_aff[2];
  const double detL = Lx * Ly * Lz;
  if (P.affine_diag) {
    const double s[3] = {detL / (Lx * Lx), detL / (Ly * Ly), detL / (Lz * Lz)};
    if (M.const_material) {
      M.kind = HODGE_SEPARABLE;
      for (int k = 0; k < 3; ++k) M.scale[k] = s[k] * c;
      return SGM_OK;
    }
    M.kind = HODGE_SCALAR;
    for (int k = 0; k < 3; ++k) M.scale[k] = s[k];
    W.resize(P.n_qp);
    for_each_qp(P, [&](size_t idx, int ex, int ey, int ez, int qx, int qy, int qz) {
      double w = P.ax[0].wq[ex * P.Q + qx] * P.ax[1].wq[ey * P.Q + qy] * P.ax[2].wq[ez * P.Q + qz];
      W[idx] = w * values[idx];
    });
    return SGM_OK;
  }
  M.kind = HODGE_FULL;
  for (int k = 0; k < 3; ++k) M.scale[k] = 1.0;
  W.resize(P.n_qp * 6);
  GeoEval G(P);
  for_each_qp(P, [&](size_t idx, int ex, int ey, int ez, int qx, int qy, int qz) {
    double F[3], D[9];
    G.eval(ex, ey, ez, qx, qy, qz, F, D);
    const double dt = det3(D);
    double w = P.ax[0].wq[ex * P.Q + qx] * P.ax[1].wq[ey * P.Q + qy] * P.ax[2].wq[ez * P.Q + qz];
    const double g = w * (values ? values[idx] : c);
    // DF^{-1} = adj(DF) / det; DF^{-1} DF^{-T} det = adj adj^T / det
    double A[9];
    A[0] = D[4] * D[8] - D[5] * D[7];
    A[1] = D[2] * D[7] - D[1] * D[8];
    A[2] = D[1] * D[5] - D[2] * D[4];
    A[3] = D[5] * D[6] - D[3] * D[8];
    A[4] = D[0] * D[8] - D[2] * D[6];
    A[5] = D[2] * D[3] - D[0] * D[5];
    A[6] = D[3] * D[7] - D[4] * D[6];
    A[7] = D[1] * D[6] - D[0] * D[7];
    A[8] = D[0] * D[4] - D[1] * D[3];
    auto m = [&](int i, int j) { return (A[i * 3 + 0] * A[j * 3 + 0] + A[i * 3 + 1] * A[j * 3 + 1] + A[i * 3 + 2] * A[j * 3 + 2]) / dt; };
    double* o = &W[idx * 6];
    o[0] = g * m(0, 0);
    o[1] = g * m(1, 1);
    o[2] = g * m(2, 2);
    o[3] = g * m(0, 1);
    o[4] = g * m(0, 2);
    o[5] = g * m(1, 2);
  });
  return SGM_OK;
}

// Greville abscissae of the untrimmed S_p on n uniform elements: g_i = mean(U[i+1 .. i+p]).
std::vector<double> greville(int p, int n) {
  const std::vector<double> U = open_knots(p, n);
  std::vector<double> g(n + p);
  for (int i = 0; i < n + p; ++i) {
    double s = 0.0;
    for (int k = 1; k <= p; ++k) s += U[i + k];
    g[i] = s / p;
  }
  return g;
}

// Geometry control points interpolating map values given at the Greville grid (reading Z18):
// per axis the collocation matrix C[j][i] = N_i(g_j) of the untrimmed S_p is inverted (dense LU
// with partial pivoting, applied mode by mode); layout [(nz+p)][(ny+p)][(nx+p)][3] in and out.
sgm_status interpolate_geometry(const int n_el[3], int p, const double* values, double* ctrl, std::string& err) {
  const int m[3] = {n_el[0] + p, n_el[1] + p, n_el[2] + p};
  std::vector<double> cur(values, values + size_t(m[0]) * m[1] * m[2] * 3), nxt(cur.size());
  for (int a = 0; a < 3; ++a) {
    const int L = m[a], n = n_el[a];
    const std::vector<double> U = open_knots(p, n), g = greville(p, n);
    std::vector<double> C(size_t(L) * L, 0.0);
    for (int j = 0; j < L; ++j) {
      int sp = p;  // knot span of g_j: U[sp] <= x < U[sp+1] (the last point uses the last span)
      while (sp < n + p - 1 && g[j] >= U[sp + 1]) ++sp;
      double N[16];
      basis_funs(U.data(), sp, g[j], p, N);
      for (int k = 0; k <= p; ++k) C[size_t(j) * L + (sp - p + k)] = N[k];
    }
    // LU with partial pivoting
    std::vector<int> piv(L);
    for (int k = 0; k < L; ++k) {
      int r = k;
      for (int i = k + 1; i < L; ++i)
        if (std::fabs(C[size_t(i) * L + k]) > std::fabs(C[size_t(r) * L + k])) r = i;
      if (!(std::fabs(C[size_t(r) * L + k]) > 0.0)) {
        err = "singular geometry collocation matrix";
        return SGM_E_SINGULAR;
      }
      piv[k] = r;
      if (r != k)
        for (int j = 0; j < L; ++j) std::swap(C[size_t(k) * L + j], C[size_t(r) * L + j]);
      for (int i = k + 1; i < L; ++i) {
        const double f = C[size_t(i) * L + k] / C[size_t(k) * L + k];
        C[size_t(i) * L + k] = f;
        for (int j = k + 1; j < L; ++j) C[size_t(i) * L + j] -= f * C[size_t(k) * L + j];
      }
    }
    // solve along axis a for every line and coordinate
    const long stride = (a == 0) ? 3 : (a == 1 ? 3L * m[0] : 3L * m[0] * m[1]);
    const long lines = long(cur.size()) / L;
    std::vector<double> v(L);
    for (long l = 0; l < lines; ++l) {
      // line l -> base offset: decompose l over the other indices (coordinate fastest)
      long rem = l, base = 0, mult = 1;
      const int dims[4] = {3, m[0], m[1], m[2]};
      for (int d = 0; d < 4; ++d) {
        if (d == a + 1) { mult *= dims[d]; continue; }
        const long idx = rem % dims[d];
        rem /= dims[d];
        base += idx * mult;
        mult *= dims[d];
      }
      for (int i = 0; i < L; ++i) v[i] = cur[base + i * stride];
      for (int k = 0; k < L; ++k) std::swap(v[k], v[piv[k]]);
      for (int i = 1; i < L; ++i)
        for (int k = 0; k < i; ++k) v[i] -= C[size_t(i) * L + k] * v[k];
      for (int i = L - 1; i >= 0; --i) {
        for (int k = i + 1; k < L; ++k) v[i] -= C[size_t(i) * L + k] * v[k];
        v[i] /= C[size_t(i) * L + i];
      }
      for (int i = 0; i < L; ++i) nxt[base + i * stride] = v[i];
    }
    cur.swap(nxt);
  }
  std::copy(cur.begin(), cur.end(), ctrl);
  return SGM_OK;
}

}  // namespace sgm
