// Persistent, warp-specialised, double-buffered line sweeps (sm_100a) -- the hot kernel.
//
// What one sweep computes (eq. kroninverse P:L571 applied mode by mode with the vec trick
// P:L575-585): for every line of every component along axis `ax`,
//     out_line = scale * A^{-1} (B in_line)
// with B a banded 1D matrix (separable Hodge Gram or pairing factor) and A = LU a banded 1D
// pairing factor (no-pivot LU, reading Z14).  The solve is the partitioned (SPIKE) form of the
// sequential banded substitution (seg_sweep.cuh): segment-local recurrences plus exact spike
// corrections.
//
// Work unit: a tile of TW = 32*LPT lines of one component; lane j of a consumer warp owns lines
// j, j+32, ... (LPT lines: independent recurrences interleave, coefficient loads are shared).
// A CTA is persistent and loops over tiles with two shared-memory slabs:
//   * producer warps stage tile t+1 into slab[(t+1)&1]: cp.async (LDGSTS) copies, or, for the
//     first pass of a half step, the fused Ampere/Faraday update (eqs. discrete2_ampere /
//     discrete2_faraday) computed from global loads, written to the state and slab;
//   * consumer warp s owns rows [s*SEG, (s+1)*SEG) of every line of the tile (SPIKE segment s) and
//     runs: band mat-vec fused with the zero-history forward substitution -> tail exchange ->
//     history scan -> spike-corrected backward substitution -> head exchange -> future scan ->
//     spike correction fused with the scaled store.
// Producer/consumer hand-off: named barriers FULL[b] / EMPTY[b]; SPIKE exchanges: a consumer-only
// named barrier.  Line-operator tables (one or two per pass) are staged once per CTA in shared
// memory; every lane of a warp reads the same table row (broadcast, 16-byte vector loads).
// Slab layouts (R = NC*SEG + P rows per line, zero beyond the line end):
//   strided axes (y, z): slab[r * TW + line]      (a warp reads 32 consecutive doubles of a row)
//   x axis             : slab[line * pitch + r]   (pitch odd >= R: conflict-free per-lane walks)
#pragma once

#include "kernels.cuh"
#include "pipe_sweep.cuh"
#include "seg_sweep.cuh"

namespace sgm {
namespace sweep {

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }

template <int N>
__device__ __forceinline__ void ldrow(double (&c)[N], const double* p) {
#pragma unroll
  for (int q = 0; q < N / 2; ++q) {
    const double2 t = ld2(p + 2 * q);
    c[2 * q] = t.x;
    c[2 * q + 1] = t.y;
  }
}

// Geometry of one component in one pass (host-computed, 32-bit: components have < 2^31 elements).
struct CompGeom {
  unsigned magic;  // floor((2^32 - 1) / X): l / X by multiply-high + one correction
  int L;       // line length
  int nlines;  // number of lines
  int X;       // strided: line l -> (l % X, l / X); x axis: unused
  int gs;      // element stride along the line
  int os;      // strided: stride of the transverse index l / X
  int rowlen;  // x axis: row length (= L)
};

struct Cfg {
  int NC, NP;     // consumer (segment) warps, producer warps
  int bulk;       // x axis only: 1 = whole-tile bulk copies (TMA engine) in and out, 0 = cp.async
  int W;          // strided slab row width (doubles)
  int rows;       // slab rows per line R = NC*SEG + P
  int pitch;      // x axis: slab pitch (odd >= rows)
  int slab;       // doubles per slab
  int tab_dbl;    // doubles per staged table
  int ntabs;      // distinct tables (1 or 2)
  int dbg;        // tuning only (SGM_PIPE_DBG): bit 0 consumers skip work, bit 1 producers skip loads
  int nitems;     // tiles over all components
  int tiles[3];   // tiles per component
  CompGeom g[3];
  // fused update (MODE 1/2): per output component c, the two curl terms
  // term t: sign * (src[t][idx_hi] - src[t][idx_lo]); see host make_update_terms
  struct Term {
    const double* src;
    int X, Y;     // src extents x, y (for index arithmetic)
    int ext_a;    // src extent along the differentiated axis (primal bound checks)
    int a;        // differentiated axis
    int sign;     // +1 / -1
  } term[3][2];
};

// l -> (l % X, l / X) without a division instruction sequence
__device__ __forceinline__ void divmod_x(const CompGeom& g, int l, int& x, int& o) {
  const unsigned ul = unsigned(l), uX = unsigned(g.X);
  unsigned q = __umulhi(ul, g.magic);
  unsigned r = ul - q * uX;
  if (r >= uX) { ++q; r -= uX; }
  x = int(r);
  o = int(q);
}

__device__ __forceinline__ int line_base(const CompGeom& g, int mode3, int l) {
  if (mode3) return l * g.rowlen;
  int x, o;
  divmod_x(g, l, x, o);
  return x + o * g.os;
}

// ---------------------------------------------------------------------------------------------
// fused Ampere / Faraday update of LPT lines of one tile (strided axis `ax`), rows pw, pw+NP, ...
//   AMPERE : d_c <- d_c + dt ((D~1 h)_c - s j_c)     dual   (dv)_k = v_{k+1} - v_k
//   FARADAY: b_c <- b_c - dt (D1 e)_c                primal (du)_k = u_k - u_{k-1}, u_{-1} = u_a = 0
// (P:L201 incidence; SURVEY 8.0 stencils).  (x, y, z) of element i of line l: ax = 2: (l%X, l/X, i);
// ax = 1: (l%X, i, l/X).
template <int PRO, int LPT>
__device__ __forceinline__ void produce_update(const SweepArgs& A, const Cfg& cfg, int c, int l0, int pw, int NP,
                                               int lane, int ax, int W, double* slab) {
  const CompGeom& g = cfg.g[c];
  const SweepComp& C = A.comp[c];
  constexpr bool DUAL = (PRO == PRO_AMPERE);
  const double dt = A.pro.dt;
  const double* jh = DUAL ? A.pro.jhat[c] : nullptr;
  const double sdt = jh ? dt * (A.pro.s_ptr ? __ldg(A.pro.s_ptr) : 1.0) : 0.0;
  const double* __restrict__ src0 = cfg.term[c][0].src;
  const double* __restrict__ src1 = cfg.term[c][1].src;
  // Per line q and term t: element offsets (from the term's src) of the "hi" and "lo" values at
  // line element 0, and masks that zero invalid primal neighbours (loads are always in bounds:
  // invalid ones are redirected to the element itself).  Along the line axis, bounds are per row.
  int st[LPT], hio[LPT][2], loo[LPT][2];
  double mhi[LPT][2], mlo[LPT][2];
  bool live[LPT];
  int tgs[2], along[2], ext_a[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const auto& T = cfg.term[c][t];
    tgs[t] = (ax == 1) ? T.X : T.X * T.Y;
    along[t] = (T.a == ax);
    ext_a[t] = T.ext_a;
  }
#pragma unroll
  for (int q = 0; q < LPT; ++q) {
    const int l = l0 + lane + 32 * q;
    live[q] = l < g.nlines;
    const int lc = live[q] ? l : g.nlines - 1;
    int x, o;
    divmod_x(g, lc, x, o);  // o = y (ax = 2) or z (ax = 1)
    st[q] = x + o * g.os;
    const int y = (ax == 2) ? o : 0, z = (ax == 2) ? 0 : o;  // line element 0
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const auto& T = cfg.term[c][t];
      const int base = x + T.X * (y + T.Y * z);
      const int da = (T.a == 0) ? 1 : (T.a == 1 ? T.X : T.X * T.Y);
      const int pa = (T.a == 0) ? x : (T.a == 1 ? y : z);
      if (DUAL) {
        hio[q][t] = base + da;  // v(pos + e_a)
        loo[q][t] = base;       // v(pos)
        mhi[q][t] = mlo[q][t] = 1.0;
      } else {
        const bool okh = along[t] || pa < T.ext_a, okl = along[t] || pa >= 1;
        hio[q][t] = okh ? base : (okl ? base - da : 0);  // u(pos)
        loo[q][t] = okl ? base - da : hio[q][t];          // u(pos - e_a)
        mhi[q][t] = okh ? 1.0 : 0.0;
        mlo[q][t] = okl ? 1.0 : 0.0;
      }
    }
  }
  double* __restrict__ state = C.in;
  constexpr int U = 4;
  for (int i0 = pw; i0 < g.L; i0 += U * NP) {
    double vh[U][LPT][2], vl[U][LPT][2], old[U][LPT], jv[U][LPT];
    // all loads of the batch first (straight-line code: U*LPT*6 loads in flight)
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int i = min(i0 + k * NP, g.L - 1);
#pragma unroll
      for (int q = 0; q < LPT; ++q) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const double* __restrict__ sp = t == 0 ? src0 : src1;
          int ih = hio[q][t] + i * tgs[t], il = loo[q][t] + i * tgs[t];
          if (!DUAL && along[t]) {
            // primal along the line: u_i (i < ext_a) and u_{i-1} (i >= 1)
            ih = (i < ext_a[t]) ? ih : il;
            il = (i >= 1) ? il : ih;
          }
          vh[k][q][t] = __ldg(sp + ih);
          vl[k][q][t] = __ldg(sp + il);
        }
        old[k][q] = state[st[q] + i * g.gs];
        jv[k][q] = jh ? __ldg(jh + st[q] + i * g.gs) : 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int i = i0 + k * NP;
#pragma unroll
      for (int q = 0; q < LPT; ++q) {
        double cu = 0.0;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          double h = vh[k][q][t], l = vl[k][q][t];
          if (!DUAL) {
            double mh = mhi[q][t], ml = mlo[q][t];
            if (along[t]) {
              mh = (i < ext_a[t]) ? 1.0 : 0.0;
              ml = (i >= 1) ? 1.0 : 0.0;
            }
            h *= mh;
            l *= ml;
          }
          cu = (t == 0) ? (h - l) : cu - (h - l);
        }
        double val;
        if (DUAL) val = fma(-sdt, jv[k][q], fma(dt, cu, old[k][q]));
        else val = fma(-dt, cu, old[k][q]);
        if (i < g.L) {
          if (live[q]) state[st[q] + i * g.gs] = val;
          slab[i * W + q * 32 + lane] = val;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
template <int P, int SEG, int LPT, int MODE, int OPS>
__global__ void __launch_bounds__(512, 1) sweep_kernel(const __grid_constant__ SweepArgs A, const __grid_constant__ Cfg cfg) {
  using RL = RowLayout<P>;
  constexpr int M = RL::M;
  constexpr int RS = RL::RS;
  constexpr int TW = 32 * LPT;
  constexpr bool XAX = (MODE == 3);
  constexpr bool band = (OPS & 1) != 0, solve = (OPS & 2) != 0;
  extern __shared__ __align__(16) double sm[];
  const int NC = cfg.NC, NP = cfg.NP;
  const int NT = (NC + NP) * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ax = XAX ? 0 : A.axis;
  const bool bulk = cfg.bulk != 0;
  double* tabs = sm;                              // [ntabs][tab_dbl]
  double* slabs = sm + cfg.ntabs * cfg.tab_dbl;   // [2][slab]
  double* tails = slabs + 2 * cfg.slab;           // [NC][M][TW]
  double* heads = tails + NC * M * TW;            // [NC][M][TW]
  unsigned long long* full_mb = reinterpret_cast<unsigned long long*>(heads + NC * M * TW);  // [2]
  const int G = gridDim.x;
  const int R = cfg.rows;
  const int W = cfg.W;  // strided slab row width

  for (int t = 0; t < cfg.ntabs; ++t) {
    const double2* src = reinterpret_cast<const double2*>(A.tabs[t]);
    double2* dst = reinterpret_cast<double2*>(tabs + t * cfg.tab_dbl);
    for (int i = threadIdx.x; i < cfg.tab_dbl / 2; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  // slabs start zeroed: positions never written by a copy hold finite values (zero or stale data),
  // and every coefficient that multiplies such a position is exactly zero
  for (int i = threadIdx.x; i < cfg.slab; i += blockDim.x) slabs[i] = slabs[cfg.slab + i] = 0.0;
  if (threadIdx.x == 0) {
    pipe::mbar_init(full_mb, 1);
    pipe::mbar_init(full_mb + 1, 1);
  }
  pipe::fence_proxy_async_smem();
  __syncthreads();

  if (warp >= NC) {
    // ================================ producers ================================
    const int pw = warp - NC;
    int it = 0;
    for (int item = blockIdx.x; item < cfg.nitems; item += G, ++it) {
      const int buf = it & 1;
      if (it >= 2) pipe::bar_sync(pipe::kBarEmpty0 + buf, NT);
      int c = 0, tile = item;
      while (c < 2 && tile >= cfg.tiles[c]) tile -= cfg.tiles[c++];
      const CompGeom& g = cfg.g[c];
      const SweepComp& C = A.comp[c];
      double* slab = slabs + buf * cfg.slab;
      const int l0 = tile * TW;
      const int cnt = min(TW, g.nlines - l0);
      if (bulk) {
        // one producer warp drives the bulk-copy engine; completion is counted on full_mb[buf]
        if (pw == 0) {
          if (lane == 0) {
            const unsigned bytes = unsigned(cnt) * unsigned(g.X) * 8u;
            pipe::mbar_arrive_expect_tx(full_mb + buf, (cfg.dbg & 2) ? 0u : bytes);
            if (!(cfg.dbg & 2)) pipe::bulk_g2s(slab, C.in + long(l0) * g.X, bytes, full_mb + buf);
          }
        }
        continue;
      }
      if (cfg.dbg & 2) {
      } else if (XAX) {
        const int pitch = cfg.pitch;
        for (int j = pw; j < TW; j += NP) {
          const int l = l0 + j;
          double* srow = slab + j * pitch;
          if (l < g.nlines) {
            const double* src = C.in + long(l) * g.rowlen;
            for (int k = lane; k < g.L; k += 32) pipe::cp_async8(srow + k, src + k);
          }
          for (int k = g.L + lane; k < R; k += 32) srow[k] = 0.0;
        }
      } else {
        if (MODE == 0) {
#pragma unroll
          for (int q = 0; q < LPT; ++q) {
            const int l = l0 + lane + 32 * q;
            double* dst = slab + pw * W + q * 32 + lane;
            if (l < g.nlines) {
              const long gstep = long(NP) * g.gs;
              const double* src = C.in + line_base(g, 0, l) + long(pw) * g.gs;
              for (int i = pw; i < g.L; i += NP, src += gstep, dst += NP * W) pipe::cp_async8(dst, src);
            } else {
              for (int i = pw; i < g.L; i += NP, dst += NP * W) *dst = 0.0;
            }
          }
        } else if (MODE == 1) {
          produce_update<PRO_AMPERE, LPT>(A, cfg, c, l0, pw, NP, lane, ax, W, slab);
        } else {
          produce_update<PRO_FARADAY, LPT>(A, cfg, c, l0, pw, NP, lane, ax, W, slab);
        }
        for (int i = g.L + pw; i < R; i += NP)
#pragma unroll
          for (int q = 0; q < LPT; ++q) slab[i * W + q * 32 + lane] = 0.0;
      }
      pipe::cp_async_wait_all();
      pipe::bar_arrive(pipe::kBarFull0 + buf, NT);
    }
    return;
  }

  // ================================ consumers ================================
  const int s = warp;
  const int r0 = s * SEG;
  int it = 0;
  for (int item = blockIdx.x; item < cfg.nitems; item += G, ++it) {
    const int buf = it & 1;
    if (bulk) pipe::mbar_wait(full_mb + buf, unsigned(it >> 1) & 1u);
    else pipe::bar_sync(pipe::kBarFull0 + buf, NT);
    int c = 0, tile = item;
    while (c < 2 && tile >= cfg.tiles[c]) tile -= cfg.tiles[c++];
    const CompGeom& g = cfg.g[c];
    const SweepComp& C = A.comp[c];
    double* slab = slabs + buf * cfg.slab;
    const double* T = tabs + (cfg.ntabs > 1 ? C.tslot : 0) * cfg.tab_dbl + r0 * RS;  // my segment's rows
    const int l0 = tile * TW;
    const int cnt = min(TW, g.nlines - l0);
    const int L = g.L;
    const int S = (L + SEG - 1) / SEG;
    const bool live = s < S;
    if (cfg.dbg & 1) {
      if (item + 2 * G < cfg.nitems) pipe::bar_arrive(pipe::kBarEmpty0 + buf, NT);
      continue;
    }
    // ---- where line q's element r lives in the slab: base[q][parity of r] + r * ES
    int cbase[LPT][2];
    constexpr int ESX = 1;
    const int ES = XAX ? ESX : W;
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
      const int j = lane + 32 * q;
      if (XAX) {
        cbase[q][0] = cbase[q][1] = j * (bulk ? g.X : cfg.pitch);  // bulk: whole-tile copy, pitch X
      } else {
        cbase[q][0] = cbase[q][1] = j;
      }
    }
    // slab index of line q, segment row k (k may be negative or >= SEG for halos); the column
    // depends on the parity of the global row r0 + k
    int cA[LPT], cB[LPT];
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
      cA[q] = (r0 & 1) ? cbase[q][1] : cbase[q][0];
      cB[q] = (r0 & 1) ? cbase[q][0] : cbase[q][1];
    }
    auto sidx = [&](int q, int k) -> int { return ((k & 1) ? cB[q] : cA[q]) + (r0 + k) * ES; };
    // ---- load segment + halos
    // w: the P original values left of the current row, in rotating slots: original row r (r >= -P,
    // relative to the segment) lives in w[(r + P) % P] (compile-time indices: no register moves).
    double v[SEG][LPT], hr[P][LPT], w[P][LPT];
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
#pragma unroll
      for (int k = 0; k < SEG; ++k) v[k][q] = live ? slab[sidx(q, k)] : 0.0;
      if (band) {
#pragma unroll
        for (int j = 0; j < P; ++j) {
          hr[j][q] = live ? slab[sidx(q, SEG + j)] : 0.0;
          w[j][q] = (live && s > 0) ? slab[sidx(q, j - P)] : 0.0;  // row j - P -> slot j
        }
      }
    }
    // ---- phase A: band mat-vec fused with the zero-history forward substitution
#pragma unroll
    for (int k = 0; k < SEG; ++k) {
      const double* row = T + k * RS;
      double y[LPT];
      if (band) {
        double cb[2 * P + 2];
        ldrow(cb, row + RL::BAND);
#pragma unroll
        for (int q = 0; q < LPT; ++q) {
          double ls = 0.0, rs = 0.0;
#pragma unroll
          for (int j = 1; j <= P; ++j) {
            ls = fma(cb[P - j], w[(k - j + P) % P][q], ls);  // original row k - j
            const double xr = (k + j < SEG) ? v[k + j][q] : hr[k + j - SEG][q];
            rs = fma(cb[P + j], xr, rs);
          }
          y[q] = fma(cb[P], v[k][q], ls + rs);
          w[k % P][q] = v[k][q];  // original row k replaces row k - P
        }
      } else {
#pragma unroll
        for (int q = 0; q < LPT; ++q) y[q] = v[k][q];
      }
      if (solve) {
        double lo[RL::LW];
        ldrow(lo, row + RL::LO);
#pragma unroll
        for (int q = 0; q < LPT; ++q) {
          double z = y[q];
#pragma unroll
          for (int j = M; j >= 1; --j)
            if (k - j >= 0) z = fma(-lo[j - 1], v[k - j][q], z);
          v[k][q] = z;
        }
      } else {
#pragma unroll
        for (int q = 0; q < LPT; ++q) v[k][q] = y[q];
      }
    }
    if (solve) {
      // ---- phase B: tails -> true history z_{r0-1..r0-M}
#pragma unroll
      for (int j = 1; j <= M; ++j)
#pragma unroll
        for (int q = 0; q < LPT; ++q) tails[(s * M + j - 1) * TW + q * 32 + lane] = v[SEG - j][q];
      pipe::bar_sync(pipe::kBarCons, NC * 32);
      double hist[M][LPT];
#pragma unroll
      for (int j = 0; j < M; ++j)
#pragma unroll
        for (int q = 0; q < LPT; ++q) hist[j][q] = 0.0;
      const double* T0 = tabs + (cfg.ntabs > 1 ? C.tslot : 0) * cfg.tab_dbl;
      for (int t = 0; t < s; ++t) {
        double nh[M][LPT];
#pragma unroll
        for (int j = 1; j <= M; ++j) {
          double f[RL::LW];
          ldrow(f, T0 + (t * SEG + SEG - j) * RS + RL::F);
#pragma unroll
          for (int q = 0; q < LPT; ++q) {
            double val = tails[(t * M + j - 1) * TW + q * 32 + lane];
#pragma unroll
            for (int i = 1; i <= M; ++i) val = fma(f[i - 1], hist[i - 1][q], val);
            nh[j - 1][q] = val;
          }
        }
#pragma unroll
        for (int j = 0; j < M; ++j)
#pragma unroll
          for (int q = 0; q < LPT; ++q) hist[j][q] = nh[j][q];
      }
      // ---- phase C: spike-corrected backward substitution (zero future); segment 0 has
      // hist = 0, the correction is applied uniformly (no divergent code path)
#pragma unroll
      for (int k = SEG - 1; k >= 0; --k) {
        const double* row = T + k * RS;
        double up[RL::UW], f[RL::LW];
        ldrow(up, row + RL::UP);
        ldrow(f, row + RL::F);
#pragma unroll
        for (int q = 0; q < LPT; ++q) {
          double z = v[k][q];
#pragma unroll
          for (int i = 1; i <= M; ++i) z = fma(f[i - 1], hist[i - 1][q], z);
          double u = z * up[0];
#pragma unroll
          for (int j = M; j >= 1; --j)
            if (k + j < SEG) u = fma(-up[j], v[k + j][q], u);
          v[k][q] = u;
        }
      }
      // ---- phase D: heads -> true future u_{r1+1..r1+M}
#pragma unroll
      for (int j = 1; j <= M; ++j)
#pragma unroll
        for (int q = 0; q < LPT; ++q) heads[(s * M + j - 1) * TW + q * 32 + lane] = v[j - 1][q];
      pipe::bar_sync(pipe::kBarCons, NC * 32);
      if (s < S - 1) {
        double fut[M][LPT];
#pragma unroll
        for (int j = 0; j < M; ++j)
#pragma unroll
          for (int q = 0; q < LPT; ++q) fut[j][q] = 0.0;
        for (int t = S - 1; t > s; --t) {
          double nf[M][LPT];
#pragma unroll
          for (int j = 1; j <= M; ++j) {
            double b[RL::LW];
            ldrow(b, T0 + (t * SEG + j - 1) * RS + RL::B);
#pragma unroll
            for (int q = 0; q < LPT; ++q) {
              double val = heads[(t * M + j - 1) * TW + q * 32 + lane];
#pragma unroll
              for (int i = 1; i <= M; ++i) val = fma(b[i - 1], fut[i - 1][q], val);
              nf[j - 1][q] = val;
            }
          }
#pragma unroll
          for (int j = 0; j < M; ++j)
#pragma unroll
            for (int q = 0; q < LPT; ++q) fut[j][q] = nf[j][q];
        }
#pragma unroll
        for (int k = 0; k < SEG; ++k) {
          double b[RL::LW];
          ldrow(b, T + k * RS + RL::B);
#pragma unroll
          for (int q = 0; q < LPT; ++q) {
            double u = v[k][q];
#pragma unroll
            for (int i = 1; i <= M; ++i) u = fma(b[i - 1], fut[i - 1][q], u);
            v[k][q] = u;
          }
        }
      }
    }
    // ---- phase E: scaled store
    const double sc = C.scale;
    if (!XAX) {
      if (live) {
#pragma unroll
        for (int q = 0; q < LPT; ++q) {
          const int l = l0 + lane + 32 * q;
          if (l < g.nlines) {
            double* dst = C.out + line_base(g, 0, l) + long(r0) * g.gs;
            const long gs = g.gs;
            if (r0 + SEG <= L) {
#pragma unroll
              for (int k = 0; k < SEG; ++k) dst[k * gs] = sc * v[k][q];
            } else {
#pragma unroll
              for (int k = 0; k < SEG; ++k)
                if (r0 + k < L) dst[k * gs] = sc * v[k][q];
            }
          }
        }
      }
    } else {
      if (!solve) pipe::bar_sync(pipe::kBarCons, NC * 32);  // every halo read before in-place writes
      if (live) {
#pragma unroll
        for (int q = 0; q < LPT; ++q)
#pragma unroll
          for (int k = 0; k < SEG; ++k)
            if (r0 + SEG <= L || r0 + k < L) slab[sidx(q, k)] = sc * v[k][q];
      }
      if (bulk) {
        pipe::fence_proxy_async_smem();
        pipe::bar_sync(pipe::kBarCons, NC * 32);
        if (threadIdx.x == 0) {
          pipe::bulk_s2g(C.out + long(l0) * g.X, slab, unsigned(cnt) * unsigned(g.X) * 8u);
          pipe::bulk_commit();
          pipe::bulk_wait_read0();  // the slab may be refilled once its contents have been read
        }
      } else {
        pipe::bar_sync(pipe::kBarCons, NC * 32);
        for (int j = s; j < TW; j += NC) {
          const int l = l0 + j;
          if (l >= g.nlines) break;
          double* dst = C.out + long(l) * g.rowlen;
          const double* srow = slab + j * cfg.pitch;
          for (int k = lane; k < L; k += 32) dst[k] = srow[k];
        }
      }
    }
    if (item + 2 * G < cfg.nitems) pipe::bar_arrive(pipe::kBarEmpty0 + buf, NT);
  }
  if (XAX && bulk && threadIdx.x == 0) pipe::bulk_wait0();
}

}  // namespace sweep
}  // namespace sgm
