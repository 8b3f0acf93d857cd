// Fused leapfrog update + first line sweep of a half step (sm_100a): the hot kernel of the fused
// schedule (SURVEY 8(a) a1+a2+a3 / a4+a5+a6, the fused P1 pass of SURVEY 8(d)).
//
// For every line of every listed component, along that component's sweep axis:
//   u      = state + dt (D~1 h - s j^)_c      (FUSE 1, eq. discrete2_ampere)
//   u      = state - dt (D1 e)_c              (FUSE 2, eq. discrete2_faraday)
//   state <- u                                 (in place: the state is read only by its own line)
//   out    = scale * dline0[t0] * dline1[t1] * A^{-1} (B u)
// with B the banded Gram factor and A = LU the banded pairing factor of the sweep axis (mode-wise
// Kronecker inverse, eq. kroninverse, vec trick P:L575-585; no-pivot LU, reading Z14),
// solved in partitioned (SPIKE) form (seg_sweep.cuh).  The curl is the integer incidence stencil
// (P:L201): each term is the difference of a source component at two points one step
// apart along the differentiated axis -- along the line (rows r, r +- 1), across lanes (t0 +- 1)
// or across lines (t1 +- 1).
//
// A CTA is persistent: NC consumer warps (one per SPIKE segment of SEG rows; lane j owns line
// t0s + j of the tile) and np producer warps.  Per tile of 32 lines the producers stream the
// state, j^ and every curl-source run the tile needs into shared memory, completion counted on
// one mbarrier: strided (y/z) lines by 16-byte LDGSTS copies, one warp per staged row of 32-34
// consecutive x (small per-row bulk copies were measured ~10x slower: the TMA engine's request
// rate, not bandwidth, bounds them), x lines by one bulk copy (TMA engine) of the tile's
// contiguous lines.  Consumers
// compute the update of their rows (and HB halo rows) from shared memory, store the updated
// state, release the staging buffers (the producer then streams the next tile while the SPIKE
// phases run on registers), and store the swept line.
#pragma once

#include "check.cuh"
#include "kernels.cuh"
#include "pipe_sweep.cuh"
#include "seg_sweep.cuh"

namespace sgm {
namespace fsweep {

constexpr int kMaxStages = 5;

// One staged source array of a component: for the tile (t1, lanes t0s + [lane_lo, lane_lo + nl)),
// rows [row_lo, row_lo + nrow) of the source line at t1 + dt1.
struct Stage {
  const double* src;
  int st0, st1, gs;     // source element strides of t0, t1 and along the line
  int dt1;              // line shift across lines (-1, 0, +1)
  int lane_lo, nl;      // staged lanes: [lane_lo, lane_lo + nl)
  int row_lo, nrow;     // staged rows (strided mode)
  int ext0, ext1;       // source extents along t0, t1 (copies are clamped to them)
  int pitch;            // strided: doubles per staged row
  int soff;             // offset (doubles) of this array in the staging area
};

// A read of the update: staged array `st`, shifted by dlane lanes and drow rows; `valid`: primal
// PEC bound on the coordinate along the differentiated axis (where: 0 row, 1 t0, 2 t1;
// lo_ok: coordinate >= 1, hi_ok: coordinate < ext).
struct Read {
  int st, dlane, drow;
};
struct Term {
  Read hi, lo;
  int where;  // differentiated axis relative to the line: 0 along, 1 = t0, 2 = t1
  int ext_a;  // source extent along it (primal bounds)
};

struct Comp {
  double* state;         // updated in place
  double* out;           // sweep output
  const double* dline[2];
  double scale;
  int xmode;             // 1: x lines (lines contiguous), 0: strided y/z lines
  int L;                 // line length
  int TD, n1;            // t0 extent (lanes) and t1 extent; tiles = n1 * ceil(TD / 32)
  int tpr;               // tiles per t1 row = ceil(TD / 32)
  int st0, st1, gs;      // state strides (t0, t1, along)
  int nst;               // staged arrays: the state (if ost >= 0), j^ (if jst >= 0), then curl sources
  int ost, jst;          // stage of the old state / of j^ (-1: none)
  int accum;             // 1: out += scale * result ((e,h) state), 0: out = scale * result
  Stage s[kMaxStages];
  Term t[2];
  int tslot;
  int tiles;
};

struct Args {
  Comp comp[3];
  int ncomp;
  const double* tabs[2];
  int ntabs, tab_dbl;
  int spike_kh, spike_kf;
  int nitems;
  int reverse;
  int stage_dbl;         // doubles of the staging area
  int np;                // producer warps
  const double* s_ptr;   // Ampere amplitude s_k (device) or null (-> 1)
  double dt;
  unsigned* ck;          // verification build (check.cuh): violation counters; unused otherwise
};

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
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mb, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(pipe::smem_u32(mb)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(pipe::smem_u32(smem)), "l"(gmem) : "memory");
}
// arrives on mb once every cp.async issued so far by this thread has completed (the mbarrier's
// expected arrival count includes this thread: .noinc)
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* mb) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(pipe::smem_u32(mb)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(pipe::smem_u32(mb)) : "memory");
}

// tile -> (component, t1, first t0)
__device__ __forceinline__ void tile_of(const Args& A, int item, int& c, int& t1, int& t0s) {
  int tile = A.reverse ? A.nitems - 1 - item : item;
  c = 0;
  while (c < A.ncomp - 1 && tile >= A.comp[c].tiles) tile -= A.comp[c++].tiles;
  const Comp& C = A.comp[c];
  t1 = tile / C.tpr;
  t0s = (tile - t1 * C.tpr) * 32;
}

template <int P, int HB, int SEG, int FUSE>
__global__ void __launch_bounds__(480, 1) fsweep_kernel(const __grid_constant__ Args A) {
  using RL = RowLayout<P>;
  constexpr int M = RL::M;
  constexpr int RS = RL::RS;
  static_assert(HB >= 1 && HB <= P, "band half-width");
  static_assert(FUSE >= 1 && FUSE <= 4, "fused kernel");
  // FUSE 1 / 2: state update (Ampere / Faraday); 3 / 4: the increments alone (the (e,h)-state step
  // e += dt S_eps(D~1 h - s j^), h -= dt S_mu(D1 e), sgm_step_eh): no state read or written
  constexpr bool DUAL = (FUSE == 1 || FUSE == 3);
  constexpr bool INC = (FUSE >= 3);
  extern __shared__ __align__(16) double sm[];
  const int NC = (blockDim.x >> 5) - A.np;  // consumer warps; the last np warps produce
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* tabs = sm;                                   // [ntabs][tab_dbl]
  double* stg = tabs + A.ntabs * A.tab_dbl;            // staging area
  double* tails = stg + A.stage_dbl;                   // [NC][M][32]
  double* heads = tails + NC * M * 32;                 // [NC][M][32]
  unsigned long long* mb = reinterpret_cast<unsigned long long*>(heads + NC * M * 32);  // tab, full, empty
  unsigned long long *tab_mb = mb, *full_mb = mb + 1, *empty_mb = mb + 2;
#ifdef SGM_CHECKED
  int* rel = reinterpret_cast<int*>(mb + 3);  // consumer-warp releases of the staging area
  if (threadIdx.x == 0) *rel = 0;
#endif
  pipe::griddep_launch_dependents();
  if (threadIdx.x == 0) {
    pipe::mbar_init(tab_mb, 1);
    pipe::mbar_init(full_mb, A.np * 32);
    pipe::mbar_init(empty_mb, NC);
  }
  pipe::fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    pipe::mbar_arrive_expect_tx(tab_mb, unsigned(A.ntabs * A.tab_dbl) * 8u);
    for (int t = 0; t < A.ntabs; ++t) pipe::bulk_g2s(tabs + t * A.tab_dbl, A.tabs[t], unsigned(A.tab_dbl) * 8u, tab_mb);
  }
  pipe::griddep_wait();  // inputs are written by the previous kernel in the stream
  const int G = gridDim.x;

  if (warp >= NC) {
    // ================================ producers ================================
    // strided stages: LDGSTS 16-byte copies, one warp per staged row (lanes on the row's chunks),
    // completion by cp.async.mbarrier.arrive.noinc of every producer thread; x-line stages: one
    // bulk copy each (TMA engine) counted as transaction bytes on the same mbarrier
    const int pw = warp - NC;
    int it = 0;
    for (int item = blockIdx.x; item < A.nitems; item += G, ++it) {
      if (it > 0) pipe::mbar_wait(empty_mb, unsigned(it - 1) & 1u);
#ifdef SGM_CHECKED
      // every consumer warp released every earlier tile; then poison the staging area
      if (pw == 0 && lane == 0 && *rel != NC * it) check::fail(A.ck, check::kFReleaseCount);
      check::jitter(unsigned(item * 64 + warp));
      for (int i = pw * 32 + lane; i < A.stage_dbl; i += A.np * 32) stg[i] = check::kPoison;
      pipe::fence_proxy_async_smem();
      pipe::bar_sync(2, A.np * 32);
#endif
      int c, t1, t0s;
      tile_of(A, item, c, t1, t0s);
      const Comp& C = A.comp[c];
      for (int si = 0; si < C.nst; ++si) {
        const Stage& S = C.s[si];
        const int tl = t1 + S.dt1;
        if (tl < 0 || tl >= S.ext1) continue;  // the shifted line does not exist: never read
        const int base0 = (t0s + S.lane_lo) * S.st0 + tl * S.st1;
        const int lo0 = tl * S.st1;  // element index of t0 = 0 on this line (row 0)
        if (C.xmode) {
          // the tile's lines are one contiguous range [base0, base0 + nl * st0) (clamped)
          if (pw == 0 && lane == 0) {
            const int G0 = base0 & ~1;
            int cs = base0 > lo0 ? base0 : lo0;
            int ce = base0 + S.nl * S.st0;
            const int hi0 = lo0 + S.ext0 * S.st0;
            ce = ce < hi0 ? ce : hi0;
            cs &= ~1;
            ce = (ce + 1) & ~1;
            if (ce > cs) {
              const unsigned bytes = unsigned(ce - cs) * 8u;
              mbar_expect_tx(full_mb, bytes);
              pipe::bulk_g2s(stg + S.soff + (cs - G0), S.src + cs, bytes, full_mb);
            }
          }
        } else {
          // one run of consecutive t0 per staged row: [g + d0, g + d1) of row r (g = lane_lo)
          const int a0 = t0s + S.lane_lo;
          const int d0 = (a0 > 0 ? a0 : 0) - a0, d1 = (a0 + S.nl < S.ext0 ? a0 + S.nl : S.ext0) - a0;
          if (d1 <= d0) continue;
          int g = base0 + (S.row_lo + pw) * S.gs;
          int dst = S.soff + pw * S.pitch;
          const int gstep = A.np * S.gs, dstep = A.np * S.pitch;
          for (int r = S.row_lo + pw; r < S.row_lo + S.nrow; r += A.np, g += gstep, dst += dstep) {
            const int cs = (g + d0) & ~1, ce = (g + d1 + 1) & ~1;
            if (2 * lane < ce - cs) cp_async16(stg + dst + (cs - (g & ~1)) + 2 * lane, S.src + cs + 2 * lane);
          }
        }
      }
      cp_async_mbar_arrive(full_mb);
    }
    return;
  }

  // ================================ consumers ================================
  const int s = warp;
  const int r0 = s * SEG;
  const double dt = A.dt;
  const double sdt = DUAL ? dt * (A.s_ptr ? __ldg(A.s_ptr) : 1.0) : 0.0;
  pipe::mbar_wait(tab_mb, 0);
  int it = 0;
  for (int item = blockIdx.x; item < A.nitems; item += G, ++it) {
    int c, t1, t0s;
    tile_of(A, item, c, t1, t0s);
    const Comp& C = A.comp[c];
    const int L = C.L;
    const int S = (L + SEG - 1) / SEG;
    const int t0 = t0s + lane;
    const bool lok = t0 < C.TD;
    const int xm = C.xmode;
    // per-tile read descriptors: the staged position of (this lane + dlane, row r + drow) is
    // q + r * rs + ((par + r * go) & 1)  (strided arrays: pitch rows, the row's copy starts at the
    // even element at or below lane_lo; x arrays: one contiguous block of lines)
    struct RD {
      int q, rs, pe, po;  // at row r0 + k: q + k * rs + (k odd ? po : pe)
    };
    auto mk = [&](const Read& R) -> RD {
      const Stage& G = C.s[R.st];
      const int b0 = (t0s + G.lane_lo) * G.st0 + (t1 + G.dt1) * G.st1;
      RD d;
      if (xm) {
        d.q = G.soff + (b0 & 1) + (lane + R.dlane - G.lane_lo) * G.st0 + R.drow + r0;
        d.rs = 1;
        d.pe = d.po = 0;
      } else {
        d.q = G.soff + (R.drow - G.row_lo) * G.pitch + (lane + R.dlane - G.lane_lo) + r0 * G.pitch;
        d.rs = G.pitch;
        const int par = b0 + (R.drow + r0) * G.gs;
        d.pe = par & 1;
        d.po = (par + G.gs) & 1;
      }
      return d;
    };
    const RD rold = mk(Read{C.ost >= 0 ? C.ost : 0, 0, 0});
    const RD rj = mk(Read{C.jst >= 0 ? C.jst : 0, 0, 0});
    const RD rh0 = mk(C.t[0].hi), rl0 = mk(C.t[0].lo), rh1 = mk(C.t[1].hi), rl1 = mk(C.t[1].lo);
    // primal PEC bounds of the transverse terms (constant per line); along-line terms check the row
    bool al[2], hok[2], lk[2];
    int exa[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const Term& T = C.t[k];
      al[k] = T.where == 0;
      const int ca = T.where == 1 ? t0 : t1;
      exa[k] = T.ext_a;
      hok[k] = ca < T.ext_a;
      lk[k] = ca >= 1;
    }
    pipe::mbar_wait(full_mb, unsigned(it) & 1u);
    // ---- the fused update of rows r0 - HB .. r0 + SEG + HB - 1 from the staged arrays
    auto upd = [&](int k) -> double {  // row r0 + k (k compile-time after unrolling)
      const int r = r0 + k;
      if (!lok || r < 0 || r >= L) return 0.0;
      auto at = [&](const RD& d) { return stg[d.q + k * d.rs + ((k & 1) ? d.po : d.pe)]; };
      const double old = INC ? 0.0 : at(rold);
      double cu[2];
      const RD* H[2] = {&rh0, &rh1};
      const RD* O[2] = {&rl0, &rl1};
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        double hi, lo;
        if (DUAL) {       // dual: (dv)_j = v_{j+1} - v_j
          hi = at(*H[t]);
          lo = at(*O[t]);
        } else {          // primal: (du)_j = u_j - u_{j-1}, u_{-1} = u_a = 0 (PEC)
          hi = (al[t] ? r < exa[t] : hok[t]) ? at(*H[t]) : 0.0;
          lo = (al[t] ? r >= 1 : lk[t]) ? at(*O[t]) : 0.0;
        }
        cu[t] = hi - lo;
      }
      const double cc = cu[0] - cu[1];
      if (DUAL) {
        const double jv = C.jst >= 0 ? at(rj) : 0.0;
        return fma(-sdt, jv, fma(dt, cc, old));
      }
      return fma(-dt, cc, old);
    };
    double v[SEG], hr[HB], w[HB];
#pragma unroll
    for (int k = 0; k < SEG; ++k) v[k] = upd(k);
#pragma unroll
    for (int j = 0; j < HB; ++j) hr[j] = upd(SEG + j);
#pragma unroll
    for (int j = 0; j < HB; ++j) w[j] = upd(j - HB);
    // staging no longer needed by this warp: release it (the producer streams the next tile)
    __syncwarp();
#ifdef SGM_CHECKED
    if (lane == 0) atomicAdd(rel, 1);
    check::jitter(unsigned(item * 64 + warp + 16));
#endif
    if (lane == 0) mbar_arrive(empty_mb);
    // updated state rows of this segment (read by no other line: stored directly)
    if (!INC && lok && s < S) {
      double* dst = C.state + (long(t0) * C.st0 + long(t1) * C.st1 + long(r0) * C.gs);
      const long gs = C.gs;
#pragma unroll
      for (int k = 0; k < SEG; ++k)
        if (r0 + k < L) dst[k * gs] = v[k];
    }
    const double* T = tabs + (A.ntabs > 1 ? C.tslot : 0) * A.tab_dbl + r0 * RS;  // my segment's rows
    // ---- phase A: band mat-vec fused with the zero-history forward substitution
#pragma unroll
    for (int k = 0; k < SEG; ++k) {
      const double* row = T + k * RS;
      constexpr int PA = (P - HB) / 2, PB = (P + HB) / 2;
      double cb[2 * P + 2];
#pragma unroll
      for (int t = PA; t <= PB; ++t) {
        const double2 c2 = ld2(row + RL::BAND + 2 * t);
        cb[2 * t] = c2.x;
        cb[2 * t + 1] = c2.y;
      }
      double ls = 0.0, rs = 0.0;
#pragma unroll
      for (int j = 1; j <= HB; ++j) {
        ls = fma(cb[P - j], w[(k - j + HB) % HB], ls);  // original row k - j
        const double xr = (k + j < SEG) ? v[k + j] : hr[k + j - SEG];
        rs = fma(cb[P + j], xr, rs);
      }
      const double y = fma(cb[P], v[k], ls + rs);
      w[k % HB] = v[k];  // original row k replaces row k - HB
      double lo[RL::LW];
      ldrow(lo, row + RL::LO);
      double z = y;
#pragma unroll
      for (int j = M; j >= 1; --j)
        if (k - j >= 0) z = fma(-lo[j - 1], v[k - j], z);
      v[k] = z;
    }
    // ---- phase B: tails -> true history z_{r0-1..r0-M}
#pragma unroll
    for (int j = 1; j <= M; ++j) tails[(s * M + j - 1) * 32 + lane] = v[SEG - j];
    pipe::bar_sync(1, NC * 32);
    double hist[M];
#pragma unroll
    for (int j = 0; j < M; ++j) hist[j] = 0.0;
    const double* T0 = tabs + (A.ntabs > 1 ? C.tslot : 0) * A.tab_dbl;
    {
      const int tb = max(0, s - A.spike_kh);  // truncated SPIKE (reading Z23)
      const double* tr = T0 + (tb * SEG + SEG - 1) * RS + RL::F;
      const double* tl = tails + tb * M * 32 + lane;
      for (int t = tb; t < s; ++t, tr += SEG * RS, tl += M * 32) {
        double nh[M];
#pragma unroll
        for (int j = 1; j <= M; ++j) {
          double f[RL::LW];
          ldrow(f, tr - (j - 1) * RS);
          double val = tl[(j - 1) * 32];
#pragma unroll
          for (int i = 1; i <= M; ++i) val = fma(f[i - 1], hist[i - 1], val);
          nh[j - 1] = val;
        }
#pragma unroll
        for (int j = 0; j < M; ++j) hist[j] = nh[j];
      }
    }
    // ---- phase C: spike-corrected backward substitution (zero future)
#pragma unroll
    for (int k = SEG - 1; k >= 0; --k) {
      const double* row = T + k * RS;
      double up[RL::UW], f[RL::LW];
      ldrow(up, row + RL::UP);
      ldrow(f, row + RL::F);
      double z = v[k];
#pragma unroll
      for (int i = 1; i <= M; ++i) z = fma(f[i - 1], hist[i - 1], z);
      double u = z * up[0];
#pragma unroll
      for (int j = M; j >= 1; --j)
        if (k + j < SEG) u = fma(-up[j], v[k + j], u);
      v[k] = u;
    }
    // ---- phase D: heads -> true future u_{r1+1..r1+M}
#pragma unroll
    for (int j = 1; j <= M; ++j) heads[(s * M + j - 1) * 32 + lane] = v[j - 1];
    pipe::bar_sync(1, NC * 32);
    if (s < S - 1) {
      double fut[M];
#pragma unroll
      for (int j = 0; j < M; ++j) fut[j] = 0.0;
      const int te = min(S - 1, s + A.spike_kf);
      const double* br = T0 + te * SEG * RS + RL::B;
      const double* hd = heads + te * M * 32 + lane;
      for (int t = te; t > s; --t, br -= SEG * RS, hd -= M * 32) {
        double nf[M];
#pragma unroll
        for (int j = 1; j <= M; ++j) {
          double b[RL::LW];
          ldrow(b, br + (j - 1) * RS);
          double val = hd[(j - 1) * 32];
#pragma unroll
          for (int i = 1; i <= M; ++i) val = fma(b[i - 1], fut[i - 1], val);
          nf[j - 1] = val;
        }
#pragma unroll
        for (int j = 0; j < M; ++j) fut[j] = nf[j];
      }
#pragma unroll
      for (int k = 0; k < SEG; ++k) {
        double b[RL::LW];
        ldrow(b, T + k * RS + RL::B);
        double u = v[k];
#pragma unroll
        for (int i = 1; i <= M; ++i) u = fma(b[i - 1], fut[i - 1], u);
        v[k] = u;
      }
    }
    // ---- phase E: scaled store
    if (lok && s < S) {
      double sc = C.scale;
      if (C.dline[0]) sc *= __ldg(C.dline[0] + t0);
      if (C.dline[1]) sc *= __ldg(C.dline[1] + t1);
      double* dst = C.out + (long(t0) * C.st0 + long(t1) * C.st1 + long(r0) * C.gs);
      const long gs = C.gs;
      if (C.accum) {
#pragma unroll
        for (int k = 0; k < SEG; ++k)
          if (r0 + k < L) dst[k * gs] = fma(sc, v[k], dst[k * gs]);
      } else if (r0 + SEG <= L) {
#pragma unroll
        for (int k = 0; k < SEG; ++k) dst[k * gs] = sc * v[k];
      } else {
#pragma unroll
        for (int k = 0; k < SEG; ++k)
          if (r0 + k < L) dst[k * gs] = sc * v[k];
      }
    }
  }
}

}  // namespace fsweep
}  // namespace sgm
