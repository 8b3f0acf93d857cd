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
// A CTA is persistent and loops over tiles with two shared-memory slabs (one when the lines are
// too long for two: loads and compute of a CTA then alternate):
//   * producer warps stage tile t+1 into slab[(t+1)&1]: cp.async (LDGSTS) copies for strided axes,
//     one bulk copy (TMA engine, mbarrier completion) per tile of whole x-lines; x tiles are also
//     stored by the producer warp (bulk copy out of the slab the consumers wrote in place);
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

#include "check.cuh"
#include "kernels.cuh"
#include "pipe_sweep.cuh"
#include "seg_sweep.cuh"

namespace sgm {
namespace sweep {

// history / future scan steps unrolled (the truncated reach is 2-3 segments at p = 3)
constexpr int kScanUnroll = 3;

#ifdef SGM_TUNING
#define SGM_TRACE(it, ev)                                                                          \
  do {                                                                                            \
    if (cfg.trace && lane == 0 && blockIdx.x < 160 && (it) < 16)                                  \
      cfg.trace[(size_t(blockIdx.x) * 16 + (it)) * 8 + (ev)] = gtimer();                          \
  } while (0)
#else
#define SGM_TRACE(it, ev) \
  do {                    \
  } while (0)
#endif

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
  int TD;      // transverse divisor: line l -> (t0, t1) = (l % TD, l / TD)
  unsigned tmagic;  // floor((2^32 - 1) / TD)
  int bpitch;  // x axis, bulk: slab pitch of this component's lines (= L, or L + 2 when L % 4 == 0)
  int lbulk;   // x axis, bulk: 1 = one bulk copy per line (padded pitch), 0 = one per tile
  int row0;    // window of a long line: first line element swept (0 = whole line)
  int slo, shi;  // rows of the (window) line that are stored: [slo, shi)
};

struct Cfg {
  int NC, NP;     // consumer (segment) warps, producer warps
  int bulk;       // x axis only: 1 = whole-tile bulk copies (TMA engine) in and out, 0 = cp.async
  int W;          // strided slab row width (doubles)
  int rows;       // slab rows per line R = NC*SEG + P
  int pitch;      // x axis: slab pitch (odd >= rows)
  int slab;       // doubles per slab
  int nslab;      // 2: double-buffered slabs; 1: one slab (lines too long for two)
  int tab_dbl;    // doubles per staged table
  int ntabs;      // distinct tables (1 or 2)
  int dbg;        // tuning only (SGM_PIPE_DBG): bit 0 consumers skip work, bit 1 producers skip loads
  int reverse;    // walk the tiles last-to-first (L2 reuse of what the previous kernel wrote last)
  int nitems;     // tiles over all components
  int tiles[3];   // tiles per component
  CompGeom g[3];
  unsigned* ck;   // verification build (check.cuh): violation counters; unused otherwise
  unsigned long long* trace;  // tuning build: timeline of this launch (check.cuh), or null
  int inject;     // verification build: fault-injection bits
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
template <int P, int HB, int SEG, int LPT, int MODE, int OPS>
__global__ void __launch_bounds__(512, (LPT == 1 ? 2 : 1)) sweep_kernel(const __grid_constant__ SweepArgs A, const __grid_constant__ Cfg cfg) {
  using RL = RowLayout<P>;
  constexpr int M = RL::M;
  constexpr int RS = RL::RS;
  constexpr int TW = 32 * LPT;
  constexpr bool XAX = (MODE == 3);
  constexpr bool band = (OPS & 1) != 0, solve = (OPS & 2) != 0;
  static_assert(HB >= 1 && HB <= P, "band half-width");
  extern __shared__ __align__(16) double sm[];
  const int NC = cfg.NC, NP = cfg.NP;
  const int NT = (NC + NP) * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool bulk = cfg.bulk != 0;
  double* tabs = sm;                              // [ntabs][tab_dbl]
  double* slabs = sm + cfg.ntabs * cfg.tab_dbl;   // [nslab][slab]
  const int NS = cfg.nslab;                       // slabs: 2 (double buffering) or 1 (long lines)
  double* tails = slabs + NS * cfg.slab;          // [NC][M][TW]
  double* heads = tails + NC * M * TW;            // [NC][M][TW]
  unsigned long long* full_mb = reinterpret_cast<unsigned long long*>(heads + NC * M * TW);  // [2] + tables
  const int G = gridDim.x;
  const int R = cfg.rows;
  const int W = cfg.W;  // strided slab row width

  unsigned long long* tab_mb = full_mb + 2;
#ifdef SGM_CHECKED
  // [0,1] item staged in slab b, [2,3] consumer-warp releases of slab b, [4,20) tails tags,
  // [20,36) heads tags (check.cuh)
  int* ckt = reinterpret_cast<int*>(full_mb + 4);
  if (threadIdx.x < check::kSmemInts) ckt[threadIdx.x] = (threadIdx.x < 2 || threadIdx.x >= 4) ? -1 : 0;
#endif
  pipe::griddep_launch_dependents();
  // slabs start zeroed: positions never written by a copy hold finite values (zero or stale data),
  // and every coefficient that multiplies such a position is exactly zero
  {
    double2* s2 = reinterpret_cast<double2*>(slabs);
    const double2 z2 = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int i = threadIdx.x; i < NS * cfg.slab / 2; i += blockDim.x) s2[i] = z2;
  }
  if (threadIdx.x == 0) {
    pipe::mbar_init(full_mb, 1);
    pipe::mbar_init(full_mb + 1, 1);
    pipe::mbar_init(tab_mb, 1);
  }
  pipe::fence_proxy_async_smem();
  __syncthreads();
  // the line-operator table(s) of this pass (constant: staged before waiting on the previous kernel)
  if (threadIdx.x == 0) {
    pipe::mbar_arrive_expect_tx(tab_mb, unsigned(cfg.ntabs * cfg.tab_dbl) * 8u);
    for (int t = 0; t < cfg.ntabs; ++t)
      pipe::bulk_g2s(tabs + t * cfg.tab_dbl, A.tabs[t], unsigned(cfg.tab_dbl) * 8u, tab_mb);
  }
  pipe::griddep_wait();  // inputs are written by the previous kernel in the stream

  if (warp >= NC) {
    // ================================ producers ================================
    const int pw = warp - NC;
    // x axis, bulk: the producer warp also stores each output tile (the consumers wrote it into the
    // slab in place and arrived on EMPTY[slab]); it waits for the copy engine to have read the
    // slab, then refills it -- the consumers never wait for a store to drain
    const bool pst = bulk;
    auto store_tile = [&](int it_s) {
      const int item_s = blockIdx.x + it_s * G;
      int c = 0, tile = cfg.reverse ? cfg.nitems - 1 - item_s : item_s;
      while (c < 2 && tile >= cfg.tiles[c]) tile -= cfg.tiles[c++];
      const CompGeom& g = cfg.g[c];
      const double* slab = slabs + (NS == 2 ? (it_s & 1) : 0) * cfg.slab;
      const int l0 = tile * TW;
      const int cnt = min(TW, g.nlines - l0);
      double* out = A.comp[c].out;
      if (g.lbulk) {
        for (int j = lane; j < cnt; j += 32) pipe::bulk_s2g(out + long(l0 + j) * g.X, slab + j * g.bpitch, unsigned(g.X) * 8u);
        pipe::bulk_commit();
        pipe::bulk_wait_read0();
      } else if (lane == 0) {
        pipe::bulk_s2g(out + long(l0) * g.X, slab, unsigned(cnt) * unsigned(g.X) * 8u);
        pipe::bulk_commit();
        pipe::bulk_wait_read0();  // the slab may be refilled once its contents have been read
      }
      __syncwarp();
    };
    int it = 0;
    for (int item = blockIdx.x; item < cfg.nitems; item += G, ++it) {
      const int buf = NS == 2 ? (it & 1) : 0;
      if (it >= NS) pipe::bar_sync(pipe::kBarEmpty0 + buf, NT);
      if (pst && it >= NS && pw == 0) store_tile(it - NS);
#ifdef SGM_CHECKED
      // every consumer warp has released every earlier use of this slab; then poison it
      if (pw == 0 && lane == 0 && ckt[2 + buf] != NC * (it / NS)) check::fail(cfg.ck, check::kReleaseCount);
      check::jitter(unsigned(item * 64 + warp));
      {
        double* ps = slabs + buf * cfg.slab;
        for (int i = pw * 32 + lane; i < cfg.slab; i += cfg.NP * 32) ps[i] = check::kPoison;
        pipe::fence_proxy_async_smem();
        if (cfg.NP > 1) pipe::bar_sync(6, cfg.NP * 32);
        else __syncwarp();
      }
#endif
      int c = 0, tile = cfg.reverse ? cfg.nitems - 1 - item : item;
      while (c < 2 && tile >= cfg.tiles[c]) tile -= cfg.tiles[c++];
      const CompGeom& g = cfg.g[c];
      const SweepComp& C = A.comp[c];
      double* slab = slabs + buf * cfg.slab;
      const int l0 = tile * TW;
      const int cnt = min(TW, g.nlines - l0);
      if (pw == 0) SGM_TRACE(it, 0);
      if (bulk) {
        // one producer warp drives the bulk-copy engine; completion is counted on full_mb[buf]
        if (pw == 0) {
          const unsigned bytes = unsigned(cnt) * unsigned(g.X) * 8u;
#ifdef SGM_CHECKED
          if (lane == 0) ckt[buf] = item;  // released to the consumers by the arrive below
#endif
          if (lane == 0) pipe::mbar_arrive_expect_tx(full_mb + buf, (cfg.dbg & 2) ? 0u : bytes);
          if (!(cfg.dbg & 2)) {
            if (g.lbulk) {
              // line by line into a padded pitch (an L % 4 == 0 pitch would put every lane's line
              // walk on the same few banks); copy completions may precede the expect: the phase
              // cannot complete before lane 0's arrival
              for (int j = lane; j < cnt; j += 32)
                pipe::bulk_g2s(slab + j * g.bpitch, C.in + long(l0 + j) * g.X, unsigned(g.X) * 8u, full_mb + buf);
            } else if (lane == 0) {
              pipe::bulk_g2s(slab, C.in + long(l0) * g.X, bytes, full_mb + buf);
            }
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
            const double* src = C.in + long(l) * g.rowlen + g.row0;
            for (int k = lane; k < g.L; k += 32) pipe::cp_async8(srow + k, src + k);
          }
          for (int k = g.L + lane; k < R; k += 32) srow[k] = 0.0;
        }
      } else {
        if (MODE == 0) {
          // rows [i0, i1) of every line of the tile; a lane copies its LPT lines, 4 rows per step
          const int rpw = (g.L + NP - 1) / NP;
          const int i0 = pw * rpw, i1 = min(g.L, i0 + rpw);
          const double* src[LPT];
          bool ok[LPT];
#pragma unroll
          for (int q = 0; q < LPT; ++q) {
            const int l = l0 + lane + 32 * q;
            ok[q] = l < g.nlines;
            src[q] = C.in + line_base(g, 0, ok[q] ? l : 0) + long(g.row0 + i0) * g.gs;
          }
          const long gs = g.gs;
          double* dst = slab + i0 * TW + lane;
          int i = i0;
          for (; i + 4 <= i1; i += 4, dst += 4 * TW) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int q = 0; q < LPT; ++q) {
                if (ok[q]) pipe::cp_async8(dst + k * TW + 32 * q, src[q]);
                src[q] += gs;
              }
          }
          for (; i < i1; ++i, dst += TW)
#pragma unroll
            for (int q = 0; q < LPT; ++q) {
              if (ok[q]) pipe::cp_async8(dst + 32 * q, src[q]);
              src[q] += gs;
            }
        }
        for (int i = g.L + pw; i < R; i += NP)
#pragma unroll
          for (int q = 0; q < LPT; ++q) slab[i * W + q * 32 + lane] = 0.0;
      }
      pipe::cp_async_wait_all();
#ifdef SGM_CHECKED
      if (pw == 0 && lane == 0) ckt[buf] = item;
#endif
      if (pw == 0) SGM_TRACE(it, 1);
      pipe::bar_arrive(pipe::kBarFull0 + buf, NT);
    }
    if (pst) {
      // the last (up to NS) output tiles
      for (int k = max(0, it - NS); k < it; ++k) {
        pipe::bar_sync(pipe::kBarEmpty0 + (NS == 2 ? (k & 1) : 0), NT);
        if (pw == 0) store_tile(k);
      }
      if (pw == 0) pipe::bulk_wait0();
    }
    return;
  }

  // ================================ consumers ================================
  const int s = warp;
  const int r0 = s * SEG;
  pipe::mbar_wait(tab_mb, 0);
  int it = 0;
  for (int item = blockIdx.x; item < cfg.nitems; item += G, ++it) {
    const int buf = NS == 2 ? (it & 1) : 0;
    if (s == 0) SGM_TRACE(it, 2);
    if (bulk) pipe::mbar_wait(full_mb + buf, unsigned(NS == 2 ? it >> 1 : it) & 1u);
    else pipe::bar_sync(pipe::kBarFull0 + buf, NT);
    if (s == 0) SGM_TRACE(it, 3);
    // release of the slab to the producers: strided passes as soon as every consumer warp holds its
    // rows in registers (the slab is dead after that: results go straight to global memory, and
    // the producers stage tile t+2 while tile t is computed); x passes after the store (the slab
    // stages the output lines)
    bool released = false;
    auto release = [&]() {
#ifdef SGM_CHECKED
      __syncwarp();
      if (lane == 0) atomicAdd(&ckt[2 + buf], 1);
#endif
      // (producer-side stores take every slab back, the last ones included)
      if ((XAX && bulk) || item + NS * G < cfg.nitems) pipe::bar_arrive(pipe::kBarEmpty0 + buf, NT);
      released = true;
    };
#ifdef SGM_CHECKED
    if (lane == 0 && ckt[buf] != item) check::fail(cfg.ck, check::kStageTag);
    check::jitter(unsigned(item * 64 + warp + 16));
    if (cfg.inject & 1) release();  // injected fault: release before reading
#endif
    int c = 0, tile = cfg.reverse ? cfg.nitems - 1 - item : item;
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
      if (!released) release();
      continue;
    }
    // ---- my lines' segment start in the slab; consecutive line elements are ES apart
    constexpr int ES = XAX ? 1 : TW;
    const int pitch = XAX ? (bulk ? g.bpitch : cfg.pitch) : 0;  // x bulk: line length (or padded)
    const double* cp[LPT];
#pragma unroll
    for (int q = 0; q < LPT; ++q) cp[q] = slab + (XAX ? (lane + 32 * q) * pitch : lane + 32 * q) + r0 * ES;
    // ---- load segment + halos.  Segments past the line end (s >= S) compute on finite padding
    // and store nothing; their spikes are never used by live segments.
    // w: the P original values left of the current row, in rotating slots: original row r (r >= -P,
    // relative to the segment) lives in w[(r + HB) % HB] (compile-time indices: no register moves).
    // HB: half-bandwidth of this pass's banded mat-vec (<= P).
    double v[SEG][LPT], hr[HB][LPT], w[HB][LPT];
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
#pragma unroll
      for (int k = 0; k < SEG; ++k) v[k][q] = cp[q][k * ES];
      if (band) {
#pragma unroll
        for (int j = 0; j < HB; ++j) hr[j][q] = cp[q][(SEG + j) * ES];
        if (s > 0) {
#pragma unroll
          for (int j = 0; j < HB; ++j) w[j][q] = cp[q][(j - HB) * ES];  // row j - HB -> slot j
        } else {
#pragma unroll
          for (int j = 0; j < HB; ++j) w[j][q] = 0.0;
        }
      }
    }
    if (!XAX && !released) release();
    // ---- phase A: band mat-vec fused with the zero-history forward substitution
#pragma unroll
    for (int k = 0; k < SEG; ++k) {
      const double* row = T + k * RS;
      double y[LPT];
      if (band) {
        // coefficients B[r][r+j], j = -HB..HB, sit at band[P + j]: load the 16-byte pairs covering them
        constexpr int PA = (P - HB) / 2, PB = (P + HB) / 2;
        double cb[2 * P + 2];
#pragma unroll
        for (int t = PA; t <= PB; ++t) {
          const double2 c2 = ld2(row + RL::BAND + 2 * t);
          cb[2 * t] = c2.x;
          cb[2 * t + 1] = c2.y;
        }
#pragma unroll
        for (int q = 0; q < LPT; ++q) {
          double ls = 0.0, rs = 0.0;
#pragma unroll
          for (int j = 1; j <= HB; ++j) {
            ls = fma(cb[P - j], w[(k - j + HB) % HB][q], ls);  // original row k - j
            const double xr = (k + j < SEG) ? v[k + j][q] : hr[k + j - SEG][q];
            rs = fma(cb[P + j], xr, rs);
          }
          y[q] = fma(cb[P], v[k][q], ls + rs);
          w[k % HB][q] = v[k][q];  // original row k replaces row k - HB
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
    if (s == 0) SGM_TRACE(it, 4);
    if (solve) {
      // ---- phase B: tails -> true history z_{r0-1..r0-M}
#pragma unroll
      for (int j = 1; j <= M; ++j)
#pragma unroll
        for (int q = 0; q < LPT; ++q) tails[(s * M + j - 1) * TW + q * 32 + lane] = v[SEG - j][q];
#ifdef SGM_CHECKED
      __syncwarp();
      if (lane == 0) ckt[4 + s] = item;
      check::jitter(unsigned(item * 64 + warp + 32));
      if (!(cfg.inject & 2))
#endif
      pipe::bar_sync(pipe::kBarCons, NC * 32);
      if (s == 0) SGM_TRACE(it, 5);
      double hist[M][LPT];
#pragma unroll
      for (int j = 0; j < M; ++j)
#pragma unroll
        for (int q = 0; q < LPT; ++q) hist[j][q] = 0.0;
      const double* T0 = tabs + (cfg.ntabs > 1 ? C.tslot : 0) * cfg.tab_dbl;
      // (truncated SPIKE: segments more than spike_kh back contribute below rounding, host-checked)
      const int tb = (cfg.dbg & 4) ? s : max(0, s - A.spike_kh);  // dbg bit 2: no history scan (timing only)
      // one step of the history recurrence from segment t (its tails, its forward spikes)
      auto hstep = [&](int t) {
#ifdef SGM_CHECKED
        if (lane == 0 && ckt[4 + t] != item) check::fail(cfg.ck, check::kTailTag);
#endif
        const double* tr = T0 + (t * SEG + SEG - 1) * RS + RL::F;  // row SEG - 1 of segment t
        const double* tl = tails + t * M * TW + lane;
        double nh[M][LPT];
#pragma unroll
        for (int j = 1; j <= M; ++j) {
          double f[RL::LW];
          ldrow(f, tr - (j - 1) * RS);
#pragma unroll
          for (int q = 0; q < LPT; ++q) {
            double val = tl[(j - 1) * TW + q * 32];
#pragma unroll
            for (int i = 1; i <= M; ++i) val = fma(f[i - 1], hist[i - 1][q], val);
            nh[j - 1][q] = val;
          }
        }
#pragma unroll
        for (int j = 0; j < M; ++j)
#pragma unroll
          for (int q = 0; q < LPT; ++q) hist[j][q] = nh[j][q];
      };
      // the last kScanUnroll steps unrolled with predication (their loads can all be issued ahead of
      // the dependent FMAs); any older steps by the loop first
      constexpr int KU = kScanUnroll;
      const int tu = (cfg.dbg & 16) ? s : max(tb, s - KU);  // dbg bit 4: no unrolled steps (tuning)
      for (int t = tb; t < tu; ++t) hstep(t);
#pragma unroll
      for (int k = 0; k < KU; ++k)
        if (s - KU + k >= tu) hstep(s - KU + k);
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
#ifdef SGM_CHECKED
      __syncwarp();
      if (lane == 0) ckt[20 + s] = item;
      check::jitter(unsigned(item * 64 + warp + 48));
#endif
      pipe::bar_sync(pipe::kBarCons, NC * 32);
      if (s < S - 1) {
        double fut[M][LPT];
#pragma unroll
        for (int j = 0; j < M; ++j)
#pragma unroll
          for (int q = 0; q < LPT; ++q) fut[j][q] = 0.0;
        const int te = (cfg.dbg & 4) ? s : min(S - 1, s + A.spike_kf);
        auto fstep = [&](int t) {
#ifdef SGM_CHECKED
          if (lane == 0 && ckt[20 + t] != item) check::fail(cfg.ck, check::kHeadTag);
#endif
          const double* br = T0 + t * SEG * RS + RL::B;  // row 0 of segment t
          const double* hd = heads + t * M * TW + lane;
          double nf[M][LPT];
#pragma unroll
          for (int j = 1; j <= M; ++j) {
            double b[RL::LW];
            ldrow(b, br + (j - 1) * RS);
#pragma unroll
            for (int q = 0; q < LPT; ++q) {
              double val = hd[(j - 1) * TW + q * 32];
#pragma unroll
              for (int i = 1; i <= M; ++i) val = fma(b[i - 1], fut[i - 1][q], val);
              nf[j - 1][q] = val;
            }
          }
#pragma unroll
          for (int j = 0; j < M; ++j)
#pragma unroll
            for (int q = 0; q < LPT; ++q) fut[j][q] = nf[j][q];
        };
        constexpr int KU = kScanUnroll;
        const int tu = (cfg.dbg & 16) ? s : min(te, s + KU);
        for (int t = te; t > tu; --t) fstep(t);
#pragma unroll
        for (int k = 0; k < KU; ++k)
          if (s + KU - k <= tu) fstep(s + KU - k);
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
    if (s == 0) SGM_TRACE(it, 6);
    // ---- phase E: scaled store (constant component scale times optional per-line diagonals)
    const double sc = C.scale;
    const bool acc = C.accum != 0;  // out += scale * result (the (e,h)-state increments)
    const bool aff = C.aw[0] != nullptr || C.aw[1] != nullptr;  // + affine boundary terms (lifting)
    double af[2] = {0.0, 0.0};
    if (aff) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
        if (C.aw[i]) af[i] = C.ac[i] * (C.as[i] ? __ldg(C.as[i]) : 1.0);
    }
    const bool unit = (sc == 1.0) && !C.dline[0] && !C.dline[1] && !acc && !aff;
    double scq[LPT];
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
      scq[q] = sc;
      if (C.dline[0] || C.dline[1]) {
        const unsigned l = unsigned(min(l0 + lane + 32 * q, g.nlines - 1));
        unsigned t1 = __umulhi(l, g.tmagic);
        unsigned t0 = l - t1 * unsigned(g.TD);
        if (t0 >= unsigned(g.TD)) { ++t1; t0 -= unsigned(g.TD); }
        if (C.dline[0]) scq[q] *= __ldg(C.dline[0] + t0);
        if (C.dline[1]) scq[q] *= __ldg(C.dline[1] + t1);
      }
    }
    if (!XAX) {
      if (live && !(cfg.dbg & 8)) {  // dbg bit 3: no stores (timing only)
#pragma unroll
        for (int q = 0; q < LPT; ++q) {
          const int l = l0 + lane + 32 * q;
          if (l < g.nlines) {
            double* dst = C.out + line_base(g, 0, l) + long(g.row0 + r0) * g.gs;
            const long gs = g.gs;
            if (acc || aff) {
              const long off = dst - C.out;
              for (int k = 0; k < SEG; ++k, dst += gs)
                if (r0 + k >= g.slo && r0 + k < g.shi) {
                  double val = acc ? fma(scq[q], v[k][q], *dst) : scq[q] * v[k][q];
                  if (C.aw[0]) val = fma(af[0], __ldg(C.aw[0] + off + k * gs), val);
                  if (C.aw[1]) val = fma(af[1], __ldg(C.aw[1] + off + k * gs), val);
                  *dst = val;
                }
            } else if (r0 >= g.slo && r0 + SEG <= g.shi && unit) {
#pragma unroll
              for (int k = 0; k < SEG; ++k, dst += gs) *dst = v[k][q];
            } else if (r0 >= g.slo && r0 + SEG <= g.shi) {
#pragma unroll
              for (int k = 0; k < SEG; ++k, dst += gs) *dst = scq[q] * v[k][q];
            } else {
#pragma unroll
              for (int k = 0; k < SEG; ++k, dst += gs)
                if (r0 + k >= g.slo && r0 + k < g.shi) *dst = scq[q] * v[k][q];
            }
          }
        }
      }
    } else {
      if (!solve) pipe::bar_sync(pipe::kBarCons, NC * 32);  // every halo read before in-place writes
      if (live && !acc && !aff) {
#pragma unroll
        for (int q = 0; q < LPT; ++q) {
          double* cw = const_cast<double*>(cp[q]);
#pragma unroll
          for (int k = 0; k < SEG; ++k)
            if (r0 + SEG <= L || r0 + k < L) cw[k] = scq[q] * v[k][q];
        }
      } else if (live) {
        // accumulate ((e,h)-state increments: the old output line, global, this CTA's lines) and/or
        // the affine boundary terms
        for (int q = 0; q < LPT; ++q) {
          double* cw = const_cast<double*>(cp[q]);
          const int l = min(l0 + lane + 32 * q, g.nlines - 1);
          const long off = long(l) * g.rowlen + g.row0 + r0;
          const double* prev = C.out + off;
          for (int k = 0; k < SEG; ++k)
            if (r0 + k < L) {
              double val = acc ? fma(scq[q], v[k][q], prev[k]) : scq[q] * v[k][q];
              if (C.aw[0]) val = fma(af[0], __ldg(C.aw[0] + off + k), val);
              if (C.aw[1]) val = fma(af[1], __ldg(C.aw[1] + off + k), val);
              cw[k] = val;
            }
        }
      }
      if (bulk) {
        // hand the output tile to the producer warp (it stores the slab, then refills it)
        pipe::fence_proxy_async_smem();
        if (!released) {
#ifdef SGM_CHECKED
          __syncwarp();
          if (lane == 0) atomicAdd(&ckt[2 + buf], 1);
#endif
          pipe::bar_arrive(pipe::kBarEmpty0 + buf, NT);
          released = true;
        }
      } else {
        pipe::bar_sync(pipe::kBarCons, NC * 32);
        for (int j = s; j < TW; j += NC) {
          const int l = l0 + j;
          if (l >= g.nlines) break;
          double* dst = C.out + long(l) * g.rowlen + g.row0;
          const double* srow = slab + j * cfg.pitch;
          for (int k = g.slo + lane; k < g.shi; k += 32) dst[k] = srow[k];
        }
      }
    }
    if (!released) release();
    if (s == 0) SGM_TRACE(it, 7);
  }
}

}  // namespace sweep
}  // namespace sgm
