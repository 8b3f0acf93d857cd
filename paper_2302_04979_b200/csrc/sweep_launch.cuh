// Host launchers of the line sweeps (template machinery; instantiated per degree in sweep_p*.cu so
// the three degrees compile in parallel).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "launch_util.cuh"
#include "seg_sweep.cuh"
#include "sweep_kernel.cuh"

namespace sgm {
namespace sweeplaunch {

// nslab: 2 double-buffered slabs, 1 a single slab (long lines); a.dry: check the fit only
template <int P, int HB, int SEG, int LPT, int MODE, int OPS>
bool launch_sweep_t(const SweepArgs& a, int nslab, cudaStream_t st) {
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
    // per-component axis (strided passes may mix y- and z-lines of different components)
    const int ax = (MODE != 3 && C.axis > 0) ? C.axis : a.axis;
    g.L = C.wlen > 0 ? C.wlen : C.ext[ax];  // a window of a long line, or the whole line
    g.row0 = C.wlen > 0 ? C.win0 : 0;
    g.slo = C.wlen > 0 ? C.slo : 0;
    g.shi = C.wlen > 0 ? C.shi : g.L;
    g.magic = 0xffffffffu / unsigned(X);
    g.nlines = X * Y * Z / C.ext[ax];
    g.X = X;
    g.rowlen = X;
    g.gs = (ax == 0) ? 1 : (ax == 1 ? X : X * Y);
    g.os = (ax == 1) ? X * Y : X;  // transverse index l / X: z (y pass) or y (z pass)
    g.TD = (ax == 0) ? Y : X;      // transverse coordinates of line l: (l % TD, l / TD)
    g.tmagic = 0xffffffffu / unsigned(g.TD);
    cfg.tiles[c] = (g.nlines + TW - 1) / TW;
    cfg.nitems += cfg.tiles[c];
    Lmax = g.L > Lmax ? g.L : Lmax;
  }
  cfg.NC = (Lmax + SEG - 1) / SEG;
  cfg.rows = cfg.NC * SEG + P;
  // x axis: a tile of whole lines is one contiguous range -> one bulk copy in and one out (TMA
  // engine), if the component bases are 16-byte aligned and the component has an even size.
  // (Strided tiles are many small row runs: measured slower on the bulk engine than cp.async.)
  bool bulk = (MODE == 3) && tune_int("SGM_BULK", 1) != 0;
  for (int c = 0; c < a.ncomp && bulk; ++c) {
    const SweepComp& C = a.comp[c];
    if ((reinterpret_cast<uintptr_t>(C.in) & 15) || (reinterpret_cast<uintptr_t>(C.out) & 15)) bulk = false;
    if ((long(C.ext[0]) * C.ext[1] * C.ext[2]) & 1) bulk = false;
    if (C.wlen > 0) bulk = false;  // a window of x-lines is not one contiguous range
  }
  cfg.bulk = bulk ? 1 : 0;
  if (bulk) cfg.NP = 1;
  else cfg.NP = tune_int("SGM_NP", 4);
  if (cfg.NP < 1) cfg.NP = 1;
  if (cfg.NC + cfg.NP > 16) cfg.NP = 16 - cfg.NC;
  if (cfg.NP < 1) return false;
  if (MODE == 3) {
    // bulk: a whole-tile copy keeps pitch = line length; a multiple of 4 would put the consumers'
    // per-lane line walks on few banks (all lanes on one bank pair at L % 16 == 0), so such lines
    // are copied one by one into pitch L + 2 (16-byte aligned rows, 4-way at worst)
    int bp_max = 0;
    for (int c = 0; c < a.ncomp; ++c) {
      sweep::CompGeom& g = cfg.g[c];
      g.lbulk = (bulk && (g.L % 4) == 0 && tune_int("SGM_LINE_BULK", 1)) ? 1 : 0;
      g.bpitch = g.lbulk ? g.L + 2 : g.L;
      bp_max = g.bpitch > bp_max ? g.bpitch : bp_max;
    }
    cfg.pitch = bulk ? bp_max : (cfg.rows | 1);
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
  cfg.dbg = tune_int("SGM_PIPE_DBG", 0);
  cfg.reverse = tune_int("SGM_SNAKE", 1) ? a.reverse : 0;
  constexpr int M = P - 1;
  cfg.nslab = nslab;
  size_t smem = (size_t(cfg.ntabs) * cfg.tab_dbl + size_t(nslab) * cfg.slab + size_t(2) * cfg.NC * M * TW + 4) *
                sizeof(double);
#ifdef SGM_CHECKED
  smem += check::kSmemInts * sizeof(int);
  cfg.ck = check_buffer();
  cfg.inject = check_inject();
#endif
  if (smem > 227 * 1024) return false;
  if (a.dry) return true;
#ifdef SGM_TUNING
  cfg.trace = trace_buffer();
#endif
  const int NT = (cfg.NC + cfg.NP) * 32;
  static unsigned long long attr_done = 0;
  if (first_on_device(attr_done))
    cudaFuncSetAttribute(sweep::sweep_kernel<P, HB, SEG, LPT, MODE, OPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep::sweep_kernel<P, HB, SEG, LPT, MODE, OPS>, NT, smem);
  if (per_sm < 1) per_sm = 1;
  const int cap = tune_int("SGM_CTAS_PER_SM", 0);
  if (cap > 0 && cap < per_sm) per_sm = cap;
  long grid = long(per_sm) * sm_count();
  if (a.share_n > 0) grid = (grid * a.share_k + a.share_n / 2) / a.share_n;
  if (grid < 1) grid = 1;
  if (grid > cfg.nitems) grid = cfg.nitems;
  if (grid < 1) grid = 1;
  launch_pdl(sweep::sweep_kernel<P, HB, SEG, LPT, MODE, OPS>, unsigned(grid), unsigned(NT), smem, st, a, cfg);
  return true;
}

// Lines of the launch over its share of the SMs: below two 64-line tiles per SM the launch is
// latency bound and 32-line tiles (one line per thread, twice the work items) finish sooner
// (64^3 p = 2/3/4 and C2 32^3: 16 / 6 / 4 / 6 % per step; from 96^3 on two lines per thread win)
inline bool few_lines(const SweepArgs& a) {
  long lines = 0;
  for (int c = 0; c < a.ncomp; ++c) {
    const SweepComp& C = a.comp[c];
    const int ax = (a.axis != 0 && C.axis > 0) ? C.axis : a.axis;
    lines += long(C.ext[0]) * C.ext[1] * C.ext[2] / C.ext[ax];
  }
  double sms = sm_count();
  if (a.share_n > 0) sms = sms * a.share_k / a.share_n;
  return lines < 2 * 64 * sms;
}

template <int P, int HB, int SEG, int MODE, int OPS>
bool launch_sweep_m(const SweepArgs& a, cudaStream_t st) {
  // two lines per thread when the register budget allows (SEG <= 17), the slabs fit and the launch
  // has enough lines; double buffering first, then a single slab (long lines)
  const int lpt = tune_int("SGM_LPT", (few_lines(a) && !a.wide) ? 1 : 2);
  for (int nslab = 2; nslab >= 1; --nslab) {
    if constexpr (SEG <= 17) {
      if (lpt == 2 && launch_sweep_t<P, HB, SEG, 2, MODE, OPS>(a, nslab, st)) return true;
    }
    if (launch_sweep_t<P, HB, SEG, 1, MODE, OPS>(a, nslab, st)) return true;
  }
  // two distinct line-operator tables that do not fit together: one launch per table (the
  // components are independent); both fits are checked before anything is launched
  if (a.tabs[1] != nullptr && a.tabs[1] != a.tabs[0]) {
    SweepArgs sub[2];
    for (int t = 0; t < 2; ++t) {
      sub[t] = a;
      sub[t].ncomp = 0;
      sub[t].tabs[0] = a.tabs[t];
      sub[t].tabs[1] = nullptr;
      for (int c = 0; c < a.ncomp; ++c)
        if (a.comp[c].tslot == t) {
          sub[t].comp[sub[t].ncomp] = a.comp[c];
          sub[t].comp[sub[t].ncomp++].tslot = 0;
        }
      sub[t].dry = 1;
      if (sub[t].ncomp > 0 && !launch_sweep_m<P, HB, SEG, MODE, OPS>(sub[t], st)) return false;
      sub[t].dry = a.dry;
    }
    for (int t = 0; t < 2; ++t)
      if (sub[t].ncomp > 0) launch_sweep_m<P, HB, SEG, MODE, OPS>(sub[t], st);
    return true;
  }
  return false;
}

template <int P, int SEG, int MODE>
bool launch_sweep_o(const SweepArgs& a, cudaStream_t st) {
  // band half-width: P - 1 for the eps-side Grams and the pairing factors, P for the mu-side Gram
  if (a.band && a.solve) {
    if (a.band_hw >= P) return launch_sweep_m<P, P, SEG, MODE, 3>(a, st);
    if (P >= 3 && a.band_hw <= P - 2) return launch_sweep_m<P, (P >= 3 ? P - 2 : 1), SEG, MODE, 3>(a, st);  // eps Gamma_C^{p-2}
    return launch_sweep_m<P, P - 1, SEG, MODE, 3>(a, st);
  } else if (a.solve) {
    return launch_sweep_m<P, P - 1, SEG, MODE, 2>(a, st);
  }
  if (a.band_hw >= P) return launch_sweep_m<P, P, SEG, MODE, 1>(a, st);
  return launch_sweep_m<P, P - 1, SEG, MODE, 1>(a, st);
}

template <int P, int SEG>
bool launch_sweep_s(const SweepArgs& a, cudaStream_t st) {
  if (a.axis == 0) return launch_sweep_o<P, SEG, 3>(a, st);
  return launch_sweep_o<P, SEG, 0>(a, st);
}

// false: no compiled configuration fits (shared memory); nothing was launched
template <int P>
bool launch_sweep_p(int seg, const SweepArgs& a, cudaStream_t st) {
  switch (seg) {
    case 12: return launch_sweep_s<P, 12>(a, st);
    case 17: return launch_sweep_s<P, 17>(a, st);
    default: return launch_sweep_s<P, 28>(a, st);
  }
}

}  // namespace sweeplaunch
}  // namespace sgm
