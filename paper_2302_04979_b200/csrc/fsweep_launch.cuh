// Host launcher of the fused update + sweep kernel (fsweep_kernel.cuh); instantiated per degree in
// sweep_p*.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "fsweep_kernel.cuh"
#include "kernels.cuh"
#include "launch_util.cuh"
#include "seg_sweep.cuh"

namespace sgm {
namespace fsweeplaunch {

inline int even_up(int v) { return (v + 1) & ~1; }

// SweepArgs (api.cu's pass description, with the curl source in a.pro) -> the kernel's parameter
// block.  Returns false when a component cannot be staged (alignment, shapes).
inline bool make_args(const SweepArgs& a, int fuse, int SEG, fsweep::Args& A, int& NC) {
  std::memset(&A, 0, sizeof(A));
  A.ncomp = a.ncomp;
  A.tabs[0] = a.tabs[0];
  A.tabs[1] = (a.tabs[1] && a.tabs[1] != a.tabs[0]) ? a.tabs[1] : nullptr;
  A.ntabs = A.tabs[1] ? 2 : 1;
  A.spike_kh = a.spike_kh;
  A.spike_kf = a.spike_kf;
  A.reverse = a.reverse;
  A.s_ptr = a.pro.s_ptr;
  A.dt = a.pro.dt;
  NC = 1;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  for (int k = 0; k < a.ncomp; ++k) {
    const SweepComp& S = a.comp[k];
    fsweep::Comp& C = A.comp[k];
    const int ax = S.axis, c = S.cidx;
    const int ta0 = (ax == 0) ? 1 : 0, ta1 = (ax == 2) ? 1 : 2;
    const long str[3] = {1, S.ext[0], long(S.ext[0]) * S.ext[1]};
    C.state = S.in;
    C.out = S.out;
    C.dline[0] = S.dline[0];
    C.dline[1] = S.dline[1];
    C.scale = S.scale;
    C.xmode = ax == 0;
    C.L = S.ext[ax];
    C.TD = S.ext[ta0];
    C.n1 = S.ext[ta1];
    C.tpr = (C.TD + 31) / 32;
    C.tiles = C.n1 * C.tpr;
    C.st0 = int(str[ta0]);
    C.st1 = int(str[ta1]);
    C.gs = int(str[ax]);
    C.tslot = (A.ntabs > 1 && S.tab == A.tabs[1]) ? 1 : 0;
    A.nitems += C.tiles;
    const int nc = (C.L + SEG - 1) / SEG;
    NC = nc > NC ? nc : NC;
    int soff = 0;
    auto add = [&](const double* src, const long* sstr, const int* se, int dt1, int lane_lo, int nl, int row_lo,
                   int nrow) -> int {
      fsweep::Stage& G = C.s[C.nst];
      G.src = src;
      G.st0 = int(sstr[ta0]);
      G.st1 = int(sstr[ta1]);
      G.gs = int(sstr[ax]);
      G.dt1 = dt1;
      G.lane_lo = lane_lo;
      G.nl = nl;
      G.row_lo = row_lo;
      G.nrow = nrow;
      G.ext0 = se[ta0];
      G.ext1 = se[ta1];
      G.pitch = even_up(nl + 2);
      G.soff = soff;
      soff += C.xmode ? even_up(nl * G.st0 + 4) : nrow * G.pitch;
      return C.nst++;
    };
    C.accum = S.accum;
    C.ost = C.jst = -1;
    if (fuse <= 2) {  // the old state (updated in place); fuse 3 / 4: increments only
      if (!al16(S.in)) return false;
      C.ost = add(S.in, str, S.ext, 0, 0, 32, 0, C.L);
    }
    const double* jh = (fuse == 1 || fuse == 3) ? a.pro.jhat[c] : nullptr;
    if (jh) {
      if (!al16(jh)) return false;
      C.jst = add(jh, str, S.ext, 0, 0, 32, 0, C.L);
    }
    // component c of the curl: d_{a1} src_{c1} - d_{a2} src_{c2}, (a1, c1) = (c+1, c+2),
    // (a2, c2) = (c+2, c+1) mod 3 (SURVEY 8.0 stencils)
    const bool dual = (fuse == 1 || fuse == 3);
    const int aa[2] = {(c + 1) % 3, (c + 2) % 3}, cc[2] = {(c + 2) % 3, (c + 1) % 3};
    for (int t = 0; t < 2; ++t) {
      const int* se = a.pro.sext[cc[t]];
      const double* src = a.pro.src[cc[t]];
      if (!al16(src)) return false;
      const long sstr[3] = {1, se[0], long(se[0]) * se[1]};
      fsweep::Term& T = C.t[t];
      const int ad = aa[t];
      T.where = ad == ax ? 0 : (ad == ta0 ? 1 : 2);
      T.ext_a = se[ad];
      if (T.where != 0 && se[ax] < C.L) return false;
      if (T.where == 0) {
        const int st = add(src, sstr, se, 0, 0, 32, 0, se[ax]);
        if (dual) T.hi = {st, 0, 1}, T.lo = {st, 0, 0};
        else T.hi = {st, 0, 0}, T.lo = {st, 0, -1};
      } else if (T.where == 1) {
        const int st = add(src, sstr, se, 0, dual ? 0 : -1, 33, 0, C.L);
        if (dual) T.hi = {st, 1, 0}, T.lo = {st, 0, 0};
        else T.hi = {st, 0, 0}, T.lo = {st, -1, 0};
      } else {
        if (dual) {
          const int s0 = add(src, sstr, se, 0, 0, 32, 0, C.L), s1 = add(src, sstr, se, 1, 0, 32, 0, C.L);
          T.hi = {s1, 0, 0};
          T.lo = {s0, 0, 0};
        } else {
          const int s0 = add(src, sstr, se, 0, 0, 32, 0, C.L), s1 = add(src, sstr, se, -1, 0, 32, 0, C.L);
          T.hi = {s0, 0, 0};
          T.lo = {s1, 0, 0};
        }
      }
    }
    A.stage_dbl = soff > A.stage_dbl ? soff : A.stage_dbl;
  }
  return true;
}

template <int P, int HB, int SEG, int FUSE>
bool launch_t(const SweepArgs& a, cudaStream_t st) {
  fsweep::Args A;
  int NC = 1;
  if (!make_args(a, FUSE, SEG, A, NC)) return false;
  A.tab_dbl = a.tab_rows * RowLayout<P>::RS;
  constexpr int M = P - 1;
  const size_t smem =
      (size_t(A.ntabs) * A.tab_dbl + A.stage_dbl + size_t(2) * NC * M * 32) * sizeof(double) + 32;
  A.ck = nullptr;
#ifdef SGM_CHECKED
  A.ck = check_buffer();
#endif
  A.np = NC <= 11 ? 4 : 15 - NC;  // producer warps (at most 15 warps per CTA)
  if (smem > 227 * 1024 || NC > 14) return false;
  if (a.dry) return true;
  auto kern = fsweep::fsweep_kernel<P, HB, SEG, FUSE>;
  static unsigned long long attr_done = 0;
  if (first_on_device(attr_done)) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const int NT = (NC + A.np) * 32;
  long grid = sm_count();
  if (a.share_n > 0) grid = (grid * a.share_k + a.share_n / 2) / a.share_n;
  if (grid > A.nitems) grid = A.nitems;
  if (grid < 1) grid = 1;
  launch_pdl(kern, unsigned(grid), unsigned(NT), smem, st, A);
  return true;
}

template <int P, int SEG>
bool launch_s(int fuse, const SweepArgs& a, cudaStream_t st) {
  // band half-width: eps fused pass Gamma_C^{p-2} (P - 2, at least 1) or Gamma_B^{p-1} (full
  // schedule, P - 1); mu fused pass Gamma_B^{p} (P) or Gamma_C^{p-1} (P - 1)
  constexpr int HLO = P >= 3 ? P - 2 : 1;
  if (fuse == 1) {
    if (a.band_hw <= HLO) return launch_t<P, HLO, SEG, 1>(a, st);
    if (a.band_hw <= P - 1) return launch_t<P, P - 1, SEG, 1>(a, st);
    return false;
  }
  if (fuse == 2) return launch_t<P, P, SEG, 2>(a, st);
  if (fuse == 3) {
    if (a.band_hw <= HLO) return launch_t<P, HLO, SEG, 3>(a, st);
    if (a.band_hw <= P - 1) return launch_t<P, P - 1, SEG, 3>(a, st);
    return false;
  }
  if (fuse == 4) return launch_t<P, P, SEG, 4>(a, st);
  return false;
}

template <int P>
bool launch_p(int seg, int fuse, const SweepArgs& a, cudaStream_t st) {
  switch (seg) {
    case 12: return launch_s<P, 12>(fuse, a, st);
    case 17: return launch_s<P, 17>(fuse, a, st);
    case 28: return launch_s<P, 28>(fuse, a, st);
    default: return false;
  }
}

}  // namespace fsweeplaunch
}  // namespace sgm
