// Persistent, warp-specialised, double-buffered line sweeps (sm_100a).
//
// What one sweep computes (eq. kroninverse P:L571 applied mode by mode with the vec trick
// P:L575-585): for every line of every component along axis `ax`,
//     out_line = scale * A^{-1} (B in_line)
// with B a banded 1D matrix (separable Hodge Gram or pairing factor) and A = LU a banded 1D
// pairing factor (no-pivot LU, reading Z14).  The solve is the partitioned (SPIKE) form of the
// sequential banded substitution: segment-local recurrences plus spike corrections (exact
// algebra; seg_sweep.cuh documents the table layout).
//
// Work unit: a tile of 32 lines of one component (lane j <-> line j).  A CTA is persistent and
// loops over tiles with two shared-memory slabs:
//   * producer warps (NP) stage tile t+1 into slab[(t+1)&1] -- cp.async (LDGSTS) copies, or, for
//     the first pass of a half step, the fused Ampere/Faraday update d <- d + dt (D~1 h - s j)
//     (b <- b - dt D1 e) computed from global loads, written back to the state and to the slab;
//   * consumer warps (NC = segments) run the banded mat-vec + SPIKE solve on slab[t&1] and store.
// Producer/consumer hand-off uses named barriers (FULL[b] / EMPTY[b]); the SPIKE exchanges use a
// consumer-only barrier.  Strided axes (y, z): slab row i holds element i of the 32 lines (lanes
// read consecutive doubles); x axis: slab row j holds line j with an odd pitch (conflict-free
// per-lane walks) and results go back through the slab for coalesced row stores.
#pragma once

#include "kernels.cuh"
#include "seg_sweep.cuh"

namespace sgm {
namespace pipe {

constexpr int kBarFull0 = 1, kBarEmpty0 = 3, kBarCons = 5;

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Geometry of one component for a sweep along `ax`.
struct LineGeom {
  long nlines;  // lines of this component
  long gs;      // element stride along the line
  int L;        // line length
  int X, Y;     // component extents x, y
};

__device__ __forceinline__ LineGeom line_geom(const SweepComp& C, int ax) {
  LineGeom g;
  g.X = C.ext[0];
  g.Y = C.ext[1];
  g.L = C.ext[ax];
  g.nlines = long(C.ext[0]) * C.ext[1] * C.ext[2] / g.L;
  g.gs = (ax == 0) ? 1 : (ax == 1 ? long(g.X) : long(g.X) * g.Y);
  return g;
}

// flat index of element 0 of line l, and its (x, y, z) decomposition helpers
__device__ __forceinline__ long line_base(const LineGeom& g, int ax, long l) {
  if (ax == 0) return l * g.X;
  if (ax == 1) return (l % g.X) + long(g.X) * g.Y * (l / g.X);
  return l;
}

}  // namespace pipe
}  // namespace sgm

namespace sgm {
namespace pipe {

// ---- mbarrier + bulk-copy (TMA engine) helpers -------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, unsigned parity) {
  const unsigned a = smem_u32(mb);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy, completion counted (bytes) on mbarrier mb; 16-byte aligned, size % 16 == 0
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mb))
               : "memory");
}
// shared -> global bulk store (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// make this thread's generic-proxy shared-memory writes visible to the async proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- programmatic dependent launch (PDL) ---------------------------------------------------------
// launch_dependents: let the next kernel in the stream be scheduled (its own griddep_wait still
// waits for this grid's completion and memory flush); griddep_wait: block until the previous
// kernel in the stream has completed.  Both are no-ops for launches without the PDL attribute.
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace pipe
}  // namespace sgm
