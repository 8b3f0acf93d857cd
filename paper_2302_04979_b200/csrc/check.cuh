// Verification build of the pipelined sweeps (-DSGM_CHECKED; build.py checked=True ->
// libsgm_checked.so).  compute-sanitizer (racecheck / synccheck) is not available on the GPU pool,
// so the producer/consumer and SPIKE-exchange protocols check themselves:
//   * hand-off tags: the producer of slab b writes the tag of the work item it staged, the
//     consumers compare it with the item they are about to read after the FULL wait (a consumer
//     that passes FULL early, or a producer that stages the wrong item, is caught);
//   * release counts: every consumer warp counts the slabs it has finished with; after the EMPTY
//     wait the producer checks that all consumer warps released every earlier use of the slab (a
//     producer that refills a slab still being read is caught);
//   * exchange tags: each consumer warp tags the tails / heads it publishes with the item number;
//     the readers of a neighbour's tails / heads check the tag after the consumer barrier;
//   * poison: before staging a tile the producers fill the slab with kPoison (finite, so that the
//     positions the coefficients multiply by exactly zero stay harmless); a staged position that
//     matters but is not (re)written, or is read before its copy landed, turns the result into
//     ~1e200 -- which the bitwise comparison with the product build and the oracle parity catch;
//   * jitter: random __nanosleep delays at every hand-off point perturb the interleaving of the
//     warps and CTAs from launch to launch (results must stay bit-identical run to run);
//   * fault injection (SGM_CHECK_INJECT, checked builds only) breaks one protocol step on purpose
//     to show that the checks above detect it: bit 0 = consumers release a slab before reading
//     their rows from it (a WAR race with the next fill), bit 1 = consumers skip the
//     barrier in front of the history scan (a RAW race on the tails).
// Violations are counted in a device buffer (count, first code) read by sgm_check_read (sgm.h).
// The product build compiles none of this.
#pragma once

#ifdef SGM_CHECKED
#include <cuda_runtime.h>

namespace sgm {
namespace check {

enum Code : unsigned {
  kStageTag = 1,     // sweep: slab tag after FULL != the item the consumer expects
  kReleaseCount = 2, // sweep: producer after EMPTY: consumer releases of the slab != expected
  kTailTag = 3,      // sweep: a neighbour's tails are not the current item's
  kHeadTag = 4,      // sweep: a neighbour's heads are not the current item's
  kFReleaseCount = 5 // fused sweep: producer after the empty mbarrier: releases != expected
};

constexpr double kPoison = 1e200;
constexpr int kSmemInts = 40;  // sweep: tag[2], rel[2], tail[16], head[16] (+ padding)

__device__ __forceinline__ void fail(unsigned* ck, unsigned code) {
  atomicAdd(ck, 1u);
  atomicCAS(ck + 1, 0u, code);
}

// a random pause of 0..~4 us at about one call in four
__device__ __forceinline__ void jitter(unsigned salt) {
  unsigned x = unsigned(clock64()) * 0x9E3779B9u ^ salt * 0x85EBCA6Bu ^ (blockIdx.x + 1u) * 0xC2B2AE35u;
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  if ((x & 3u) == 0u) __nanosleep((x >> 8) & 4095u);
}

}  // namespace check

// host side (api.cu): the library's device violation buffer (allocated on first use) and the
// fault-injection bits (SGM_CHECK_INJECT)
unsigned* check_buffer();
int check_inject();

}  // namespace sgm
#endif

#ifdef SGM_TUNING
#include <cuda_runtime.h>
#include <cstddef>
namespace sgm {
#ifdef SGM_TUNING
// tuning build: timeline of one selected sweep launch, [cta < 160][tile < 16][event < 8]
constexpr size_t kTraceLen = size_t(160) * 16 * 8;
unsigned long long* trace_buffer();
extern unsigned long long* g_trace_ptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif
}  // namespace sgm
#endif
