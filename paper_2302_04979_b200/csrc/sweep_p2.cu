// Line-sweep launchers for degree p = 2 (see sweep_launch.cuh).
#include "sweep_launch.cuh"
#include "fsweep_launch.cuh"

namespace sgm {
bool launch_sweep_p2(int seg, const SweepArgs& a, cudaStream_t st) { return sweeplaunch::launch_sweep_p<2>(seg, a, st); }
bool launch_fsweep_p2(int seg, int fuse, const SweepArgs& a, cudaStream_t st) {
  return fsweeplaunch::launch_p<2>(seg, fuse, a, st);
}
}  // namespace sgm
