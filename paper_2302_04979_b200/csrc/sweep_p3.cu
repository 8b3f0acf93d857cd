// Line-sweep launchers for degree p = 3 (see sweep_launch.cuh).
#include "sweep_launch.cuh"
#include "fsweep_launch.cuh"

namespace sgm {
bool launch_sweep_p3(int seg, const SweepArgs& a, cudaStream_t st) { return sweeplaunch::launch_sweep_p<3>(seg, a, st); }
bool launch_fsweep_p3(int seg, int fuse, const SweepArgs& a, cudaStream_t st) {
  return fsweeplaunch::launch_p<3>(seg, fuse, a, st);
}
}  // namespace sgm
