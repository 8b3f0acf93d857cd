// Line-sweep launchers for degree p = 4 (see sweep_launch.cuh).
#include "sweep_launch.cuh"

namespace sgm {
void launch_sweep_p4(int seg, const SweepArgs& a, cudaStream_t st) { sweeplaunch::launch_sweep_p<4>(seg, a, st); }
}  // namespace sgm
