// Line-sweep launchers for the table layout p + 1 = 5 (see sweep_launch.cuh): only the scheme-1
// eps star at p = 4 uses it (the LU of Gamma_B^4 has half-bandwidth 4).
#include "sweep_launch.cuh"

namespace sgm {
bool launch_sweep_p5(int seg, const SweepArgs& a, cudaStream_t st) { return sweeplaunch::launch_sweep_p<5>(seg, a, st); }
}  // namespace sgm
