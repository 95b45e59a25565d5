// Generic-chain kernel instantiations: any descriptor up to 16 DoF, runtime
// task / control mode / substeps.
#include "launch.hpp"

namespace sg {

template <class CH>
static cudaError_t launch_generic(const StepParams& P, const LaunchArgs& a) {
  if (a.reset) return launch_reset<CH, -1>(P, a.stream);
  if (a.team_warps >= 2) return launch_team<CH, -1, -1, 0, 2>(P, a.k_steps, a.gen, a.stream);
  return launch_team<CH, -1, -1, 0, 1>(P, a.k_steps, a.gen, a.stream);
}

cudaError_t launch_generic8(const StepParams& P, const LaunchArgs& a) { return launch_generic<GenericChain<8>>(P, a); }
cudaError_t launch_generic16(const StepParams& P, const LaunchArgs& a) { return launch_generic<GenericChain<16>>(P, a); }

}  // namespace sg
