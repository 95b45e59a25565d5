// Kernel instantiations for the PSM chain structure (assets/robots/psm.robot).
#include "launch.hpp"

namespace sg {

cudaError_t launch_psm(const StepParams& P, const LaunchArgs& a) {
  if (a.task == kTaskPath) return launch_fixed<PsmChain, kTaskPath, kModePosition, 4>(P, a);
  if (a.task == kTaskTrack) return launch_fixed<PsmChain, kTaskTrack, kModePosition, 4>(P, a);
  return launch_fixed<PsmChain, kTaskTarget, kModePosition, 4>(P, a);
}

}  // namespace sg
