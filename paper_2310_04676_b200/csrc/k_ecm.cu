// Kernel instantiations for the ECM chain structure (assets/robots/ecm.robot).
#include "launch.hpp"

namespace sg {

cudaError_t launch_ecm(const StepParams& P, const LaunchArgs& a) {
  if (a.task == kTaskPath) return launch_fixed<EcmChain, kTaskPath, kModePosition, 4>(P, a);
  if (a.task == kTaskTrack) return launch_fixed<EcmChain, kTaskTrack, kModePosition, 4>(P, a);
  return launch_fixed<EcmChain, kTaskTarget, kModePosition, 4>(P, a);
}

}  // namespace sg
