// Kernel instantiations for the STAR chain structure (assets/robots/star.robot).
#include "launch.hpp"

namespace sg {

cudaError_t launch_star(const StepParams& P, const LaunchArgs& a) {
  if (a.task == kTaskPath) return launch_fixed<StarChain, kTaskPath, kModePosition, 4>(P, a);
  if (a.task == kTaskTrack) return launch_fixed<StarChain, kTaskTrack, kModePosition, 4>(P, a);
  return launch_fixed<StarChain, kTaskTarget, kModePosition, 4>(P, a);
}

}  // namespace sg
