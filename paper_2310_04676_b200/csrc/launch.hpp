// Per-chain kernel launchers (one translation unit per chain structure so the
// instantiations compile in parallel).
#pragma once

#include "kernels.cuh"

namespace sg {

enum ChainId : int { kChainGeneric8 = 0, kChainGeneric16 = 1, kChainPsm = 2, kChainEcm = 3, kChainStar = 4 };

// One entry point per chain structure. task: kTaskTarget / kTaskPath.
// team_warps: warps per 32-env team (1, 2 or 4; generic chains 1 or 2).
// Specialised chains are instantiated for position control with 4 substeps
// (the reference defaults); anything else runs on the generic chains with
// runtime mode / substeps.
struct LaunchArgs {
  int k_steps;
  bool gen;
  bool reset;
  int task;
  int team_warps;
  cudaStream_t stream;
  int layout = kLayoutAuto;  // TeamLayout (kernels.cuh)
};

cudaError_t launch_generic8(const StepParams& P, const LaunchArgs& a);
cudaError_t launch_generic16(const StepParams& P, const LaunchArgs& a);
cudaError_t launch_psm(const StepParams& P, const LaunchArgs& a);
cudaError_t launch_ecm(const StepParams& P, const LaunchArgs& a);
cudaError_t launch_star(const StepParams& P, const LaunchArgs& a);

template <class CH, int TASK, int MODE, int SUB>
inline cudaError_t launch_fixed(const StepParams& P, const LaunchArgs& a) {
  if (a.reset) return launch_reset<CH, TASK>(P, a.stream);
  switch (a.team_warps) {
    case 1: return launch_team<CH, TASK, MODE, SUB, 1>(P, a.k_steps, a.gen, a.stream);
    case 2: return launch_team<CH, TASK, MODE, SUB, 2>(P, a.k_steps, a.gen, a.stream, a.layout);
    case 3: return launch_team<CH, TASK, MODE, SUB, 3>(P, a.k_steps, a.gen, a.stream);
    default: return launch_team<CH, TASK, MODE, SUB, 4>(P, a.k_steps, a.gen, a.stream);
  }
}

}  // namespace sg
