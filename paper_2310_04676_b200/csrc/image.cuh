// ImageMatching on the device (proj/src/envs.cpp:269-295 sample_scene /
// render_row, 333-335 reset, 464-473 render phase, 513-523 reward; renderer
// proj/src/render.cpp:34-67). One warp owns one env: lane d < A integrates
// DoF d, every lane evaluates the camera FK, and the warp renders the env's
// w*h image (pixel p -> lane p % 32), reduces the L1 image error and writes
// the observation row [q | qdot | tip | q_target | target image | current
// image] with coalesced stores.
//
// Layout in HBM: joint state DoF-major [A][n]; tips [3][n]; per-env scene
// [n][16] (3 spheres x {cx, cy, cz, radius, albedo}); target image [n][w*h];
// target camera [n][12] (R row-major, p) kept for inspection.
#pragma once

#include "kernels.cuh"

namespace sg {

constexpr int kImWarps = 8;  // envs (warps) per CTA

struct ImParams {
  RobotTable robot;
  float cam_R[9];  // trailing fixed rotations x tip orientation: camera frame in the last DoF frame
  int32_t A, O, W, H, wh, episode_len, substeps, control_mode;
  int32_t chain, pad1;  // ChainId of the camera FK (launch.hpp): specialised structure or generic
  int64_t n;
  float f, inv_f, near_, far_, dt_sub, pad0;  // f: focal length in pixels, 0.5 w / tan(fov / 2)
  double sigma, radius, center[3];
  // state
  float* q;  // [A][n]
  float* qd;
  float* qt;
  float* tips;  // [3][n]
  int32_t* step_count;
  int32_t* hold_count;
  int64_t* episode_count;
  uint64_t* rng_state;
  uint64_t* rng_inc;
  float* scenes;   // [n][16]
  float* target;   // [n][wh]
  float* tcam;     // [n][12]
  // StepResult
  float* obs;  // [n][O]
  float* tobs;
  float* rewards;
  float* task_error;
  uint8_t* terminated;
  uint8_t* timed_out;
  unsigned long long* sat_total;
  unsigned long long* ended_total;
  int32_t* err;
  const float* actions;  // [n][A] caller actions (device)
  // bench stream: act_state[i] = state at env i's row start; lane d's draw is
  // that state advanced d times (pow_*), the next row start G*A draws later
  uint64_t* act_state;
  float* act_buf;
  uint64_t act_inc, jump_mult, jump_add;
  uint64_t pow_mult[kMaxDof], pow_add[kMaxDof];
};

cudaError_t launch_image(const ImParams& P, int k_steps, bool gen, bool reset, cudaStream_t st);

}  // namespace sg
