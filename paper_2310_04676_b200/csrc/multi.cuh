// MultiToolReaching on the device (proj/src/envs.cpp:101-116, 118-223,
// 304-360, 362-408, 540-593): T robots per env (bimanual PSM pairs, trimanual
// PSM + PSM + ECM camera), one SimBatch per tool with its own PCG32 stream
// (stream id = tool * 2^32 + global row, dynamics.cpp:238), tool-major action
// and observation columns, every tip mapped through the tool's base pose.
//
// Layout in HBM: q / qdot / q_target DoF-major [A][n] over the concatenated
// tool DoFs (column c of the action row = DoF row c), tips / goals [3T][n],
// PCG32 state / inc [T][n]; StepResult row-major like the single-tool env.
#pragma once

#include "kernels.cuh"

namespace sg {

constexpr int kMaxTools = 4;      // device path: up to 4 tools of <= 8 DoF each
constexpr int kMaxToolDof = 8;
constexpr int kMtWarps = 4;       // reset kernel: warps per CTA, each stages its own 32 rows

struct ToolEnc {
  RobotTable robot;   // build_table: fixed joints folded, tip offset in the last DoF frame
  float base_R[9];    // tool base rotation (row-major) and position (Pose, envs.hpp:59)
  float base_p[3];
  float view[3];      // (pending fixed rotation * tip rotation) * (0, 0, -1): camera axis in the last DoF frame
  int32_t camera;     // models_[t].name == "ecm" (envs.cpp:339, 545)
  int32_t off;        // first action / DoF column of the tool
  double center[3];   // workspace centre: base.transform_point(FK(mid)) (envs.cpp:159-161)
  uint64_t col_mult, col_add;  // bench stream: advance by `off` draws (row start -> the tool's first column)
  int32_t chain;               // ChainId (launch.hpp): compile-time structure of the tool's FK, or generic
  int32_t pad[3];
};

struct MtParams {
  ToolEnc tool[kMaxTools];
  int32_t T, A, O, Os;  // tools, action dim, obs dim, padded shared-memory row stride (odd)
  int32_t scorer, pad_s;  // team warp that scores (the tool with the fewest DoFs)
  int32_t episode_len, success_hold, substeps, control_mode;
  int64_t n;
  float rho, success_radius, dt_sub;
  float collision_threshold, collision_penalty, view_penalty;
  double goal_sigma, radius;
  // state
  float* q;   // [A][n]
  float* qd;
  float* qt;
  float* goals;  // [3T][n]
  float* tips;   // [3T][n]
  int32_t* step_count;
  int32_t* hold_count;
  int64_t* episode_count;
  uint64_t* rng_state;  // [T][n]
  uint64_t* rng_inc;
  // StepResult
  float* obs;   // [n][O]
  float* tobs;
  float* rewards;
  float* task_error;
  uint8_t* terminated;
  uint8_t* timed_out;
  unsigned long long* sat_total;
  unsigned long long* ended_total;
  int32_t* err;
  const float* actions;  // [n][A] caller actions (device)
  // bench stream (bench.cpp:31-35): act_state[i] = stream state at env i's
  // next row start; a row is A consecutive draws, the next step's row start
  // is G*A draws later (jump_mult / jump_add)
  uint64_t* act_state;
  float* act_buf;  // [n][A]
  uint64_t act_inc, jump_mult, jump_add;
};

cudaError_t launch_multi(const MtParams& P, int k_steps, bool gen, bool reset, cudaStream_t st);

}  // namespace sg
