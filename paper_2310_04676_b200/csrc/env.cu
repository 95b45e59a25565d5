// Host side of the drop-in boundary: env object, device allocation, kernel
// launch, and the extern "C" entry points declared in include/sg_env.h.
//
// Mirrors VecTaskEnv construction (proj/src/envs.cpp:118-223): config
// validation (:65-81), gain resolution (:142-158, default_dynamics_config
// dynamics.cpp:69-86, DynamicsConfig::validate :44-67), SimBatch seeding
// (dynamics.cpp:225-241), workspace centre = FK(mid) (:161-162), observation
// layout (:166-192). The step itself is one fused kernel (kernels.cuh).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <array>
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "launch.hpp"
#include "multi.cuh"
#include "image.cuh"
#include "robot.hpp"
#include "sg_env.h"

namespace {

thread_local std::string g_last_error;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw sg::SimError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)
// driver-API calls (stream memory operations)
#define CU(x)                                                                                    \
  do {                                                                                           \
    const CUresult r_ = (x);                                                                     \
    if (r_ != CUDA_SUCCESS)                                                                      \
      throw sg::SimError(std::string("CUDA driver error ") + std::to_string((int)r_) + " in " #x); \
  } while (0)

// ---- host PCG32 (rng.hpp:25-83) for stream seeding and jump tables --------
struct HostPcg {
  uint64_t state = 0, inc = 0;
  uint32_t next() {
    const uint64_t old = state;
    state = old * sg::kPcgMult + inc;
    const uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
    const uint32_t rot = static_cast<uint32_t>(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  void seed(uint64_t initstate, uint64_t initseq) {
    state = 0;
    inc = (initseq << 1u) | 1u;
    next();
    state += initstate;
    next();
  }
};

uint64_t splitmix64(uint64_t& x) {
  x += 0x9e3779b97f4a7c15ULL;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

HostPcg make_stream(uint64_t seed, uint64_t id) {
  uint64_t x = seed ^ (0x2545f4914f6cdd1dULL * (id + 1));
  const uint64_t a = splitmix64(x);
  const uint64_t b = splitmix64(x);
  HostPcg r;
  r.seed(a, b);
  return r;
}

// Affine map s -> mult * s + add equal to k PCG32 advances with increment inc.
void pcg_jump(uint64_t k, uint64_t inc, uint64_t& mult, uint64_t& add) {
  uint64_t acc_m = 1, acc_a = 0, cur_m = sg::kPcgMult, cur_a = inc;
  while (k) {
    if (k & 1) {
      acc_m *= cur_m;
      acc_a = acc_a * cur_m + cur_a;
    }
    cur_a = (cur_m + 1) * cur_a;
    cur_m *= cur_m;
    k >>= 1;
  }
  mult = acc_m;
  add = acc_a;
}

template <typename T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  CK(cudaMalloc(&p, count * sizeof(T)));
  CK(cudaMemset(p, 0, count * sizeof(T)));
  return static_cast<T*>(p);
}

using Mat3 = std::array<double, 9>;

Mat3 quat_to_mat(const sg::Quat& q) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  return {1 - 2 * (y * y + z * z), 2 * (x * y - w * z),     2 * (x * z + w * y),
          2 * (x * y + w * z),     1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
          2 * (x * z - w * y),     2 * (y * z + w * x),     1 - 2 * (x * x + y * y)};
}

Mat3 mat_mul(const Mat3& a, const Mat3& b) {
  Mat3 o{};
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o[r * 3 + c] = a[r * 3] * b[c] + a[r * 3 + 1] * b[3 + c] + a[r * 3 + 2] * b[6 + c];
  return o;
}

sg::Vec3 mat_vec(const Mat3& a, const sg::Vec3& v) {
  return {a[0] * v[0] + a[1] * v[1] + a[2] * v[2], a[3] * v[0] + a[4] * v[1] + a[5] * v[2],
          a[6] * v[0] + a[7] * v[1] + a[8] * v[2]};
}

bool is_identity(const Mat3& m) {
  const Mat3 I{1, 0, 0, 0, 1, 0, 0, 0, 1};
  return m == I;
}

// Packs the chain per actuated joint. A pending rigid transform (p, R)
// accumulates fixed joints (fk_walk: p += R*o; R = R*R_o) and is folded into
// the next actuated joint's origin, or into the tool tip at the end.
sg::RobotTable build_table(const sg::RobotModel& m, double dt_sub, const std::vector<double>& kp,
                           const std::vector<double>& kd, const std::vector<double>& inertia,
                           const std::vector<double>& damping) {
  if (m.dof_count > sg::kMaxDof)
    throw sg::ConfigError("robot '" + m.name + "' has more than " + std::to_string(sg::kMaxDof) + " DoF");
  sg::RobotTable t;
  std::memset(&t, 0, sizeof(t));
  t.dof = m.dof_count;
  t.jaw = m.jaw_dof();
  sg::Vec3 pend_p{0, 0, 0};
  Mat3 pend_R{1, 0, 0, 0, 1, 0, 0, 0, 1};
  int d = 0;
  for (const auto& j : m.joints) {
    const Mat3 Rj = quat_to_mat(j.origin_rotation);
    const sg::Vec3 o = mat_vec(pend_R, j.origin_translation);
    const sg::Vec3 p{pend_p[0] + o[0], pend_p[1] + o[1], pend_p[2] + o[2]};
    // exact identity when the quaternion is (1,0,0,0) (every builtin origin)
    const bool ident_j = j.origin_rotation == sg::Quat{1, 0, 0, 0};
    const Mat3 Rc = ident_j ? pend_R : mat_mul(pend_R, Rj);
    if (j.kind == sg::JointKind::Fixed) {
      pend_p = p;
      pend_R = Rc;
      continue;
    }
    auto& e = t.j[d++];
    e.kind = static_cast<int32_t>(j.kind);
    e.axis_code = 6;
    for (int k = 0; k < 3; ++k) {
      const int o1 = (k + 1) % 3, o2 = (k + 2) % 3;
      if (j.axis[o1] == 0.0 && j.axis[o2] == 0.0) {
        if (j.axis[k] == 1.0) e.axis_code = k;
        if (j.axis[k] == -1.0) e.axis_code = k + 3;
      }
    }
    for (int k = 0; k < 3; ++k) {
      e.axis[k] = static_cast<float>(j.axis[k]);
      e.o[k] = static_cast<float>(p[k]);
      if (p[k] != 0.0) e.flags |= 1 << k;
    }
    if (!is_identity(Rc)) {
      e.flags |= 8;
      for (int k = 0; k < 9; ++k) e.R[k] = static_cast<float>(Rc[k]);
    }
    pend_p = {0, 0, 0};
    pend_R = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  }
  // tip = pending o (p + R * tip_xyz); the tip orientation does not move the point
  const sg::Vec3 tt = mat_vec(pend_R, m.tip_position);
  for (int k = 0; k < 3; ++k) {
    const double v = pend_p[k] + tt[k];
    t.tip[k] = static_cast<float>(v);
    if (v != 0.0) t.tip_flags |= 1 << k;
  }
  for (int dd = 0; dd < m.dof_count; ++dd) {
    const auto& j = m.dof_joint(dd);
    t.lo[dd] = static_cast<float>(j.limit_lo);
    t.hi[dd] = static_cast<float>(j.limit_hi);
    t.vel[dd] = static_cast<float>(j.velocity_limit);
    t.eff[dd] = static_cast<float>(j.effort_limit);
    t.lo_d[dd] = j.limit_lo;
    t.hi_d[dd] = j.limit_hi;
    t.kp[dd] = static_cast<float>(kp[dd]);
    t.kd[dd] = static_cast<float>(kd[dd]);
    t.damping[dd] = static_cast<float>(damping[dd]);
    t.dt_over_inertia[dd] = static_cast<float>(dt_sub / inertia[dd]);
  }
  return t;
}

// Warps per team (kernels.cuh env_step_kernel): 2 measured best for PSM
// (16,384 envs), ECM (65,536) and STAR (16,384) alike (tools/ab.sh); the
// generic chains use 2 as well. SG_TEAM_WARPS overrides (tuning, A/B).
int team_warps_for(int chain) {
  const char* s = std::getenv("SG_TEAM_WARPS");
  int v = s ? std::atoi(s) : 2;
  if (chain < sg::kChainPsm) return v >= 2 ? 2 : 1;
  return v >= 4 ? 4 : (v < 1 ? 1 : v);
}

// Team layout of the specialised two-warp kernels (kernels.cuh TeamLayout):
// automatic unless SG_TEAM_LAYOUT=legacy|packed (tests exercise both layouts
// at every size; A/B measurements).
int team_layout_from_env() {
  const char* s = std::getenv("SG_TEAM_LAYOUT");
  if (!s) return sg::kLayoutAuto;
  if (std::string(s) == "legacy") return sg::kLayoutLegacy;
  if (std::string(s) == "packed") return sg::kLayoutPacked;
  return sg::kLayoutAuto;
}

// NVTX range around every host-side entry point (header-only NVTX3: a no-op
// unless a profiler injects itself), so a timeline shows each C-ABI call.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <typename F>
int guard(F&& f) {
  try {
    f();
    return SG_OK;
  } catch (const sg::SimError& e) {
    g_last_error = e.what();
    return SG_ERR_SIM;
  } catch (const sg::ConfigError& e) {
    g_last_error = e.what();
    return SG_ERR_CONFIG;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SG_ERR_SIM;
  }
}

}  // namespace

struct sg_robot {
  sg::RobotModel model;
  sg::RobotTable table;
};

struct sg_env {
  sg::RobotModel model;
  sg_env_config cfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  sg::StepParams P{};
  int A = 0, O = 0;
  int64_t n = 0;
  double center[3]{};
  double radius = 0;
  std::vector<std::pair<std::string, std::pair<int, int>>> layout;
  float* d_actions_in = nullptr;  // staging for sg_env_step_host
  unsigned long long last_sat = 0;
  unsigned long long last_ended = 0;
  // device {sat_total, ended slot A, err, ended slot B, ticket, pad...}
  unsigned long long* counters = nullptr;
  unsigned long long* h_counters = nullptr;  // pinned, mapped: {sat_total, ended, err} of the last host step
  // zero-copy host step: teams reading their action rows over PCIe at once
  // (SG_HOST_READ_WINDOW, 0 = all at once). 128 of 512 teams (PSM 16K): later
  // teams' reads overlap earlier teams' result writes, 63.5 -> 62.0 us per
  // step (tools/gpu_r3a.sh: 64 / 256 / 384 no better)
  int read_window = std::getenv("SG_HOST_READ_WINDOW") ? std::atoi(std::getenv("SG_HOST_READ_WINDOW")) : 128;
  // zero-copy host step: observation rows by the copy engine in chunks of
  // teams, each chunk's copy starting as soon as its teams are done
  // (SG_HOST_CE_CHUNKS, 0 = the kernel writes them over PCIe itself).
  // Parity-tested but slower (PSM 16K: 62.9 us per step zero-copy, 85 / 99 /
  // 124 / 172 us with 2 / 4 / 8 / 16 chunks: every chunk's stream wait +
  // copy costs more than the copy engine gains over the SMs' PCIe writes)
  int ce_chunks = std::getenv("SG_HOST_CE_CHUNKS") ? std::atoi(std::getenv("SG_HOST_CE_CHUNKS")) : 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copy_done = nullptr;
  unsigned int* d_chunks = nullptr;  // [64] counts | [64] flags
  unsigned long long* d_status = nullptr;    // device alias of h_counters
  int host_slot = 0;                          // ended slot of the next host step
  bool bench_ready = false;
  // MultiToolReaching (multi.cuh): its own parameter block and buffers
  bool multi = false;
  sg::MtParams M{};
  std::vector<sg::RobotModel> tools;
  std::vector<std::array<double, 7>> bases;    // per tool: xyz, quaternion wxyz
  std::vector<std::array<double, 3>> centers;  // per tool workspace centre
  // ImageMatching (image.cuh)
  bool image = false;
  sg::ImParams I{};
  bool own_kernel() const { return multi || image; }  // task kernels outside the env_step family

  ~sg_env() {
    cudaSetDevice(device);
    cudaStreamSynchronize(stream);
    if (copy_stream) {
      cudaStreamSynchronize(copy_stream);
      cudaStreamDestroy(copy_stream);
      cudaEventDestroy(copy_done);
      cudaFree(d_chunks);
    }
    if (h_counters) cudaFreeHost(h_counters);
    const auto& p = P.p;
    void* bufs[] = {p.q,   p.qd,       p.qt,         p.goals,      p.tips,     p.step_count, p.hold_count,
                    p.episode_count, p.wp_idx,     p.wp_len,     p.wps,      p.rng_state,  p.rng_inc,
                    p.obs, p.tobs,     p.rewards,    p.task_error, p.terminated, p.timed_out, counters,
                    p.act_state, p.act_buf, d_actions_in, p.rec_valid, p.rec_q, p.rec_len, p.rec_err, p.rec_rng,
                    p.rec_wps, p.goal_spawn, p.goal_vel};
    for (void* b : bufs)
      if (b) cudaFree(b);
    if (multi) {
      void* mb[] = {M.q, M.qd, M.qt, M.goals, M.tips, M.step_count, M.hold_count, M.episode_count, M.rng_state,
                    M.rng_inc, M.obs, M.tobs, M.rewards, M.task_error, M.terminated, M.timed_out, M.act_state,
                    M.act_buf};
      for (void* b : mb)
        if (b) cudaFree(b);
    }
    if (image) {
      void* ib[] = {I.q, I.qd, I.qt, I.tips, I.step_count, I.hold_count, I.episode_count, I.rng_state, I.rng_inc,
                    I.scenes, I.target, I.tcam, I.obs, I.tobs, I.rewards, I.task_error, I.terminated, I.timed_out,
                    I.act_state, I.act_buf};
      for (void* b : ib)
        if (b) cudaFree(b);
    }
  }
  int32_t* err_word() const { return multi ? M.err : (image ? I.err : P.p.err); }
  void launch_mt(int k_steps, bool gen, bool reset) {
    if (image) CK(sg::launch_image(I, k_steps, gen, reset, stream));
    else CK(sg::launch_multi(M, k_steps, gen, reset, stream));
  }

  int chain = sg::kChainGeneric8;
  int team_warps = 1;
  int team_layout = sg::kLayoutAuto;
  // Zero-copy host steps wait for the launch's completion flag (h_status[3])
  // instead of cudaStreamSynchronize: 65.6 vs 69.6 us per PSM 16K step
  // (tools/gpu_r2g.sh). SG_HOST_POLL=0 restores the synchronize (A/B).
  bool host_poll = true;
  unsigned long long host_seq = 0;

  void launch(int k_steps, bool gen, bool reset) {
    sg::LaunchArgs a{k_steps, gen, reset, P.task.task, team_warps, stream, team_layout};
    cudaError_t e = cudaSuccess;
    switch (chain) {
      case sg::kChainPsm: e = sg::launch_psm(P, a); break;
      case sg::kChainEcm: e = sg::launch_ecm(P, a); break;
      case sg::kChainStar: e = sg::launch_star(P, a); break;
      case sg::kChainGeneric16: e = sg::launch_generic16(P, a); break;
      default: e = sg::launch_generic8(P, a); break;
    }
    CK(e);
  }
  // Fused multi-step launches of a PathFollowing env first bring the reset
  // records up to date (path_record_kernel, kernels.cuh): the launch's reset
  // bursts then install precomputed resets. Single steps reset inline.
  void launch_step(int k_steps, bool gen) {
    if (k_steps > 1 && P.p.rec_valid) {
      const unsigned grid = static_cast<unsigned>((n + sg::kRecEnvsPerBlock - 1) / sg::kRecEnvsPerBlock);
      sg::path_record_kernel<<<grid, sg::kRecThreads, 0, stream>>>(P);
      CK(cudaGetLastError());
    }
    launch(k_steps, gen, false);
  }
  void launch_reset() { launch(0, false, true); }

  // DoF block [b, e) of team warp s (kernels.cuh: Block)
  // (blocks are cut from the chain's compile-time DoF count: A for the fixed
  // chains, 8/16 for the generic ones, whose warps skip DoFs >= A)
  void warp_block(int s, int& b, int& e) const {
    const int D = chain == sg::kChainGeneric8 ? 8 : (chain == sg::kChainGeneric16 ? 16 : A);
    const int b0 = sg::dof_block_begin(D, team_warps, s);
    b = std::min(b0, A);
    e = std::min(b0 + sg::dof_block_size(D, team_warps, s), A);
  }

  void views(sg_step_views* out) const {
    if (!out) return;
    if (image) {
      out->observations = I.obs;
      out->terminal_observations = I.tobs;
      out->rewards = I.rewards;
      out->task_error = I.task_error;
      out->terminated = I.terminated;
      out->timed_out = I.timed_out;
      out->action_saturations_total = I.sat_total;
      out->n_envs = n;
      out->obs_dim = O;
      out->action_dim = A;
      return;
    }
    if (multi) {
      out->observations = M.obs;
      out->terminal_observations = M.tobs;
      out->rewards = M.rewards;
      out->task_error = M.task_error;
      out->terminated = M.terminated;
      out->timed_out = M.timed_out;
      out->action_saturations_total = M.sat_total;
      out->n_envs = n;
      out->obs_dim = O;
      out->action_dim = A;
      return;
    }
    out->observations = P.p.obs;
    out->terminal_observations = P.p.tobs;
    out->rewards = P.p.rewards;
    out->task_error = P.p.task_error;
    out->terminated = P.p.terminated;
    out->timed_out = P.p.timed_out;
    out->action_saturations_total = P.p.sat_total;
    out->n_envs = n;
    out->obs_dim = O;
    out->action_dim = A;
  }

  // Synchronise and convert the device error word (errors.hpp semantics).
  void check() {
    CK(cudaStreamSynchronize(stream));
    int32_t err = 0;
    CK(cudaMemcpy(&err, err_word(), sizeof(err), cudaMemcpyDeviceToHost));
    raise(err);
  }
  void raise(int32_t err) {
    if (!err) return;
    CK(cudaMemset(err_word(), 0, sizeof(int32_t)));
    if (err & sg::kErrNonFiniteAction) throw sg::SimError("dynamics.step: non-finite action entry");
    if (err & sg::kErrNonFiniteReward) throw sg::SimError("env.step: non-finite reward");
    if (err & sg::kErrGoalSampling)
      throw sg::ConfigError("goal sampling rejected 1000 candidates; workspace_radius is misconfigured for goal_sigma");
    if (err & sg::kErrWaypointCap) throw sg::SimError("env: waypoint table capacity exceeded");
    throw sg::SimError("env: device error " + std::to_string(err));
  }
};

namespace {

void validate_env_config(const sg_env_config& c) {  // envs.cpp:65-81
  if (c.n_envs < 1) throw sg::ConfigError("env.n_envs must be >= 1");
  if (c.episode_len < 1) throw sg::ConfigError("env.episode_len must be >= 1");
  if (!(c.goal_sigma > 0.0)) throw sg::ConfigError("env.goal_sigma must be > 0");
  if (!(c.success_radius > 0.0)) throw sg::ConfigError("env.success_radius must be > 0");
  if (!(c.reward_scale < 0.0)) throw sg::ConfigError("env.reward_scale (rho) must be < 0");
  if (!(c.path_penalty > 0.0)) throw sg::ConfigError("env.path_penalty (alpha) must be > 0");
  if (c.success_hold < 1) throw sg::ConfigError("env.success_hold must be >= 1");
  if (!(c.goal_offset_clip > 0.0)) throw sg::ConfigError("env.goal_offset_clip must be > 0");
  if (!(c.waypoint_spacing > 0.0)) throw sg::ConfigError("env.waypoint_spacing must be > 0");
  if (c.workspace_radius < 0.0) throw sg::ConfigError("env.workspace_radius must be >= 0");
  if (c.tracking_vel_noise_std < 0.0) throw sg::ConfigError("env.tracking_vel_noise_std must be >= 0");
  if (!(c.tracking_vel_clamp > 0.0)) throw sg::ConfigError("env.tracking_vel_clamp must be > 0");
  if (c.collision_threshold < 0.0) throw sg::ConfigError("env.collision_threshold must be >= 0");
  if (c.collision_penalty < 0.0) throw sg::ConfigError("env.collision_penalty must be >= 0");
  if (c.view_penalty < 0.0) throw sg::ConfigError("env.view_penalty must be >= 0");
}

const char* task_name(int t) {
  switch (t) {
    case SG_TASK_TARGET_REACHING: return "target_reaching";
    case SG_TASK_ACTIVE_TRACKING: return "active_tracking";
    case SG_TASK_IMAGE_MATCHING: return "image_matching";
    case SG_TASK_PATH_FOLLOWING: return "path_following";
    case SG_TASK_MULTI_TOOL_REACHING: return "multi_tool_reaching";
  }
  return "?";
}

std::vector<double> resolve_gain(const double* v, int32_t count, const std::vector<double>& fallback, int dof,
                                 const char* name) {
  if (count < 0) throw sg::ConfigError(std::string("dynamics.") + name + ": negative length");
  if (count == 0) return fallback;
  if (count == 1) return std::vector<double>(dof, v[0]);
  return std::vector<double>(v, v + count);
}

template <class CH>
bool chain_matches(const sg::RobotTable& t) {
  if (t.dof != CH::kDof || t.tip_flags != CH::kTipFlags || t.jaw != CH::kJaw) return false;
  for (int d = 0; d < CH::kDof; ++d) {
    const auto& j = t.j[d];
    if (j.axis_code == 6) return false;
    // the specialised kernels evaluate sin/cos without range reduction
    if (j.kind == sg::kRevolute && (t.lo_d[d] < -M_PI || t.hi_d[d] > M_PI)) return false;
    if (sg::jsig(j.kind, j.axis_code, j.flags & 7, (j.flags >> 3) & 1) != CH::kSig[d]) return false;
  }
  return true;
}

int select_chain(const sg::RobotTable& t, int control_mode, int substeps) {
  if (control_mode == SG_CONTROL_POSITION && substeps == 4) {
    if (chain_matches<sg::PsmChain>(t)) return sg::kChainPsm;
    if (chain_matches<sg::EcmChain>(t)) return sg::kChainEcm;
    if (chain_matches<sg::StarChain>(t)) return sg::kChainStar;
  }
  return t.dof <= 8 ? sg::kChainGeneric8 : sg::kChainGeneric16;
}

// DynamicsConfig resolution for one robot (envs.cpp:142-158: empty gain
// vectors -> default_dynamics_config, dynamics.cpp:69-86; one value ->
// broadcast) and DynamicsConfig::validate (dynamics.cpp:44-67).
struct ResolvedDyn {
  sg_dynamics_config dc;
  std::vector<double> kp, kd, inertia, damping;
  double dt_sub;
};

ResolvedDyn resolve_dynamics(const sg_dynamics_config* dyn, const sg::RobotModel& m) {
  sg_dynamics_config dc;
  sg_dynamics_config_init(&dc);
  if (dyn) dc = *dyn;
  const int dof = m.dof_count;
  std::vector<double> dkp(dof), dkd(dof), dinert(dof), ddamp(dof);
  for (int d = 0; d < dof; ++d) {
    const double mass = m.dof_joint(d).kind == sg::JointKind::Prismatic ? 0.5 : 0.05;
    dinert[d] = mass;
    dkp[d] = 380.0 * mass;
    dkd[d] = 2.0 * std::sqrt(dkp[d] * mass);
    ddamp[d] = 0.1 * dkd[d];
  }
  auto kp = resolve_gain(dc.kp, dc.n_kp, dkp, dof, "kp");
  auto kd = resolve_gain(dc.kd, dc.n_kd, dkd, dof, "kd");
  auto inertia = resolve_gain(dc.inertia, dc.n_inertia, dinert, dof, "inertia");
  auto damping = resolve_gain(dc.damping, dc.n_damping, ddamp, dof, "damping");
  if (!(dc.control_dt > 0.0)) throw sg::ConfigError("dynamics.control_dt must be > 0");
  if (dc.substeps < 1) throw sg::ConfigError("dynamics.substeps must be >= 1");
  if (dc.control_mode < 0 || dc.control_mode > 2) throw sg::ConfigError("unknown control mode");
  auto check_vec = [&](const std::vector<double>& v, const char* name, bool positive) {
    if (static_cast<int>(v.size()) != dof)
      throw sg::ConfigError(std::string("dynamics.") + name + " must have one entry per DoF (" +
                            std::to_string(dof) + "), got " + std::to_string(v.size()));
    for (size_t i = 0; i < v.size(); ++i) {
      if (positive && !(v[i] > 0.0))
        throw sg::ConfigError(std::string("dynamics.") + name + "[" + std::to_string(i) + "] must be > 0");
      if (!positive && v[i] < 0.0)
        throw sg::ConfigError(std::string("dynamics.") + name + "[" + std::to_string(i) + "] must be >= 0");
    }
  };
  check_vec(kp, "kp", true);
  check_vec(kd, "kd", true);
  check_vec(inertia, "inertia", true);
  check_vec(damping, "damping", false);
  return ResolvedDyn{dc, kp, kd, inertia, damping, dc.control_dt / dc.substeps};
}

// Eigen's quaternion * vector (_transformVector): uv = 2 (u x v); v + w uv + u x uv.
sg::Vec3 quat_rotate(const double* q, const sg::Vec3& v) {
  const double u[3] = {q[1], q[2], q[3]};
  double uv[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
  for (double& x : uv) x += x;
  const double c[3] = {u[1] * uv[2] - u[2] * uv[1], u[2] * uv[0] - u[0] * uv[2], u[0] * uv[1] - u[1] * uv[0]};
  return {v[0] + q[0] * uv[0] + c[0], v[1] + q[0] * uv[1] + c[1], v[2] + q[0] * uv[2] + c[2]};
}

// default_tool_bases (envs.cpp:101-116): xyz + quaternion (w, x, y, z).
std::vector<std::array<double, 7>> default_tool_bases(size_t n_tools, double r) {
  std::vector<std::array<double, 7>> b(n_tools, std::array<double, 7>{0, 0, 0, 1, 0, 0, 0});
  if (n_tools == 1) return b;
  const double dx = 0.7 * r;
  b[0][0] = -dx;
  b[1][0] = dx;
  if (n_tools >= 3) {  // camera arm behind the scene, pitched toward it
    b[2][1] = -2.0 * r;
    b[2][2] = 0.5 * r;
    const sg::Quat q = sg::quat_from_rpy(0.9, 0.0, 0.0);
    for (int k = 0; k < 4; ++k) b[2][3 + k] = q[k];
  }
  for (size_t t = 3; t < n_tools; ++t) b[t][1] = (static_cast<double>(t) - 1.0) * 2.0 * dx;
  return b;
}

// Rotation between the last actuated joint's frame and the tool-tip frame:
// the trailing fixed joints' origin rotations times the tip orientation
// (fk_walk, robot_model.cpp:371-395). build_table folds the trailing
// translations into the tip offset; the camera axis needs the rotation too.
Mat3 trailing_tip_rotation(const sg::RobotModel& m) {
  Mat3 R{1, 0, 0, 0, 1, 0, 0, 0, 1};
  for (const auto& j : m.joints) {
    if (j.kind != sg::JointKind::Fixed) {
      R = {1, 0, 0, 0, 1, 0, 0, 0, 1};
      continue;
    }
    if (!(j.origin_rotation == sg::Quat{1, 0, 0, 0})) R = mat_mul(R, quat_to_mat(j.origin_rotation));
  }
  if (!(m.tip_orientation == sg::Quat{1, 0, 0, 0})) R = mat_mul(R, quat_to_mat(m.tip_orientation));
  return R;
}

// VecTaskEnv construction for MultiToolReaching (envs.cpp:118-223): per-tool
// gain resolution and SimBatch (stream salt = tool), tool bases, workspace
// centres through the bases, tool-major observation layout.
std::unique_ptr<sg_env> make_multi_env(const sg_env_config& cfg, const sg_dynamics_config* dyn,
                                       std::vector<sg::RobotModel> models, int device) {
  const int T = static_cast<int>(models.size());
  if (T > sg::kMaxTools)
    throw sg::ConfigError("multi_tool_reaching: the device path supports at most " + std::to_string(sg::kMaxTools) +
                          " robots");
  auto env = std::make_unique<sg_env>();
  env->multi = true;
  env->cfg = cfg;
  env->device = device;
  CK(cudaSetDevice(device));
  env->n = cfg.n_envs;
  env->radius = cfg.workspace_radius > 0.0 ? cfg.workspace_radius : 3.0 * cfg.goal_sigma;  // envs.cpp:134
  if (cfg.n_tool_bases == 0) {
    env->bases = default_tool_bases(T, env->radius);
  } else {
    if (cfg.n_tool_bases != T || !cfg.tool_bases)
      throw sg::ConfigError("env.tool_bases must have one entry per robot");
    for (int t = 0; t < T; ++t) {
      std::array<double, 7> b;
      for (int k = 0; k < 7; ++k) b[k] = cfg.tool_bases[7 * t + k];
      env->bases.push_back(b);
    }
  }
  auto& M = env->M;
  M.T = T;
  int A = 0;
  ResolvedDyn rd0{};
  for (int t = 0; t < T; ++t) {
    const sg::RobotModel& m = models[t];
    if (m.dof_count > sg::kMaxToolDof)
      throw sg::ConfigError("multi_tool_reaching: robot '" + m.name + "' has more than " +
                            std::to_string(sg::kMaxToolDof) + " DoF (device path limit)");
    const ResolvedDyn rd = resolve_dynamics(dyn, m);
    if (t == 0) rd0 = rd;
    sg::ToolEnc& E = M.tool[t];
    E.robot = build_table(m, rd.dt_sub, rd.kp, rd.kd, rd.inertia, rd.damping);
    const auto& b = env->bases[t];
    const Mat3 bR = quat_to_mat(sg::Quat{b[3], b[4], b[5], b[6]});
    for (int k = 0; k < 9; ++k) E.base_R[k] = static_cast<float>(bR[k]);
    for (int k = 0; k < 3; ++k) E.base_p[k] = static_cast<float>(b[k]);
    const sg::Vec3 view = mat_vec(trailing_tip_rotation(m), sg::Vec3{0.0, 0.0, -1.0});
    for (int k = 0; k < 3; ++k) E.view[k] = static_cast<float>(view[k]);
    E.camera = m.name == "ecm" ? 1 : 0;  // envs.cpp:339, 545
    E.chain = chain_matches<sg::PsmChain>(E.robot)    ? sg::kChainPsm
              : chain_matches<sg::EcmChain>(E.robot)  ? sg::kChainEcm
              : chain_matches<sg::StarChain>(E.robot) ? sg::kChainStar
                                                      : sg::kChainGeneric8;
    E.off = A;
    A += m.dof_count;
    // workspace centre: tool_bases_[t].transform_point(FK(mid).position) (envs.cpp:159-161)
    const sg::Vec3 tip = sg::forward_kinematics_position(m, m.mid_configuration());
    const sg::Vec3 rt = quat_rotate(b.data() + 3, tip);
    const std::array<double, 3> c{b[0] + rt[0], b[1] + rt[1], b[2] + rt[2]};
    env->centers.push_back(c);
    for (int k = 0; k < 3; ++k) E.center[k] = c[k];
  }
  for (int k = 0; k < 3; ++k) env->center[k] = env->centers[0][k];
  M.A = A;
  M.scorer = 0;
  for (int t = 1; t < T; ++t)  // the least-loaded tool warp also scores
    if (models[t].dof_count <= models[M.scorer].dof_count) M.scorer = t;
  M.O = 3 * A + 6 * T;  // envs.cpp:166-192
  M.Os = M.O | 1;
  M.episode_len = cfg.episode_len;
  M.success_hold = cfg.success_hold;
  M.substeps = rd0.dc.substeps;
  M.control_mode = rd0.dc.control_mode;
  M.n = env->n;
  M.rho = static_cast<float>(cfg.reward_scale);
  M.success_radius = static_cast<float>(cfg.success_radius);
  M.dt_sub = static_cast<float>(rd0.dt_sub);
  M.collision_threshold = static_cast<float>(cfg.collision_threshold);
  M.collision_penalty = static_cast<float>(cfg.collision_penalty);
  M.view_penalty = static_cast<float>(cfg.view_penalty);
  M.goal_sigma = cfg.goal_sigma;
  M.radius = env->radius;
  env->A = A;
  env->O = M.O;

  int off = 0;
  auto add = [&](const char* name, int len) {
    env->layout.push_back({name, {off, len}});
    off += len;
  };
  add("dof_pos", A);
  add("dof_vel", A);
  add("tip_pos", 3 * T);
  add("dof_target", A);
  add("goal", 3 * T);

  const int64_t n = env->n;
  M.q = dalloc<float>(n * A);
  M.qd = dalloc<float>(n * A);
  M.qt = dalloc<float>(n * A);
  M.goals = dalloc<float>(n * 3 * T);
  M.tips = dalloc<float>(n * 3 * T);
  M.step_count = dalloc<int32_t>(n);
  M.hold_count = dalloc<int32_t>(n);
  M.episode_count = dalloc<int64_t>(n);
  M.rng_state = dalloc<uint64_t>(n * T);
  M.rng_inc = dalloc<uint64_t>(n * T);
  M.obs = dalloc<float>(n * M.O);
  M.tobs = dalloc<float>(n * M.O);
  M.rewards = dalloc<float>(n);
  M.task_error = dalloc<float>(n);
  M.terminated = dalloc<uint8_t>(n);
  M.timed_out = dalloc<uint8_t>(n);
  env->counters = dalloc<unsigned long long>(8);
  M.sat_total = env->counters;
  M.ended_total = env->counters + 1;
  M.err = reinterpret_cast<int32_t*>(env->counters + 2);
  CK(cudaHostAlloc(&env->h_counters, 4 * sizeof(unsigned long long), cudaHostAllocMapped));
  std::memset(env->h_counters, 0, 4 * sizeof(unsigned long long));
  // SimBatch::create per tool (dynamics.cpp:225-241): mid configuration at
  // rest, stream id = tool * 2^32 + global row
  std::vector<float> qh(static_cast<size_t>(n) * A);
  std::vector<uint64_t> st(static_cast<size_t>(n) * T), inc(static_cast<size_t>(n) * T);
  for (int t = 0; t < T; ++t) {
    const auto mid = models[t].mid_configuration();
    for (int d = 0; d < models[t].dof_count; ++d)
      for (int64_t i = 0; i < n; ++i) qh[(M.tool[t].off + d) * n + i] = static_cast<float>(mid[d]);
    for (int64_t i = 0; i < n; ++i) {
      const HostPcg r =
          make_stream(cfg.seed, (static_cast<uint64_t>(t) << 32) + static_cast<uint64_t>(cfg.row_offset + i));
      st[t * n + i] = r.state;
      inc[t * n + i] = r.inc;
    }
  }
  CK(cudaMemcpy(M.q, qh.data(), qh.size() * sizeof(float), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(M.qt, qh.data(), qh.size() * sizeof(float), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(M.rng_state, st.data(), st.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(M.rng_inc, inc.data(), inc.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
  env->d_actions_in = dalloc<float>(n * A);
  env->tools = std::move(models);
  env->model = env->tools[0];
  CK(cudaDeviceSynchronize());
  return env;
}

// VecTaskEnv construction for ImageMatching (envs.cpp:118-223 with
// RenderConfig::validate, render.cpp:24-32): single robot, identity tool
// base, per-env scene / target image / target camera, observation
// [q | qdot | tip | q_target | target image | current image].
std::unique_ptr<sg_env> make_image_env(const sg_env_config& cfg, const sg_dynamics_config* dyn,
                                       std::vector<sg::RobotModel> models, int device) {
  if (cfg.render_width < 8 || cfg.render_height < 8) throw sg::ConfigError("render: width and height must be >= 8");
  if (!(cfg.render_near > 0.0) || !(cfg.render_near < cfg.render_far))
    throw sg::ConfigError("render: require 0 < near < far");
  if (!(cfg.render_fov > 0.0) || !(cfg.render_fov < 3.1)) throw sg::ConfigError("render: fov must be in (0, pi)");
  auto env = std::make_unique<sg_env>();
  env->image = true;
  env->cfg = cfg;
  env->device = device;
  CK(cudaSetDevice(device));
  env->model = std::move(models[0]);
  const sg::RobotModel& m = env->model;
  const ResolvedDyn rd = resolve_dynamics(dyn, m);
  auto& I = env->I;
  I.robot = build_table(m, rd.dt_sub, rd.kp, rd.kd, rd.inertia, rd.damping);
  const Mat3 cr = trailing_tip_rotation(m);
  for (int k = 0; k < 9; ++k) I.cam_R[k] = static_cast<float>(cr[k]);
  // the camera FK only needs the chain structure (any control mode)
  I.chain = chain_matches<sg::PsmChain>(I.robot)    ? sg::kChainPsm
            : chain_matches<sg::EcmChain>(I.robot)  ? sg::kChainEcm
            : chain_matches<sg::StarChain>(I.robot) ? sg::kChainStar
            : I.robot.dof <= 8                      ? sg::kChainGeneric8
                                                    : sg::kChainGeneric16;
  env->n = cfg.n_envs;
  env->A = m.dof_count;
  I.A = m.dof_count;
  I.W = cfg.render_width;
  I.H = cfg.render_height;
  I.wh = I.W * I.H;
  I.O = 3 * I.A + 3 + 2 * I.wh;  // envs.cpp:185-188
  env->O = I.O;
  I.episode_len = cfg.episode_len;
  I.substeps = rd.dc.substeps;
  I.control_mode = rd.dc.control_mode;
  I.n = env->n;
  const double f = 0.5 * cfg.render_width / std::tan(0.5 * cfg.render_fov);  // render.cpp:39
  I.f = static_cast<float>(f);
  I.inv_f = static_cast<float>(1.0 / f);
  I.near_ = static_cast<float>(cfg.render_near);
  I.far_ = static_cast<float>(cfg.render_far);
  I.dt_sub = static_cast<float>(rd.dt_sub);
  I.sigma = cfg.goal_sigma;
  env->radius = cfg.workspace_radius > 0.0 ? cfg.workspace_radius : 3.0 * cfg.goal_sigma;  // envs.cpp:134
  I.radius = env->radius;
  const sg::Vec3 c = sg::forward_kinematics_position(m, m.mid_configuration());  // envs.cpp:159-161
  for (int k = 0; k < 3; ++k) env->center[k] = I.center[k] = c[k];
  int off = 0;
  auto add = [&](const char* name, int len) {
    env->layout.push_back({name, {off, len}});
    off += len;
  };
  add("dof_pos", I.A);
  add("dof_vel", I.A);
  add("tip_pos", 3);
  add("dof_target", I.A);
  add("target_image", I.wh);
  add("current_image", I.wh);
  const int64_t n = env->n;
  const int A = I.A;
  I.q = dalloc<float>(n * A);
  I.qd = dalloc<float>(n * A);
  I.qt = dalloc<float>(n * A);
  I.tips = dalloc<float>(n * 3);
  I.step_count = dalloc<int32_t>(n);
  I.hold_count = dalloc<int32_t>(n);
  I.episode_count = dalloc<int64_t>(n);
  I.rng_state = dalloc<uint64_t>(n);
  I.rng_inc = dalloc<uint64_t>(n);
  I.scenes = dalloc<float>(n * 16);
  I.target = dalloc<float>(static_cast<size_t>(n) * I.wh);
  I.tcam = dalloc<float>(n * 12);
  I.obs = dalloc<float>(static_cast<size_t>(n) * I.O);
  I.tobs = dalloc<float>(static_cast<size_t>(n) * I.O);
  I.rewards = dalloc<float>(n);
  I.task_error = dalloc<float>(n);
  I.terminated = dalloc<uint8_t>(n);
  I.timed_out = dalloc<uint8_t>(n);
  env->counters = dalloc<unsigned long long>(8);
  I.sat_total = env->counters;
  I.ended_total = env->counters + 1;
  I.err = reinterpret_cast<int32_t*>(env->counters + 2);
  CK(cudaHostAlloc(&env->h_counters, 4 * sizeof(unsigned long long), cudaHostAllocMapped));
  std::memset(env->h_counters, 0, 4 * sizeof(unsigned long long));
  {  // SimBatch::create (dynamics.cpp:225-241), stream id = global row
    const auto mid = m.mid_configuration();
    std::vector<float> qh(static_cast<size_t>(n) * A);
    for (int d = 0; d < A; ++d)
      for (int64_t i = 0; i < n; ++i) qh[d * n + i] = static_cast<float>(mid[d]);
    CK(cudaMemcpy(I.q, qh.data(), qh.size() * sizeof(float), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(I.qt, qh.data(), qh.size() * sizeof(float), cudaMemcpyHostToDevice));
    std::vector<uint64_t> st(n), inc(n);
    for (int64_t i = 0; i < n; ++i) {
      const HostPcg r = make_stream(cfg.seed, static_cast<uint64_t>(cfg.row_offset + i));
      st[i] = r.state;
      inc[i] = r.inc;
    }
    CK(cudaMemcpy(I.rng_state, st.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(I.rng_inc, inc.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice));
  }
  env->d_actions_in = dalloc<float>(n * A);
  CK(cudaDeviceSynchronize());
  return env;
}

std::unique_ptr<sg_env> make_env(const sg_env_config& cfg, const sg_dynamics_config* dyn,
                                 std::vector<sg::RobotModel> models, int device) {
  validate_env_config(cfg);
  if (models.empty()) throw sg::ConfigError("env: at least one robot is required");
  if (cfg.task == SG_TASK_MULTI_TOOL_REACHING) {
    if (models.size() < 2) throw sg::ConfigError("multi_tool_reaching requires >= 2 robots");
  } else if (models.size() != 1) {
    throw sg::ConfigError(std::string(task_name(cfg.task)) + " requires exactly 1 robot");
  }
  if (cfg.task == SG_TASK_MULTI_TOOL_REACHING) return make_multi_env(cfg, dyn, std::move(models), device);
  if (cfg.task == SG_TASK_IMAGE_MATCHING) {
    if (cfg.n_tool_bases != 0) throw sg::ConfigError("env.tool_bases: only supported for multi_tool_reaching");
    return make_image_env(cfg, dyn, std::move(models), device);
  }
  if (cfg.n_tool_bases != 0 && cfg.n_tool_bases != 1)
    throw sg::ConfigError("env.tool_bases must have one entry per robot");
  if (cfg.n_tool_bases == 1) {  // the single-tool kernels work in the robot base frame
    const double ident[7] = {0, 0, 0, 1, 0, 0, 0};
    if (!cfg.tool_bases || !std::equal(ident, ident + 7, cfg.tool_bases))
      throw sg::ConfigError("env.tool_bases: a non-identity base is only supported for multi_tool_reaching");
  }
  if (cfg.task != SG_TASK_TARGET_REACHING && cfg.task != SG_TASK_PATH_FOLLOWING &&
      cfg.task != SG_TASK_ACTIVE_TRACKING)
    throw sg::ConfigError(std::string("task '") + task_name(cfg.task) + "' is not on the sg_env device path");

  auto env = std::make_unique<sg_env>();
  env->model = std::move(models[0]);
  const sg::RobotModel& m = env->model;
  env->cfg = cfg;
  env->device = device;
  CK(cudaSetDevice(device));
  env->n = cfg.n_envs;
  env->A = m.dof_count;
  env->O = 3 * m.dof_count + 6;

  const ResolvedDyn rd = resolve_dynamics(dyn, m);
  const int dof = m.dof_count;
  const double dt_sub = rd.dt_sub;
  const sg_dynamics_config& dc = rd.dc;

  auto& P = env->P;
  P.robot = build_table(m, dt_sub, rd.kp, rd.kd, rd.inertia, rd.damping);

  // ---- task params ------------------------------------------------------------
  env->radius = cfg.workspace_radius > 0.0 ? cfg.workspace_radius : 3.0 * cfg.goal_sigma;  // envs.cpp:134
  const sg::Vec3 c = sg::forward_kinematics_position(m, m.mid_configuration());           // envs.cpp:161-162
  for (int k = 0; k < 3; ++k) env->center[k] = c[k];
  auto& T = P.task;
  T.task = cfg.task;
  T.episode_len = cfg.episode_len;
  T.success_hold = cfg.success_hold;
  T.substeps = dc.substeps;
  T.control_mode = dc.control_mode;
  T.n = env->n;
  T.rho = static_cast<float>(cfg.reward_scale);
  T.neg_alpha = static_cast<float>(-cfg.path_penalty);
  T.success_radius = static_cast<float>(cfg.success_radius);
  T.dt_sub = static_cast<float>(dt_sub);
  T.goal_sigma = cfg.goal_sigma;
  T.radius = env->radius;
  for (int k = 0; k < 3; ++k) T.center[k] = env->center[k];
  T.spacing = cfg.waypoint_spacing;
  T.goal_offset_clip = static_cast<float>(cfg.goal_offset_clip);
  T.track_noise_std = static_cast<float>(cfg.tracking_vel_noise_std);
  T.track_vel_clamp = static_cast<float>(cfg.tracking_vel_clamp);
  // Path length bound: |S'(u)| <= 3|a|u^2 + 2|b|u + |c| integrates to
  // |a| + |b| + |c| <= (0.5 + 0.5 + 0.3) * sqrt(3) (coefficient ranges of
  // sample_path, envs.cpp:244-246); shrinking only shortens the path.
  T.wp_cap = cfg.task == SG_TASK_PATH_FOLLOWING
                 ? static_cast<int32_t>(std::floor(1.3 * std::sqrt(3.0) / cfg.waypoint_spacing)) + 4
                 : 0;

  // ---- layout (envs.cpp:166-192) ---------------------------------------------
  int off = 0;
  auto add = [&](const char* name, int len) {
    env->layout.push_back({name, {off, len}});
    off += len;
  };
  add("dof_pos", dof);
  add("dof_vel", dof);
  add("tip_pos", 3);
  add("dof_target", dof);
  add(cfg.task == SG_TASK_PATH_FOLLOWING ? "waypoint" : "goal", 3);

  // ---- device state (SoA) -------------------------------------------------------
  const int64_t n = env->n;
  auto& p = P.p;
  p.q = dalloc<float>(n * dof);
  p.qd = dalloc<float>(n * dof);
  p.qt = dalloc<float>(n * dof);
  p.goals = dalloc<float>(n * 3);
  p.tips = dalloc<float>(n * 3);
  p.step_count = dalloc<int32_t>(n);
  p.hold_count = dalloc<int32_t>(n);
  p.episode_count = dalloc<int64_t>(n);
  p.wp_idx = dalloc<int32_t>(n);
  p.wp_len = dalloc<int32_t>(n);
  p.wps = T.wp_cap ? dalloc<float>(static_cast<size_t>(n) * T.wp_cap * 3) : nullptr;
  if (cfg.task == SG_TASK_ACTIVE_TRACKING) {
    p.goal_spawn = dalloc<float>(n * 3);
    p.goal_vel = dalloc<float>(n * 3);
  }
  if (T.wp_cap) {  // PathFollowing reset records (kernels.cuh path_record_kernel)
    p.rec_valid = dalloc<uint8_t>(n);
    p.rec_q = dalloc<float>(n * dof);
    p.rec_len = dalloc<int32_t>(n);
    p.rec_err = dalloc<int32_t>(n);
    p.rec_rng = dalloc<uint64_t>(n);
    p.rec_wps = dalloc<float>(static_cast<size_t>(n) * T.wp_cap * 3);
  }
  p.rng_state = dalloc<uint64_t>(n);
  p.rng_inc = dalloc<uint64_t>(n);
  p.obs = dalloc<float>(n * env->O);
  p.tobs = dalloc<float>(n * env->O);
  p.rewards = dalloc<float>(n);
  p.task_error = dalloc<float>(n);
  p.terminated = dalloc<uint8_t>(n);
  p.timed_out = dalloc<uint8_t>(n);
  // device counters in one 64-byte block: {saturation total, ended rows of
  // host-step slot A, error word, ended rows of slot B, CTA ticket, ended rows
  // of device steps, saturations of host-step slot A, of slot B}. The host
  // step reads its slot through a mapped pinned status the kernel's last CTA
  // fills (no copy, no memset); device steps never touch the host slots.
  env->counters = dalloc<unsigned long long>(8);
  p.sat_total = env->counters;
  p.ended_total = env->counters + 5;
  p.err = reinterpret_cast<int32_t*>(env->counters + 2);
  CK(cudaHostAlloc(&env->h_counters, 4 * sizeof(unsigned long long), cudaHostAllocMapped));
  std::memset(env->h_counters, 0, 4 * sizeof(unsigned long long));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&env->d_status), env->h_counters, 0));
  p.act_state = nullptr;
  p.act_buf = nullptr;
  // SimBatch::create (dynamics.cpp:225-241): mid configuration at rest, stream
  // id = salt * 2^32 + global row (single tool: salt 0).
  {
    const auto mid = m.mid_configuration();
    std::vector<float> qh(static_cast<size_t>(n) * dof);
    for (int d = 0; d < dof; ++d)
      for (int64_t i = 0; i < n; ++i) qh[d * n + i] = static_cast<float>(mid[d]);
    CK(cudaMemcpy(p.q, qh.data(), qh.size() * sizeof(float), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p.qt, qh.data(), qh.size() * sizeof(float), cudaMemcpyHostToDevice));
    std::vector<uint64_t> st(n), inc(n);
    for (int64_t i = 0; i < n; ++i) {
      HostPcg r = make_stream(cfg.seed, static_cast<uint64_t>(cfg.row_offset + i));
      st[i] = r.state;
      inc[i] = r.inc;
    }
    CK(cudaMemcpy(p.rng_state, st.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p.rng_inc, inc.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice));
  }
  env->d_actions_in = dalloc<float>(n * dof);
  // kernel selection: compile-time chain structure when the descriptor's
  // structure matches a builtin one and the dynamics are the reference
  // defaults' shape (position control, 4 substeps); generic chain otherwise
  // (every single-robot task, ActiveTracking included, has specialised instantiations)
  env->chain = select_chain(P.robot, dc.control_mode, dc.substeps);
  env->team_warps = team_warps_for(env->chain);
  env->team_layout = team_layout_from_env();
  if (const char* f = std::getenv("SG_HOST_POLL")) env->host_poll = std::atoi(f) != 0;
  CK(cudaDeviceSynchronize());
  return env;
}

}  // namespace

extern "C" {

const char* sg_last_error(void) { return g_last_error.c_str(); }
const char* sg_version(void) { return "sg_env 0.1 (sm_100a)"; }

void sg_env_config_init(sg_env_config* c) {  // envs.hpp:42-63
  std::memset(c, 0, sizeof(*c));
  c->task = SG_TASK_TARGET_REACHING;
  c->n_envs = 1024;
  c->episode_len = 300;
  c->goal_sigma = 0.05;
  c->goal_offset_clip = 0.2;
  c->reward_scale = -1.0;
  c->path_penalty = 1.0;
  c->success_radius = 0.005;
  c->success_hold = 10;
  c->workspace_radius = 0.0;
  c->waypoint_spacing = 0.02;
  c->tracking_vel_noise_std = 0.01;
  c->tracking_vel_clamp = 0.01;
  c->collision_threshold = 0.01;
  c->collision_penalty = 1.0;
  c->view_penalty = 0.1;
  c->seed = 0;
  c->row_offset = 0;
  c->render_width = 32;  // render.hpp:31-36
  c->render_height = 32;
  c->render_fov = 1.0471975511965976;
  c->render_near = 0.005;
  c->render_far = 2.0;
}

void sg_dynamics_config_init(sg_dynamics_config* d) {  // dynamics.hpp:34-44
  std::memset(d, 0, sizeof(*d));
  d->control_dt = 0.01;
  d->substeps = 4;
  d->control_mode = SG_CONTROL_POSITION;
}

int sg_env_create(const sg_env_config* cfg, const sg_dynamics_config* dyn, const char* const* robots,
                  int32_t n_robots, int32_t device, sg_env** out) {
  return guard([&] {
    if (!cfg || !out) throw sg::ConfigError("sg_env_create: null argument");
    std::vector<sg::RobotModel> models;
    for (int i = 0; i < n_robots; ++i) models.push_back(sg::resolve_robot(robots[i]));
    *out = make_env(*cfg, dyn, std::move(models), device).release();
  });
}

int sg_env_create_from_text(const sg_env_config* cfg, const sg_dynamics_config* dyn, const char* const* texts,
                            const char* const* origins, int32_t n_robots, int32_t device, sg_env** out) {
  return guard([&] {
    if (!cfg || !out) throw sg::ConfigError("sg_env_create_from_text: null argument");
    std::vector<sg::RobotModel> models;
    for (int i = 0; i < n_robots; ++i)
      models.push_back(sg::parse_robot(texts[i], origins && origins[i] ? origins[i] : "inline"));
    *out = make_env(*cfg, dyn, std::move(models), device).release();
  });
}

void sg_env_destroy(sg_env* env) { delete env; }

int sg_env_set_stream(sg_env* env, void* stream) {
  return guard([&] { env->stream = static_cast<cudaStream_t>(stream); });
}

int sg_env_dims(const sg_env* env, int64_t* n, int32_t* obs_dim, int32_t* action_dim) {
  return guard([&] {
    if (n) *n = env->n;
    if (obs_dim) *obs_dim = env->O;
    if (action_dim) *action_dim = env->A;
  });
}

int32_t sg_env_layout_count(const sg_env* env) { return static_cast<int32_t>(env->layout.size()); }

int sg_env_layout_field(const sg_env* env, int32_t index, const char** name, int32_t* offset, int32_t* length) {
  return guard([&] {
    if (index < 0 || index >= static_cast<int32_t>(env->layout.size()))
      throw sg::ConfigError("layout field index out of range");
    const auto& f = env->layout[index];
    if (name) *name = f.first.c_str();
    if (offset) *offset = f.second.first;
    if (length) *length = f.second.second;
  });
}

int sg_env_workspace(const sg_env* env, double* center3, double* radius) {
  return guard([&] {
    for (int k = 0; k < 3; ++k) center3[k] = env->center[k];
    *radius = env->radius;
  });
}

int sg_env_tools(const sg_env* env, int32_t* n_tools, double* centers, double* bases, int32_t* dofs) {
  return guard([&] {
    const int T = env->multi ? env->M.T : 1;
    if (n_tools) *n_tools = T;
    for (int t = 0; t < T; ++t) {
      for (int k = 0; k < 3; ++k)
        if (centers) centers[3 * t + k] = env->multi ? env->centers[t][k] : env->center[k];
      for (int k = 0; k < 7; ++k)
        if (bases) bases[7 * t + k] = env->multi ? env->bases[t][k] : (k == 3 ? 1.0 : 0.0);
      if (dofs) dofs[t] = env->multi ? env->tools[t].dof_count : env->A;
    }
  });
}

int sg_env_images(const sg_env* env, float** d_target, float** d_scenes, float** d_target_cameras, int32_t* width,
                  int32_t* height) {
  return guard([&] {
    if (!env->image) throw sg::ConfigError("sg_env_images: not an image_matching env");
    if (d_target) *d_target = env->I.target;
    if (d_scenes) *d_scenes = env->I.scenes;
    if (d_target_cameras) *d_target_cameras = env->I.tcam;
    if (width) *width = env->I.W;
    if (height) *height = env->I.H;
  });
}

int sg_env_reset(sg_env* env, sg_step_views* out) {
  NvtxRange nvtx("sg_env_reset");
  return guard([&] {
    CK(cudaSetDevice(env->device));
    if (env->own_kernel()) env->launch_mt(0, false, true);
    else env->launch_reset();
    env->views(out);
  });
}

int sg_env_reset_host(sg_env* env, float* h_observations) {
  NvtxRange nvtx("sg_env_reset_host");
  return guard([&] {
    if (!h_observations) throw sg::SimError("env.reset: null observation buffer");
    CK(cudaSetDevice(env->device));
    if (env->own_kernel()) env->launch_mt(0, false, true);
    else env->launch_reset();
    sg_step_views v;
    env->views(&v);
    CK(cudaMemcpyAsync(h_observations, v.observations, env->n * env->O * sizeof(float), cudaMemcpyDeviceToHost,
                       env->stream));
    env->check();
  });
}

// Pinned, mapped host allocations made by sg_host_alloc: host base -> {bytes,
// device alias base}. A host step resolves its buffers here without a CUDA
// call per pointer (cudaPointerGetAttributes only for foreign buffers).
namespace {
struct HostAlloc {
  size_t bytes;
  uintptr_t dev;
};
std::mutex g_host_mu;
std::map<uintptr_t, HostAlloc> g_host_allocs;
}  // namespace

int sg_host_alloc(size_t bytes, void** out) {
  return guard([&] {
    if (!out) throw sg::ConfigError("sg_host_alloc: null output pointer");
    *out = nullptr;
    CK(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable | cudaHostAllocMapped));
    void* dev = nullptr;
    CK(cudaHostGetDevicePointer(&dev, *out, 0));
    std::lock_guard<std::mutex> lk(g_host_mu);
    g_host_allocs[reinterpret_cast<uintptr_t>(*out)] = HostAlloc{bytes ? bytes : 1, reinterpret_cast<uintptr_t>(dev)};
  });
}

int sg_host_free(void* p) {
  return guard([&] {
    if (!p) return;
    {
      std::lock_guard<std::mutex> lk(g_host_mu);
      g_host_allocs.erase(reinterpret_cast<uintptr_t>(p));
    }
    CK(cudaFreeHost(p));
  });
}

int sg_env_step_into(sg_env* env, const float* d_actions, const sg_step_out* dst, sg_step_views* out) {
  NvtxRange nvtx("sg_env_step_into");
  return guard([&] {
    if (!d_actions) throw sg::SimError("env.step: action shape mismatch");
    CK(cudaSetDevice(env->device));
    const sg_step_out none{};
    const sg_step_out& d = dst ? *dst : none;
    if (env->own_kernel()) {  // task kernels: step, then device copies into the caller's buffers
      env->M.actions = d_actions;
      env->I.actions = d_actions;
      env->launch_mt(1, false, false);
      sg_step_views v;
      env->views(&v);
      const auto cp = [&](void* to, const void* from, size_t bytes) {
        if (to) CK(cudaMemcpyAsync(to, from, bytes, cudaMemcpyDeviceToDevice, env->stream));
      };
      cp(d.observations, v.observations, env->n * env->O * sizeof(float));
      cp(d.rewards, v.rewards, env->n * sizeof(float));
      cp(d.task_error, v.task_error, env->n * sizeof(float));
      cp(d.terminated, v.terminated, env->n);
      cp(d.timed_out, v.timed_out, env->n);
      env->views(out);
      return;
    }
    // the step kernel writes these fields only: point it at the caller's
    // buffers for this launch (restored on every exit path)
    if (d.observations && (reinterpret_cast<uintptr_t>(d.observations) & 15u) != 0)
      throw sg::ConfigError("sg_env_step_into: observations must be 16-byte aligned");
    auto& p = env->P.p;
    struct Restore {
      sg::EnvPtrs& p;
      float *obs, *rewards, *task_error;
      uint8_t *terminated, *timed_out;
      ~Restore() {
        p.obs = obs;
        p.rewards = rewards;
        p.task_error = task_error;
        p.terminated = terminated;
        p.timed_out = timed_out;
      }
    } restore{p, p.obs, p.rewards, p.task_error, p.terminated, p.timed_out};
    if (d.observations) p.obs = d.observations;
    if (d.rewards) p.rewards = d.rewards;
    if (d.task_error) p.task_error = d.task_error;
    if (d.terminated) p.terminated = d.terminated;
    if (d.timed_out) p.timed_out = d.timed_out;
    env->P.actions = d_actions;
    env->P.actions_aligned = (reinterpret_cast<uintptr_t>(d_actions) & 15u) == 0;
    env->launch_step(1, false);
    env->views(out);
  });
}

int sg_env_step(sg_env* env, const float* d_actions, sg_step_views* out) {
  NvtxRange nvtx("sg_env_step");
  return guard([&] {
    if (!d_actions) throw sg::SimError("env.step: action shape mismatch");
    CK(cudaSetDevice(env->device));
    if (env->own_kernel()) {
      env->M.actions = d_actions;
      env->I.actions = d_actions;
      env->launch_mt(1, false, false);
      env->views(out);
      return;
    }
    env->P.actions = d_actions;
    env->P.actions_aligned = (reinterpret_cast<uintptr_t>(d_actions) & 15u) == 0;
    env->launch_step(1, false);
    env->views(out);
  });
}

// cuStreamWaitValue32 through the runtime's driver entry-point lookup (the
// library does not link libcuda, so it still loads on a machine without a
// driver for the CPU-side tests).
using StreamWaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static StreamWaitValue32Fn stream_wait_value32() {
  static StreamWaitValue32Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      throw sg::SimError("host step: cuStreamWaitValue32 unavailable");
    return reinterpret_cast<StreamWaitValue32Fn>(p);
  }();
  return fn;
}

// Device alias of a host pointer the GPU can address directly (pinned memory
// from cudaMallocHost / cudaHostAlloc / cudaHostRegister; under UVA the alias
// equals the host address), or nullptr for pageable memory.
static void* mapped_alias(const void* h) {
  if (!h) return nullptr;
  {
    const uintptr_t u = reinterpret_cast<uintptr_t>(h);
    std::lock_guard<std::mutex> lk(g_host_mu);
    auto it = g_host_allocs.upper_bound(u);
    if (it != g_host_allocs.begin()) {
      --it;
      if (u - it->first < it->second.bytes) return reinterpret_cast<void*>(it->second.dev + (u - it->first));
    }
  }
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// Host step of the MultiToolReaching / ImageMatching kernels: staged copies
// around one launch, counters read back with the result (the zero-copy
// publication path is the single-tool env_step family's).
static void task_step_host(sg_env* env, const float* h_actions, sg_host_result* out) {
  const int64_t n = env->n;
  const int O = env->O;
  auto& s = env->stream;
  CK(cudaMemcpyAsync(env->d_actions_in, h_actions, n * env->A * sizeof(float), cudaMemcpyHostToDevice, s));
  env->M.actions = env->d_actions_in;
  env->I.actions = env->d_actions_in;
  // counters before the launch ({sat, ended} into h_counters[2..3]) and after
  // it: this step's deltas, whatever device steps ran since the last host step
  CK(cudaMemcpyAsync(env->h_counters + 2, env->counters, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  env->launch_mt(1, false, false);
  sg_step_views v;
  env->views(&v);
  if (out) {
    if (out->observations)
      CK(cudaMemcpyAsync(out->observations, v.observations, n * O * sizeof(float), cudaMemcpyDeviceToHost, s));
    if (out->rewards) CK(cudaMemcpyAsync(out->rewards, v.rewards, n * sizeof(float), cudaMemcpyDeviceToHost, s));
    if (out->task_error)
      CK(cudaMemcpyAsync(out->task_error, v.task_error, n * sizeof(float), cudaMemcpyDeviceToHost, s));
    if (out->terminated) CK(cudaMemcpyAsync(out->terminated, v.terminated, n, cudaMemcpyDeviceToHost, s));
    if (out->timed_out) CK(cudaMemcpyAsync(out->timed_out, v.timed_out, n, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaMemcpyAsync(env->h_counters, env->counters, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const unsigned long long sat = env->h_counters[0] - env->h_counters[2];
  const unsigned long long ended = env->h_counters[1] - env->h_counters[3];
  int32_t err = 0;
  CK(cudaMemcpy(&err, env->counters + 2, sizeof(err), cudaMemcpyDeviceToHost));
  env->raise(err);
  if (out && out->terminal_observations && ended != 0)
    CK(cudaMemcpy(out->terminal_observations, v.terminal_observations, n * O * sizeof(float),
                  cudaMemcpyDeviceToHost));
  env->last_ended += ended;
  env->last_sat += sat;
  if (out) out->action_saturations = static_cast<int64_t>(sat);
}

int sg_env_step_host(sg_env* env, const float* h_actions, sg_host_result* out) {
  NvtxRange nvtx("sg_env_step_host");
  return guard([&] {
    if (!h_actions) throw sg::SimError("env.step: action shape mismatch");
    CK(cudaSetDevice(env->device));
    if (env->own_kernel()) return task_step_host(env, h_actions, out);
    const int64_t n = env->n;
    const int O = env->O;
    auto& s = env->stream;
    auto& p = env->P.p;
    // Zero-copy when every buffer is pinned: the kernel reads the actions over
    // PCIe and writes the StepResult rows straight into the caller's buffers
    // (one launch, no copy-engine round trips). Pageable buffers: staged copies.
    bool zc = true;
    void* a_act = mapped_alias(h_actions);
    zc &= a_act != nullptr;
    float* host_f[4] = {nullptr, nullptr, nullptr, nullptr};
    uint8_t* host_u[2] = {nullptr, nullptr};
    if (out) {
      float* const fs[4] = {out->observations, out->terminal_observations, out->rewards, out->task_error};
      uint8_t* const us[2] = {out->terminated, out->timed_out};
      for (int k = 0; k < 4 && zc; ++k)
        if (fs[k]) zc &= (host_f[k] = static_cast<float*>(mapped_alias(fs[k]))) != nullptr;
      for (int k = 0; k < 2 && zc; ++k)
        if (us[k]) zc &= (host_u[k] = static_cast<uint8_t*>(mapped_alias(us[k]))) != nullptr;
      // obs rows are stored as float4 runs
      zc &= (reinterpret_cast<uintptr_t>(host_f[0]) & 15u) == 0 && (reinterpret_cast<uintptr_t>(host_f[1]) & 15u) == 0;
    }
    // rows ended in THIS step: alternate between two counter slots; the
    // launch zeroes the other one for the next host step
    const int slot = env->host_slot;
    env->host_slot ^= 1;
    p.ended_total = env->counters + (slot ? 3 : 1);
    p.ended_clear = env->counters + (slot ? 1 : 3);
    p.sat_step = env->counters + (slot ? 7 : 6);
    p.sat_clear = env->counters + (slot ? 6 : 7);
    p.ticket = reinterpret_cast<unsigned int*>(env->counters + 4);
    p.h_status = env->d_status;
    if (zc) {
      env->P.actions = static_cast<const float*>(a_act);
      env->P.actions_aligned = (reinterpret_cast<uintptr_t>(a_act) & 15u) == 0;
      p.h_obs = host_f[0];
      p.h_tobs = host_f[1];
      p.h_rewards = host_f[2];
      p.h_task_error = host_f[3];
      p.h_terminated = host_u[0];
      p.h_timed_out = host_u[1];
      p.h_seq = ++env->host_seq;
      // rolling PCIe read window (kernels.cuh StepParams::read_gate): only
      // (a team waits only on teams dispatched before it: CTAs start in index order)
      const int64_t teams = (n + 31) / 32;
      if (env->read_window > 0 && teams <= (int64_t)sg::sm_count() * 8) {
        p.read_gate = reinterpret_cast<unsigned int*>(env->counters + 4) + 1;
        p.read_window = env->read_window;
      }
      // observation rows by the copy engine, chunk by chunk (the legacy
      // one-team-per-CTA layout: chunk = block range)
      const int64_t teams_total = (n + 31) / 32;
      const int chunks = (int)std::min<int64_t>(std::min(env->ce_chunks, 64), teams_total);
      const bool ce = chunks > 0 && host_f[0] != nullptr && env->team_layout != sg::kLayoutPacked &&
                      !env->own_kernel();
      int chunk_teams = 0;
      if (ce) {
        if (!env->copy_stream) {
          CK(cudaStreamCreateWithFlags(&env->copy_stream, cudaStreamNonBlocking));
          CK(cudaEventCreateWithFlags(&env->copy_done, cudaEventDisableTiming));
          CK(cudaMalloc(&env->d_chunks, 128 * sizeof(unsigned int)));
          CK(cudaMemset(env->d_chunks, 0, 128 * sizeof(unsigned int)));
        }
        chunk_teams = (int)((teams_total + chunks - 1) / chunks);
        p.chunk_count = env->d_chunks;
        p.chunk_flag = env->d_chunks + 64;
        p.chunk_teams = chunk_teams;
        p.h_obs = nullptr;  // rows stay in HBM (P.p.obs) for the copy engine
      }
      env->launch_step(1, false);
      if (ce) {
        const unsigned seq = static_cast<unsigned>(p.h_seq);
        for (int c = 0; c * chunk_teams < teams_total; ++c) {
          const int64_t r0 = (int64_t)c * chunk_teams * 32, r1 = std::min<int64_t>(n, r0 + (int64_t)chunk_teams * 32);
          CU(stream_wait_value32()(env->copy_stream, reinterpret_cast<CUdeviceptr>(env->d_chunks + 64 + c), seq,
                                   CU_STREAM_WAIT_VALUE_GEQ));
          CK(cudaMemcpyAsync(out->observations + r0 * O, p.obs + r0 * O, (r1 - r0) * O * sizeof(float),
                             cudaMemcpyDeviceToHost, env->copy_stream));
        }
        CK(cudaEventRecord(env->copy_done, env->copy_stream));
        p.chunk_count = p.chunk_flag = nullptr;
      }
      p.read_gate = nullptr;
      p.h_obs = p.h_tobs = p.h_rewards = p.h_task_error = nullptr;
      p.h_terminated = p.h_timed_out = nullptr;
    } else {
      CK(cudaMemcpyAsync(env->d_actions_in, h_actions, n * env->A * sizeof(float), cudaMemcpyHostToDevice, s));
      env->P.actions = env->d_actions_in;
      env->P.actions_aligned = 1;
      env->launch_step(1, false);
      if (out) {
        if (out->observations)
          CK(cudaMemcpyAsync(out->observations, p.obs, n * O * sizeof(float), cudaMemcpyDeviceToHost, s));
        if (out->rewards) CK(cudaMemcpyAsync(out->rewards, p.rewards, n * sizeof(float), cudaMemcpyDeviceToHost, s));
        if (out->task_error)
          CK(cudaMemcpyAsync(out->task_error, p.task_error, n * sizeof(float), cudaMemcpyDeviceToHost, s));
        if (out->terminated) CK(cudaMemcpyAsync(out->terminated, p.terminated, n, cudaMemcpyDeviceToHost, s));
        if (out->timed_out) CK(cudaMemcpyAsync(out->timed_out, p.timed_out, n, cudaMemcpyDeviceToHost, s));
      }
    }
    p.h_status = nullptr;
    p.ended_clear = p.sat_step = p.sat_clear = nullptr;
    p.ended_total = env->counters + 5;
    if (zc && env->host_poll) {
      // The launch's last CTA writes the status and then h_status[3] = seq
      // behind system fences that order every CTA's result rows before it:
      // the result is complete once the flag arrives. cudaStreamQuery every
      // 256 polls catches a failed launch (the flag would never come).
      volatile unsigned long long* hs = env->h_counters;
      for (unsigned spins = 1; hs[3] != env->host_seq; ++spins) {
        if ((spins & 255u) == 0) {
          const cudaError_t e = cudaStreamQuery(s);
          if (e == cudaSuccess) {
            if (hs[3] != env->host_seq) throw sg::SimError("host step: completion flag missing after the launch");
            break;
          }
          if (e != cudaErrorNotReady) CK(e);
        }
      }
    } else {
      CK(cudaStreamSynchronize(s));
    }
    if (zc && env->copy_done && env->ce_chunks > 0 && out && out->observations)
      CK(cudaEventSynchronize(env->copy_done));  // the copy engine's observation rows
    const unsigned long long sat = env->h_counters[0], ended = env->h_counters[1];  // this step's
    env->raise(static_cast<int32_t>(env->h_counters[2] & 0xffffffffu));
    // terminal_observations are only meaningful on ended rows (envs.hpp:87);
    // staged path: copied only on steps where some row ended (1 step in 300
    // under random actions); zero-copy path: the kernel wrote the ended rows
    if (!zc && out && out->terminal_observations && ended != 0)
      CK(cudaMemcpy(out->terminal_observations, p.tobs, n * O * sizeof(float), cudaMemcpyDeviceToHost));
    env->last_ended += ended;
    env->last_sat += sat;
    if (out) out->action_saturations = static_cast<int64_t>(sat);
  });
}

int sg_env_host_counters(const sg_env* env, uint64_t* ended_rows_total, uint64_t* saturations_total) {
  return guard([&] {
    if (ended_rows_total) *ended_rows_total = env->last_ended;
    if (saturations_total) *saturations_total = env->last_sat;
  });
}

int sg_env_task_error(const sg_env* env, float** d) {
  return guard([&] { *d = env->multi ? env->M.task_error : (env->image ? env->I.task_error : env->P.p.task_error); });
}

int sg_env_state(const sg_env* env, sg_state_views* o) {
  return guard([&] {
    std::memset(o, 0, sizeof(*o));
    if (env->multi) {
      const auto& M = env->M;
      o->q = M.q;
      o->qdot = M.qd;
      o->q_target = M.qt;
      o->goals = M.goals;
      o->tips = M.tips;
      o->step_count = M.step_count;
      o->hold_count = M.hold_count;
      o->episode_count = M.episode_count;
      o->rng_state = M.rng_state;
      o->rng_inc = M.rng_inc;
      o->dof = env->A;
      o->n_envs = env->n;
      o->n_tools = M.T;
      return;
    }
    o->n_tools = 1;
    if (env->image) {
      const auto& I = env->I;
      o->q = I.q;
      o->qdot = I.qd;
      o->q_target = I.qt;
      o->tips = I.tips;
      o->step_count = I.step_count;
      o->hold_count = I.hold_count;
      o->episode_count = I.episode_count;
      o->rng_state = I.rng_state;
      o->rng_inc = I.rng_inc;
      o->dof = env->A;
      o->n_envs = env->n;
      return;
    }
    const auto& p = env->P.p;
    o->q = p.q;
    o->qdot = p.qd;
    o->q_target = p.qt;
    o->goals = p.goals;
    o->tips = p.tips;
    o->step_count = p.step_count;
    o->hold_count = p.hold_count;
    o->episode_count = p.episode_count;
    o->waypoint_idx = p.wp_idx;
    o->waypoint_len = p.wp_len;
    o->waypoints = p.wps;
    o->rng_state = p.rng_state;
    o->rng_inc = p.rng_inc;
    o->waypoint_cap = env->P.task.wp_cap;
    o->dof = env->A;
    o->n_envs = env->n;
  });
}

int sg_env_synchronize(sg_env* env) {
  return guard([&] {
    CK(cudaSetDevice(env->device));
    env->check();
  });
}

int sg_env_bench_begin(sg_env* env, uint64_t seed, int64_t first_step, int64_t global_n) {
  return guard([&] {
    CK(cudaSetDevice(env->device));
    if (global_n < env->n + env->cfg.row_offset) throw sg::ConfigError("bench: global_n_envs smaller than this shard");
    if (env->image) {  // one stream state per env at its row start; lane d reads draw d of the row
      auto& I = env->I;
      if (!I.act_state) {
        I.act_state = dalloc<uint64_t>(env->n);
        I.act_buf = dalloc<float>(env->n * env->A);
      }
      const HostPcg r = make_stream(seed, 0xac7104);  // bench.cpp:115
      sg::JumpTable J;
      for (int b = 0; b < 64; ++b) pcg_jump(1ULL << b, r.inc, J.mult[b], J.add[b]);
      const uint64_t A = static_cast<uint64_t>(env->A);
      I.act_inc = r.inc;
      pcg_jump(static_cast<uint64_t>(global_n) * A, r.inc, I.jump_mult, I.jump_add);
      for (int d = 0; d < sg::kMaxDof; ++d) pcg_jump(d, r.inc, I.pow_mult[d], I.pow_add[d]);
      const unsigned grid = static_cast<unsigned>((env->n + 127) / 128);
      sg::bench_seed_kernel<<<grid, 128, 0, env->stream>>>(I.act_state, env->n, r.state,
                                                           static_cast<uint64_t>(first_step) * global_n * A,
                                                           env->cfg.row_offset, env->A, J);
      CK(cudaGetLastError());
      env->bench_ready = true;
      return;
    }
    if (env->multi) {  // one stream state per env at its row start; A consecutive draws per row
      auto& M = env->M;
      if (!M.act_state) {
        M.act_state = dalloc<uint64_t>(env->n);
        M.act_buf = dalloc<float>(env->n * env->A);
      }
      const HostPcg r = make_stream(seed, 0xac7104);  // bench.cpp:115
      sg::JumpTable J;
      for (int b = 0; b < 64; ++b) pcg_jump(1ULL << b, r.inc, J.mult[b], J.add[b]);
      const uint64_t A = static_cast<uint64_t>(env->A);
      M.act_inc = r.inc;
      pcg_jump(static_cast<uint64_t>(global_n) * A, r.inc, M.jump_mult, M.jump_add);
      for (int t = 0; t < M.T; ++t)  // a tool warp's first draw of the row: `off` draws after the row start
        pcg_jump(static_cast<uint64_t>(M.tool[t].off), r.inc, M.tool[t].col_mult, M.tool[t].col_add);
      const unsigned grid = static_cast<unsigned>((env->n + 127) / 128);
      sg::bench_seed_kernel<<<grid, 128, 0, env->stream>>>(M.act_state, env->n, r.state,
                                                           static_cast<uint64_t>(first_step) * global_n * A,
                                                           env->cfg.row_offset, env->A, J);
      CK(cudaGetLastError());
      env->bench_ready = true;
      return;
    }
    auto& p = env->P.p;
    if (!p.act_state) {
      p.act_state = dalloc<uint64_t>(static_cast<size_t>(env->n) * sg::kMaxTeamWarps);
      p.act_buf = dalloc<float>(env->n * env->A);
    }
    const HostPcg r = make_stream(seed, 0xac7104);  // bench.cpp:115
    sg::JumpTable J;
    for (int b = 0; b < 64; ++b) pcg_jump(1ULL << b, r.inc, J.mult[b], J.add[b]);
    const uint64_t A = static_cast<uint64_t>(env->A);
    const uint64_t first_draw = static_cast<uint64_t>(first_step) * static_cast<uint64_t>(global_n) * A;
    env->P.bench.inc = r.inc;
    // warp s draws DoFs [b0, e0) of each row: it keeps the state at draw
    // first + g*A + b0, reads draw b0 + j by a j-advance, and moves on by
    // global_n*A per step
    pcg_jump(static_cast<uint64_t>(global_n) * A, r.inc, env->P.bench.jump_mult, env->P.bench.jump_add);
    for (int j = 0; j < sg::kMaxDof; ++j) pcg_jump(j, r.inc, env->P.bench.pow_mult[j], env->P.bench.pow_add[j]);
    for (int s = 0; s < env->team_warps; ++s) {
      int b0, e0;
      env->warp_block(s, b0, e0);
      const int bs = 128;
      const unsigned grid = static_cast<unsigned>((env->n + bs - 1) / bs);
      sg::bench_seed_kernel<<<grid, bs, 0, env->stream>>>(p.act_state + static_cast<size_t>(s) * env->n, env->n,
                                                          r.state, first_draw + static_cast<uint64_t>(b0),
                                                          env->cfg.row_offset, env->A, J);
      CK(cudaGetLastError());
    }
    env->bench_ready = true;
  });
}

int sg_env_bench_step(sg_env* env, int32_t k_steps) {
  NvtxRange nvtx("sg_env_bench_step");
  return guard([&] {
    if (!env->bench_ready) throw sg::ConfigError("sg_env_bench_step before sg_env_bench_begin");
    if (k_steps < 1) throw sg::ConfigError("bench: k_steps must be >= 1");
    CK(cudaSetDevice(env->device));
    if (env->own_kernel()) env->launch_mt(k_steps, true, false);
    else env->launch_step(k_steps, true);
  });
}

int sg_env_bench_actions(const sg_env* env, float** d_actions) {
  return guard([&] {
    float* buf = env->multi ? env->M.act_buf : (env->image ? env->I.act_buf : env->P.p.act_buf);
    if (!buf) throw sg::ConfigError("sg_env_bench_actions before sg_env_bench_begin");
    *d_actions = buf;
  });
}

// ---- robot utilities ----------------------------------------------------------
int sg_robot_parse(const char* text, const char* origin, sg_robot** out) {
  return guard([&] {
    auto r = std::make_unique<sg_robot>();
    r->model = sg::parse_robot(text, origin ? origin : "inline");
    std::vector<double> ones(r->model.dof_count, 1.0);
    r->table = build_table(r->model, 0.0025, ones, ones, ones, ones);
    *out = r.release();
  });
}

int sg_robot_resolve(const char* name_or_path, sg_robot** out) {
  return guard([&] {
    auto r = std::make_unique<sg_robot>();
    r->model = sg::resolve_robot(name_or_path);
    std::vector<double> ones(r->model.dof_count, 1.0);
    r->table = build_table(r->model, 0.0025, ones, ones, ones, ones);
    *out = r.release();
  });
}

void sg_robot_destroy(sg_robot* r) { delete r; }

int sg_robot_dof(const sg_robot* r, int32_t* dof, int32_t* jaw) {
  return guard([&] {
    if (dof) *dof = r->model.dof_count;
    if (jaw) *jaw = r->model.jaw_dof();
  });
}

int sg_robot_fk(const sg_robot* r, const float* d_q, int64_t n, float* d_pos, void* stream) {
  return guard([&] {
    if (n <= 0) return;
    int32_t* d_err = nullptr;
    CK(cudaMalloc(&d_err, sizeof(int32_t)));
    CK(cudaMemsetAsync(d_err, 0, sizeof(int32_t), static_cast<cudaStream_t>(stream)));
    const int b = 128;
    const unsigned grid = static_cast<unsigned>((n + b - 1) / b);
    if (r->model.dof_count <= 8)
      sg::fk_batch_kernel<8><<<grid, b, 0, static_cast<cudaStream_t>(stream)>>>(r->table, d_q, n, d_pos, d_err);
    else
      sg::fk_batch_kernel<16><<<grid, b, 0, static_cast<cudaStream_t>(stream)>>>(r->table, d_q, n, d_pos, d_err);
    cudaError_t le = cudaGetLastError();
    int32_t err = 0;
    cudaError_t ce = cudaMemcpyAsync(&err, d_err, sizeof(err), cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream));
    cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    cudaFree(d_err);
    CK(le);
    CK(ce);
    if (err) throw sg::SimError("forward_kinematics: joint value outside limits");
  });
}

}  // extern "C"
