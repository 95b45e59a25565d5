// C++ drop-in over the C-ABI (include/sg_env.h): the method set of the
// reference's BatchedEnv / VecTaskEnv (proj/include/scalpel/envs.hpp:107-179),
// namespace scalpel_b200 in place of scalpel. Header-only; link libsg_env.so.
//
// Differences a caller sees: buffers are fp32 device
// memory (row-major n_envs x dim, the reference's MatrixXdR layout) owned by
// the env; step() takes device actions (or host actions via step_host());
// device-detected errors surface at the next synchronising call.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../sg_env.h"

namespace scalpel_b200 {

class ConfigError : public std::runtime_error {  // errors.hpp:23-26 (exit code 2)
 public:
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
class SimError : public std::runtime_error {  // errors.hpp:44-47 (exit code 1)
 public:
  explicit SimError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(int rc) {
  if (rc == SG_OK) return;
  if (rc == SG_ERR_CONFIG) throw ConfigError(sg_last_error());
  throw SimError(sg_last_error());
}

// geometry.hpp Pose: position + unit quaternion (w, x, y, z).
struct Pose {
  double position[3] = {0.0, 0.0, 0.0};
  double orientation[4] = {1.0, 0.0, 0.0, 0.0};
};

// quat_from_rpy (geometry.hpp:45-49): AngleAxis(yaw, Z) * AngleAxis(pitch, Y) *
// AngleAxis(roll, X) -- the reference's JSON tool_bases / origin `rpy`.
inline Pose pose_from_xyz_rpy(double x, double y, double z, double roll, double pitch, double yaw) {
  const double cr = std::cos(0.5 * roll), sr = std::sin(0.5 * roll), cp = std::cos(0.5 * pitch),
               sp = std::sin(0.5 * pitch), cy = std::cos(0.5 * yaw), sy = std::sin(0.5 * yaw);
  // (qz * qy) * qx
  const double w1 = cy * cp, x1 = -sy * sp, y1 = cy * sp, z1 = sy * cp;
  Pose p;
  p.position[0] = x;
  p.position[1] = y;
  p.position[2] = z;
  p.orientation[0] = w1 * cr - x1 * sr;
  p.orientation[1] = w1 * sr + x1 * cr;
  p.orientation[2] = y1 * cr + z1 * sr;
  p.orientation[3] = z1 * cr - y1 * sr;
  return p;
}

// envs.hpp:42-63 defaults; tool_bases (envs.hpp:59) kept as Poses and handed
// to the C-ABI as xyz + wxyz rows.
struct EnvConfig : sg_env_config {
  EnvConfig() { sg_env_config_init(this); }
  EnvConfig(const EnvConfig& o) : sg_env_config(o), bases_(o.bases_) { repoint(); }
  EnvConfig& operator=(const EnvConfig& o) {
    static_cast<sg_env_config&>(*this) = o;
    bases_ = o.bases_;
    repoint();
    return *this;
  }
  void set_tool_bases(const std::vector<Pose>& bases) {
    bases_.clear();
    for (const auto& b : bases) {
      bases_.insert(bases_.end(), b.position, b.position + 3);
      bases_.insert(bases_.end(), b.orientation, b.orientation + 4);
    }
    repoint();
  }

 private:
  void repoint() {
    tool_bases = bases_.empty() ? nullptr : bases_.data();
    n_tool_bases = static_cast<int32_t>(bases_.size() / 7);
  }
  std::vector<double> bases_;
};
struct DynamicsConfig : sg_dynamics_config {  // dynamics.hpp:34-44 defaults
  DynamicsConfig() { sg_dynamics_config_init(this); }
};

// StepResult (envs.hpp:82-89) as device views.
struct StepResult {
  const float* observations = nullptr;
  const float* rewards = nullptr;
  const uint8_t* terminated = nullptr;
  const uint8_t* timed_out = nullptr;
  const float* terminal_observations = nullptr;
};

struct ObservationField {
  std::string name;
  int offset = 0;
  int length = 0;
};

class BatchedEnv {  // envs.hpp:107-118
 public:
  virtual ~BatchedEnv() = default;
  virtual int64_t n_envs() const = 0;
  virtual int obs_dim() const = 0;
  virtual int action_dim() const = 0;
  virtual const float* reset() = 0;
  virtual const StepResult& step(const float* d_actions) = 0;
  virtual const float* task_error() const = 0;
};

class VecTaskEnv : public BatchedEnv {
 public:
  // robots: builtin names ("psm", "ecm", "star") or .robot paths.
  VecTaskEnv(const EnvConfig& cfg, const std::vector<std::string>& robots,
             const DynamicsConfig& dyn = DynamicsConfig(), int device = 0) {
    std::vector<const char*> names;
    for (const auto& r : robots) names.push_back(r.c_str());
    check(sg_env_create(&cfg, &dyn, names.data(), static_cast<int32_t>(names.size()), device, &env_));
    int32_t o = 0, a = 0;
    check(sg_env_dims(env_, &n_, &o, &a));
    obs_dim_ = o;
    action_dim_ = a;
  }
  ~VecTaskEnv() override { sg_env_destroy(env_); }
  VecTaskEnv(const VecTaskEnv&) = delete;
  VecTaskEnv& operator=(const VecTaskEnv&) = delete;

  int64_t n_envs() const override { return n_; }
  int obs_dim() const override { return obs_dim_; }
  int action_dim() const override { return action_dim_; }

  void set_stream(void* cuda_stream) { check(sg_env_set_stream(env_, cuda_stream)); }

  const float* reset() override {
    check(sg_env_reset(env_, &views_));
    fill();
    return views_.observations;
  }
  const StepResult& step(const float* d_actions) override {
    check(sg_env_step(env_, d_actions, &views_));
    fill();
    return result_;
  }
  // Host actions -> host StepResult (synchronous; reports device errors).
  int64_t step_host(const float* h_actions, sg_host_result* out) {
    check(sg_env_step_host(env_, h_actions, out));
    return out ? out->action_saturations : 0;
  }
  const float* task_error() const override {
    float* p = nullptr;
    check(sg_env_task_error(env_, &p));
    return p;
  }
  void synchronize() { check(sg_env_synchronize(env_)); }

  std::vector<ObservationField> layout() const {  // envs.cpp:166-192
    std::vector<ObservationField> out;
    for (int32_t i = 0; i < sg_env_layout_count(env_); ++i) {
      const char* name = nullptr;
      int32_t off = 0, len = 0;
      check(sg_env_layout_field(env_, i, &name, &off, &len));
      out.push_back({name, off, len});
    }
    return out;
  }
  // MultiToolReaching geometry: VecTaskEnv::tool_base (envs.hpp:144) and the
  // per-tool workspace centres (envs.cpp:159-161).
  int n_tools() const {
    int32_t t = 0;
    check(sg_env_tools(env_, &t, nullptr, nullptr, nullptr));
    return t;
  }
  Pose tool_base(int tool) const {
    const int t = n_tools();
    if (tool < 0 || tool >= t) throw ConfigError("tool index out of range");
    std::vector<double> b(7 * static_cast<size_t>(t));
    check(sg_env_tools(env_, nullptr, nullptr, b.data(), nullptr));
    Pose p;
    for (int k = 0; k < 3; ++k) p.position[k] = b[7 * tool + k];
    for (int k = 0; k < 4; ++k) p.orientation[k] = b[7 * tool + 3 + k];
    return p;
  }
  sg_env* handle() { return env_; }

 private:
  void fill() {
    result_.observations = views_.observations;
    result_.rewards = views_.rewards;
    result_.terminated = views_.terminated;
    result_.timed_out = views_.timed_out;
    result_.terminal_observations = views_.terminal_observations;
  }
  sg_env* env_ = nullptr;
  int64_t n_ = 0;
  int obs_dim_ = 0, action_dim_ = 0;
  sg_step_views views_{};
  StepResult result_{};
};

}  // namespace scalpel_b200
