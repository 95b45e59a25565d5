// fp64 host-matrix drop-in for the reference's BatchedEnv surface
// (proj/include/scalpel/envs.hpp:82-118):
//
//   const MatrixXdR&  reset();
//   const StepResult& step(const Eigen::Ref<const MatrixXdR>& actions);
//   const VectorXd&   task_error() const;
//
// with StepResult = {MatrixXdR observations, VectorXd rewards,
// vector<uint8_t> terminated, timed_out, MatrixXdR terminal_observations,
// int64_t action_saturations}, in namespace scalpel_b200::host with the
// reference's names (BatchedEnv, VecTaskEnv, StepResult, EnvConfig,
// DynamicsConfig, RenderConfig, RobotModel / resolve_robot, ThreadPool,
// Pcg32 / make_stream, ConfigError / SimError). A caller written against the
// reference (Trainer takes BatchedEnv&, ppo.hpp:108; bench_sim constructs
// VecTaskEnv(cfg, {resolve_robot(name)}, dyn, render, &pool), bench.cpp:97-135)
// compiles unchanged after `namespace scalpel = scalpel_b200::host;`:
//
//  * with Eigen on the include path (or SG_WITH_EIGEN defined) MatrixXdR /
//    VectorXd ARE Eigen's types and step() takes Eigen::Ref<const MatrixXdR>;
//  * without Eigen, scalpel_b200::MatrixXdR / VectorXd are minimal row-major
//    fp64 containers with the accessors those callers use (rows, cols, size,
//    data, operator(), row-pointer access, setZero / resize).
//
// Each call converts the fp64 actions into a pinned fp32 staging buffer, runs
// ONE sg_env_step_host (the kernel reads the actions over PCIe and writes the
// StepResult rows into pinned fp32 buffers), then widens the result into the
// fp64 members the reference exposes. Terminal observations are widened only
// on rows that ended (they are defined on ended rows only, envs.hpp:87).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "env.hpp"
#include "rng.hpp"

#if !defined(SG_WITH_EIGEN) && defined(__has_include)
#if __has_include(<Eigen/Dense>)
#define SG_WITH_EIGEN 1
#endif
#endif
#ifdef SG_WITH_EIGEN
#include <Eigen/Dense>
#endif

namespace scalpel_b200 {
namespace host {

using scalpel_b200::ConfigError;
using scalpel_b200::DynamicsConfig;
using scalpel_b200::EnvConfig;
using scalpel_b200::make_stream;
using scalpel_b200::Pcg32;
using scalpel_b200::SimError;

// Constructor-compatibility types: a robot is named by a builtin ("psm",
// "ecm", "star") or a .robot path and parsed by the library
// (robot_model.cpp:337-349); the reference's render settings and host thread
// pool have no role on the device path.
struct RobotModel {
  std::string name_or_path;
};
inline RobotModel resolve_robot(const std::string& name_or_path) {
  sg_robot* r = nullptr;  // validate now, like the reference (ConfigError / ParseError)
  check(sg_robot_resolve(name_or_path.c_str(), &r));
  sg_robot_destroy(r);
  return RobotModel{name_or_path};
}
struct RenderConfig {};
class ThreadPool {
 public:
  explicit ThreadPool(int = 0) {}
};

#ifdef SG_WITH_EIGEN
using MatrixXdR = Eigen::Matrix<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>;
using VectorXd = Eigen::VectorXd;
using ActionsRef = Eigen::Ref<const MatrixXdR>;
#else
// Row-major fp64 matrix: the MatrixXdR accessors the reference's callers use.
class MatrixXdR {
 public:
  MatrixXdR() = default;
  MatrixXdR(int64_t rows, int64_t cols) { resize(rows, cols); }
  void resize(int64_t rows, int64_t cols) {
    rows_ = rows;
    cols_ = cols;
    v_.assign(static_cast<size_t>(rows * cols), 0.0);
  }
  void setZero() { std::fill(v_.begin(), v_.end(), 0.0); }
  int64_t rows() const { return rows_; }
  int64_t cols() const { return cols_; }
  int64_t size() const { return rows_ * cols_; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(int64_t r, int64_t c) { return v_[static_cast<size_t>(r * cols_ + c)]; }
  double operator()(int64_t r, int64_t c) const { return v_[static_cast<size_t>(r * cols_ + c)]; }
  const double* row_ptr(int64_t r) const { return v_.data() + r * cols_; }

 private:
  int64_t rows_ = 0, cols_ = 0;
  std::vector<double> v_;
};
class VectorXd {
 public:
  VectorXd() = default;
  explicit VectorXd(int64_t n) { resize(n); }
  void resize(int64_t n) { v_.assign(static_cast<size_t>(n), 0.0); }
  int64_t size() const { return static_cast<int64_t>(v_.size()); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator[](int64_t i) { return v_[static_cast<size_t>(i)]; }
  double operator[](int64_t i) const { return v_[static_cast<size_t>(i)]; }
  double& operator()(int64_t i) { return v_[static_cast<size_t>(i)]; }
  double operator()(int64_t i) const { return v_[static_cast<size_t>(i)]; }

 private:
  std::vector<double> v_;
};
using ActionsRef = const MatrixXdR&;
#endif

struct StepResult {  // envs.hpp:82-89
  MatrixXdR observations;  // ended rows already re-observed post-reset
  VectorXd rewards;
  std::vector<uint8_t> terminated;
  std::vector<uint8_t> timed_out;
  MatrixXdR terminal_observations;  // valid on ended rows
  int64_t action_saturations = 0;
};

// The reference's abstract surface with its host fp64 types (envs.hpp:107-118).
class BatchedEnv {
 public:
  virtual ~BatchedEnv() = default;
  virtual int64_t n_envs() const = 0;
  virtual int obs_dim() const = 0;
  virtual int action_dim() const = 0;
  virtual const MatrixXdR& reset() = 0;
  virtual const StepResult& step(ActionsRef actions) = 0;
  virtual const VectorXd& task_error() const = 0;
};

class VecTaskEnv : public BatchedEnv {
 public:
  VecTaskEnv(const EnvConfig& cfg, const std::vector<RobotModel>& models, const DynamicsConfig& dyn = DynamicsConfig(),
             const RenderConfig& = RenderConfig(), ThreadPool* = nullptr, int device = 0)
      : env_(cfg, names(models), dyn, device) {
    n_ = env_.n_envs();
    o_ = env_.obs_dim();
    a_ = env_.action_dim();
    act_ = pinned(n_ * a_);
    obs_ = pinned(n_ * o_);
    tobs_ = pinned(n_ * o_);
    rew_ = pinned(n_);
    err_ = pinned(n_);
    void* p = nullptr;
    check(sg_host_alloc(static_cast<size_t>(2 * n_), &p));
    flags_ = static_cast<uint8_t*>(p);
    res_.observations.resize(n_, o_);
    res_.terminal_observations.resize(n_, o_);
    res_.rewards.resize(n_);
    res_.terminated.assign(static_cast<size_t>(n_), 0);
    res_.timed_out.assign(static_cast<size_t>(n_), 0);
    task_error_.resize(n_);
  }
  ~VecTaskEnv() override {
    for (void* p : {static_cast<void*>(act_), static_cast<void*>(obs_), static_cast<void*>(tobs_),
                    static_cast<void*>(rew_), static_cast<void*>(err_), static_cast<void*>(flags_)})
      sg_host_free(p);
  }
  VecTaskEnv(const VecTaskEnv&) = delete;
  VecTaskEnv& operator=(const VecTaskEnv&) = delete;

  int64_t n_envs() const override { return n_; }
  int obs_dim() const override { return o_; }
  int action_dim() const override { return a_; }

  const MatrixXdR& reset() override {  // envs.cpp:425-435
    check(sg_env_reset_host(env_.handle(), obs_));
    widen(obs_, res_.observations.data(), n_ * o_);
    return res_.observations;
  }

  const StepResult& step(ActionsRef actions) override {  // envs.cpp:437-617
    if (actions.rows() != n_ || actions.cols() != a_) throw SimError("env.step: action shape mismatch");
    for (int64_t i = 0; i < n_; ++i)  // element access: an Eigen::Ref may carry an outer stride
      for (int j = 0; j < a_; ++j) act_[i * a_ + j] = static_cast<float>(actions(i, j));
    sg_host_result out{};
    out.observations = obs_;
    out.terminal_observations = tobs_;
    out.rewards = rew_;
    out.task_error = err_;
    out.terminated = flags_;
    out.timed_out = flags_ + n_;
    check(sg_env_step_host(env_.handle(), act_, &out));
    widen(obs_, res_.observations.data(), n_ * o_);
    widen(rew_, res_.rewards.data(), n_);
    widen(err_, task_error_.data(), n_);
    std::memcpy(res_.terminated.data(), flags_, static_cast<size_t>(n_));
    std::memcpy(res_.timed_out.data(), flags_ + n_, static_cast<size_t>(n_));
    for (int64_t i = 0; i < n_; ++i)
      if (flags_[i] | flags_[n_ + i]) widen(tobs_ + i * o_, res_.terminal_observations.data() + i * o_, o_);
    res_.action_saturations = out.action_saturations;
    return res_;
  }

  const VectorXd& task_error() const override { return task_error_; }
  scalpel_b200::VecTaskEnv& device_env() { return env_; }

 private:
  static std::vector<std::string> names(const std::vector<RobotModel>& models) {
    std::vector<std::string> out;
    for (const auto& m : models) out.push_back(m.name_or_path);
    return out;
  }
  float* pinned(int64_t count) {
    void* p = nullptr;
    check(sg_host_alloc(static_cast<size_t>(count) * sizeof(float), &p));
    return static_cast<float*>(p);
  }
  static void widen(const float* s, double* d, int64_t count) {
    for (int64_t k = 0; k < count; ++k) d[k] = static_cast<double>(s[k]);
  }

  scalpel_b200::VecTaskEnv env_;
  int64_t n_ = 0;
  int o_ = 0, a_ = 0;
  float *act_ = nullptr, *obs_ = nullptr, *tobs_ = nullptr, *rew_ = nullptr, *err_ = nullptr;
  uint8_t* flags_ = nullptr;
  StepResult res_;
  VectorXd task_error_;
};

}  // namespace host
}  // namespace scalpel_b200
