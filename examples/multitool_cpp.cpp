// Trimanual MultiToolReaching through the C++ drop-in (include/sg/env.hpp):
// the reference's config JSON {"env": {"task": "multi_tool_reaching",
// "tool_bases": [{"xyz": [...], "rpy": [...]}, ...]}, "robots": ["psm", "psm",
// "ecm"]} expressed on scalpel_b200::EnvConfig. Host-buffer steps, random
// actions, prints the mean reward per step.
//   g++ -std=c++17 -Iinclude examples/multitool_cpp.cpp -Lpaper_2310_04676_b200/lib -lsg_env
#include <cstdio>
#include <random>
#include <vector>

#include "sg/env.hpp"

int main() {
  using namespace scalpel_b200;
  EnvConfig cfg;
  cfg.task = SG_TASK_MULTI_TOOL_REACHING;
  cfg.n_envs = 1024;
  cfg.set_tool_bases({pose_from_xyz_rpy(-0.105, 0.0, 0.0, 0, 0, 0), pose_from_xyz_rpy(0.105, 0.0, 0.0, 0, 0, 0),
                      pose_from_xyz_rpy(0.0, -0.3, 0.075, 0.9, 0, 0)});  // default_tool_bases(3, 0.15)
  try {
    VecTaskEnv env(cfg, {"psm", "psm", "ecm"});
    std::printf("tools %d  action_dim %d  obs_dim %d\n", env.n_tools(), env.action_dim(), env.obs_dim());
    const int64_t n = env.n_envs();
    std::vector<float> act(n * env.action_dim()), obs(n * env.obs_dim()), rew(n);
    std::mt19937 gen(0);
    std::uniform_real_distribution<float> u(-1.f, 1.f);
    env.reset();
    for (int s = 0; s < 10; ++s) {
      for (auto& a : act) a = u(gen);
      sg_host_result out{};
      out.observations = obs.data();
      out.rewards = rew.data();
      env.step_host(act.data(), &out);
      double m = 0;
      for (float r : rew) m += r;
      std::printf("step %d mean reward %.5f\n", s, m / n);
    }
  } catch (const ConfigError& e) {
    std::printf("ConfigError: %s\n", e.what());
    return 2;
  } catch (const SimError& e) {
    std::printf("SimError: %s\n", e.what());
    return 1;
  }
  return 0;
}
