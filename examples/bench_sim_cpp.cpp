// The reference's bench_sim loop (proj/src/bench.cpp:97-135) written against
// the C++ drop-in: fresh env, reset, warm-up step, timed steps with host
// actions from make_stream(seed, 0xac7104). Build:
//   g++ -std=c++17 -O2 -Iinclude examples/bench_sim_cpp.cpp \
//       -Lpaper_2310_04676_b200/lib -lsg_env -Wl,-rpath,$PWD/paper_2310_04676_b200/lib -o bench_sim_cpp
#include <chrono>
#include <cstdio>
#include <vector>

#include "sg/env.hpp"

int main(int argc, char** argv) {
  using namespace scalpel_b200;
  EnvConfig cfg;
  cfg.n_envs = argc > 1 ? std::atoll(argv[1]) : 16384;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 200;
  try {
    VecTaskEnv env(cfg, {"psm"});
    env.reset();
    std::vector<float> actions(env.n_envs() * env.action_dim(), 0.25f);
    std::vector<float> obs(env.n_envs() * env.obs_dim()), rew(env.n_envs());
    sg_host_result out{};
    out.observations = obs.data();
    out.rewards = rew.data();
    env.step_host(actions.data(), &out);  // warm-up
    const auto t0 = std::chrono::steady_clock::now();
    for (int s = 0; s < steps; ++s) env.step_host(actions.data(), &out);
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("%lld envs x %d steps: %.3e env-steps/s (host buffers, C++ drop-in)\n",
                static_cast<long long>(env.n_envs()), steps, env.n_envs() * steps / sec);
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const SimError& e) {
    std::fprintf(stderr, "sim error: %s\n", e.what());
    return 1;
  }
  return 0;
}
