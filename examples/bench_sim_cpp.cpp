// The reference's bench_sim protocol (proj/src/bench.cpp:97-135) through the
// fp64 host drop-in (include/sg/host_env.hpp): the body below is the
// reference's loop -- fresh VecTaskEnv, reset, actions filled row-major from
// make_stream(seed, 0xac7104) (bench.cpp:31-35), one warm-up step, then timed
// steps -- with `namespace scalpel = scalpel_b200::host;` as the only change.
// Build:
//   g++ -std=c++17 -O2 -Iinclude examples/bench_sim_cpp.cpp -Lpaper_2310_04676_b200/lib -lsg_env
//       -Wl,-rpath,$PWD/paper_2310_04676_b200/lib -o bench_sim_cpp
//   ./bench_sim_cpp [n_envs=16384] [steps=200] [seed=0]
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "sg/host_env.hpp"

namespace scalpel = scalpel_b200::host;

int main(int argc, char** argv) {
  using namespace scalpel;
  EnvConfig cfg;
  cfg.n_envs = argc > 1 ? std::atoll(argv[1]) : 16384;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 200;
  cfg.seed = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 0;
  try {
    VecTaskEnv env(cfg, {resolve_robot("psm")}, DynamicsConfig(), RenderConfig());
    Pcg32 action_rng = make_stream(cfg.seed, 0xac7104);
    MatrixXdR actions(env.n_envs(), env.action_dim());
    env.reset();
    fill_uniform_actions(action_rng, actions);
    env.step(actions);  // warm-up: timing starts after the first step
    int64_t done = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int s = 0; s < steps; ++s) {
      fill_uniform_actions(action_rng, actions);
      env.step(actions);  // observations and rewards computed, then ignored
      done += env.n_envs();
    }
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("%lld envs x %d steps: %.3e env-steps/s (bench_sim protocol, fp64 host matrices, C++ drop-in)\n",
                static_cast<long long>(env.n_envs()), steps, done / sec);
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const SimError& e) {
    std::fprintf(stderr, "sim error: %s\n", e.what());
    return 1;
  }
  return 0;
}
