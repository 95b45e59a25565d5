// The reference's bench_sim loop (bench.cpp:97-135) written against the fp64
// host drop-in (include/sg/host_env.hpp): reset, then steps with actions from
// make_stream(seed, 0xac7104) (bench.cpp:31-35). Writes the last step's
// StepResult and the run's counters to a binary file that
// tests/test_gpu_cpp.py compares with the fp64 oracle.
//   host_env_parity <out.bin> <n_envs> <steps> <seed>
#include <cstdio>
#include <cstdlib>

#include "sg/host_env.hpp"
#include "sg/rng.hpp"

namespace scalpel = scalpel_b200::host;  // the only line a reference caller adds

int main(int argc, char** argv) {
  using namespace scalpel;
  if (argc < 5) return 2;
  EnvConfig cfg;
  cfg.n_envs = std::atoll(argv[2]);
  cfg.seed = std::strtoull(argv[4], nullptr, 10);
  const int steps = std::atoi(argv[3]);
  ThreadPool pool(4);
  VecTaskEnv env(cfg, {resolve_robot("psm")}, DynamicsConfig(), RenderConfig(), &pool);
  BatchedEnv& base = env;  // callers hold the abstract surface, like Trainer (ppo.hpp:108)
  const MatrixXdR& obs0 = base.reset();
  double first = obs0(0, 0);
  Pcg32 rng = make_stream(cfg.seed, 0xac7104);
  MatrixXdR actions(base.n_envs(), base.action_dim());
  int64_t ended = 0, sat = 0;
  const StepResult* r = nullptr;
  for (int s = 0; s < steps; ++s) {
    fill_uniform_actions(rng, actions);
    r = &base.step(actions);
    for (int64_t i = 0; i < base.n_envs(); ++i) ended += r->terminated[i] | r->timed_out[i];
    sat += r->action_saturations;
  }
  FILE* f = std::fopen(argv[1], "wb");
  if (!f) return 3;
  const int64_t head[4] = {base.n_envs(), base.obs_dim(), ended, sat};
  std::fwrite(head, sizeof(head), 1, f);
  std::fwrite(&first, sizeof(double), 1, f);
  std::fwrite(r->observations.data(), sizeof(double), base.n_envs() * base.obs_dim(), f);
  std::fwrite(r->rewards.data(), sizeof(double), base.n_envs(), f);
  std::fwrite(base.task_error().data(), sizeof(double), base.n_envs(), f);
  std::fwrite(r->terminated.data(), 1, base.n_envs(), f);
  std::fwrite(r->timed_out.data(), 1, base.n_envs(), f);
  std::fwrite(r->terminal_observations.data(), sizeof(double), base.n_envs() * base.obs_dim(), f);
  std::fclose(f);
  return 0;
}
