/*
 * sg_env.h — C-ABI drop-in boundary for the batched environment step
 * (B200-native replacement of the reference "scalpel" VecTaskEnv hot path).
 *
 * Plain pointers and sizes only: no torch, no Eigen, no C++ types. Device
 * buffers are owned by the env handle; views returned by reset/step stay
 * valid until the next call on the same handle (ownership rule of the
 * reference: `reset()`/`step()` return const refs to member buffers,
 * proj/include/scalpel/envs.hpp:113-114,177).
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/proj):
 *   sg_env_create            VecTaskEnv::VecTaskEnv        src/envs.cpp:118-223
 *                            + make_env / resolve_robot      src/config.cpp:366-370,
 *                                                             src/robot_model.cpp:337-349
 *   sg_env_destroy           ~VecTaskEnv
 *   sg_env_dims              BatchedEnv::n_envs/obs_dim/action_dim  include/scalpel/envs.hpp:110-112
 *   sg_env_layout_*          VecTaskEnv::layout()          include/scalpel/envs.hpp:137, src/envs.cpp:166-192
 *   sg_env_tools             VecTaskEnv::tool_base / workspace centres  include/scalpel/envs.hpp:144,
 *                                                             src/envs.cpp:101-116,136-161
 *   sg_env_images            TaskState image-matching fields         include/scalpel/envs.hpp:73-76
 *   sg_env_reset             BatchedEnv::reset()           src/envs.cpp:425-435
 *   sg_env_step              BatchedEnv::step(actions)     src/envs.cpp:437-617
 *   sg_env_step_host         BatchedEnv::step on host buffers (same call a host-side
 *                            caller such as Trainer::iterate, src/ppo.cpp:279, makes)
 *   sg_env_task_error        BatchedEnv::task_error()      include/scalpel/envs.hpp:117
 *   sg_env_bench_*           bench_sim's action stream + step loop  src/bench.cpp:31-35,97-135
 *   sg_robot_*               parse_robot / forward_kinematics_batch  src/robot_model.cpp:191-283,404-443
 *   sg_policy_*              Policy ctor / forward (tensor cores)   src/policy.cpp:42-161
 *   sg_elu_*, sg_ppo_gather  ppo_update minibatch gather + ELU fwd/bwd  src/ppo.cpp:157-224, src/policy.cpp:33,163-218
 *   sg_ppo_loss              ppo_loss_and_grad (loss, metrics, analytic gradients)  src/ppo.cpp:76-155
 *   sg_last_error            exception message (what()) of the reference's
 *                            ConfigError / ParseError / SimError  include/scalpel/errors.hpp:23-48
 *
 * Error convention (tools/main.cpp:246-255 exit codes): every int-returning
 * entry point returns SG_OK (0), SG_ERR_SIM (1: SimError — shape mismatch,
 * non-finite action or reward, out-of-limit FK input) or SG_ERR_CONFIG
 * (2: ConfigError/ParseError — bad config or descriptor, goal sampling
 * exhaustion). The message is thread-local, read with sg_last_error().
 * Device-detected errors (non-finite action/reward, goal-sampling exhaustion)
 * are latched in a device error word and reported by the next synchronising
 * call (sg_env_step_host, sg_env_synchronize).
 */
#ifndef SG_ENV_H
#define SG_ENV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_OK 0
#define SG_ERR_SIM 1
#define SG_ERR_CONFIG 2

/* Task enum, same order as scalpel::Task (include/scalpel/envs.hpp:31-37). */
enum {
  SG_TASK_TARGET_REACHING = 0,
  SG_TASK_ACTIVE_TRACKING = 1,
  SG_TASK_IMAGE_MATCHING = 2,
  SG_TASK_PATH_FOLLOWING = 3,
  SG_TASK_MULTI_TOOL_REACHING = 4
};

/* scalpel::ControlMode (include/scalpel/dynamics.hpp:27). */
enum { SG_CONTROL_POSITION = 0, SG_CONTROL_VELOCITY = 1, SG_CONTROL_TORQUE = 2 };

/* scalpel::EnvConfig (include/scalpel/envs.hpp:42-63); defaults from
 * sg_env_config_init. row_offset = global index of this handle's row 0, so
 * per-env RNG streams are seeded by GLOBAL env id (multi-GPU sharding: rank r
 * of an N-per-rank job passes row_offset = r*N and is bit-identical to the
 * same rows of a single-device run). */
typedef struct sg_env_config {
  int32_t task;
  int32_t episode_len;
  int64_t n_envs;
  double goal_sigma;
  double goal_offset_clip;
  double reward_scale;
  double path_penalty;
  double success_radius;
  int32_t success_hold;
  int32_t reserved0;
  double workspace_radius;
  double waypoint_spacing;
  double tracking_vel_noise_std;
  double tracking_vel_clamp;
  double collision_threshold;
  double collision_penalty;
  double view_penalty;
  uint64_t seed;
  int64_t row_offset;
  /* MultiToolReaching tool base poses (EnvConfig::tool_bases, envs.hpp:59):
   * n_tool_bases x 7 doubles (x, y, z, qw, qx, qy, qz); 0 -> the reference's
   * default_tool_bases (envs.cpp:101-116), otherwise one per robot
   * ("env.tool_bases must have one entry per robot", envs.cpp:137-139). */
  const double* tool_bases;
  int32_t n_tool_bases;
  int32_t reserved1;
  /* ImageMatching camera (RenderConfig, render.hpp:31-38; defaults 32 x 32,
   * 60 deg horizontal fov, near 0.005, far 2.0). */
  int32_t render_width;
  int32_t render_height;
  double render_fov;
  double render_near;
  double render_far;
} sg_env_config;

/* scalpel::DynamicsConfig (include/scalpel/dynamics.hpp:34-44). Gain arrays
 * follow VecTaskEnv's resolution rule (src/envs.cpp:145-153): length 0 ->
 * per-robot defaults, 1 -> broadcast, dof -> per-DoF. */
typedef struct sg_dynamics_config {
  double control_dt;
  int32_t substeps;
  int32_t control_mode;
  const double* kp;
  int32_t n_kp;
  int32_t n_kd;
  const double* kd;
  const double* inertia;
  int32_t n_inertia;
  int32_t n_damping;
  const double* damping;
} sg_dynamics_config;

/* Device views of one StepResult (include/scalpel/envs.hpp:82-89), fp32 /
 * u8, row-major n_envs x obs_dim like the reference's MatrixXdR. Rows of ended
 * envs in `observations` are already post-reset; `terminal_observations` is
 * valid on ended rows only. `action_saturations_total` is a device u64 that
 * accumulates StepDiagnostics::saturated_actions over the handle's lifetime
 * (per-step value = difference of consecutive reads). */
typedef struct sg_step_views {
  float* observations;
  float* terminal_observations;
  float* rewards;
  float* task_error;
  uint8_t* terminated;
  uint8_t* timed_out;
  unsigned long long* action_saturations_total;
  int64_t n_envs;
  int32_t obs_dim;
  int32_t action_dim;
} sg_step_views;

/* Caller-owned DEVICE destinations of one step's results (sg_env_step_into):
 * observations row-major n_envs x obs_dim (stride obs_dim), the per-env
 * fields n_envs long. NULL fields go to the env's own buffers. */
typedef struct sg_step_out {
  float* observations;
  float* rewards;
  float* task_error;
  uint8_t* terminated;
  uint8_t* timed_out;
} sg_step_out;

/* Host copy of one StepResult (sg_env_step_host). Any pointer may be NULL
 * to skip that field's device->host copy. */
typedef struct sg_host_result {
  float* observations;
  float* terminal_observations;
  float* rewards;
  float* task_error;
  uint8_t* terminated;
  uint8_t* timed_out;
  int64_t action_saturations; /* this step */
} sg_host_result;

/* Device state views (SimBatch + TaskState, include/scalpel/sim_batch.hpp:28-41,
 * envs.hpp:66-80) for parity tests and integration. Joint arrays are DoF-major
 * structure-of-arrays: element (row, dof) lives at [dof * n_envs + row].
 * goals/tips: [k * n_envs + row], k = 0..2. Waypoint table: row-major
 * [row][waypoint_cap][3]. */
typedef struct sg_state_views {
  float* q;
  float* qdot;
  float* q_target;
  float* goals;
  float* tips;
  int32_t* step_count;
  int32_t* hold_count;
  int64_t* episode_count;
  int32_t* waypoint_idx;
  int32_t* waypoint_len;
  float* waypoints;
  uint64_t* rng_state;
  uint64_t* rng_inc;
  int32_t waypoint_cap;
  int32_t dof;
  int64_t n_envs;
  int32_t n_tools; /* MultiToolReaching: goals/tips are [3*n_tools][n], rng [n_tools][n] */
  int32_t reserved;
} sg_state_views;

typedef struct sg_env sg_env;

void sg_env_config_init(sg_env_config* cfg);
void sg_dynamics_config_init(sg_dynamics_config* dyn);

/* robots[i] is a builtin name ("psm", "ecm", "star") or a path to a .robot
 * descriptor (resolve_robot semantics). device: CUDA ordinal. */
int sg_env_create(const sg_env_config* cfg, const sg_dynamics_config* dyn,
                  const char* const* robots, int32_t n_robots, int32_t device, sg_env** out);
/* Same, from descriptor texts; origins[i] names the text in ParseError messages. */
int sg_env_create_from_text(const sg_env_config* cfg, const sg_dynamics_config* dyn,
                            const char* const* texts, const char* const* origins,
                            int32_t n_robots, int32_t device, sg_env** out);
void sg_env_destroy(sg_env* env);

/* cudaStream_t as void*; NULL = the legacy default stream. */
int sg_env_set_stream(sg_env* env, void* stream);
int sg_env_dims(const sg_env* env, int64_t* n_envs, int32_t* obs_dim, int32_t* action_dim);
int32_t sg_env_layout_count(const sg_env* env);
int sg_env_layout_field(const sg_env* env, int32_t index, const char** name, int32_t* offset,
                        int32_t* length);
int sg_env_workspace(const sg_env* env, double* center3, double* radius);
/* Per-tool geometry (VecTaskEnv::tool_base / workspace centres, envs.hpp:144,
 * envs.cpp:159-161): n_tools, and when non-NULL centers (3 per tool), bases
 * (7 per tool: xyz, quaternion wxyz), dofs (1 per tool). Single-robot tasks
 * report one tool with the identity base. */
int sg_env_tools(const sg_env* env, int32_t* n_tools, double* centers, double* bases, int32_t* dofs);
/* ImageMatching task state (TaskState::target_images / scenes / target_cameras,
 * envs.hpp:73-76) as device views: target images n x (w*h) fp32, scenes
 * n x 16 fp32 (3 spheres x {cx, cy, cz, radius, albedo}, 1 pad), target
 * cameras n x 12 fp32 (rotation row-major, position). SG_ERR_CONFIG for
 * other tasks. */
int sg_env_images(const sg_env* env, float** d_target, float** d_scenes, float** d_target_cameras, int32_t* width,
                  int32_t* height);

int sg_env_reset(sg_env* env, sg_step_views* out);
/* VecTaskEnv::reset() returning host observations (envs.cpp:425-435,
 * `const MatrixXdR& reset()`): reset on the device, copy the n_envs x obs_dim
 * fp32 observation rows into h_observations (pinned or pageable), synchronise
 * and report errors. */
int sg_env_reset_host(sg_env* env, float* h_observations);
/* Page-locked host memory for the host-step buffers (zero-copy path of
 * sg_env_step_host); any FFI caller can use it instead of its own allocator. */
int sg_host_alloc(size_t bytes, void** out);
int sg_host_free(void* p);
/* d_actions: device, row-major n_envs x action_dim fp32 (stride = action_dim). */
int sg_env_step(sg_env* env, const float* d_actions, sg_step_views* out);
/* sg_env_step writing the step's observations / rewards / task_error / flags
 * straight into caller device buffers (a trainer's rollout-buffer slot:
 * ppo.cpp:280-299 stores exactly these), instead of the env's own buffers
 * and a copy per field. terminal_observations stay env-owned (views). */
int sg_env_step_into(sg_env* env, const float* d_actions, const sg_step_out* dst, sg_step_views* out);
/* Host actions (pinned or pageable): H2D copy, step, D2H copy of the fields
 * requested in `out`, synchronise, report errors. terminal_observations is
 * copied only on steps where at least one row ended (it is defined on ended
 * rows only); otherwise the host buffer is left untouched. */
int sg_env_step_host(sg_env* env, const float* h_actions, sg_host_result* out);
int sg_env_task_error(const sg_env* env, float** d_task_error);
/* Running totals over the sg_env_step_host calls so far (host side, no sync):
 * rows that ended (terminated or timed out) and saturated action entries in
 * those host steps; device-side steps (sg_env_step, bench) are not counted. */
int sg_env_host_counters(const sg_env* env, uint64_t* ended_rows_total, uint64_t* saturations_total);
int sg_env_state(const sg_env* env, sg_state_views* out);
/* Waits for the env stream and converts the device error word. */
int sg_env_synchronize(sg_env* env);

/* Bench workload of bench_sim (src/bench.cpp:31-35,97-135): actions are draw
 * #(s*G*A + g*A + d) of make_stream(seed, 0xac7104) for step s, GLOBAL env g,
 * DoF d — the reference's serial row-major fill, reproduced bit-for-bit on the
 * device by PCG32 jump-ahead. global_n_envs/row_offset describe the sharding
 * (single device: n_envs / 0). first_step: index of the next step (0 = the
 * untimed warm-up step of bench_sim). */
int sg_env_bench_begin(sg_env* env, uint64_t seed, int64_t first_step, int64_t global_n_envs);
/* k_steps fused steps in ONE launch: per step, generate the actions (also
 * written to the env's action buffer), step, write the full StepResult and
 * auto-reset. Equivalent to k_steps calls of sg_env_step with those actions. */
int sg_env_bench_step(sg_env* env, int32_t k_steps);
/* Device buffer the bench generator writes (n_envs x action_dim fp32). */
int sg_env_bench_actions(const sg_env* env, float** d_actions);

/* Robot-model utilities. */
typedef struct sg_robot sg_robot;
int sg_robot_parse(const char* text, const char* origin, sg_robot** out);
int sg_robot_resolve(const char* name_or_path, sg_robot** out);
void sg_robot_destroy(sg_robot* robot);
int sg_robot_dof(const sg_robot* robot, int32_t* dof, int32_t* jaw_dof);
/* Batched FK on the device: d_q row-major n x dof fp32 -> d_pos n x 3 fp32.
 * Out-of-limit rows (check_q, src/robot_model.cpp:353-367) raise SG_ERR_SIM. */
int sg_robot_fk(const sg_robot* robot, const float* d_q, int64_t n, float* d_pos, void* stream);

/* Policy MLP forward on the tensor cores (tcgen05, BF16 in / FP32 accumulate):
 * Policy::forward (src/policy.cpp:110-161) for the reference's default
 * 256/128/64 ELU actor and critic trunks. d_flat is the reference's flat
 * parameter vector (policy.cpp:42-63) in fp32 on the device; load_params
 * packs it into bf16 UMMA images (call after every parameter update). */
typedef struct sg_policy sg_policy;
int sg_policy_create(int32_t obs_dim, int32_t action_dim, const int32_t* hidden, int32_t n_hidden,
                     int32_t device, sg_policy** out);
void sg_policy_destroy(sg_policy* policy);
int sg_policy_param_count(const sg_policy* policy, int64_t* count, int64_t* log_std_offset);
int sg_policy_load_params(sg_policy* policy, const float* d_flat, void* stream);
/* Policy::init_params (policy.cpp:87-102) on the host into h_flat (param_count fp32). */
int sg_policy_init_params(const sg_policy* policy, uint64_t seed, double init_log_std, float* h_flat);
/* d_obs: n x obs_stride fp32 (e.g. the env's observation view) -> d_mean
 * (n x action_dim), d_value (n). */
int sg_policy_forward(const sg_policy* policy, const float* d_obs, int64_t n, int32_t obs_stride,
                      float* d_mean, float* d_value, void* stream);
/* Bootstrap values (ppo.cpp:304-313): V(terminal obs) for rows with
 * timed_out && !terminated, 0 elsewhere; tiles without such rows skip all
 * tensor-core work. */
int sg_policy_bootstrap(const sg_policy* policy, const float* d_terminal_obs, int64_t n, int32_t obs_stride,
                        const uint8_t* d_timed_out, const uint8_t* d_terminated, float* d_value, void* stream);
/* Rollout sampling (ppo.cpp:262-277): actions = mean + exp(clamp(log_std)) * z,
 * logp = sum(-z^2/2 - log_std - log(2 pi)/2), z drawn from the trainer stream
 * (stream_state/inc = make_stream(seed, 0x7261696e)) at u32 draw
 * *d_draw_pos + step_offset + 2*(e*A + i), i.e. the reference's serial order. */
int sg_policy_sample(const float* d_mean, int64_t n, int32_t action_dim, const float* d_log_std_raw,
                     uint64_t stream_state, uint64_t stream_inc, const uint64_t* d_draw_pos,
                     uint64_t step_offset, float* d_actions, float* d_logp, void* stream);
/* Forward + rollout sampling in ONE tensor-core launch (the trainer's per-step
 * policy call, ppo.cpp:262-277): sg_policy_forward's value (and mean, when
 * d_mean != NULL) plus sg_policy_sample's actions / logp from the same draws,
 * bit-identical to the two separate calls. action_dim <= 16. */
int sg_policy_act(const sg_policy* policy, const float* d_obs, int64_t n, int32_t obs_stride,
                  const float* d_log_std_raw, uint64_t stream_state, uint64_t stream_inc, const uint64_t* d_draw_pos,
                  uint64_t step_offset, float* d_actions, float* d_logp, float* d_mean, float* d_value, void* stream);
/* sg_policy_act for rollout step t that also computes step t-1's timeout
 * bootstrap values (sg_policy_bootstrap's result: V(d_boot_obs row) where
 * d_timed_out && !d_terminated, else 0, into d_boot_value) in the same
 * launch: tiles with such rows run the critic trunk again on the terminal
 * rows, the others only write zeros. Bit-identical to the two calls. */
int sg_policy_act_bootstrap(const sg_policy* policy, const float* d_obs, int64_t n, int32_t obs_stride,
                            const float* d_log_std_raw, uint64_t stream_state, uint64_t stream_inc,
                            const uint64_t* d_draw_pos, uint64_t step_offset, float* d_actions, float* d_logp,
                            float* d_mean, float* d_value, const float* d_boot_obs, int32_t boot_stride,
                            const uint8_t* d_timed_out, const uint8_t* d_terminated, float* d_boot_value,
                            void* stream);
/* The stream part of sg_policy_sample ahead of the forward (it depends on
 * the trainer stream and log-std only): for every (env e, dim i) the draw at
 * *d_draw_pos + step_offset + 2*(e*A + i) -> d_scaled_noise[e*A + i] =
 * exp(clamp(log_std_i)) * z (fp64) and d_logp[e] = sum_i(-z^2/2 - log_std_i
 * - log(2 pi)/2) (dim order). Lets the trainer draw step t+1's noise on a
 * second stream while the env step produces step t+1's observations. */
int sg_policy_noise(const sg_policy* policy, int64_t n, const float* d_log_std_raw, uint64_t stream_state,
                    uint64_t stream_inc, const uint64_t* d_draw_pos, uint64_t step_offset, double* d_scaled_noise,
                    float* d_logp, void* stream);
/* Forward + actions from sg_policy_noise's output: actions = (float)(mean +
 * d_scaled_noise), bit-identical to sg_policy_act on the same draws. */
int sg_policy_act_noise(const sg_policy* policy, const float* d_obs, int64_t n, int32_t obs_stride,
                        const double* d_scaled_noise, float* d_actions, float* d_mean, float* d_value, void* stream);
/* The PPO update's minibatch forward (ppo.cpp:157-224 -> Policy::forward) on
 * the tensor cores, for the backward pass: bf16 observation rows d_obs_bf16
 * (n x obs_stride, obs_stride >= 32 and a multiple of 8, columns >= obs_dim
 * zero) -> every hidden activation, bf16 row-major per trunk (actor, critic):
 * d_h1 [2][n][256], d_h2 [2][n][128], d_h3 [2][n][64], and the last layer's
 * padded outputs d_out [2][n][8] (actor mean; critic value in column 0).
 * Uses the parameters of the last sg_policy_load_params. */
int sg_policy_train_forward(const sg_policy* policy, const void* d_obs_bf16, int64_t n, int32_t obs_stride, void* d_h1,
                            void* d_h2, void* d_h3, void* d_out, void* stream);
/* W^T images for sg_policy_dgrad_elu, packed from a flat fp32 parameter
 * vector: image i (i = trunk*3 + layer - 1, hidden layers 1..3) holds
 * W_i^T (in_dim[i] rows x out_dim[i] rounded up to 16 columns, bf16, the
 * UMMA K-major layout) at the byte offset of the images before it
 * (in_dim * round16(out_dim) * 2 bytes each); w_off[i] = offset of W_i
 * [out x in] row-major in d_flat. */
int sg_policy_pack_wt(const float* d_flat, const int64_t* w_off, const int32_t* out_dim, const int32_t* in_dim,
                      uint8_t* d_images, void* stream);
/* Weight gradient of one layer of the update's minibatch (Policy::backward,
 * policy.cpp:163-218): d_grad [out x in] fp32 = d_dy^T d_x over m rows, with
 * d_dy bf16 [m x out] and d_x bf16 [m x in] row-major (out x in of the
 * 256/128/64 trunk with padded obs / outputs: 256x32, 128x256, 64x128, 8x64).
 * parts CTAs each reduce a slice of rows on the tensor cores into
 * d_partial (parts * out * in fp32), then one pass sums them into d_grad. */
int sg_policy_wgrad(const void* d_dy, int32_t out_dim, const void* d_x, int32_t in_dim, int64_t m, float* d_partial,
                    int32_t parts, float* d_grad, void* stream);
/* Backward through one hidden layer of the update's minibatch
 * (Policy::backward, policy.cpp:163-218): d_dz = (d_dy W) * ELU'(d_h), where
 * ELU'(h) = h > 0 ? 1 : h + 1 from the stored output h; d_dy bf16 [m x k]
 * (row stride dy_stride), d_wt_image one sg_policy_pack_wt image, d_h /
 * d_dz bf16 [m x n_in]. One tensor-core launch (fp32 accumulation, one
 * rounding), instead of a GEMM writing d_dy W plus an elementwise pass.
 * Shapes of the 256/128/64 trunk: (n_in, k) = (256, 128), (128, 64), (64, <= 16). */
int sg_policy_dgrad_elu(const void* d_dy, int32_t dy_stride, int32_t k, const void* d_wt_image, int32_t n_in,
                        const void* d_h, void* d_dz, int64_t m, void* stream);
/* The whole backward through hidden layer l of the update's minibatch
 * (Policy::backward, policy.cpp:163-218) in one launch: d_dz = (d_dy W) *
 * ELU'(d_h) as sg_policy_dgrad_elu (same shapes), plus, when not NULL,
 * d_colsum[n_in] (fp32) += the column sums of d_dz (the bias gradient of
 * layer l-1) and d_wgrad[k x n_in] (fp32, row-major) += d_dy^T d_h (the
 * weight gradient of layer l; d_h is layer l's input). d_h / d_dz move
 * through TMA (16-byte aligned, row stride n_in). With d_x0 (bf16 [m x 32],
 * the input of layer l-1 = the 256-wide first layer's input, only for
 * n_in = 256), d_wgrad0[256 x 32] (fp32) += d_dz^T d_x0 as well -- the
 * first layer's weight gradient -- and d_dz (may be NULL) is not written. */
int sg_policy_layer_backward(const void* d_dy, int32_t dy_stride, int32_t k, const void* d_wt_image, int32_t n_in,
                             const void* d_h, void* d_dz, int64_t m, float* d_colsum, float* d_wgrad,
                             const void* d_x0, int32_t x0_width, float* d_wgrad0, void* stream);
/* The last two layers of one trunk's update backward (Policy::backward,
 * policy.cpp:163-218) in one launch: with dY_3 = d_dy3 (bf16 [m x k3], k3 <=
 * 8, row stride dy3_stride), h_3 / h_2 the stored outputs (bf16 [m x 64] /
 * [m x 128]) and the sg_policy_pack_wt images of W_3 (64 x 16) and W_2
 * (128 x 64): d_db3 += 1^T dY_3, d_dw3 [k3 x 64] += dY_3^T h_3, dZ_2 =
 * (dY_3 W_3) * ELU'(h_3) (kept on chip), d_db2 += 1^T dZ_2, d_dw2 [64 x 128]
 * += dZ_2^T h_2, d_dz1 [m x 128] = (dZ_2 W_2) * ELU'(h_2) (written) and
 * d_db1 += 1^T dZ_1. All fp32 gradients accumulate. */
int sg_policy_backward_tail(const void* d_dy3, int32_t dy3_stride, int32_t k3, const void* d_wt3_image,
                            const void* d_wt2_image, const void* d_h3, const void* d_h2, void* d_dz1, int64_t m,
                            float* d_db3, float* d_dw3, float* d_db2, float* d_dw2, float* d_db1, void* stream);
/* Flat-parameter layout sg_policy_load_params packs from: per (trunk, layer)
 * (actor layers 0..3 then critic) the offsets of W [out x in] row-major and
 * of b, the row stride in_dim[layer] and the row count out_dim[trunk*4 + l]
 * (a trainer's padded copy, e.g. obs width 27 -> 32, outputs 7 -> 8; padded
 * entries must be zero). Default: the reference layout (policy.cpp:42-63). */
int sg_policy_set_param_layout(sg_policy* policy, const int64_t* w_off, const int64_t* b_off, const int32_t* in_dim,
                               const int32_t* out_dim);
/* compute_gae (rollout.cpp:42-66, time-major [n_steps][n_envs]) without the
 * normalisation, plus episode statistics (ppo.cpp:286-303) accumulated into
 * d_stats4 = {reward_sum, episode_reward_sum, final_error_sum, episodes}. */
int sg_compute_gae(const float* d_rewards, const float* d_values, const uint8_t* d_terminated,
                   const uint8_t* d_timed_out, const float* d_bootstrap, const float* d_last_values,
                   const float* d_task_error, int32_t n_steps, int64_t n_envs, double gamma, double lambda,
                   float* d_advantages, float* d_returns, float* d_ep_acc, double* d_stats4, void* stream);
/* ppo_update's optimizer step (ppo.cpp:199-207) on a flat fp32 parameter
 * vector: global-norm clip of d_grad to max_grad_norm (when larger), Adam with
 * the reference's bias correction (Adam::step, ppo.cpp:56-64; m, v state,
 * step counter *d_step incremented on device), box projection of the log-std
 * segment [log_std_offset, +log_std_n) to [log_std_min, log_std_max], d_grad
 * zeroed, and (if non-NULL) a bf16 copy of the new parameters written to
 * d_bf16_mirror. d_grad_sq: two floats, [0] scratch (the squared norm),
 * [1] a sticky flag set to 1 when the gradient norm is not finite; the
 * parameters and moments are then left unchanged (the reference throws
 * "ppo_update: non-finite loss", ppo.cpp:193-199; the caller clears [1] and
 * raises after its next synchronisation). Graph-capturable. */
int sg_adam_step(float* d_params, float* d_grad, float* d_m, float* d_v, void* d_bf16_mirror, int64_t n,
                 float* d_grad_sq, int32_t* d_step, double lr, double beta1, double beta2, double eps,
                 double max_grad_norm, int64_t log_std_offset, int32_t log_std_n, double log_std_min,
                 double log_std_max, void* stream);
/* PPO update helpers around the library GEMMs (Trainer::update / ppo_update,
 * ppo.cpp:157-224; Policy::backward, policy.cpp:163-218). dtype 0 = fp32,
 * 1 = bf16; count a multiple of 4 (fp32) / 8 (bf16) elements, 16-byte aligned.
 * ELU forward h = z > 0 ? z : expm1(z) (may run in place); backward from the
 * output: dz = dh * (h > 0 ? 1 : h + 1). Graph-capturable. */
int sg_elu_forward(const void* d_z, void* d_h, int64_t count, int32_t dtype, void* stream);
int sg_elu_backward(const void* d_h, const void* d_dh, void* d_dz, int64_t count, int32_t dtype, void* stream);
/* ELU backward fused with the next-lower layer's bias gradient, bf16 row-major
 * [m x n] (n a multiple of 8): d_dz = d_dh * ELU'(d_h) and d_colsum[c] +=
 * sum over rows of d_dz[., c] (fp32 atomics: d_colsum is the bias gradient,
 * zero before the minibatch). d_h == NULL: a plain column sum of d_dh (the
 * last layer's bias gradient); d_dz == NULL: no dz output. */
int sg_elu_backward_colsum(const void* d_h, const void* d_dh, void* d_dz, int64_t m, int32_t n, float* d_colsum,
                           void* stream);
/* Minibatch gather (ppo.cpp:173-190): rows d_idx[0..m) of the rollout buffer:
 * obs (obs_w fp32 per row) into d_obs_out rows of obs_out_w >= obs_w (fp32, or
 * bf16 when obs_bf16; columns past obs_w zero), actions (A fp32), old
 * log-probs, advantages, returns. */
int sg_ppo_gather(const int64_t* d_idx, int64_t m, const float* d_obs, int32_t obs_w, void* d_obs_out,
                  int32_t obs_out_w, int32_t obs_bf16, const float* d_act, int32_t A, float* d_act_out,
                  const float* d_logp,
                  float* d_logp_out, const float* d_adv, float* d_adv_out, const float* d_ret, float* d_ret_out,
                  void* stream);
/* The data part of ppo_loss_and_grad (ppo.cpp:90-154) in one pass over a
 * minibatch of B samples: d_mean / d_value are the padded last-layer outputs
 * (row strides mstride >= A, vstride >= 1; dtype 0 fp32, 1 bf16), log-std
 * clamped to [ls_min, ls_max]; writes the analytic gradients d_dmean /
 * d_dvalue (same layout and dtype, padded columns zero) and d_dlog_std (A,
 * zero outside the box), d_out = {loss, policy_loss, value_loss, entropy, kl,
 * clip_fraction}; d_acc: 4 + A floats of scratch. A <= 16. */
int sg_ppo_loss(const void* d_mean, int32_t mstride, const void* d_value, int32_t vstride, int32_t dtype,
                const float* d_log_std_raw, const float* d_act, const float* d_old_logp, const float* d_adv,
                const float* d_ret, int64_t B, int32_t A, double clip_eps, double value_coef, double entropy_coef,
                double ls_min, double ls_max, void* d_dmean, void* d_dvalue, float* d_dlog_std, float* d_acc,
                float* d_out, void* stream);
/* Policy checkpoints in the reference's versioned binary format
 * (save_checkpoint / load_checkpoint, src/policy.cpp:220-295): "SCLPCKP1",
 * u32 version 1, obs_dim, action_dim, n_hidden, hidden[], length-prefixed
 * robot and task names, u64 param count, the flat parameter vector as
 * little-endian fp64 (reference layout, policy.cpp:42-63). load: any pointer
 * may be NULL (header-only read); hidden must hold 64 entries; the reference's
 * ConfigError messages (not a checkpoint, version, corrupt, truncated, count
 * mismatch) come back as SG_ERR_CONFIG. */
int sg_checkpoint_save(const char* path, int32_t obs_dim, int32_t action_dim, const int32_t* hidden,
                       int32_t n_hidden, const char* robot, const char* task, const double* h_params,
                       int64_t param_count);
int sg_checkpoint_load(const char* path, int32_t* obs_dim, int32_t* action_dim, int32_t* hidden, int32_t* n_hidden,
                       char* robot, int32_t robot_cap, char* task, int32_t task_cap, double* h_params,
                       int64_t params_cap, int64_t* param_count);
const char* sg_policy_last_error(void);

const char* sg_last_error(void);
const char* sg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SG_ENV_H */
