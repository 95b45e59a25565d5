/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C11 + pthreads) of the reference "scalpel" hot path
 * (/root/reference/proj, C++20/Eigen, not buildable here: Eigen3 and vendor/
 * are absent). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library, and only as the
 * checker or the timed CPU baseline — never as the product path.
 *
 * Two builds come from the same source: libsg_oracle_f64.so (SGO_REAL=double,
 * the parity oracle, faithful to the reference's fp64 arithmetic) and
 * libsg_oracle_f32.so (SGO_REAL=float for state/FK/reward, fp64 for the reset
 * math exactly like the device) which measures intrinsic fp32 drift and sets
 * the parity tolerances.
 *
 * Pinning: see DESIGN.md §Oracle. The reference's own known-answer tests are
 * re-run against this code in tests/test_oracle_*.py (PCG32 KAT, FK vs
 * 4x4 homogeneous-matrix oracle at 1e-9, dynamics properties, spline KATs).
 */
#ifndef SG_ORACLE_H
#define SG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:25-83 ---------------------------------------------------- */
typedef struct { uint64_t state, inc; } sgo_pcg32;

void sgo_pcg32_seed(sgo_pcg32* r, uint64_t initstate, uint64_t initseq);
uint32_t sgo_pcg32_next(sgo_pcg32* r);
double sgo_pcg32_uniform(sgo_pcg32* r, double lo, double hi);
double sgo_pcg32_normal(sgo_pcg32* r);
void sgo_make_stream(uint64_t seed, uint64_t stream_id, sgo_pcg32* out);
/* bench.cpp:31-35 — row-major fill from one stream. */
void sgo_fill_uniform_actions(sgo_pcg32* r, double* actions, int64_t count);
void sgo_fill_normals(sgo_pcg32* r, double* z, int64_t count);

/* ---- robot_model.hpp:29-61 -------------------------------------------- */
#define SGO_MAX_JOINTS 32
enum { SGO_REVOLUTE = 0, SGO_PRISMATIC = 1, SGO_FIXED = 2 };

typedef struct {
  char name[64];
  int32_t kind;
  double axis[3];
  double origin_xyz[3];
  double origin_quat[4]; /* w x y z */
  double limit_lo, limit_hi, velocity_limit, effort_limit;
} sgo_joint;

typedef struct {
  char name[64];
  int32_t n_joints;
  sgo_joint joints[SGO_MAX_JOINTS];
  double tip_xyz[3];
  double tip_quat[4];
  int32_t jaw_joint; /* -1: none */
  int32_t dof;
  int32_t dof_to_joint[SGO_MAX_JOINTS];
} sgo_robot;

/* Returns 0 on success, 2 on ConfigError/ParseError (message in err). */
int sgo_parse_robot(const char* text, const char* origin, sgo_robot* out, char* err, int errlen);
int sgo_jaw_dof(const sgo_robot* m);
/* Forward kinematics in SGO_REAL precision; pos[3], quat[4] (w,x,y,z). */
void sgo_fk(const sgo_robot* m, const double* q, double* pos, double* quat);
/* 4x4 homogeneous-matrix oracle with Rodrigues rotations (test_robot_model.cpp:27-56). */
void sgo_fk_matrix(const sgo_robot* m, const double* q, double* mat16);

/* ---- dynamics.hpp:34-49 ----------------------------------------------- */
enum { SGO_POSITION = 0, SGO_VELOCITY = 1, SGO_TORQUE = 2 };
typedef struct {
  double control_dt;
  int32_t substeps;
  int32_t control_mode;
  double kp[SGO_MAX_JOINTS], kd[SGO_MAX_JOINTS], inertia[SGO_MAX_JOINTS], damping[SGO_MAX_JOINTS];
} sgo_dyn;
void sgo_default_dynamics(const sgo_robot* m, sgo_dyn* out);

/* Standalone SimBatch (sim_batch.hpp:28-41) for the dynamics KATs. State is
 * SGO_REAL internally; exposed through double views filled on demand. */
typedef struct sgo_sim sgo_sim;
sgo_sim* sgo_sim_create(const sgo_robot* m, int64_t n, uint64_t seed, uint64_t salt);
void sgo_sim_destroy(sgo_sim* s);
/* returns 0 ok, 1 SimError (non-finite action); *saturated receives the count */
int sgo_sim_step(sgo_sim* s, const double* actions, const sgo_dyn* cfg, int64_t* saturated);
void sgo_sim_reset_rows(sgo_sim* s, const uint8_t* mask);
void sgo_sim_get(const sgo_sim* s, double* q, double* qdot, double* q_target);
void sgo_sim_set(sgo_sim* s, const double* q, const double* qdot, const double* q_target);

/* ---- spline.hpp / spline.cpp ------------------------------------------ */
/* coeffs = a[3], b[3], c[3], d[3]. Returns waypoint count (may exceed cap:
 * only the first cap are written), -2 on ConfigError. */
int sgo_spline_waypoints(const double* coeffs, double t0, double t1, double spacing, double* out,
                         int cap);
double sgo_spline_arc_length(const double* coeffs, double t0, double t1, int subdivisions);

/* ---- envs.hpp:42-63 --------------------------------------------------- */
enum { SGO_TARGET_REACHING = 0, SGO_ACTIVE_TRACKING = 1, SGO_IMAGE_MATCHING = 2,
       SGO_PATH_FOLLOWING = 3, SGO_MULTI_TOOL = 4 };
typedef struct {
  int32_t task;
  int64_t n_envs;
  int32_t episode_len;
  double goal_sigma, goal_offset_clip, reward_scale, path_penalty, success_radius;
  int32_t success_hold;
  double workspace_radius, waypoint_spacing;
  double tracking_vel_noise_std, tracking_vel_clamp;
  uint64_t seed;
  int64_t row_offset; /* global id of row 0: stream id = row_offset + row */
  /* MultiToolReaching (envs.hpp:56-58) */
  double collision_threshold, collision_penalty, view_penalty;
  /* ImageMatching: RenderConfig (render.hpp:31-38) */
  int32_t render_w, render_h;
  double render_fov, render_near, render_far;
} sgo_env_cfg;
void sgo_env_cfg_default(sgo_env_cfg* c);

typedef struct sgo_env sgo_env;
/* threads: pool lanes (0 = hardware_concurrency, 1 = serial). NULL dyn -> defaults. */
sgo_env* sgo_env_create(const sgo_env_cfg* c, const sgo_robot* m, const sgo_dyn* dyn, int threads,
                        char* err, int errlen);
void sgo_env_destroy(sgo_env* e);
int sgo_env_obs_dim(const sgo_env* e);
int sgo_env_action_dim(const sgo_env* e);
int sgo_env_lanes(const sgo_env* e);
int sgo_env_reset(sgo_env* e);
/* 0 ok, 1 SimError (non-finite action / reward), 2 ConfigError (goal sampling). */
int sgo_env_step(sgo_env* e, const double* actions);
const char* sgo_env_error(const sgo_env* e);

/* Views, all converted to double (row-major, n_envs rows). */
void sgo_env_get_obs(const sgo_env* e, double* obs, double* terminal_obs);
void sgo_env_get_result(const sgo_env* e, double* rewards, uint8_t* terminated, uint8_t* timed_out,
                        double* task_error, int64_t* saturations);
void sgo_env_get_state(const sgo_env* e, double* q, double* qdot, double* q_target, double* tips,
                       double* goals);
void sgo_env_get_counters(const sgo_env* e, int32_t* step_count, int32_t* hold_count,
                          int64_t* episode_count, int32_t* waypoint_idx, int32_t* waypoint_len);
void sgo_env_get_rng(const sgo_env* e, uint64_t* state, uint64_t* inc);
/* waypoints of one row, returns count */
int sgo_env_get_waypoints(const sgo_env* e, int64_t row, double* out, int cap);
void sgo_env_workspace(const sgo_env* e, double* center3, double* radius);
int64_t sgo_env_goal_draws(const sgo_env* e); /* total sample_goal attempts so far */
/* overwrite state (for adversarial tests) */
void sgo_env_set_state(sgo_env* e, const double* q, const double* qdot, const double* q_target);

/* ---- render.cpp:34-67 ------------------------------------------------- */
/* Pinhole render of spheres (n x {cx, cy, cz, radius, albedo}) from the camera
 * pose (pos[3], quat wxyz); out: w*h row-major, top row first. */
void sgo_render(const double* cam_pos, const double* cam_quat, int w, int h, double fov, double near_,
                double far_, const double* spheres, int n_spheres, double* out);
/* ImageMatching views: target / current images n x w*h, scenes n x 15,
 * target cameras n x 7 (xyz, wxyz). */
void sgo_env_get_images(const sgo_env* e, double* target, double* current, double* scenes,
                        double* target_cameras);

/* ---- MultiToolReaching: envs.cpp:101-116 (bases, min separation), 118-223
 * (ctor), 304-360 (reset_row), 362-408 (observe), 437-617 (step), 540-587
 * (reward). One SimBatch per tool, stream id = tool * 2^32 + global row. */
#define SGO_MAX_TOOLS 8
typedef struct { double xyz[3]; double quat[4]; /* w x y z */ } sgo_pose;
/* default_tool_bases (envs.cpp:101-116) */
void sgo_default_tool_bases(int n_tools, double workspace_radius, sgo_pose* out);
/* multi_tool_min_separation (envs.cpp:90-99) over tips[n][3]; +inf below 2 */
double sgo_multi_tool_min_separation(const double* tips, int n);
typedef struct sgo_mt_env sgo_mt_env;
/* models: n_tools contiguous robots; bases: NULL -> defaults; dyn: NULL ->
 * per-robot defaults, else n_tools entries. */
sgo_mt_env* sgo_mt_env_create(const sgo_env_cfg* c, const sgo_robot* models, int n_tools,
                              const sgo_pose* bases, const sgo_dyn* dyn, int threads, char* err,
                              int errlen);
void sgo_mt_env_destroy(sgo_mt_env* e);
/* total action / observation dims; dofs[t] = DoF of tool t (n_tools entries) */
void sgo_mt_env_dims(const sgo_mt_env* e, int* action_dim, int* obs_dim, int* dofs);
int sgo_mt_env_reset(sgo_mt_env* e);
int sgo_mt_env_step(sgo_mt_env* e, const double* actions);
const char* sgo_mt_env_error(const sgo_mt_env* e);
void sgo_mt_env_get_obs(const sgo_mt_env* e, double* obs, double* terminal_obs);
void sgo_mt_env_get_result(const sgo_mt_env* e, double* rewards, uint8_t* terminated,
                           uint8_t* timed_out, double* task_error, int64_t* saturations);
/* q/qdot/q_target: n x action_dim (tool-major columns); tips/goals: n x 3T;
 * axes: n x 3T camera view axes (orientation * (0,0,-1)) */
void sgo_mt_env_get_state(const sgo_mt_env* e, double* q, double* qdot, double* q_target,
                          double* tips, double* goals, double* axes);
void sgo_mt_env_get_counters(const sgo_mt_env* e, int32_t* step_count, int32_t* hold_count,
                             int64_t* episode_count);
/* rng: n_tools x n */
void sgo_mt_env_get_rng(const sgo_mt_env* e, uint64_t* state, uint64_t* inc);
void sgo_mt_env_workspace(const sgo_mt_env* e, double* centers3t, double* radius, double* bases7t);

/* ---- bench.cpp:97-135 ------------------------------------------------- */
/* Runs the reference protocol: fresh env per run (seed+run), reset, warm-up
 * step, then steps until total_steps transitions; run_seconds[r] receives the
 * timed region. Returns 0 or an error code. */
int sgo_bench_sim(const sgo_env_cfg* c, const sgo_robot* m, int64_t total_steps, int runs,
                  int threads, double* run_seconds, int64_t* run_steps);

#ifdef __cplusplus
}
#endif
#endif
