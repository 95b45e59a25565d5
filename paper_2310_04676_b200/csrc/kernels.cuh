// sm_100a device code for the batched environment step.
//
// One fused kernel per step (or per K fused steps): PD dynamics + limit
// projection (proj/src/dynamics.cpp:99-204) -> FK tip (robot_model.cpp:371-402)
// -> reward / hold / waypoint advance / flags (envs.cpp:478-593) -> observation
// (envs.cpp:362-408) -> terminal copy + masked auto-reset + re-observe
// (envs.cpp:604-615, reset_row :304-360). One thread owns one env; the state
// lives in registers for the whole launch and in DoF-major SoA fp32 in HBM
// between launches. Observation rows (row-major, the contract layout) are
// staged through shared memory and written with coalesced 16-byte stores.
//
// Precision: state / FK / reward in fp32 (parity within a stated tolerance).
// Reset math (PCG32 draws, Box-Muller, goal rejection, spline arc-length
// table) in fp64 with explicit round-to-nearest intrinsics (no FMA
// contraction) so reset decisions and waypoint counts match the fp64 oracle.
#pragma once

#include <cstdint>

namespace sg {

constexpr int kMaxDof = 16;
constexpr int kGoalRejectionLimit = 1000;  // envs.cpp:29
constexpr int kSplineSubdiv = 1000;        // spline.cpp:24
constexpr uint64_t kPcgMult = 6364136223846793005ULL;

enum : int32_t { kRevolute = 0, kPrismatic = 1, kFixed = 2 };
enum : int32_t { kTaskTarget = 0, kTaskPath = 3 };
enum : int32_t { kModePosition = 0, kModeVelocity = 1, kModeTorque = 2 };
enum : int32_t {
  kErrNonFiniteAction = 1,
  kErrNonFiniteReward = 2,
  kErrGoalSampling = 4,
  kErrWaypointCap = 8,
  kErrFkLimit = 16,
};

// Per-DoF joint table, packed on the host from RobotModel. Fixed joints are
// folded into the next DoF joint's origin transform (and trailing ones into
// the tool tip), so entry d is exactly the d-th actuated joint and every array
// index in the kernel is a compile-time constant (no local-memory spills).
// axis_code 0..5 = +x,+y,+z,-x,-y,-z (every builtin joint), 6 = generic axis.
// flags: bit0..2 origin translation x/y/z != 0, bit3 origin rotation is not
// the identity.
struct JointEnc {
  int32_t kind;
  int32_t axis_code;
  int32_t flags;
  int32_t pad;
  float o[3];
  float axis[3];
  float R[9];
};

struct RobotTable {
  int32_t dof;
  int32_t jaw;        // DoF index of the jaw, -1 if none
  int32_t tip_flags;  // bit0..2 nonzero tip xyz components
  int32_t pad;
  JointEnc j[kMaxDof];
  float tip[3];
  float lo[kMaxDof], hi[kMaxDof], vel[kMaxDof], eff[kMaxDof];
  float kp[kMaxDof], kd[kMaxDof], damping[kMaxDof], dt_over_inertia[kMaxDof];
  double lo_d[kMaxDof], hi_d[kMaxDof];
};

struct TaskParams {
  int32_t task;
  int32_t episode_len;
  int32_t success_hold;
  int32_t substeps;
  int32_t control_mode;
  int32_t wp_cap;
  int64_t n;
  float rho;            // reward_scale
  float neg_alpha;      // -path_penalty
  float success_radius;
  float dt_sub;
  double goal_sigma;
  double radius;        // workspace radius
  double center[3];
  double spacing;
};

struct EnvPtrs {
  float* q;       // [dof][n]
  float* qd;
  float* qt;
  float* goals;   // [3][n]
  float* tips;    // [3][n]
  int32_t* step_count;
  int32_t* hold_count;
  int64_t* episode_count;
  int32_t* wp_idx;
  int32_t* wp_len;
  float* wps;     // [n][wp_cap][3]
  uint64_t* rng_state;
  uint64_t* rng_inc;
  // StepResult
  float* obs;     // [n][O]
  float* tobs;
  float* rewards;
  float* task_error;
  uint8_t* terminated;
  uint8_t* timed_out;
  unsigned long long* sat_total;
  int32_t* err;
  // bench action stream (per-env PCG state positioned at the env's next draw)
  uint64_t* act_state;
  float* act_buf;  // [n][A]
};

struct BenchStream {
  uint64_t inc;
  uint64_t jump_mult;  // advance by (global_n - 1) * A draws after an env's A draws
  uint64_t jump_add;
};

struct StepParams {
  RobotTable robot;
  TaskParams task;
  EnvPtrs p;
  BenchStream bench;
  const float* actions;  // [n][A] row-major (non-bench path)
  int32_t actions_aligned;
};

// ---------------------------------------------------------------------------
// PCG32 (rng.hpp:25-83), fp64 draws without FMA contraction.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pcg_next(uint64_t& s, uint64_t inc) {
  const uint64_t old = s;
  s = old * kPcgMult + inc;
  const uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
  const uint32_t rot = static_cast<uint32_t>(old >> 59u);
  return (xs >> rot) | (xs << ((32u - rot) & 31u));
}

__device__ __forceinline__ double pcg_uniform(uint64_t& s, uint64_t inc, double lo, double hi) {
  const double u = static_cast<double>(pcg_next(s, inc)) * 0x1.0p-32;
  return __dadd_rn(lo, __dmul_rn(__dadd_rn(hi, -lo), u));
}

__device__ __forceinline__ double pcg_normal(uint64_t& s, uint64_t inc) {
  const double u1 = __dmul_rn(__dadd_rn(static_cast<double>(pcg_next(s, inc)), 0.5), 0x1.0p-32);
  const double u2 = static_cast<double>(pcg_next(s, inc)) * 0x1.0p-32;
  return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(6.283185307179586477, u2)));
}

__device__ __forceinline__ double norm3_rn(double x, double y, double z) {
  return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

// ---------------------------------------------------------------------------
// Forward kinematics in fp32 (fk_walk, robot_model.cpp:371-395), rotation as a
// 3x3 matrix; warp-uniform branches on the joint codes (every thread of the
// grid walks the same chain).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void rot_cols(float (&m)[9], int ca, int cb, float c, float s) {
  // columns (ca, cb) <- (c*col_a + s*col_b, c*col_b - s*col_a); ca/cb constant after inlining
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const float a = m[r * 3 + ca], b = m[r * 3 + cb];
    m[r * 3 + ca] = c * a + s * b;
    m[r * 3 + cb] = c * b - s * a;
  }
}

template <int DMAX>
__device__ __forceinline__ void fk_tip(const RobotTable& R, const float (&q)[DMAX], float (&tip)[3]) {
  float m[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};  // row-major
  float p0 = 0.f, p1 = 0.f, p2 = 0.f;
#pragma unroll
  for (int d = 0; d < DMAX; ++d) {
    if (d >= R.dof) break;
    const JointEnc& J = R.j[d];
    const int fl = J.flags;
    // p += R * origin_translation
    if (fl & 1) { p0 += m[0] * J.o[0]; p1 += m[3] * J.o[0]; p2 += m[6] * J.o[0]; }
    if (fl & 2) { p0 += m[1] * J.o[1]; p1 += m[4] * J.o[1]; p2 += m[7] * J.o[1]; }
    if (fl & 4) { p0 += m[2] * J.o[2]; p1 += m[5] * J.o[2]; p2 += m[8] * J.o[2]; }
    if (fl & 8) {  // R = R * R_origin
      float t[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          t[r * 3 + c] = m[r * 3 + 0] * J.R[0 * 3 + c] + m[r * 3 + 1] * J.R[1 * 3 + c] + m[r * 3 + 2] * J.R[2 * 3 + c];
#pragma unroll
      for (int k = 0; k < 9; ++k) m[k] = t[k];
    }
    const float qv = q[d];
    const int code = J.axis_code;
    if (J.kind == kRevolute) {
      // 2*pi range reduction then the SFU sin/cos (abs err ~2^-21.4 on
      // [-pi, pi]): FK never feeds back into the decoupled joint dynamics, so
      // this only perturbs the observed tip by ~1e-7 m.
      const float red = fmaf(-6.28318530717958647692f, rintf(qv * 0.15915494309189533577f), qv);
      float s, c;
      __sincosf(red, &s, &c);
      if (code == 2) rot_cols(m, 0, 1, c, s);        // +z
      else if (code == 5) rot_cols(m, 0, 1, c, -s);  // -z
      else if (code == 0) rot_cols(m, 1, 2, c, s);   // +x
      else if (code == 3) rot_cols(m, 1, 2, c, -s);  // -x
      else if (code == 1) rot_cols(m, 2, 0, c, s);   // +y: col2' = c*col2 + s*col0, col0' = c*col0 - s*col2
      else if (code == 4) rot_cols(m, 2, 0, c, -s);  // -y
      else {  // generic axis: Rodrigues  Rr = I + s K + (1 - c) K^2
        const float kx = J.axis[0], ky = J.axis[1], kz = J.axis[2], omc = 1.f - c;
        const float rr[9] = {1.f + omc * (-ky * ky - kz * kz), -s * kz + omc * kx * ky, s * ky + omc * kx * kz,
                             s * kz + omc * kx * ky, 1.f + omc * (-kx * kx - kz * kz), -s * kx + omc * ky * kz,
                             -s * ky + omc * kx * kz, s * kx + omc * ky * kz, 1.f + omc * (-kx * kx - ky * ky)};
        float t[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int cc = 0; cc < 3; ++cc)
            t[r * 3 + cc] = m[r * 3 + 0] * rr[0 * 3 + cc] + m[r * 3 + 1] * rr[1 * 3 + cc] + m[r * 3 + 2] * rr[2 * 3 + cc];
#pragma unroll
        for (int k = 0; k < 9; ++k) m[k] = t[k];
      }
    } else {  // prismatic: p += R * (axis * q)
      if (code == 0 || code == 3) {
        const float v = code == 3 ? -qv : qv;
        p0 += m[0] * v; p1 += m[3] * v; p2 += m[6] * v;
      } else if (code == 1 || code == 4) {
        const float v = code == 4 ? -qv : qv;
        p0 += m[1] * v; p1 += m[4] * v; p2 += m[7] * v;
      } else if (code == 2 || code == 5) {
        const float v = code == 5 ? -qv : qv;
        p0 += m[2] * v; p1 += m[5] * v; p2 += m[8] * v;
      } else {
        const float a0 = J.axis[0] * qv, a1 = J.axis[1] * qv, a2 = J.axis[2] * qv;
        p0 += m[0] * a0 + m[1] * a1 + m[2] * a2;
        p1 += m[3] * a0 + m[4] * a1 + m[5] * a2;
        p2 += m[6] * a0 + m[7] * a1 + m[8] * a2;
      }
    }
  }
  const int tf = R.tip_flags;
  if (tf & 1) { p0 += m[0] * R.tip[0]; p1 += m[3] * R.tip[0]; p2 += m[6] * R.tip[0]; }
  if (tf & 2) { p0 += m[1] * R.tip[1]; p1 += m[4] * R.tip[1]; p2 += m[7] * R.tip[1]; }
  if (tf & 4) { p0 += m[2] * R.tip[2]; p1 += m[5] * R.tip[2]; p2 += m[8] * R.tip[2]; }
  tip[0] = p0;
  tip[1] = p1;
  tip[2] = p2;
}

// ---------------------------------------------------------------------------
// Spline (spline.hpp:24-36, spline.cpp:40-72) in fp64, streaming: the
// 1001-point cumulative chord table is regenerated on the fly in the same
// summation order, so no per-thread table is needed.
// ---------------------------------------------------------------------------
struct Spline {
  double c[12];  // a[3], b[3], c[3], d[3]; t0 = 0, t1 = 1
};

__device__ __forceinline__ void spline_eval(const Spline& s, double t, double (&o)[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double v = __dadd_rn(__dmul_rn(s.c[k], t), s.c[3 + k]);
    v = __dadd_rn(__dmul_rn(v, t), s.c[6 + k]);
    o[k] = __dadd_rn(__dmul_rn(v, t), s.c[9 + k]);
  }
}

__device__ __forceinline__ double dist3_rn(const double (&a)[3], const double (&b)[3]) {
  return norm3_rn(__dadd_rn(a[0], -b[0]), __dadd_rn(a[1], -b[1]), __dadd_rn(a[2], -b[2]));
}

// Writes waypoints (fp32) for one row; returns the count (<= cap), or -1 if
// the table capacity is exceeded.
__device__ __noinline__ int spline_waypoints_stream(const Spline& s, double spacing, float* out, int cap) {
  const double span = 1.0;  // t1 - t0 (sample_path, envs.cpp:248-249)
  double prev[3], p[3];
  spline_eval(s, 0.0, prev);
  double total = 0.0;
  for (int k = 1; k <= kSplineSubdiv; ++k) {
    spline_eval(s, __dmul_rn(span, (double)k) / (double)kSplineSubdiv, p);
    total = __dadd_rn(total, dist3_rn(p, prev));
    prev[0] = p[0]; prev[1] = p[1]; prev[2] = p[2];
  }
  int count = 0;
  double p0[3];
  spline_eval(s, 0.0, p0);
  out[0] = (float)p0[0]; out[1] = (float)p0[1]; out[2] = (float)p0[2];
  count = 1;
  if (total <= 1e-12) return count;
  int seg = 0;
  double cum_seg = 0.0, p_seg[3] = {p0[0], p0[1], p0[2]}, p_next[3];
  spline_eval(s, __dmul_rn(span, 1.0) / (double)kSplineSubdiv, p_next);
  double cum_next = __dadd_rn(cum_seg, dist3_rn(p_next, p_seg));
  const double limit = __dadd_rn(total, -1e-12);
  for (double sv = spacing; sv < limit; sv = __dadd_rn(sv, spacing)) {
    while (seg + 1 < kSplineSubdiv && cum_next < sv) {
      ++seg;
      cum_seg = cum_next;
      p_seg[0] = p_next[0]; p_seg[1] = p_next[1]; p_seg[2] = p_next[2];
      spline_eval(s, __dmul_rn(span, (double)(seg + 1)) / (double)kSplineSubdiv, p_next);
      cum_next = __dadd_rn(cum_seg, dist3_rn(p_next, p_seg));
    }
    const double seg_len = __dadd_rn(cum_next, -cum_seg);
    const double frac = seg_len > 0.0 ? __dadd_rn(sv, -cum_seg) / seg_len : 0.0;
    const double t = __dmul_rn(span, __dadd_rn((double)seg, frac)) / (double)kSplineSubdiv;
    double w[3];
    spline_eval(s, t, w);
    if (count >= cap) return -1;
    out[3 * count + 0] = (float)w[0];
    out[3 * count + 1] = (float)w[1];
    out[3 * count + 2] = (float)w[2];
    ++count;
  }
  double pe[3];
  spline_eval(s, __dmul_rn(span, (double)kSplineSubdiv) / (double)kSplineSubdiv, pe);
  if (count >= cap) return -1;
  out[3 * count + 0] = (float)pe[0];
  out[3 * count + 1] = (float)pe[1];
  out[3 * count + 2] = (float)pe[2];
  return count + 1;
}

// sample_goal (envs.cpp:230-239). The reference builds the offset with
// Eigen::Vector3d(n(), n(), n()); g++ evaluates constructor arguments
// right-to-left, so the first draw is z (oracle/probe_eval_order.cpp).
__device__ __forceinline__ bool sample_goal(uint64_t& s, uint64_t inc, const TaskParams& T, double (&g)[3]) {
  for (int attempt = 0; attempt < kGoalRejectionLimit; ++attempt) {
    const double nz = __dmul_rn(T.goal_sigma, pcg_normal(s, inc));
    const double ny = __dmul_rn(T.goal_sigma, pcg_normal(s, inc));
    const double nx = __dmul_rn(T.goal_sigma, pcg_normal(s, inc));
    g[0] = __dadd_rn(T.center[0], nx);
    g[1] = __dadd_rn(T.center[1], ny);
    g[2] = __dadd_rn(T.center[2], nz);
    if (norm3_rn(__dadd_rn(g[0], -T.center[0]), __dadd_rn(g[1], -T.center[1]), __dadd_rn(g[2], -T.center[2])) <=
        T.radius)
      return true;
  }
  return false;
}

// reset_row (envs.cpp:304-360) for one env. Out of line (rare path) and
// communicating through HBM only, so the caller's state arrays stay in
// registers: the caller reloads q/qdot/q_target/goal/tip/waypoint idx+len
// after the call. Returns an error bit (0 on success).
template <int DMAX>
__device__ __noinline__ int reset_env(const StepParams& P, int64_t i) {
  const RobotTable& R = P.robot;
  const TaskParams& T = P.task;
  const int64_t n = T.n;
  uint64_t s = P.p.rng_state[i];
  const uint64_t inc = P.p.rng_inc[i];
  int err = 0;
  float q[DMAX], qd[DMAX], qt[DMAX], goal[3], tip[3];
  int32_t wp_idx = 0, wp_len = 0;
#pragma unroll
  for (int d = 0; d < DMAX; ++d) {
    if (d < R.dof) {
      const double quarter = __dmul_rn(0.25, __dadd_rn(R.hi_d[d], -R.lo_d[d]));
      q[d] = (float)pcg_uniform(s, inc, __dadd_rn(R.lo_d[d], quarter), __dadd_rn(R.hi_d[d], -quarter));
      qd[d] = 0.f;
      qt[d] = q[d];
    }
  }
  fk_tip<DMAX>(R, q, tip);
  if (T.task == kTaskPath) {
    // sample_path (envs.cpp:241-267)
    Spline sp;
#pragma unroll
    for (int k = 0; k < 3; ++k) sp.c[k] = pcg_uniform(s, inc, -0.5, 0.5);
#pragma unroll
    for (int k = 0; k < 3; ++k) sp.c[3 + k] = pcg_uniform(s, inc, -0.5, 0.5);
#pragma unroll
    for (int k = 0; k < 3; ++k) sp.c[6 + k] = pcg_uniform(s, inc, -0.3, 0.3);
    double d[3];
    if (!sample_goal(s, inc, T, d)) err |= kErrGoalSampling;
    sp.c[9] = d[0]; sp.c[10] = d[1]; sp.c[11] = d[2];
    double max_off = 0.0;
    for (int k = 0; k <= 100; ++k) {
      double pt[3];
      spline_eval(sp, __dmul_rn(0.01, (double)k), pt);
      const double off = dist3_rn(pt, d);
      max_off = max_off > off ? max_off : off;
    }
    const double ctr[3] = {T.center[0], T.center[1], T.center[2]};
    const double allowed = __dadd_rn(T.radius, -dist3_rn(d, ctr));
    if (max_off > 0.0 && max_off > allowed) {
      const double scale = __dmul_rn(0.95, allowed > 0.0 ? allowed : 0.0) / max_off;
#pragma unroll
      for (int k = 0; k < 9; ++k) sp.c[k] = __dmul_rn(sp.c[k], scale);
    }
    float* table = P.p.wps + i * (int64_t)T.wp_cap * 3;
    int cnt = spline_waypoints_stream(sp, T.spacing, table, T.wp_cap);
    if (cnt < 0) {
      err |= kErrWaypointCap;
      cnt = T.wp_cap;
    }
    wp_len = cnt;
    wp_idx = 0;
    goal[0] = table[0];
    goal[1] = table[1];
    goal[2] = table[2];
  } else {
    double g[3];
    if (!sample_goal(s, inc, T, g)) err |= kErrGoalSampling;
    goal[0] = (float)g[0];
    goal[1] = (float)g[1];
    goal[2] = (float)g[2];
  }
  P.p.rng_state[i] = s;
  P.p.step_count[i] = 0;
  P.p.hold_count[i] = 0;
  P.p.episode_count[i] += 1;
#pragma unroll
  for (int d = 0; d < DMAX; ++d) {
    if (d < R.dof) {
      P.p.q[d * n + i] = q[d];
      P.p.qd[d * n + i] = qd[d];
      P.p.qt[d * n + i] = qt[d];
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    P.p.goals[k * n + i] = goal[k];
    P.p.tips[k * n + i] = tip[k];
  }
  if (T.task == kTaskPath) {
    P.p.wp_idx[i] = wp_idx;
    P.p.wp_len[i] = wp_len;
  }
  return err;
}

// Reload one env's state from HBM into registers (after reset_env).
template <int DMAX>
__device__ __forceinline__ void load_env(const StepParams& P, int64_t i, float (&q)[DMAX], float (&qd)[DMAX],
                                         float (&qt)[DMAX], float (&goal)[3], float (&tip)[3], int32_t& wi,
                                         int32_t& wl) {
  const int64_t n = P.task.n;
#pragma unroll
  for (int d = 0; d < DMAX; ++d) {
    if (d < P.robot.dof) {
      q[d] = P.p.q[d * n + i];
      qd[d] = P.p.qd[d * n + i];
      qt[d] = P.p.qt[d * n + i];
    } else {
      q[d] = qd[d] = qt[d] = 0.f;
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    goal[k] = P.p.goals[k * n + i];
    tip[k] = P.p.tips[k * n + i];
  }
  if (P.task.task == kTaskPath) {
    wi = P.p.wp_idx[i];
    wl = P.p.wp_len[i];
  }
}

// ---------------------------------------------------------------------------
// Block-cooperative coalesced copies between shared staging and global rows.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void block_store(float* __restrict__ g, const float* __restrict__ s, int count) {
  if ((reinterpret_cast<uintptr_t>(g) & 15u) == 0) {
    const int n4 = count >> 2;
    float4* g4 = reinterpret_cast<float4*>(g);
    const float4* s4 = reinterpret_cast<const float4*>(s);
    for (int k = threadIdx.x; k < n4; k += blockDim.x) g4[k] = s4[k];
    for (int k = (n4 << 2) + threadIdx.x; k < count; k += blockDim.x) g[k] = s[k];
  } else {
    for (int k = threadIdx.x; k < count; k += blockDim.x) g[k] = s[k];
  }
}

__device__ __forceinline__ void block_load(float* __restrict__ s, const float* __restrict__ g, int count,
                                           bool aligned) {
  if (aligned) {
    const int n4 = count >> 2;
    const float4* g4 = reinterpret_cast<const float4*>(g);
    float4* s4 = reinterpret_cast<float4*>(s);
    for (int k = threadIdx.x; k < n4; k += blockDim.x) s4[k] = __ldg(g4 + k);
    for (int k = (n4 << 2) + threadIdx.x; k < count; k += blockDim.x) s[k] = __ldg(g + k);
  } else {
    for (int k = threadIdx.x; k < count; k += blockDim.x) s[k] = __ldg(g + k);
  }
}

// ---------------------------------------------------------------------------
// The fused step kernel. GEN_ACTIONS: actions are the bench stream
// (bench.cpp:31-35) generated in-kernel and written to p.act_buf; otherwise
// they are read from P.actions.
// ---------------------------------------------------------------------------
template <int DMAX, bool GEN_ACTIONS>
__global__ void __launch_bounds__(128) env_step_kernel(const __grid_constant__ StepParams P, int k_steps) {
  extern __shared__ __align__(16) float smem[];
  const RobotTable& R = P.robot;
  const TaskParams& T = P.task;
  const int A = R.dof;
  const int O = 3 * A + 6;
  const int64_t n = T.n;
  const int64_t row0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t i = row0 + threadIdx.x;
  const bool active = i < n;
  const int rows = (int)min((int64_t)blockDim.x, n - row0);
  float* s_obs = smem;                             // blockDim * O
  float* s_act = smem + (size_t)blockDim.x * O;    // blockDim * A (16B aligned: blockDim*O*4 % 16 == 0)

  float q[DMAX], qd[DMAX], qt[DMAX], goal[3], tip[3];
  int32_t sc = 0, hc = 0, wi = 0, wl = 0;
  uint64_t act_s = 0;
  if (active) {
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
      if (d < A) {
        q[d] = P.p.q[d * n + i];
        qd[d] = P.p.qd[d * n + i];
        qt[d] = P.p.qt[d * n + i];
      } else {
        q[d] = qd[d] = qt[d] = 0.f;
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) goal[k] = P.p.goals[k * n + i];
    sc = P.p.step_count[i];
    hc = P.p.hold_count[i];
    if (T.task == kTaskPath) {
      wi = P.p.wp_idx[i];
      wl = P.p.wp_len[i];
    }
    if (GEN_ACTIONS) act_s = P.p.act_state[i];
  } else {
#pragma unroll
    for (int d = 0; d < DMAX; ++d) q[d] = qd[d] = qt[d] = 0.f;
    goal[0] = goal[1] = goal[2] = 0.f;
  }
  tip[0] = tip[1] = tip[2] = 0.f;

  for (int step = 0; step < k_steps; ++step) {
    // ---- actions ---------------------------------------------------------
    float a[DMAX];
    if (GEN_ACTIONS) {
#pragma unroll
      for (int d = 0; d < DMAX; ++d) {
        a[d] = 0.f;
        if (d < A && active) {
          const uint32_t u = pcg_next(act_s, P.bench.inc);
          // uniform(-1, 1) = -1 + 2 * (u * 2^-32), exact in fp64, one rounding to fp32
          a[d] = (float)(-1.0 + 2.0 * ((double)u * 0x1.0p-32));
          s_act[threadIdx.x * A + d] = a[d];
        }
      }
      if (active) act_s = act_s * P.bench.jump_mult + P.bench.jump_add;
      __syncthreads();
      block_store(P.p.act_buf + row0 * A, s_act, rows * A);
    } else {
      __syncthreads();
      block_load(s_act, P.actions + row0 * A, rows * A, P.actions_aligned != 0);
      __syncthreads();
#pragma unroll
      for (int d = 0; d < DMAX; ++d) a[d] = (d < A && active) ? s_act[threadIdx.x * A + d] : 0.f;
    }

    // ---- dynamics (dynamics.cpp:133-185) ----------------------------------
    int sat = 0, bad = 0;
    if (active) {
#pragma unroll
      for (int d = 0; d < DMAX; ++d) {
        if (d >= A) continue;
        float ad = a[d];
        if (!isfinite(ad)) {
          bad = 1;
          continue;
        }
        if (ad < -1.f || ad > 1.f) {
          ad = ad < -1.f ? -1.f : 1.f;
          ++sat;
        }
        const float lo = R.lo[d], hi = R.hi[d], vl = R.vel[d], ef = R.eff[d];
        float v_target = 0.f, tau_cmd = 0.f;
        const auto rescale = [](float x, float l, float h) {
          if (x >= 1.f) return h;
          if (x <= -1.f) return l;
          return l + 0.5f * (x + 1.f) * (h - l);
        };
        if (T.control_mode == kModePosition) {
          qt[d] = (d == R.jaw) ? (ad > 0.f ? hi : lo) : rescale(ad, lo, hi);
        } else if (T.control_mode == kModeVelocity) {
          v_target = rescale(ad, -vl, vl);
        } else {
          tau_cmd = rescale(ad, -ef, ef);
        }
        const float kp = R.kp[d], kd = R.kd[d], damp = R.damping[d], gain = R.dt_over_inertia[d];
        const float dt = T.dt_sub;
        float qq = q[d], vv = qd[d];
        for (int s = 0; s < T.substeps; ++s) {
          float tau;
          if (T.control_mode == kModePosition) tau = kp * (qt[d] - qq) - kd * vv;
          else if (T.control_mode == kModeVelocity) tau = kd * (v_target - vv);
          else tau = tau_cmd;
          tau = fminf(fmaxf(tau, -ef), ef);
          vv += (tau - damp * vv) * gain;
          vv = fminf(fmaxf(vv, -vl), vl);
          qq += vv * dt;
          if (qq < lo) {
            qq = lo;
            vv = 0.f;
          } else if (qq > hi) {
            qq = hi;
            vv = 0.f;
          }
        }
        q[d] = qq;
        qd[d] = vv;
      }
    }
    // saturation count: warp-aggregated, one atomic per warp with work
    {
      const unsigned wsat = __reduce_add_sync(0xffffffffu, (unsigned)sat);
      if (wsat && (threadIdx.x & 31) == 0) atomicAdd(P.p.sat_total, (unsigned long long)wsat);
      if (__any_sync(0xffffffffu, bad) && bad) atomicOr(P.p.err, kErrNonFiniteAction);
    }

    // ---- FK + reward + flags (envs.cpp:456-463, 478-593) ------------------
    bool ended = false;
    if (active) {
      fk_tip<DMAX>(R, q, tip);
      sc += 1;
      float reward, dist;
      bool goal_met;
      {
        const float dx = tip[0] - goal[0], dy = tip[1] - goal[1], dz = tip[2] - goal[2];
        dist = sqrtf(dx * dx + dy * dy + dz * dz);
      }
      if (T.task == kTaskPath) {
        reward = T.neg_alpha * dist;
        float dcur = dist;
        const float* table = P.p.wps + i * (int64_t)T.wp_cap * 3;
        while (wi + 1 < wl && dcur < T.success_radius) {
          ++wi;
          goal[0] = table[3 * wi + 0];
          goal[1] = table[3 * wi + 1];
          goal[2] = table[3 * wi + 2];
          const float dx = tip[0] - goal[0], dy = tip[1] - goal[1], dz = tip[2] - goal[2];
          dcur = sqrtf(dx * dx + dy * dy + dz * dz);
        }
        goal_met = (wi + 1 == wl) && dcur < T.success_radius;
      } else {
        reward = T.rho * dist;
        hc = dist < T.success_radius ? hc + 1 : 0;
        goal_met = hc >= T.success_hold;
      }
      if (!isfinite(reward)) atomicOr(P.p.err, kErrNonFiniteReward);
      const bool timed_out = sc >= T.episode_len;
      P.p.rewards[i] = reward;
      P.p.task_error[i] = dist;
      P.p.terminated[i] = goal_met ? 1 : 0;
      P.p.timed_out[i] = timed_out ? 1 : 0;
      ended = goal_met || timed_out;
    }

    // ---- observation (envs.cpp:362-408) -----------------------------------
    const auto stage_obs = [&]() {
      if (!active) return;
      float* o = s_obs + threadIdx.x * O;
      int off = 0;
#pragma unroll
      for (int d = 0; d < DMAX; ++d)
        if (d < A) o[off + d] = q[d];
      off += A;
#pragma unroll
      for (int d = 0; d < DMAX; ++d)
        if (d < A) o[off + d] = qd[d];
      off += A;
      o[off + 0] = tip[0];
      o[off + 1] = tip[1];
      o[off + 2] = tip[2];
      off += 3;
#pragma unroll
      for (int d = 0; d < DMAX; ++d)
        if (d < A) o[off + d] = qt[d];
      off += A;
      o[off + 0] = goal[0];
      o[off + 1] = goal[1];
      o[off + 2] = goal[2];
    };
    stage_obs();
    // ---- ended rows: terminal obs, masked reset, re-observe ----------------
    const int any_ended = __syncthreads_or(ended);
    if (any_ended) {
      // pre-reset observation rows of ended envs -> terminal_observations
      // (envs.cpp:606-611); each warp copies its own ended rows, one row per
      // pass with the lanes spread over the row (coalesced).
      const unsigned m = __ballot_sync(0xffffffffu, ended);
      const int lane = threadIdx.x & 31;
      const int wbase = threadIdx.x & ~31;
      for (unsigned mm = m; mm; mm &= mm - 1) {
        const int src = wbase + __ffs(mm) - 1;
        const int64_t row = row0 + src;
        for (int k = lane; k < O; k += 32) P.p.tobs[row * O + k] = s_obs[src * O + k];
      }
      __syncwarp();
      if (ended) {
        const int e = reset_env<DMAX>(P, i);
        if (e) atomicOr(P.p.err, e);
        load_env<DMAX>(P, i, q, qd, qt, goal, tip, wi, wl);
        sc = 0;
        hc = 0;
        stage_obs();
      }
    }
    __syncthreads();
    block_store(P.p.obs + row0 * O, s_obs, rows * O);
  }

  if (active) {
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
      if (d < A) {
        P.p.q[d * n + i] = q[d];
        P.p.qd[d * n + i] = qd[d];
        P.p.qt[d * n + i] = qt[d];
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      P.p.goals[k * n + i] = goal[k];
      P.p.tips[k * n + i] = tip[k];
    }
    P.p.step_count[i] = sc;
    P.p.hold_count[i] = hc;
    if (T.task == kTaskPath) {
      P.p.wp_idx[i] = wi;
      P.p.wp_len[i] = wl;
    }
    if (GEN_ACTIONS) P.p.act_state[i] = act_s;
  }
}

// reset() (envs.cpp:425-435): every row through reset_row, episode_count := 0,
// observe, clear flags and rewards.
template <int DMAX>
__global__ void __launch_bounds__(128) env_reset_kernel(const __grid_constant__ StepParams P) {
  extern __shared__ __align__(16) float smem[];
  const RobotTable& R = P.robot;
  const TaskParams& T = P.task;
  const int A = R.dof;
  const int O = 3 * A + 6;
  const int64_t n = T.n;
  const int64_t row0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t i = row0 + threadIdx.x;
  const int rows = (int)min((int64_t)blockDim.x, n - row0);
  if (i < n) {
    float q[DMAX], qd[DMAX], qt[DMAX], goal[3], tip[3];
    int32_t wi = 0, wl = 0;
    const int e = reset_env<DMAX>(P, i);
    if (e) atomicOr(P.p.err, e);
    load_env<DMAX>(P, i, q, qd, qt, goal, tip, wi, wl);
    P.p.episode_count[i] = 0;
    P.p.terminated[i] = 0;
    P.p.timed_out[i] = 0;
    P.p.rewards[i] = 0.f;
    float* o = smem + threadIdx.x * O;
    int off = 0;
    for (int d = 0; d < A; ++d) o[off++] = q[d];
    for (int d = 0; d < A; ++d) o[off++] = qd[d];
    for (int k = 0; k < 3; ++k) o[off++] = tip[k];
    for (int d = 0; d < A; ++d) o[off++] = qt[d];
    for (int k = 0; k < 3; ++k) o[off++] = goal[k];
  }
  __syncthreads();
  block_store(P.p.obs + row0 * O, smem, rows * O);
}

// Positions the per-env bench action stream at draw (first_step*G + g)*A,
// g = row_offset + i (jump-ahead, O(log k) table of PCG32 powers).
struct JumpTable {
  uint64_t mult[64];
  uint64_t add[64];
};

__global__ void bench_seed_kernel(uint64_t* act_state, int64_t n, uint64_t base_state, uint64_t first_draw,
                                  int64_t row_offset, int32_t A, const __grid_constant__ JumpTable J) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t k = first_draw + (uint64_t)(row_offset + i) * (uint64_t)A;
  uint64_t s = base_state;
  for (int b = 0; k; ++b, k >>= 1)
    if (k & 1) s = s * J.mult[b] + J.add[b];
  act_state[i] = s;
}

// Batched FK (forward_kinematics_batch, robot_model.cpp:404-443) with check_q.
template <int DMAX>
__global__ void fk_batch_kernel(const __grid_constant__ RobotTable R, const float* __restrict__ q_in, int64_t n,
                                float* __restrict__ pos, int32_t* err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float q[DMAX], tip[3];
  bool bad = false;
#pragma unroll
  for (int d = 0; d < DMAX; ++d) {
    q[d] = d < R.dof ? q_in[i * R.dof + d] : 0.f;
    if (d < R.dof) {
      const double v = q[d];
      if (v < R.lo_d[d] - 1e-9 || v > R.hi_d[d] + 1e-9) bad = true;  // check_q, kEps 1e-9
    }
  }
  if (bad) atomicOr(err, kErrFkLimit);
  fk_tip<DMAX>(R, q, tip);
  pos[i * 3 + 0] = tip[0];
  pos[i * 3 + 1] = tip[1];
  pos[i * 3 + 2] = tip[2];
}

}  // namespace sg
