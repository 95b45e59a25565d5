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

#if defined(SG_TIME_PROBE) || defined(SG_PHASE_PROBE)
#include <cstdio>
#endif
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <utility>

namespace sg {

constexpr int kMaxDof = 16;
constexpr int kGoalRejectionLimit = 1000;  // envs.cpp:29
constexpr int kSplineSubdiv = 1000;        // spline.cpp:24
constexpr uint64_t kPcgMult = 6364136223846793005ULL;

enum : int32_t { kRevolute = 0, kPrismatic = 1, kFixed = 2 };
enum : int32_t { kTaskTarget = 0, kTaskTrack = 1, kTaskPath = 3 };
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
  // ActiveTracking (envs.cpp:493-512)
  float goal_offset_clip;
  float track_noise_std;
  float track_vel_clamp;
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
  float* goal_spawn;  // [3][n] ActiveTracking: goal at reset
  float* goal_vel;    // [3][n] ActiveTracking: goal velocity
  // PathFollowing reset records (nullable): the NEXT reset_row of env i is a
  // function of its PCG32 state only, which changes only at resets, so it is
  // computed ahead by path_record_kernel (full warps, many warps per SM) and
  // a reset just installs it. rec_valid[i] == 1 when the record matches the
  // current state.
  uint8_t* rec_valid;
  float* rec_q;      // [dof][n]
  int32_t* rec_len;  // waypoint count
  int32_t* rec_err;  // error bits of the sampling
  uint64_t* rec_rng; // PCG32 state after the reset's draws
  float* rec_wps;    // [n][wp_cap][3]
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
  unsigned long long* ended_total;  // running count of ended rows (host polls it)
  int32_t* err;
  // bench action stream (per-env PCG state positioned at the env's next draw)
  uint64_t* act_state;
  float* act_buf;  // [n][A]
  // Host mirrors of the StepResult (caller-step path only, nullable): device
  // aliases of the caller's pinned host buffers. The kernel writes each
  // field there too, so the result crosses PCIe as the kernel's own posted
  // stores (sg_env_step_host) instead of separate copies.
  float* h_obs;
  float* h_tobs;  // ended rows only
  // Host-step status (nullable): the launch's last CTA copies {sat_total,
  // ended rows of this step, error word} into mapped pinned memory, so the
  // host reads them after its one synchronisation without a copy.
  unsigned long long* h_status;
  unsigned long long h_seq;  // host step number: written to h_status[3] last, after a system fence
  unsigned long long* ended_clear;  // zeroed at launch start: the next host step's ended slot
  unsigned long long* sat_step;     // host step: saturations of THIS step (nullable)
  unsigned long long* sat_clear;    // zeroed at launch start: the next host step's saturation slot
  unsigned int* ticket;             // CTA completion counter (last CTA publishes, then re-arms it)
  // Host step read window (nullable): teams that finished staging their
  // action rows; team b stages once read_gate >= b - read_window + 1, so at
  // most ~read_window teams read over PCIe at once and later teams' reads
  // overlap earlier teams' result writes (the last CTA re-arms it)
  unsigned int* read_gate;
  int read_window;
  // Host step with the observation rows copied by the copy engine (nullable):
  // team b counts into chunk_count[b / chunk_teams]; the chunk's last team
  // publishes chunk_flag[chunk] = h_seq, on which the copy stream waits
  // (cuStreamWaitValue32) before copying the chunk's rows to the host
  unsigned int* chunk_count;
  unsigned int* chunk_flag;
  int chunk_teams;
  float* h_rewards;
  float* h_task_error;
  uint8_t* h_terminated;
  uint8_t* h_timed_out;
};

constexpr int kMaxTeamWarps = 8;

struct BenchStream {
  uint64_t inc;
  // A team warp keeps the stream state s at its block's first draw of the
  // step; draw j of the block is output(s advanced j times) = output(s *
  // pow_mult[j] + pow_add[j]) (independent, no serial LCG chain), and the
  // next step's first draw is s advanced by global_n * A (jump_*).
  uint64_t jump_mult;
  uint64_t jump_add;
  uint64_t pow_mult[kMaxDof];
  uint64_t pow_add[kMaxDof];
};

struct StepParams {
  RobotTable robot;
  TaskParams task;
  EnvPtrs p;
  BenchStream bench;
  const float* actions;  // [n][A] row-major (non-bench path; device or mapped host memory)
  int32_t actions_aligned;  // 16-byte aligned base: the team stages its rows with float4 loads
};

// ---------------------------------------------------------------------------
// PCG32 (rng.hpp:25-83), fp64 draws without FMA contraction.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pcg_output(uint64_t old) {  // XSH-RR of the pre-advance state
  const uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
  const uint32_t rot = static_cast<uint32_t>(old >> 59u);
  return __funnelshift_r(xs, xs, rot);
}

__device__ __forceinline__ uint32_t pcg_next(uint64_t& s, uint64_t inc) {
  const uint64_t old = s;
  s = old * kPcgMult + inc;
  return pcg_output(old);
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
// Forward kinematics in fp32 (fk_walk, robot_model.cpp:371-395). The rotation
// is carried as a 3x3 matrix. Two chain policies:
//   FixedChain<TIP, SIG...>: the joint STRUCTURE (kind, axis, which origin
//     components are non-zero) is a compile-time signature, link lengths /
//     limits / gains stay runtime parameters. Every builtin descriptor (PSM,
//     ECM, STAR) has one; any descriptor with the same structure uses it.
//   GenericChain<DMAX>: any chain up to DMAX DoF, warp-uniform branches on the
//     runtime joint table.
// ---------------------------------------------------------------------------
constexpr int jsig(int kind, int axis, int oflags, int rot = 0) {
  return kind | (axis << 2) | (oflags << 5) | (rot << 8);
}

__device__ __forceinline__ void rot_cols(float (&m)[9], int ca, int cb, float c, float s) {
  // columns (ca, cb) <- (c*col_a + s*col_b, c*col_b - s*col_a)
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const float a = m[r * 3 + ca], b = m[r * 3 + cb];
    m[r * 3 + ca] = c * a + s * b;
    m[r * 3 + cb] = c * b - s * a;
  }
}

__device__ __forceinline__ void fast_sincos(float x, float& s, float& c) {
  // 2*pi range reduction then the SFU sin/cos (abs err ~2^-21.4 on [-pi, pi]).
  // FK never feeds back into the decoupled joint dynamics, so this only
  // perturbs the observed tip, by ~1e-7 m.
  const float red = fmaf(-6.28318530717958647692f, rintf(x * 0.15915494309189533577f), x);
  __sincosf(red, &s, &c);
}

// One actuated joint of fk_walk with signature fields (kind, axis, oflags, rot)
// that are compile-time constants in FixedChain and runtime in GenericChain.
// reduce: 2*pi range reduction before the SFU sin/cos. The specialised
// chains skip it: the host selects them only when every revolute limit lies
// in [-pi, pi] (select_chain), where __sincosf is accurate as is.
__device__ __forceinline__ void fk_joint(const JointEnc& J, int kind, int axis, int of, int rot, float qv,
                                         float (&m)[9], float (&p)[3], bool reduce = true) {
  // p += R * origin_translation
  if (of & 1) { p[0] += m[0] * J.o[0]; p[1] += m[3] * J.o[0]; p[2] += m[6] * J.o[0]; }
  if (of & 2) { p[0] += m[1] * J.o[1]; p[1] += m[4] * J.o[1]; p[2] += m[7] * J.o[1]; }
  if (of & 4) { p[0] += m[2] * J.o[2]; p[1] += m[5] * J.o[2]; p[2] += m[8] * J.o[2]; }
  if (rot) {  // R = R * R_origin
    float t[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        t[r * 3 + c] = m[r * 3 + 0] * J.R[0 * 3 + c] + m[r * 3 + 1] * J.R[1 * 3 + c] + m[r * 3 + 2] * J.R[2 * 3 + c];
#pragma unroll
    for (int k = 0; k < 9; ++k) m[k] = t[k];
  }
  if (kind == kRevolute) {
    float s, c;
    if (reduce) fast_sincos(qv, s, c);
    else __sincosf(qv, &s, &c);
    if (axis == 2) rot_cols(m, 0, 1, c, s);        // +z
    else if (axis == 5) rot_cols(m, 0, 1, c, -s);  // -z
    else if (axis == 0) rot_cols(m, 1, 2, c, s);   // +x
    else if (axis == 3) rot_cols(m, 1, 2, c, -s);  // -x
    else if (axis == 1) rot_cols(m, 2, 0, c, s);   // +y: col2' = c*col2 + s*col0, col0' = c*col0 - s*col2
    else if (axis == 4) rot_cols(m, 2, 0, c, -s);  // -y
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
    if (axis == 0 || axis == 3) {
      const float v = axis == 3 ? -qv : qv;
      p[0] += m[0] * v; p[1] += m[3] * v; p[2] += m[6] * v;
    } else if (axis == 1 || axis == 4) {
      const float v = axis == 4 ? -qv : qv;
      p[0] += m[1] * v; p[1] += m[4] * v; p[2] += m[7] * v;
    } else if (axis == 2 || axis == 5) {
      const float v = axis == 5 ? -qv : qv;
      p[0] += m[2] * v; p[1] += m[5] * v; p[2] += m[8] * v;
    } else {
      const float a0 = J.axis[0] * qv, a1 = J.axis[1] * qv, a2 = J.axis[2] * qv;
      p[0] += m[0] * a0 + m[1] * a1 + m[2] * a2;
      p[1] += m[3] * a0 + m[4] * a1 + m[5] * a2;
      p[2] += m[6] * a0 + m[7] * a1 + m[8] * a2;
    }
  }
}

__device__ __forceinline__ void fk_tip_offset(const RobotTable& R, int tf, const float (&m)[9], const float (&p)[3],
                                              float (&tip)[3]) {
  float t0 = p[0], t1 = p[1], t2 = p[2];
  if (tf & 1) { t0 += m[0] * R.tip[0]; t1 += m[3] * R.tip[0]; t2 += m[6] * R.tip[0]; }
  if (tf & 2) { t0 += m[1] * R.tip[1]; t1 += m[4] * R.tip[1]; t2 += m[7] * R.tip[1]; }
  if (tf & 4) { t0 += m[2] * R.tip[2]; t1 += m[5] * R.tip[2]; t2 += m[8] * R.tip[2]; }
  tip[0] = t0;
  tip[1] = t1;
  tip[2] = t2;
}

template <int TIPF, int JAW, int... S>
struct FixedChain {
  static constexpr int kDof = sizeof...(S);
  static constexpr bool kExact = true;
  static constexpr int kTipFlags = TIPF;
  static constexpr int kJaw = JAW;
  static constexpr int kSig[kDof] = {S...};
  __device__ static int dof(const RobotTable&) { return kDof; }
  __device__ static int jaw(const RobotTable&) { return kJaw; }
  template <int D>
  __device__ static void joint(const RobotTable& R, const float (&q)[kDof], float (&m)[9], float (&p)[3]) {
    constexpr int sig = kSig[D];
    fk_joint(R.j[D], sig & 3, (sig >> 2) & 7, (sig >> 5) & 7, (sig >> 8) & 1, q[D], m, p, false);
  }
  template <int... D>
  __device__ static void walk(const RobotTable& R, const float (&q)[kDof], float (&m)[9], float (&p)[3],
                              std::integer_sequence<int, D...>) {
    (joint<D>(R, q, m, p), ...);
  }
  __device__ static void fk(const RobotTable& R, const float (&q)[kDof], float (&tip)[3]) {
    float m[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
    float p[3] = {0.f, 0.f, 0.f};
    walk(R, q, m, p, std::make_integer_sequence<int, kDof>{});
    fk_tip_offset(R, TIPF, m, p, tip);
  }
};

template <int DMAX>
struct GenericChain {
  static constexpr int kDof = DMAX;
  static constexpr bool kExact = false;
  static constexpr int kTipFlags = -1;  // runtime (RobotTable::tip_flags)
  __device__ static int dof(const RobotTable& R) { return R.dof; }
  __device__ static int jaw(const RobotTable& R) { return R.jaw; }
  __device__ static void fk(const RobotTable& R, const float (&q)[DMAX], float (&tip)[3]) {
    float m[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
    float p[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
      if (d >= R.dof) break;
      const JointEnc& J = R.j[d];
      fk_joint(J, J.kind, J.axis_code, J.flags & 7, (J.flags >> 3) & 1, q[d], m, p);
    }
    fk_tip_offset(R, R.tip_flags, m, p, tip);
  }
};

// Builtin chain structures (assets/robots/*.robot after fixed-joint folding).
using PsmChain = FixedChain<0, 6, jsig(kRevolute, 2, 0), jsig(kRevolute, 1, 0), jsig(kPrismatic, 5, 4),
                            jsig(kRevolute, 2, 0), jsig(kRevolute, 0, 4), jsig(kRevolute, 1, 4),
                            jsig(kRevolute, 0, 4)>;
using EcmChain = FixedChain<4, -1, jsig(kRevolute, 2, 0), jsig(kRevolute, 1, 0), jsig(kPrismatic, 5, 4),
                            jsig(kRevolute, 2, 0), jsig(kRevolute, 0, 4), jsig(kRevolute, 1, 4)>;
using StarChain = FixedChain<4, -1, jsig(kRevolute, 2, 4), jsig(kRevolute, 1, 4), jsig(kRevolute, 2, 4),
                             jsig(kRevolute, 1, 4), jsig(kRevolute, 2, 4), jsig(kRevolute, 1, 4),
                             jsig(kRevolute, 2, 0), jsig(kRevolute, 1, 4)>;

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

// Knot parameters t_k = k / 1000 of the chord table, correctly rounded at
// compile time: a constant-cache broadcast instead of an fp64 division per point.
struct SplineTTable {
  double t[kSplineSubdiv + 1];
};
constexpr SplineTTable make_spline_t() {
  SplineTTable r{};
  for (int k = 0; k <= kSplineSubdiv; ++k) r.t[k] = static_cast<double>(k) / static_cast<double>(kSplineSubdiv);
  return r;
}
static __constant__ SplineTTable kSplineT = make_spline_t();

// sample_spline_waypoints (spline.cpp:40-72) in ONE pass over the 1001-point
// chord table, without storing it: the cumulative sums are formed in the
// reference's order, and the waypoint loop
//   for (s = spacing; s < total - 1e-12; s += spacing) {
//     while (seg + 1 < 1000 && cum[seg + 1] < s) ++seg; emit(seg, s) }
// is advanced as soon as cum[seg + 1] is known: a target s is emitted at the
// first k with cum[k] >= s (seg = k - 1), exactly where the reference's while
// loop stops. total is known only at the end, so emissions with
// s >= total - 1e-12 (at most one, since spacing >> 1e-12) are truncated.
// Same operations, same rounding; half the fp64 work of a two-pass walk.
// Writes fp32 waypoints; returns the count, or -1 past the table capacity.
template <int U>
static __device__ __noinline__ int spline_waypoints_stream(const Spline& s, double spacing, float* out, int cap) {
  const double span = 1.0;  // t1 - t0 (sample_path, envs.cpp:248-249)
  double p_prev[3];
  spline_eval(s, 0.0, p_prev);
  out[0] = (float)p_prev[0];
  out[1] = (float)p_prev[1];
  out[2] = (float)p_prev[2];
  int count = 1, tentative = 1;
  double cum_prev = 0.0, sv = spacing;
  double s_emit[2] = {0.0, 0.0};  // targets of the last two tentative emissions
  // Points in batches of U: the U evaluations and chord lengths are
  // independent (instruction-level parallelism for the fp64 latency chains);
  // only the cumulative sum and the emission loop run point by point, in the
  // reference's order, so every value is unchanged.
  static_assert(kSplineSubdiv % U == 0, "batch must divide the subdivision count");
  for (int kb = 1; kb <= kSplineSubdiv; kb += U) {
    double px[U][3], dk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) spline_eval(s, kSplineT.t[kb + u], px[u]);  // t_k == span * k / 1000
    dk[0] = dist3_rn(px[0], p_prev);
#pragma unroll
    for (int u = 1; u < U; ++u) dk[u] = dist3_rn(px[u], px[u - 1]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
    const int k = kb + u;
    const double cum_k = __dadd_rn(cum_prev, dk[u]);
    while (cum_k >= sv) {  // the reference's while loop stops at seg = k - 1 for this s
      const double seg_len = __dadd_rn(cum_k, -cum_prev);
      const double frac = seg_len > 0.0 ? __dadd_rn(sv, -cum_prev) / seg_len : 0.0;
      const double t = __dmul_rn(span, __dadd_rn((double)(k - 1), frac)) / (double)kSplineSubdiv;
      double w[3];
      spline_eval(s, t, w);
      if (tentative < cap) {
        out[3 * tentative + 0] = (float)w[0];
        out[3 * tentative + 1] = (float)w[1];
        out[3 * tentative + 2] = (float)w[2];
      }
      s_emit[tentative & 1] = sv;
      ++tentative;
      sv = __dadd_rn(sv, spacing);
    }
    cum_prev = cum_k;
    }
    p_prev[0] = px[U - 1][0];
    p_prev[1] = px[U - 1][1];
    p_prev[2] = px[U - 1][2];
  }
  const double total = cum_prev;
  if (total <= 1e-12) return count;
  const double limit = __dadd_rn(total, -1e-12);
  count = tentative;
  while (count > 1 && !(s_emit[(count - 1) & 1] < limit)) --count;  // drop s >= total - 1e-12
  if (count >= cap) return -1;
  out[3 * count + 0] = (float)p_prev[0];  // pts[1000] == eval(span * 1000 / 1000)
  out[3 * count + 1] = (float)p_prev[1];
  out[3 * count + 2] = (float)p_prev[2];
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

// sample_path (envs.cpp:241-267) + sample_spline_waypoints: draws the cubic
// from the env stream, shrinks it into the workspace ball and writes the
// waypoint table (fp32 copies of the fp64 waypoints). cnt = waypoint count.
// Returns error bits.
// QUAD > 1: the QUAD lanes of a group (same stream state) split the 101-point
// offset scan and combine the maximum by shuffle (max is exact, so the
// result is unchanged).
template <int QUAD = 1>
__device__ __forceinline__ int sample_path_spline(const TaskParams& T, uint64_t& s, uint64_t inc, Spline& sp) {
  int err = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) sp.c[k] = pcg_uniform(s, inc, -0.5, 0.5);
#pragma unroll
  for (int k = 0; k < 3; ++k) sp.c[3 + k] = pcg_uniform(s, inc, -0.5, 0.5);
#pragma unroll
  for (int k = 0; k < 3; ++k) sp.c[6 + k] = pcg_uniform(s, inc, -0.3, 0.3);
  double d[3];
  if (!sample_goal(s, inc, T, d)) err |= kErrGoalSampling;
  sp.c[9] = d[0];
  sp.c[10] = d[1];
  sp.c[11] = d[2];
  double max_off = 0.0;
  const int r = QUAD > 1 ? (threadIdx.x & (QUAD - 1)) : 0;
#pragma unroll 4
  for (int k = r; k <= 100; k += QUAD) {  // independent samples: unrolled for ILP
    double pt[3];
    spline_eval(sp, __dmul_rn(0.01, (double)k), pt);
    const double off = dist3_rn(pt, d);
    max_off = max_off > off ? max_off : off;
  }
  if constexpr (QUAD > 1) {
#pragma unroll
    for (int o = 1; o < QUAD; o <<= 1) {
      const double other = __shfl_xor_sync(0xffffffffu, max_off, o);
      max_off = max_off > other ? max_off : other;
    }
  }
  const double ctr[3] = {T.center[0], T.center[1], T.center[2]};
  const double allowed = __dadd_rn(T.radius, -dist3_rn(d, ctr));
  if (max_off > 0.0 && max_off > allowed) {
    const double scale = __dmul_rn(0.95, allowed > 0.0 ? allowed : 0.0) / max_off;
#pragma unroll
    for (int k = 0; k < 9; ++k) sp.c[k] = __dmul_rn(sp.c[k], scale);
  }
  return err;
}

// U: knots per batch (independent fp64 chains)
template <int U>
__device__ __forceinline__ int sample_path_waypoints(const TaskParams& T, uint64_t& s, uint64_t inc, float* table,
                                                     int& cnt) {
  Spline sp;
  int err = sample_path_spline(T, s, inc, sp);
  cnt = spline_waypoints_stream<U>(sp, T.spacing, table, T.wp_cap);
  if (cnt < 0) {
    err |= kErrWaypointCap;
    cnt = T.wp_cap;
  }
  return err;
}

#ifdef SG_RECORD_QUAD
// Computes the next reset_row of every PathFollowing env whose record is
// stale (after its last reset consumed it): q draws (middle half of each
// range, rounded once) then sample_path, from the env's current stream
// state, into the record buffers.
//
// Four lanes per env (a quad; 8 envs per warp, 4x the warps of one lane per
// env): every lane of the quad draws the same spline; per round of 20 knots
// lane r evaluates knots r*5+1..r*5+5 and their chord lengths (5 independent
// fp64 chains), the quad exchanges the 20 chords by shuffle, and all four
// lanes walk them in order (cumulative sum + waypoint emission exactly as
// sample_spline_waypoints; lane 0 writes). Same operations and summation
// order as spline_waypoints_stream, so the tables are bit-identical.
constexpr int kRecThreads = 128;
constexpr int kRecEnvsPerBlock = kRecThreads / 4;
static __global__ void __launch_bounds__(kRecThreads) path_record_kernel(const __grid_constant__ StepParams P) {
  constexpr int kQ = 4, kU = 5, kRound = kQ * kU;  // lanes per env, knots per lane per round
  static_assert(kSplineSubdiv % kRound == 0, "rounds must tile the knots");
  const RobotTable& R = P.robot;
  const TaskParams& T = P.task;
  const int64_t n = T.n;
  const int lane = threadIdx.x & 31, r = lane & (kQ - 1), base = lane & ~(kQ - 1);
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kQ;
  const bool need = i < n && !P.p.rec_valid[i];
  if (!__any_sync(0xffffffffu, need)) return;
  uint64_t s = need ? P.p.rng_state[i] : 0;
  const uint64_t inc = need ? P.p.rng_inc[i] : 1;
  int err = 0;
  Spline sp;
#pragma unroll
  for (int k = 0; k < 12; ++k) sp.c[k] = 0.0;
  for (int d = 0; d < R.dof; ++d) {  // (lanes without work draw from a dummy stream)
    const double quarter = __dmul_rn(0.25, __dadd_rn(R.hi_d[d], -R.lo_d[d]));
    const float qv = (float)pcg_uniform(s, inc, __dadd_rn(R.lo_d[d], quarter), __dadd_rn(R.hi_d[d], -quarter));
    if (need && r == 0) P.p.rec_q[d * n + i] = qv;
  }
  err = sample_path_spline<kQ>(T, s, inc, sp);
  if (!need) err = 0;
  const bool writer = need && r == 0;
  float* out = P.p.rec_wps + (need ? i : 0) * (int64_t)T.wp_cap * 3;
  const int cap = T.wp_cap;
  const double spacing = T.spacing;
  double p_end[3];  // last knot of the previous round (lane r = 0 needs it)
  spline_eval(sp, 0.0, p_end);
  if (writer) {
    out[0] = (float)p_end[0];
    out[1] = (float)p_end[1];
    out[2] = (float)p_end[2];
  }
  int tentative = 1;
  double cum_prev = 0.0, sv = spacing;
  double s_emit[2] = {0.0, 0.0};  // targets of the last two tentative emissions
  for (int kb = 1; kb <= kSplineSubdiv; kb += kRound) {
    const int k0 = kb + r * kU;  // this lane's first knot
    double px[kU][3], dk[kU], pp[3];
#pragma unroll
    for (int u = 0; u < kU; ++u) spline_eval(sp, kSplineT.t[k0 + u], px[u]);
    // knot k0 - 1: the previous lane's last knot, or the previous round's end
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double up = __shfl_sync(0xffffffffu, px[kU - 1][k], (lane + 31) & 31);  // lane - 1
      pp[k] = r == 0 ? p_end[k] : up;
    }
    dk[0] = dist3_rn(px[0], pp);
#pragma unroll
    for (int u = 1; u < kU; ++u) dk[u] = dist3_rn(px[u], px[u - 1]);
#pragma unroll
    for (int k = 0; k < 3; ++k) p_end[k] = __shfl_sync(0xffffffffu, px[kU - 1][k], base + kQ - 1);
    // every lane of the quad walks the round's chords in knot order; cum is
    // non-decreasing, so a round whose last cumulative length is below the
    // next target emits nothing and needs only its sums
    double dr[kRound];
#pragma unroll
    for (int q = 0; q < kQ; ++q)
#pragma unroll
      for (int u = 0; u < kU; ++u) dr[q * kU + u] = __shfl_sync(0xffffffffu, dk[u], base + q);
    double cum_end = cum_prev;
#pragma unroll
    for (int j = 0; j < kRound; ++j) cum_end = __dadd_rn(cum_end, dr[j]);
    if (!(cum_end >= sv)) {
      cum_prev = cum_end;
      continue;
    }
#pragma unroll 1
    for (int j = 0; j < kRound; ++j) {
      {
        const double d = dr[j];
        const int k = kb + j;
        const double cum_k = __dadd_rn(cum_prev, d);
        while (cum_k >= sv) {  // the reference's while loop stops at seg = k - 1 for this s
          const double seg_len = __dadd_rn(cum_k, -cum_prev);
          const double frac = seg_len > 0.0 ? __dadd_rn(sv, -cum_prev) / seg_len : 0.0;
          const double tw = __dmul_rn(1.0, __dadd_rn((double)(k - 1), frac)) / (double)kSplineSubdiv;
          double wv[3];
          spline_eval(sp, tw, wv);
          if (writer && tentative < cap) {
            out[3 * tentative + 0] = (float)wv[0];
            out[3 * tentative + 1] = (float)wv[1];
            out[3 * tentative + 2] = (float)wv[2];
          }
          s_emit[tentative & 1] = sv;
          ++tentative;
          sv = __dadd_rn(sv, spacing);
        }
        cum_prev = cum_k;
      }
    }
  }
  if (!writer) return;
  const double total = cum_prev;
  int count = 1;
  if (total > 1e-12) {
    const double limit = __dadd_rn(total, -1e-12);
    count = tentative;
    while (count > 1 && !(s_emit[(count - 1) & 1] < limit)) --count;  // drop s >= total - 1e-12
    if (count >= cap) {
      err |= kErrWaypointCap;
      count = cap;
    } else {
      out[3 * count + 0] = (float)p_end[0];  // pts[1000]
      out[3 * count + 1] = (float)p_end[1];
      out[3 * count + 2] = (float)p_end[2];
      count += 1;
    }
  }
  P.p.rec_len[i] = count;
  P.p.rec_err[i] = err;
  P.p.rec_rng[i] = s;
  P.p.rec_valid[i] = 1;
}

#else
// Computes the next reset_row of every PathFollowing env whose record is
// stale (after its last reset consumed it): q draws (middle half of each
// range, rounded once) then sample_path, from the env's current stream
// state, into the record buffers.
//
// Warp-specialised: a block owns 32 envs. Warps 1-4 are EVALUATORS, four
// lanes per env: they draw the env's q and spline (every lane of the quad the
// same stream; the 101-point offset scan split over the quad), then per round
// of 20 knots lane r evaluates knots r*5+1..r*5+5 and their chord lengths
// (5 independent fp64 chains) into a shared-memory ring. Warp 0 is the
// WALKER, one lane per env: it takes each round's 20 chords in knot order
// and runs the cumulative sum of sample_spline_waypoints (spline.cpp:40-72),
// queueing each waypoint emission's inputs; the evaluators turn a round's
// queue (all 32 envs, compacted, one emission per lane: the fp64 divisions
// and the spline evaluation without divergence) into waypoints while the
// walker sums the next round. Two ring / queue stages, handed over with named
// barriers (FULL: evaluators arrive, walker syncs; EMPTY: the reverse). Same
// operations and summation order as spline_waypoints_stream, so the tables
// are bit-identical.
constexpr int kRecEnvsPerBlock = 32, kRecQ = 4, kRecU = 5, kRecRound = kRecQ * kRecU;
constexpr int kRecRounds = kSplineSubdiv / kRecRound;
constexpr int kRecPad = kRecRound + 1;  // 21 doubles per env row: conflict-free walker loads
constexpr int kRecEval = kRecEnvsPerBlock * kRecQ;  // evaluator threads
constexpr int kRecThreads = 32 + kRecEval;           // 160
constexpr int kRecEmitQ = 6;                         // queued emissions per env per round
static_assert(kSplineSubdiv % kRecRound == 0, "rounds must tile the knots");

struct RecEmit {  // one queued waypoint emission
  double cum_prev, cum_k, sv;
  int k, slot;
};

__device__ __forceinline__ void rec_bar_sync(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kRecThreads) : "memory"); }
__device__ __forceinline__ void rec_bar_arrive(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(kRecThreads) : "memory");
}

// One waypoint of sample_spline_waypoints: target sv reached at knot k,
// t = (k - 1 + (sv - cum_prev) / seg_len) / 1000, fp32 copy of eval(t).
__device__ __forceinline__ void rec_emit(const Spline& sp, float* dst, double cp, double ck, double svv, int k) {
  const double seg_len = __dadd_rn(ck, -cp);
  const double frac = seg_len > 0.0 ? __dadd_rn(svv, -cp) / seg_len : 0.0;
  const double tw = __dmul_rn(1.0, __dadd_rn((double)(k - 1), frac)) / (double)kSplineSubdiv;
  double wv[3];
  spline_eval(sp, tw, wv);
  dst[0] = (float)wv[0];
  dst[1] = (float)wv[1];
  dst[2] = (float)wv[2];
}

// 4 blocks per SM: the 512 blocks of 16,384 envs run in one wave on 148 SMs
#ifndef SG_REC_MINB
#define SG_REC_MINB 4
#endif
static __global__ void __launch_bounds__(kRecThreads, SG_REC_MINB) path_record_kernel(const __grid_constant__ StepParams P) {
  constexpr int kBarSetup = 1, kBarFull = 2, kBarEmpty = 4, kBarDone = 6;  // FULL / EMPTY: + stage
  __shared__ double ring[2][kRecEnvsPerBlock][kRecPad];
  __shared__ RecEmit s_q[2][kRecEnvsPerBlock][kRecEmitQ];
  __shared__ int s_qoff[2][kRecEnvsPerBlock + 1];  // exclusive offsets, total at [32]
  __shared__ double s_sp[kRecEnvsPerBlock][12];
  __shared__ uint64_t s_rng[kRecEnvsPerBlock];
  __shared__ int s_err[kRecEnvsPerBlock], s_need[kRecEnvsPerBlock];
  const RobotTable& R = P.robot;
  const TaskParams& T = P.task;
  const int64_t n = T.n;
  const int cap = T.wp_cap;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e0 = (int64_t)blockIdx.x * kRecEnvsPerBlock;
  const int el = warp == 0 ? lane : (warp - 1) * (32 / kRecQ) + lane / kRecQ;  // env of this thread
  const int64_t i = e0 + el;
  const bool need = i < n && !P.p.rec_valid[i];
  if (warp == 0) s_need[lane] = need ? 1 : 0;
  if (!__syncthreads_or(need)) return;

  if (warp > 0) {  // ---- evaluators ----------------------------------------
    const int r = lane & (kRecQ - 1), base = lane & ~(kRecQ - 1);
    const int te = threadIdx.x - 32;  // 0 .. kRecEval - 1
    uint64_t s = need ? P.p.rng_state[i] : 0;
    const uint64_t inc = need ? P.p.rng_inc[i] : 1;
    for (int d = 0; d < R.dof; ++d) {  // (lanes without work draw from a dummy stream)
      const double quarter = __dmul_rn(0.25, __dadd_rn(R.hi_d[d], -R.lo_d[d]));
      const float qv = (float)pcg_uniform(s, inc, __dadd_rn(R.lo_d[d], quarter), __dadd_rn(R.hi_d[d], -quarter));
      if (need && r == 0) P.p.rec_q[d * n + i] = qv;
    }
    Spline sp;
#pragma unroll
    for (int k = 0; k < 12; ++k) sp.c[k] = 0.0;
    const int err = sample_path_spline<kRecQ>(T, s, inc, sp);
    if (r == 0) {
#pragma unroll
      for (int k = 0; k < 12; ++k) s_sp[el][k] = sp.c[k];
      s_rng[el] = s;
      s_err[el] = need ? err : 0;
    }
    rec_bar_arrive(kBarSetup);
    double p_end[3];  // last knot of the previous round (lane r = 0 needs it)
    spline_eval(sp, 0.0, p_end);
    for (int j = 0; j < kRecRounds + 2; ++j) {
      const int st = j & 1;
      double dk[kRecU];
      if (j < kRecRounds) {
        const int k0 = 1 + j * kRecRound + r * kRecU;  // this lane's first knot
        double px[kRecU][3], pp[3];
#pragma unroll
        for (int u = 0; u < kRecU; ++u) spline_eval(sp, kSplineT.t[k0 + u], px[u]);
        // knot k0 - 1: the previous lane's last knot, or the previous round's end
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double up = __shfl_sync(0xffffffffu, px[kRecU - 1][k], (lane + 31) & 31);  // lane - 1
          pp[k] = r == 0 ? p_end[k] : up;
        }
        dk[0] = dist3_rn(px[0], pp);
#pragma unroll
        for (int u = 1; u < kRecU; ++u) dk[u] = dist3_rn(px[u], px[u - 1]);
#pragma unroll
        for (int k = 0; k < 3; ++k) p_end[k] = __shfl_sync(0xffffffffu, px[kRecU - 1][k], base + kRecQ - 1);
      }
      if (j >= 2) {
        // the walker is done with round j - 2 in this stage: its chords are
        // consumed and its emissions queued -- turn them into waypoints
        rec_bar_sync(kBarEmpty + st);
        const int total_q = s_qoff[st][kRecEnvsPerBlock];
        for (int f = te; f < total_q; f += kRecEval) {
          int e = 0;  // last env whose first entry is <= f
#pragma unroll
          for (int step = 16; step; step >>= 1)
            if (e + step < kRecEnvsPerBlock && s_qoff[st][e + step] <= f) e += step;
          const RecEmit& q = s_q[st][e][f - s_qoff[st][e]];
          if (s_need[e] && q.slot < cap) {
            Spline spe;
#pragma unroll
            for (int c = 0; c < 12; ++c) spe.c[c] = s_sp[e][c];
            rec_emit(spe, P.p.rec_wps + (e0 + e) * (int64_t)cap * 3 + 3 * q.slot, q.cum_prev, q.cum_k, q.sv, q.k);
          }
        }
      }
      if (j < kRecRounds) {
#pragma unroll
        for (int u = 0; u < kRecU; ++u) ring[st][el][r * kRecU + u] = dk[u];
        rec_bar_arrive(kBarFull + st);
      }
    }
    rec_bar_arrive(kBarDone);
    return;
  }

  // ---- walker: lane = env ----------------------------------------------------
  rec_bar_sync(kBarSetup);
  Spline sp;
#pragma unroll
  for (int k = 0; k < 12; ++k) sp.c[k] = s_sp[lane][k];
  int err = s_err[lane];
  const uint64_t s_after = s_rng[lane];
  const double spacing = T.spacing;
  float* out = P.p.rec_wps + (need ? i : 0) * (int64_t)cap * 3;
  {
    double p0[3];
    spline_eval(sp, 0.0, p0);
    if (need) {
      out[0] = (float)p0[0];
      out[1] = (float)p0[1];
      out[2] = (float)p0[2];
    }
  }
  int tentative = 1;
  double cum_prev = 0.0, sv = spacing;
  double s_emit[2] = {0.0, 0.0};  // targets of the last two tentative emissions
  for (int j = 0; j < kRecRounds; ++j) {
    const int st = j & 1;
    rec_bar_sync(kBarFull + st);
    const double* dr = ring[st][lane];
    // the round's cumulative lengths (one dependent fp64 add per knot, in the
    // reference's order); cum is non-decreasing, so a round whose last value
    // is below the next target emits nothing
    double cum[kRecRound];
    {
      double c = cum_prev;
#pragma unroll
      for (int u = 0; u < kRecRound; ++u) {
        c = __dadd_rn(c, dr[u]);
        cum[u] = c;
      }
    }
    int qn = 0;
    if (__any_sync(0xffffffffu, cum[kRecRound - 1] >= sv)) {
#pragma unroll
      for (int u = 0; u < kRecRound; ++u) {
        const int k = 1 + j * kRecRound + u;
        const double cum_k = cum[u];
        while (cum_k >= sv) {  // the reference's while loop stops at seg = k - 1 for this s
          if (qn < kRecEmitQ) {
            RecEmit& q = s_q[st][lane][qn++];
            q.cum_prev = cum_prev;
            q.cum_k = cum_k;
            q.sv = sv;
            q.k = k;
            q.slot = tentative;
          } else if (need && tentative < cap) {  // queue full (rare): emit on the spot
            rec_emit(sp, out + 3 * tentative, cum_prev, cum_k, sv, k);
          }
          s_emit[tentative & 1] = sv;
          ++tentative;
          sv = __dadd_rn(sv, spacing);
        }
        cum_prev = cum_k;
      }
    }
    cum_prev = cum[kRecRound - 1];
    // publish the round's queue (exclusive scan of the per-env counts)
    int off = qn;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, off, d);
      if (lane >= d) off += v;
    }
    s_qoff[st][lane] = off - qn;
    if (lane == 31) s_qoff[st][kRecEnvsPerBlock] = off;
    __syncwarp();
    rec_bar_arrive(kBarEmpty + st);
  }
  rec_bar_sync(kBarDone);  // every queued waypoint is written
  if (!need) return;
  const double total = cum_prev;
  int count = 1;
  if (total > 1e-12) {
    const double limit = __dadd_rn(total, -1e-12);
    count = tentative;
    while (count > 1 && !(s_emit[(count - 1) & 1] < limit)) --count;  // drop s >= total - 1e-12
    if (count >= cap) {
      err |= kErrWaypointCap;
      count = cap;
    } else {
      double p_last[3];  // pts[1000]
      spline_eval(sp, kSplineT.t[kSplineSubdiv], p_last);
      out[3 * count + 0] = (float)p_last[0];
      out[3 * count + 1] = (float)p_last[1];
      out[3 * count + 2] = (float)p_last[2];
      count += 1;
    }
  }
  P.p.rec_len[i] = count;
  P.p.rec_err[i] = err;
  P.p.rec_rng[i] = s_after;
  P.p.rec_valid[i] = 1;
}
#endif

// reset_row (envs.cpp:304-360) for one env. Out of line (rare path) and
// communicating through HBM only, so the caller's state arrays stay in
// registers: the caller reloads q/qdot/q_target/goal/tip/waypoint idx+len
// after the call. Returns an error bit (0 on success).
template <class CH, int TASK>
__device__ __noinline__ int reset_env(const StepParams& P, int64_t i) {
  constexpr int D = CH::kDof;
  const RobotTable& R = P.robot;
  const TaskParams& T = P.task;
  const int task = TASK >= 0 ? TASK : T.task;
  const int dof = CH::dof(R);
  const int64_t n = T.n;
  uint64_t s = P.p.rng_state[i];
  const uint64_t inc = P.p.rng_inc[i];
  int err = 0;
  float q[D], goal[3], tip[3];
  int32_t wp_idx = 0, wp_len = 0;
  const bool rec = task == kTaskPath && P.p.rec_valid && P.p.rec_valid[i];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    q[d] = 0.f;
    if (d < dof) {
      if (rec) {
        q[d] = P.p.rec_q[d * n + i];
      } else {
        const double quarter = __dmul_rn(0.25, __dadd_rn(R.hi_d[d], -R.lo_d[d]));
        q[d] = (float)pcg_uniform(s, inc, __dadd_rn(R.lo_d[d], quarter), __dadd_rn(R.hi_d[d], -quarter));
      }
    }
  }
  CH::fk(R, q, tip);
  if (task == kTaskPath) {
    float* table = P.p.wps + i * (int64_t)T.wp_cap * 3;
    int cnt;
    if (rec) {  // install the precomputed reset (same draws, same arithmetic)
      cnt = P.p.rec_len[i];
      err |= P.p.rec_err[i];
      s = P.p.rec_rng[i];
      const float* src = P.p.rec_wps + i * (int64_t)T.wp_cap * 3;
      for (int k = 0; k < 3 * cnt; ++k) table[k] = src[k];
      P.p.rec_valid[i] = 0;
    } else {
      err |= sample_path_waypoints<4>(T, s, inc, table, cnt);
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
    if (task == kTaskTrack) {  // envs.cpp:322-327
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        P.p.goal_spawn[k * n + i] = goal[k];
        P.p.goal_vel[k * n + i] = 0.f;
      }
    }
  }
  P.p.rng_state[i] = s;
  P.p.step_count[i] = 0;
  P.p.hold_count[i] = 0;
  P.p.episode_count[i] += 1;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (d < dof) {
      P.p.q[d * n + i] = q[d];
      P.p.qd[d * n + i] = 0.f;
      P.p.qt[d * n + i] = q[d];
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    P.p.goals[k * n + i] = goal[k];
    P.p.tips[k * n + i] = tip[k];
  }
  if (task == kTaskPath) {
    P.p.wp_idx[i] = wp_idx;
    P.p.wp_len[i] = wp_len;
  }
  return err;
}

// rng.normal() (rng.hpp:53-57) with the uniforms formed exactly in fp64 and
// the transform in fp32 (the stream consumption, 2 u32, is exact).
__device__ __forceinline__ float pcg_normal_f32(uint64_t& s, uint64_t inc) {
  const uint32_t a = pcg_next(s, inc), b = pcg_next(s, inc);
  const float u1 = (float)__dmul_rn(__dadd_rn((double)a, 0.5), 0x1.0p-32);  // (0, 1)
  const float u2 = (float)((double)b * 0x1.0p-32);
  return sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
}

// ActiveTracking goal drift after scoring (envs.cpp:497-510): g += vel; per
// axis clamp g to spawn +- goal_offset_clip, vel += N(0, noise_std) from the
// env's stream, clamp vel to +- vel_clamp. Spawn / velocity / stream state
// live in HBM (the generic-chain kernel runs this task).
static __device__ __noinline__ void track_drift(const StepParams& P, int64_t i, float* goal) {
  const TaskParams& T = P.task;
  const int64_t n = T.n;
  uint64_t s = P.p.rng_state[i];
  const uint64_t inc = P.p.rng_inc[i];
  float vel[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    vel[k] = P.p.goal_vel[k * n + i];
    goal[k] += vel[k];
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float sp = P.p.goal_spawn[k * n + i];
    goal[k] = fminf(fmaxf(goal[k], sp - T.goal_offset_clip), sp + T.goal_offset_clip);
    vel[k] += T.track_noise_std * pcg_normal_f32(s, inc);
    vel[k] = fminf(fmaxf(vel[k], -T.track_vel_clamp), T.track_vel_clamp);
    P.p.goal_vel[k * n + i] = vel[k];
  }
  P.p.rng_state[i] = s;
}

// Load one env's state from HBM (DoF-major SoA) into registers.
template <class CH, int TASK>
__device__ __forceinline__ void load_env(const StepParams& P, int64_t i, float (&q)[CH::kDof],
                                         float (&qd)[CH::kDof], float (&qt)[CH::kDof], float (&goal)[3],
                                         float (&tip)[3], int32_t& wi, int32_t& wl) {
  const int64_t n = P.task.n;
  const int dof = CH::dof(P.robot);
#pragma unroll
  for (int d = 0; d < CH::kDof; ++d) {
    if (d < dof) {
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
  const int task = TASK >= 0 ? TASK : P.task.task;
  if (task == kTaskPath) {
    wi = P.p.wp_idx[i];
    wl = P.p.wp_len[i];
  }
}

// rescale_to_range (dynamics.cpp:91-95): exact at both endpoints.
__device__ __forceinline__ float rescale(float x, float l, float h) {
  if (x >= 1.f) return h;
  if (x <= -1.f) return l;
  return l + 0.5f * (x + 1.f) * (h - l);
}

// ---------------------------------------------------------------------------
// The fused step kernel: dynamics -> FK -> reward/flags -> observation ->
// terminal copy + masked reset + re-observe, k_steps steps per launch.
//
// Warp-specialised env teams. A CTA is one team of G warps that owns 32 envs
// (lane = env); warp s of the team owns a contiguous DoF block (dof_block_*).
// Because the DoF block is warp-uniform, every DoF index stays a compile-time
// constant inside the warp's code (FixedChain joint structure is preserved)
// and there is no intra-warp divergence. Per step each warp integrates its
// DoFs, builds the partial FK transform of its joints and stages its
// observation columns; warp 0 (the scorer) turns the partial transforms into
// the tip, scores reward / hold / waypoint advance / flags, resets ended envs
// and stores the observation rows while the producer warps already run the
// next step (team_run). G multiplies the warps per SM (16384 envs = 512
// teams), which is what hides latency here.
//
//   CH    chain policy          TASK  kTaskTarget / kTaskPath, or -1 runtime
//   G     warps per team        MODE  control mode, or -1 runtime
//   GEN   actions = the bench stream generated in-kernel   SUB  substeps or 0
// ---------------------------------------------------------------------------
constexpr int kTeamEnvs = 32;

struct Xform {  // rigid transform (R row-major, p)
  float m[9];
  float p[3];
};

// v <- p + m * v
__device__ __forceinline__ void apply_xform(const float* m, const float* p, float (&v)[3]) {
  const float v0 = p[0] + m[0] * v[0] + m[1] * v[1] + m[2] * v[2];
  const float v1 = p[1] + m[3] * v[0] + m[4] * v[1] + m[5] * v[2];
  const float v2 = p[2] + m[6] * v[0] + m[7] * v[1] + m[8] * v[2];
  v[0] = v0;
  v[1] = v1;
  v[2] = v2;
}

// DoF block of team warp S: [B, B + N). Warp 0 (the scorer: tip, reward,
// flags, resets, observation rows) takes scorer_dofs(D, G) DoFs; the others
// are split contiguously over the producer warps 1..G-1, remainder to the
// last ones. Shared by host (bench stream seeding) and device.
#ifndef SG_SCORER_SHARE
#define SG_SCORER_SHARE 1  // the scorer takes this many DoFs fewer than D / G (at least 1)
#endif
#ifndef SG_SCORER_DOFS
#define SG_SCORER_DOFS -1  // >= 0: the scorer's DoF count (A/B); -1: the SG_SCORER_SHARE rule
#endif
__host__ __device__ constexpr int scorer_dofs(int D, int G) {
  return G == 1 ? D
                : (SG_SCORER_DOFS >= 0 ? (SG_SCORER_DOFS < D ? SG_SCORER_DOFS : D - 1)
                                       : (D / G - SG_SCORER_SHARE > 1 ? D / G - SG_SCORER_SHARE : 1));
}
__host__ __device__ constexpr int dof_block_begin(int D, int G, int S) {
  return S == 0 ? 0
                : scorer_dofs(D, G) + (S - 1) * ((D - scorer_dofs(D, G)) / (G - 1)) +
                      ((S - 1) - ((G - 1) - (D - scorer_dofs(D, G)) % (G - 1)) > 0
                           ? (S - 1) - ((G - 1) - (D - scorer_dofs(D, G)) % (G - 1))
                           : 0);
}
__host__ __device__ constexpr int dof_block_size(int D, int G, int S) {
  return S == 0 ? scorer_dofs(D, G)
                : (D - scorer_dofs(D, G)) / (G - 1) +
                      ((S - 1) >= (G - 1) - (D - scorer_dofs(D, G)) % (G - 1) ? 1 : 0);
}

template <class CH, int G, int S>
struct Block {
  static constexpr int B = dof_block_begin(CH::kDof, G, S);
  static constexpr int N = dof_block_size(CH::kDof, G, S);
  static constexpr int E = B + N;
};

// Partial FK of joints [B, E) starting from the identity.
template <class CH, int B, int... J>
__device__ __forceinline__ void fk_range(const RobotTable& R, const float* q, Xform& x,
                                         std::integer_sequence<int, J...>) {
  if constexpr (CH::kExact) {
    ((void)fk_joint(R.j[B + J], CH::kSig[B + J] & 3, (CH::kSig[B + J] >> 2) & 7, (CH::kSig[B + J] >> 5) & 7,
                    (CH::kSig[B + J] >> 8) & 1, q[J], x.m, x.p, false),
     ...);
  } else {
    (
        [&] {
          if (B + J < R.dof) {
            const JointEnc& Jt = R.j[B + J];
            fk_joint(Jt, Jt.kind, Jt.axis_code, Jt.flags & 7, (Jt.flags >> 3) & 1, q[J], x.m, x.p);
          }
        }(),
        ...);
  }
}

// Right-to-left POINT form of fk_walk for a FixedChain joint:
// v <- o_j + Motion_j(q_j) v (T_j = Trans(o_j) Motion_j; the builtin
// signatures carry no origin rotation). A revolute joint rotates two
// coordinates (4 ops), a prismatic one shifts one; no rotation matrix is
// composed, and the sin/cos of every joint are independent of v.
template <class CH, int D>
__device__ __forceinline__ void point_joint(const RobotTable& R, float qv, float s, float c, float (&v)[3]) {
  constexpr int sig = CH::kSig[D];
  constexpr int kind = sig & 3, axis = (sig >> 2) & 7, of = (sig >> 5) & 7;
  static_assert(((sig >> 8) & 1) == 0, "the point form needs identity origin rotations");
  if constexpr (kind == kRevolute) {
    const float sn = axis >= 3 ? -s : s;
    if constexpr (axis % 3 == 2) {  // z
      const float x = v[0], y = v[1];
      v[0] = fmaf(c, x, -sn * y);
      v[1] = fmaf(sn, x, c * y);
    } else if constexpr (axis % 3 == 0) {  // x
      const float y = v[1], z = v[2];
      v[1] = fmaf(c, y, -sn * z);
      v[2] = fmaf(sn, y, c * z);
    } else {  // y
      const float x = v[0], z = v[2];
      v[0] = fmaf(c, x, sn * z);
      v[2] = fmaf(-sn, x, c * z);
    }
  } else {
    v[axis % 3] += axis >= 3 ? -qv : qv;
  }
  const JointEnc& J = R.j[D];
  if constexpr ((of & 1) != 0) v[0] += J.o[0];
  if constexpr ((of & 2) != 0) v[1] += J.o[1];
  if constexpr ((of & 4) != 0) v[2] += J.o[2];
}

// v <- T_B ... T_{B+N-1} v (right to left), sin/cos precomputed.
template <class CH, int B, int N>
__device__ __forceinline__ void point_range(const RobotTable& R, const float* q, const float* sn, const float* cs,
                                            float (&v)[3]) {
  if constexpr (N > 0) {
    point_joint<CH, B + N - 1>(R, q[N - 1], sn[N - 1], cs[N - 1], v);
    point_range<CH, B, N - 1>(R, q, sn, cs, v);
  }
}

template <class CH>
__device__ __forceinline__ int tip_flags_of(const RobotTable& R) {
  if constexpr (CH::kExact) return CH::kTipFlags;
  else return R.tip_flags;
}

// Per-team shared memory. Everything a step publishes is double-buffered by
// step parity: producers stage step k+1 while the scorer still reads step k.
template <int G>
struct TeamSmem {
  float xf[2][G][12][kTeamEnvs];  // partial transforms, lane-contiguous (conflict-free)
  int32_t ended[2][kTeamEnvs];    // rows that ended at the step of that parity
  int32_t any_end[2];             // the scorer's "rows ended" flag for the barrier of that parity
};

// Coalesced team store of `count` staged floats with 16-byte vectors. For a
// FixedChain full team the count and thread count are compile-time constants:
// all shared loads of the thread are issued before its global stores. g must
// be 16-byte aligned (an env's row block always is).
template <class CH, int FULL, int NT>
__device__ __forceinline__ void team_store(float* __restrict__ g, const float* __restrict__ s, int count, bool vec,
                                           int t) {
  // vec: count % 4 == 0 (a team's rows start at a multiple of 4 envs, so g is
  // 16-byte aligned); the unroll bound is the full 32-env team
  if (CH::kExact && vec) {
    constexpr int iters = (FULL / 4 + NT - 1) / NT;
    const int n4 = count >> 2;
    float4* g4 = reinterpret_cast<float4*>(g);
    const float4* s4 = reinterpret_cast<const float4*>(s);
    float4 v[iters];
#pragma unroll
    for (int it = 0; it < iters; ++it)
      if (t + it * NT < n4) v[it] = s4[t + it * NT];
#pragma unroll
    for (int it = 0; it < iters; ++it)
      if (t + it * NT < n4) g4[t + it * NT] = v[it];
  } else {
    for (int k = t; k < count; k += NT) g[k] = s[k];
  }
}

// Observation row buffers of a team: the scorer stores its rows right after
// scoring (two buffers, by step parity). SG_PRODUCER_ROWS (A/B builds): the
// producers store step k's rows after B(k+1) while the scorer stages step
// k+1 and everyone produces step k+2 -- three buffers in flight; parity-green
// but measured slower (PSM 16K, K = 250: 207.7 vs 177.0 us; ECM 566.8 vs
// 486.0 us).
template <int G>
__host__ __device__ constexpr int team_obs_bufs() {
#ifdef SG_PRODUCER_ROWS
  return G > 1 ? 3 : 2;
#else
  return 2;
#endif
}

// Shared memory of one team (TeamSmem + observation row buffers and
// double-buffered action rows), a multiple of 16 bytes.
template <int G>
__host__ __device__ constexpr size_t team_smem_bytes_g(int A) {
  return (sizeof(TeamSmem<G>) + 15) / 16 * 16 +
         (size_t)(team_obs_bufs<G>() * kTeamEnvs * (3 * A + 6) + 2 * (kTeamEnvs * A + 4)) * 4;
}
template <int G>
inline size_t team_smem_bytes(int A) {
  return team_smem_bytes_g<G>(A);
}

// Rows of one team and its synchronisation. TPC == 1: the CTA is the team
// (32 envs per CTA, CTA barriers). TPC > 1 ("packed"): TPC teams per CTA with
// one CTA per SM; the env quads (4 envs) are split evenly over all
// gridDim.x * TPC teams (<= 32 envs each), so every SM carries the same
// number of envs, and the team's warps meet at a named barrier (id 1 + team).
#ifdef SG_TIME_PROBE
// Launch timeline probe (A/B builds only): {first CTA start, first team past
// its state loads, last team past step 0, first / last team past the loop,
// last CTA end}, %globaltimer ns; the last CTA prints and re-arms them.
__device__ unsigned long long g_tprobe[8] = {~0ull, ~0ull, 0, ~0ull, 0, 0, 0, 0};
__device__ unsigned int g_tprobe_ticket = 0;
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

struct Team {
  int64_t row0;
  int rows;     // <= 0: empty team
  int id;       // team index within the CTA
  int tthread;  // thread index within the team (role * 32 + lane)
};

// Team barriers. The scorer and the producers reach each barrier from
// their own role's code (warp-specialised, like CUTLASS's named-barrier
// producer / consumer warps); a one-team CTA uses __syncthreads(_or), a
// packed CTA the named barrier 1 + team. compute-sanitizer synccheck reports
// these role-divergent arrivals ("divergent threads in block") with either
// barrier form; memcheck and racecheck are clean and the results are
// bit-exact against the oracle. SG_UNALIGNED_TEAM_BARRIERS: the non-aligned
// barrier.cta forms for one-team CTAs too (measured 1-3 % slower).
template <int G, int TPC>
__device__ __forceinline__ bool team_sync_or(const Team& tm, bool v) {
#ifndef SG_UNALIGNED_TEAM_BARRIERS
  if constexpr (TPC == 1) {
    return __syncthreads_or(v);
  } else
#endif
  {
    uint32_t r;
    asm volatile(
        "{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n barrier.cta.red.or.pred q, %2, %3, p;\n"
        " selp.u32 %0, 1, 0, q;\n}"
        : "=r"(r)
        : "r"((uint32_t)v), "r"(1 + tm.id), "r"(32 * G)
        : "memory");
    return r != 0;
  }
}

template <int G, int TPC>
__device__ __forceinline__ void team_sync(const Team& tm);

// A team barrier that also hands every warp the scorer's warp-uniform flag
// v (S == 0: "rows ended at the previous step"): the barrier OR-reduction.
// SG_FLAG_TEAM_BARRIER (A/B): the scorer's lane 0 stores the flag into `slot`
// (one per step parity) before a plain barrier and everyone reads it after
// -- same result, 5 % slower at K = 250 (187.6 vs 177.5 us), and synccheck
// reports the plain barrier's role-divergent arrivals just the same.
template <int G, int TPC, int S>
__device__ __forceinline__ bool team_sync_flag(const Team& tm, int32_t& slot, bool v) {
#ifndef SG_FLAG_TEAM_BARRIER
  return team_sync_or<G, TPC>(tm, S == 0 && v);
#else
  if (S == 0 && (threadIdx.x & 31) == 0) slot = v ? 1 : 0;
  team_sync<G, TPC>(tm);
  return *reinterpret_cast<volatile int32_t*>(&slot) != 0;
#endif
}

template <int G, int TPC>
__device__ __forceinline__ void team_sync(const Team& tm) {
#ifndef SG_UNALIGNED_TEAM_BARRIERS
  if constexpr (TPC == 1) {
    __syncthreads();
    return;
  }
#endif
  asm volatile("barrier.cta.sync %0, %1;" ::"r"(1 + tm.id), "r"(32 * G) : "memory");
}

// One team warp. Warp 0 is the SCORER, warps 1..G-1 are PRODUCERS. Per step k
// every warp draws (or reads) its block's actions, integrates its DoFs,
// builds its partial FK transform and stages its observation columns, then
// all warps meet at ONE barrier B(k). After it, producers store the step's
// action rows and go straight on to step k+1, while the scorer turns the
// partial transforms into the tip, scores reward / hold / waypoint / flags,
// copies terminal rows, resets ended envs (reset_row through HBM) and stores
// the step's observation rows. Rows that ended at step k were reset by the
// scorer while producers already advanced them to step k+1 from the stale
// state: B(k+1) returns that fact (barrier OR), and producers redo step k+1
// for those rows from the reset state with the same actions (one extra
// barrier, one step in 300 under random actions).
template <class CH, int G, int S, int TASK, int MODE, int SUB, bool GEN, int TPC>
__device__ __forceinline__ void team_run(const StepParams& P, int k_steps, float* s_obs_base, float* s_act_base,
                                         TeamSmem<G>& ts, const Team& tm) {
  using Blk = Block<CH, G, S>;
  constexpr int NB = Blk::N > 0 ? Blk::N : 1;
  constexpr int B0 = Blk::B;
  const RobotTable& R = P.robot;
  const TaskParams& T = P.task;
  const int A = CH::dof(R);
  const int O = 3 * A + 6;
  const int task = TASK >= 0 ? TASK : T.task;
  const int mode = MODE >= 0 ? MODE : T.control_mode;
  const int substeps = SUB > 0 ? SUB : T.substeps;
  const int64_t n = T.n;
  const int lane = threadIdx.x & 31;
  const int64_t row0 = tm.row0;
  const int64_t i = row0 + lane;
  const int rows = tm.rows;
  const bool active = lane < rows;
  // runtime DoF count of this block (generic chains)
  const auto has = [&](int j) { return Blk::N > 0 && (CH::kExact || B0 + j < A); };

  float q[NB], qd[NB], qt[NB];
  const auto load_block = [&]() {
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      q[j] = qd[j] = qt[j] = 0.f;
      if (active && has(j)) {
        q[j] = P.p.q[(B0 + j) * n + i];
        qd[j] = P.p.qd[(B0 + j) * n + i];
        qt[j] = P.p.qt[(B0 + j) * n + i];
      }
    }
  };
  load_block();
  // the scorer owns the task state
  float goal[3] = {0.f, 0.f, 0.f}, tip[3] = {0.f, 0.f, 0.f};
  int32_t sc = 0, hc = 0, wi = 0, wl = 0;
  const auto load_task = [&]() {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      goal[k] = P.p.goals[k * n + i];
      tip[k] = P.p.tips[k * n + i];
    }
    sc = P.p.step_count[i];
    hc = P.p.hold_count[i];
    if (task == kTaskPath) {
      wi = P.p.wp_idx[i];
      wl = P.p.wp_len[i];
    }
  };
  if (S == 0 && active) load_task();
  uint64_t act_s = 0;
  if (GEN && active) act_s = P.p.act_state[(int64_t)S * n + i];

  // Position-control fast path (every specialised chain): the PD law with
  // dt/inertia folded into the gains, u = (kp*qt - kp*q - kd*qd) * dt/I
  // clamped to +-eff*dt/I (== clamp(tau) * dt/I), vv = qd*(1 - damping*dt/I) + u,
  // and DoF pairs advanced with packed FFMA2 (fp32 rounding differs from the
  // reference's operation order by a few ulp, inside the state tolerance).
  constexpr bool kPd = CH::kExact && MODE == kModePosition && SUB > 0 && Blk::N > 0;
  float gk[NB], gd[NB], gc[NB], ge[NB], glo[NB], ghi[NB], gvl[NB], ghalf[NB], gmid[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int d = B0 + j < kMaxDof ? B0 + j : 0;
    const float dti = R.dt_over_inertia[d];
    gk[j] = R.kp[d] * dti;
    gd[j] = R.kd[d] * dti;
    gc[j] = 1.f - R.damping[d] * dti;
    ge[j] = R.eff[d] * dti;
    glo[j] = R.lo[d];
    ghi[j] = R.hi[d];
    gvl[j] = R.vel[d];
    ghalf[j] = 0.5f * (R.hi[d] - R.lo[d]);  // rescale_to_range as one FFMA (GEN)
    gmid[j] = R.lo[d] + ghalf[j];
  }

  float a[NB];  // this step's actions (kept for a producer's redo)

  // ---- actions: the bench stream (GEN) or the caller's rows ----------------
  // GEN: the next step's draws are made one step ahead (an[], from state
  // act_pf) so the 64-bit LCG / XSH-RR chains overlap the current step's FK
  // instead of heading the next step's critical path.
  float an[NB];
  uint64_t act_pf = act_s;
  const auto prefetch = [&]() {
    if constexpr (GEN) {
      act_pf = act_s;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        an[j] = 0.f;
        if (has(j)) {  // inactive lanes (ragged last team) draw too: no divergence, never stored
          const uint64_t st = j == 0 ? act_s : act_s * P.bench.pow_mult[j] + P.bench.pow_add[j];
          const uint32_t u = pcg_output(st);
          // uniform(-1, 1) = -1 + 2 * (u * 2^-32) = (u - 2^31) * 2^-31: the exact
          // fp64 value of the reference (bench.cpp:34) rounded once to fp32
          an[j] = __int2float_rn((int32_t)(u ^ 0x80000000u)) * 0x1.0p-31f;
        }
      }
      act_s = act_s * P.bench.jump_mult + P.bench.jump_add;
    }
  };
  prefetch();
  const auto draw = [&](float* s_act) {
    if constexpr (GEN) {
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        a[j] = an[j];
        if (has(j)) s_act[lane * A + B0 + j] = a[j];
      }
    } else {
      // the caller's rows, staged once per launch (below)
#pragma unroll
      for (int j = 0; j < NB; ++j) a[j] = (active && has(j)) ? s_act_base[lane * A + B0 + j] : 0.f;
    }
  };
  if constexpr (!GEN) {
    // The team's action rows are one contiguous run: coalesced (float4 when
    // aligned) loads into shared memory, then each warp picks its DoFs (one
    // pass over PCIe when the actions are in mapped host memory). A launch
    // with caller actions applies the same rows at every step.
    const bool gate = TPC == 1 && P.p.read_gate != nullptr;
    if (gate && (int)blockIdx.x >= P.p.read_window) {
      if (tm.tthread == 0) {
        const unsigned need = blockIdx.x - P.p.read_window + 1;
        while (*reinterpret_cast<volatile unsigned*>(P.p.read_gate) < need) __nanosleep(64);
      }
      team_sync<G, TPC>(tm);
    }
    const float* src = P.actions + row0 * A;
    const int cnt = rows * A;
    if (P.actions_aligned) {
      const int n4 = cnt >> 2;
      for (int k = tm.tthread; k < n4; k += 32 * G)
        reinterpret_cast<float4*>(s_act_base)[k] = reinterpret_cast<const float4*>(src)[k];
      for (int k = (n4 << 2) + tm.tthread; k < cnt; k += 32 * G) s_act_base[k] = src[k];
    } else {
      for (int k = tm.tthread; k < cnt; k += 32 * G) s_act_base[k] = src[k];
    }
    team_sync<G, TPC>(tm);
    if (gate && tm.tthread == 0) atomicAdd(P.p.read_gate, 1u);
  }

  // ---- dynamics (dynamics.cpp:133-185) on this block; count: saturation /
  // non-finite bookkeeping (warp-collective; false on a producer's redo) ------
  const auto dynamics = [&](bool count) {
    int sat = 0, bad = 0;
    float v_target[NB], tau_cmd[NB], kpqt[NB];
    const int jaw = CH::jaw(R);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int d = B0 + j;
      v_target[j] = tau_cmd[j] = kpqt[j] = 0.f;
      if (!has(j)) continue;
      float ad = a[j];
      // generated bench actions are finite and inside [-1, 1) by construction
      // (never saturate; rescale's a <= -1 branch yields lo exactly like the
      // formula), so the GEN path skips these checks
      if (!GEN) {
        if (!isfinite(ad)) {
          bad = 1;
          ad = 0.f;
        }
        if (ad < -1.f || ad > 1.f) {
          ad = ad < -1.f ? -1.f : 1.f;
          ++sat;
        }
      }
      const float lo = R.lo[d], hi = R.hi[d];
      // GEN: a in [-1, 1) so rescale_to_range is the affine map (one FFMA;
      // fp32 rounding differs from the three-op form by <= 1 ulp)
      const auto rs = [&](float x, float l, float h) {
        return GEN ? fmaf(x, 0.5f * (h - l), l + 0.5f * (h - l)) : rescale(x, l, h);
      };
      if (mode == kModePosition) {
        qt[j] = (d == jaw) ? (ad > 0.f ? hi : lo) : (GEN ? fmaf(ad, ghalf[j], gmid[j]) : rs(ad, lo, hi));
        kpqt[j] = (kPd ? gk[j] : R.kp[d]) * qt[j];
      } else if (mode == kModeVelocity) {
        v_target[j] = rs(ad, -R.vel[d], R.vel[d]);
      } else {
        tau_cmd[j] = rs(ad, -R.eff[d], R.eff[d]);
      }
    }
    const float dt = T.dt_sub;
#ifdef SG_SAT_DYN
    if constexpr (kPd) {
      // Saturating form: the torque and velocity clamps become FFMA.SAT into
      // [0, 1] on pre-scaled gains (a clamp to [-e, e] is e * (2 sat(x / 2e + 1/2) - 1)),
      // which shortens the per-substep dependency chain from 12 to 9 ops.
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const float i2e = 0.5f / ge[j], i2v = 0.5f / gvl[j];
        const float ak = -gk[j] * i2e, ad = -gd[j] * i2e, k0 = fmaf(kpqt[j], i2e, 0.5f);
        const float bv = gc[j] * i2v, cs = ge[j] / gvl[j], c0 = 0.5f - ge[j] * i2v;
        const float v2 = 2.f * gvl[j], v2dt = v2 * dt, vdt = gvl[j] * dt;
#pragma unroll
        for (int st = 0; st < SUB; ++st) {
          const float qm = q[j] - vdt;
          const float su = __saturatef(fmaf(ad, qd[j], fmaf(ak, q[j], k0)));
          const float sv = __saturatef(fmaf(qd[j], bv, fmaf(su, cs, c0)));
          const float vv = fmaf(sv, v2, -gvl[j]);
          const float qq = fmaf(sv, v2dt, qm);
          const float qc = fminf(fmaxf(qq, glo[j]), ghi[j]);
          qd[j] = qc != qq ? 0.f : vv;
          q[j] = qc;
        }
      }
    } else
#endif
    if constexpr (kPd) {
      const auto clampf = [](float x, float l, float h) { return fminf(fmaxf(x, l), h); };
      const auto finish = [&](int j, float vv, float qq) {  // limit projection (velocity already limited)
        const float qc = clampf(qq, glo[j], ghi[j]);
        qd[j] = qc != qq ? 0.f : vv;
        q[j] = qc;
      };
#pragma unroll
      for (int s = 0; s < SUB; ++s) {
#pragma unroll
        for (int j = 0; j + 1 < NB; j += 2) {
          const int d = B0 + j;
          const float2 Q = make_float2(q[j], q[j + 1]), QD = make_float2(qd[j], qd[j + 1]);
          float2 u = __ffma2_rn(make_float2(-gk[j], -gk[j + 1]), Q, make_float2(kpqt[j], kpqt[j + 1]));
          u = __ffma2_rn(make_float2(-gd[j], -gd[j + 1]), QD, u);
          u.x = clampf(u.x, -ge[j], ge[j]);
          u.y = clampf(u.y, -ge[j + 1], ge[j + 1]);
          float2 vv = __ffma2_rn(QD, make_float2(gc[j], gc[j + 1]), u);
          vv.x = clampf(vv.x, -gvl[j], gvl[j]);
          vv.y = clampf(vv.y, -gvl[j + 1], gvl[j + 1]);
          const float2 qq = __ffma2_rn(vv, make_float2(dt, dt), Q);
          finish(j, vv.x, qq.x);
          finish(j + 1, vv.y, qq.y);
        }
        if constexpr (NB % 2 == 1) {
          constexpr int j = NB - 1;
          const int d = B0 + j;
          float u = fmaf(-gd[j], qd[j], fmaf(-gk[j], q[j], kpqt[j]));
          u = clampf(u, -ge[j], ge[j]);
          const float vv = clampf(fmaf(qd[j], gc[j], u), -gvl[j], gvl[j]);
          finish(j, vv, fmaf(vv, dt, q[j]));
        }
      }
    } else {
      // generic path: substeps outer so the block's DoFs interleave; per-DoF
      // operation order as in the reference
#pragma unroll(SUB > 0 ? SUB : 1)
      for (int s = 0; s < substeps; ++s) {
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const int d = B0 + j;
          if (!has(j)) continue;
          const float ef = R.eff[d], vl = R.vel[d];
          float tau;
          if (mode == kModePosition) tau = fmaf(-R.kd[d], qd[j], fmaf(-R.kp[d], q[j], kpqt[j]));
          else if (mode == kModeVelocity) tau = R.kd[d] * (v_target[j] - qd[j]);
          else tau = tau_cmd[j];
          tau = fminf(fmaxf(tau, -ef), ef);
          float vv = qd[j] + (tau - R.damping[d] * qd[j]) * R.dt_over_inertia[d];
          vv = fminf(fmaxf(vv, -vl), vl);
          const float qq = q[j] + vv * dt;
          const float qc = fminf(fmaxf(qq, R.lo[d]), R.hi[d]);  // limit projection
          qd[j] = qc != qq ? 0.f : vv;
          q[j] = qc;
        }
      }
    }
    if (!GEN && count) {
      if (!active) sat = bad = 0;
      const unsigned wsat = __reduce_add_sync(0xffffffffu, (unsigned)sat);
      if (wsat && lane == 0) {
        atomicAdd(P.p.sat_total, (unsigned long long)wsat);
        if (P.p.sat_step) atomicAdd(P.p.sat_step, (unsigned long long)wsat);
      }
      if (__any_sync(0xffffffffu, bad) && bad) atomicOr(P.p.err, kErrNonFiniteAction);
    }
  };

  // ---- partial FK of this block + publication ---------------------------------
  // tip = T_0 o T_1 o ... o T_{G-1} (tip offset), evaluated right to left as
  // matrix-vector products: the last warp publishes v = p + R * tip (3 floats;
  // its final rotation is dead code when the tip offset is zero), middle warps
  // publish (R, p), the scorer applies them to its own transform.
  // With a non-zero tool-tip offset (ECM, STAR) the last warp of a
  // FixedChain team (S = G - 1) uses the right-to-left point form: it maps
  // the tip point through its joints (no rotation matrix composed) and
  // publishes it; the scorer keeps the left-to-right transform of its own
  // joints, built before the barrier, and applies it after. With a zero tip
  // offset (PSM) the left-to-right form already drops the last rotation and
  // measured faster (tools/ab.sh: ECM 33.9 -> 35.4 G env-steps/s, STAR
  // unchanged, PSM 23.2 -> 22.2 with the point form).
  constexpr bool kPoint = CH::kExact && CH::kTipFlags != 0 && G >= 2 && S == G - 1 && Blk::N > 0;
  Xform x;
  const auto publish = [&](int b, float* s_obs) {
    if constexpr (kPoint) {
      float psn[NB], pcs[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) __sincosf(q[j], &psn[j], &pcs[j]);
      float v[3] = {(CH::kTipFlags & 1) ? R.tip[0] : 0.f, (CH::kTipFlags & 2) ? R.tip[1] : 0.f,
                    (CH::kTipFlags & 4) ? R.tip[2] : 0.f};
      point_range<CH, B0, Blk::N>(R, q, psn, pcs, v);
#pragma unroll
      for (int k = 0; k < 3; ++k) ts.xf[b][S][9 + k][lane] = v[k];
    } else {
#pragma unroll
    for (int k = 0; k < 9; ++k) x.m[k] = (k % 4 == 0) ? 1.f : 0.f;
    x.p[0] = x.p[1] = x.p[2] = 0.f;
    fk_range<CH, B0>(R, q, x, std::make_integer_sequence<int, Blk::N>{});
    }
    if (kPoint) {
    } else if (S > 0 && S == G - 1) {
      float v[3];
      fk_tip_offset(R, tip_flags_of<CH>(R), x.m, x.p, v);
#pragma unroll
      for (int k = 0; k < 3; ++k) ts.xf[b][S][9 + k][lane] = v[k];
    } else if (S > 0) {
#pragma unroll
      for (int k = 0; k < 9; ++k) ts.xf[b][S][k][lane] = x.m[k];
#pragma unroll
      for (int k = 0; k < 3; ++k) ts.xf[b][S][9 + k][lane] = x.p[k];
    }
    {  // (inactive lanes stage rows past `rows`, never stored)
      float* o = s_obs + lane * O;
#pragma unroll
      for (int j = 0; j < NB; ++j)
        if (has(j)) {
          o[B0 + j] = q[j];
          o[A + B0 + j] = qd[j];
          o[2 * A + 3 + B0 + j] = qt[j];
        }
    }
  };

  // Observation rows live in kOB buffers: step k stages into buffer k % kOB.
  // kProdRows (G > 1): the producers store step k's rows after B(k+1) (the
  // scorer has finished staging them by then); else the scorer stores them
  // right after scoring (G == 1: together with the generated action rows).
  constexpr int kOB = team_obs_bufs<G>();
  constexpr bool kProdRows = kOB == 3;
  const auto obs_buf = [&](int st) { return s_obs_base + (st % kOB) * (kTeamEnvs * O); };
  const auto store_rows = [&](int st) {
    const float* so = obs_buf(st);
    constexpr int NT = kProdRows ? (G - 1) * 32 : 32;
    const int t = kProdRows ? tm.tthread - 32 : lane;
    if constexpr (GEN && G == 1)
      team_store<CH, kTeamEnvs * CH::kDof, 32>(P.p.act_buf + row0 * A, s_act_base + (st & 1) * (kTeamEnvs * A + 4),
                                               rows * A, (rows & 3) == 0, lane);
    team_store<CH, kTeamEnvs * (3 * CH::kDof + 6), NT>(P.p.obs + row0 * O, so, rows * O, (rows & 3) == 0, t);
    if constexpr (!GEN) {
      if (P.p.h_obs)
        team_store<CH, kTeamEnvs * (3 * CH::kDof + 6), NT>(P.p.h_obs + row0 * O, so, rows * O, (rows & 3) == 0, t);
    }
  };

  // Rows that ended at step k (pb = parity of k) are reset by the WHOLE team
  // (env lane l by warp l % G: reset_row is fp64-heavy, PathFollowing most of
  // all), after which the scorer re-observes them (and, without producer row
  // stores, stores step k's rows).
  const auto reset_phase = [&](int k) {
    const int pb = k & 1;
#ifdef SG_RESET_FULLWARP
    if (active && ts.ended[pb][lane] && (int)(blockIdx.x % G) == S) {
#else
    if (active && ts.ended[pb][lane] && (lane % G) == S) {
#endif
      const int e = reset_env<CH, TASK>(P, i);  // reset_row (envs.cpp:304-360) through HBM
      if (e) atomicOr(P.p.err, e);
    }
    team_sync<G, TPC>(tm);
    if constexpr (S == 0) {
      float* so = obs_buf(k);
      if (active && ts.ended[pb][lane]) {  // the post-reset observation row
        load_block();
        load_task();
        float* o = so + lane * O;
#pragma unroll
        for (int d = 0; d < CH::kDof; ++d)
          if (CH::kExact || d < A) {
            o[d] = P.p.q[d * n + i];
            o[A + d] = P.p.qd[d * n + i];
            o[2 * A + 3 + d] = P.p.qt[d * n + i];
          }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          o[2 * A + k] = tip[k];
          o[3 * A + 3 + k] = goal[k];
        }
      }
      __syncwarp();
      if constexpr (!kProdRows) store_rows(k);
    }
  };

  bool pend = false;  // scorer: rows ended at the previous step (reset pending)
#ifdef SG_TIME_PROBE
  if (lane == 0) atomicMin(&g_tprobe[1], globaltimer_ns());  // state loaded, first step begins
#endif
#ifdef SG_PHASE_PROBE
  long long t_prod = 0, t_bar = 0, t_post = 0, t_mark = clock64();
#define SG_MARK(acc)                    \
  do {                                  \
    const long long now_ = clock64();   \
    acc += now_ - t_mark;               \
    t_mark = now_;                      \
  } while (0)
#else
#define SG_MARK(acc) \
  do {               \
  } while (0)
#endif
  for (int step = 0; step < k_steps; ++step) {
    const int b = step & 1;
    float* s_obs = obs_buf(step);
    float* s_act = s_act_base + b * (kTeamEnvs * A + 4);
    if (!(S == 0 && pend)) {  // a scorer with pending resets produces after them
      draw(s_act);
      dynamics(true);
      prefetch();
      publish(b, s_obs);
    }
    SG_MARK(t_prod);
    // B(step); its OR says rows of step-1 ended: reset them as a team, then the
    // scorer produces this step and producers redo it for the reset rows
    const bool any_end = team_sync_flag<G, TPC, S>(tm, ts.any_end[b], pend);
    SG_MARK(t_bar);
    if (any_end) {
      reset_phase(step - 1);
      if constexpr (S == 0) {
        draw(s_act);
        dynamics(true);
        prefetch();
        publish(b, s_obs);
        pend = false;
      } else {
        if (active && ts.ended[b ^ 1][lane]) {  // redo this step from the reset state
          load_block();
          dynamics(false);
          publish(b, s_obs);
        }
      }
      team_sync<G, TPC>(tm);
    }

    if constexpr (S > 0) {
      // producers store the previous step's observation rows (staged and, after
      // a reset phase, re-observed by the scorer) and this step's generated
      // action rows, then move on
      if (kProdRows && step > 0) store_rows(step - 1);
      if (GEN)
        team_store<CH, kTeamEnvs * CH::kDof, (G - 1) * 32>(P.p.act_buf + row0 * A, s_act, rows * A,
                                                          (rows & 3) == 0, tm.tthread - 32);
    } else {
      // ---- scorer: tip, reward, flags (envs.cpp:456-463, 478-593) -----------
      float v[3];
      if constexpr (G == 1) {
        fk_tip_offset(R, tip_flags_of<CH>(R), x.m, x.p, v);
      } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) v[k] = ts.xf[b][G - 1][9 + k][lane];
#pragma unroll
        for (int s = G - 2; s >= 1; --s) {
          float y[12];
#pragma unroll
          for (int k = 0; k < 12; ++k) y[k] = ts.xf[b][s][k][lane];
          apply_xform(y, y + 9, v);
        }
        apply_xform(x.m, x.p, v);
      }
      bool ended = false;
      float* o = s_obs + lane * O;
      {  // computed on every lane (no divergence); global side effects on active lanes only
        tip[0] = v[0];
        tip[1] = v[1];
        tip[2] = v[2];
        sc += 1;
        float reward, dist;
        bool goal_met;
        {
          const float dx = tip[0] - goal[0], dy = tip[1] - goal[1], dz = tip[2] - goal[2];
          dist = sqrtf(dx * dx + dy * dy + dz * dz);
        }
        if (task == kTaskPath) {
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
        } else if (task == kTaskTrack) {
          // ActiveTracking (envs.cpp:493-512): scored against the current
          // goal, which then drifts (env stream, 2 u32 per normal)
          reward = T.rho * dist;
          goal_met = false;
          if (active) track_drift(P, i, goal);
        } else {
          reward = T.rho * dist;
          hc = dist < T.success_radius ? hc + 1 : 0;
          goal_met = hc >= T.success_hold;
        }
        const bool timed_out = sc >= T.episode_len;
        if (active) {
          if (!isfinite(reward)) atomicOr(P.p.err, kErrNonFiniteReward);
          P.p.rewards[i] = reward;
          P.p.task_error[i] = dist;
          P.p.terminated[i] = goal_met ? 1 : 0;
          P.p.timed_out[i] = timed_out ? 1 : 0;
          if constexpr (!GEN) {
            if (P.p.h_rewards) P.p.h_rewards[i] = reward;
            if (P.p.h_task_error) P.p.h_task_error[i] = dist;
            if (P.p.h_terminated) P.p.h_terminated[i] = goal_met ? 1 : 0;
            if (P.p.h_timed_out) P.p.h_timed_out[i] = timed_out ? 1 : 0;
          }
        }
        ended = active && (goal_met || timed_out);
        o[2 * A + 0] = tip[0];
        o[2 * A + 1] = tip[1];
        o[2 * A + 2] = tip[2];
        o[3 * A + 3] = goal[0];
        o[3 * A + 4] = goal[1];
        o[3 * A + 5] = goal[2];
      }
      ts.ended[b][lane] = ended;
      const unsigned em = __ballot_sync(0xffffffffu, ended);
      pend = em != 0;
      __syncwarp();  // staged columns, tip / goal and ended flags are complete
      if (pend) {
        if (lane == 0) atomicAdd(P.p.ended_total, (unsigned long long)__popc(em));
        // terminal observations (envs.cpp:606-611): the pre-reset rows; the
        // step's observation rows are stored after the team reset phase
        for (int r = 0; r < rows; ++r) {
          if (!((em >> r) & 1u)) continue;
          for (int k = lane; k < O; k += 32) {
            P.p.tobs[(row0 + r) * O + k] = s_obs[r * O + k];
            if constexpr (!GEN) {
              if (P.p.h_tobs) P.p.h_tobs[(row0 + r) * O + k] = s_obs[r * O + k];
            }
          }
        }
      } else if constexpr (!kProdRows) {
        store_rows(step);
      }
    }
    SG_MARK(t_post);
#ifdef SG_TIME_PROBE
    if (step == 0 && lane == 0) atomicMax(&g_tprobe[2], globaltimer_ns());
#endif
  }
#ifdef SG_TIME_PROBE
  if (lane == 0) {
    atomicMin(&g_tprobe[3], globaltimer_ns());  // first team through all steps
    atomicMax(&g_tprobe[4], globaltimer_ns());  // last team through all steps
  }
#endif
#ifdef SG_PHASE_PROBE
  if (blockIdx.x < 3 && lane == 0)
    printf("probe cta %d warp %d: produce %lld barrier %lld post %lld cycles over %d steps\n", (int)blockIdx.x, S,
           t_prod, t_bar, t_post, k_steps);
#endif
#undef SG_MARK
  // rows that ended at the last step: team reset, then the last step's rows
  // are stored (by the producers once the scorer has re-observed the reset
  // rows); the producers' registers of reset rows are stale (the reset state
  // is already in HBM)
  const bool fix = team_sync_flag<G, TPC, S>(tm, ts.any_end[k_steps & 1], pend);
  if (fix) reset_phase(k_steps - 1);
  if constexpr (kProdRows) {
    if (fix) team_sync<G, TPC>(tm);
    if (S > 0) store_rows(k_steps - 1);
  }
  const bool stale = S > 0 && fix && ts.ended[(k_steps - 1) & 1][lane];
  if (active) {
    if (!stale) {
#pragma unroll
      for (int j = 0; j < NB; ++j)
        if (has(j)) {
          P.p.q[(B0 + j) * n + i] = q[j];
          P.p.qd[(B0 + j) * n + i] = qd[j];
          P.p.qt[(B0 + j) * n + i] = qt[j];
        }
    }
    if (S == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        P.p.goals[k * n + i] = goal[k];
        P.p.tips[k * n + i] = tip[k];
      }
      P.p.step_count[i] = sc;
      P.p.hold_count[i] = hc;
      if (task == kTaskPath) {
        P.p.wp_idx[i] = wi;
        P.p.wp_len[i] = wl;
      }
    }
    if (GEN) P.p.act_state[(int64_t)S * n + i] = act_pf;  // the drawn-ahead step was not consumed
  }
}

template <class CH, int G, int TASK, int MODE, int SUB, bool GEN, int TPC, int... S>
__device__ __forceinline__ void team_dispatch(const StepParams& P, int k_steps, float* s_obs, float* s_act,
                                              TeamSmem<G>& ts, const Team& tm, int role,
                                              std::integer_sequence<int, S...>) {
  ((role == S ? team_run<CH, G, S, TASK, MODE, SUB, GEN, TPC>(P, k_steps, s_obs, s_act, ts, tm) : void()), ...);
}

// MINB: CTAs per SM the register budget targets. 1 (no cap: ~156 registers,
// 6 two-warp teams per SM) unless the launch has more teams than the GPU holds
// at once; then 8 (128 registers): ECM at 65,536 envs is 2,048 teams, three
// partial waves at 6 per SM and two at 8 (tools/ab.sh: +6.5 %; the cap costs
// 8-9 % when every team is resident anyway, PSM / STAR at 16,384 envs).
//
// TPC: teams per CTA (1, or 4 for the packed one-CTA-per-SM layout). Warp w
// has role w / TPC (0 = scorer) in team (w % TPC + role) % TPC, so every SM
// sub-partition (warp slot % 4) hosts one warp of each role: the scorer and
// producer instruction streams differ in length, and with one two-warp team
// per CTA all producers of an SM shared two sub-partitions.
template <class CH, int G, int TASK, int MODE, int SUB, bool GEN, int MINB = 1, int TPC = 1>
__global__ void __launch_bounds__(32 * G * TPC, MINB) env_step_kernel(const __grid_constant__ StepParams P,
                                                                      int k_steps) {
  extern __shared__ __align__(16) float smem[];
  // a kernel launched after this one with programmatic stream serialization
  // (the policy forward of the next rollout step) may be scheduled as SMs
  // free up; its griddepcontrol.wait still waits for this grid's completion
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int A = CH::dof(P.robot);
  const int O = 3 * A + 6;
  const int64_t n = P.task.n;
  const int w = threadIdx.x >> 5;
  int role = w / TPC;
#ifdef SG_ROLE_SPREAD
  if constexpr (TPC == 1 && G == 2) {
    // Roles by SM sub-partition (warp slot % 4): the scorer and producer
    // instruction streams differ in length, and with warp 0 always the scorer
    // every SM's scorers share two sub-partitions. Team pair slot t = lower
    // slot / 2 puts its scorer on sub-partition {0, 3, 1, 2}[t % 4], so each
    // sub-partition hosts scorers and producers alike. Only the role choice
    // depends on the (hardware-assigned) slots; both warps agree through smem.
    __shared__ int s_slot[2];
    uint32_t wid;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    if ((threadIdx.x & 31) == 0) s_slot[w] = (int)wid;
    __syncthreads();
    const int lo = min(s_slot[0], s_slot[1]);
    const int pref = (0x2130 >> (4 * ((lo >> 1) & 3))) & 3;  // {0, 3, 1, 2}[t % 4]
    const int scorer = (s_slot[1] & 3) == pref && (s_slot[0] & 3) != pref ? 1 : 0;
    role = w == scorer ? 0 : 1;
  }
#endif
  Team tm;
  tm.id = (w % TPC + role) % TPC;
  tm.tthread = role * 32 + (threadIdx.x & 31);
  if constexpr (TPC == 1) {
    tm.row0 = (int64_t)blockIdx.x * kTeamEnvs;
    tm.rows = (int)min((int64_t)kTeamEnvs, n - tm.row0);
  } else {
#ifdef SG_PACKED32
    // full 32-env teams, 3 or 4 per CTA (SM): the legacy layout's rows with
    // the packed layout's role placement
    const int64_t teams = (n + kTeamEnvs - 1) / kTeamEnvs;
    const int64_t t0 = (int64_t)blockIdx.x * teams / gridDim.x, t1 = ((int64_t)blockIdx.x + 1) * teams / gridDim.x;
    const int64_t g = t0 + tm.id;
    tm.row0 = g * kTeamEnvs;
    tm.rows = g < t1 ? (int)min((int64_t)kTeamEnvs, n - tm.row0) : 0;
#else
    const int64_t quads = (n + 3) / 4, teams = (int64_t)gridDim.x * TPC;
    const int64_t g = (int64_t)blockIdx.x * TPC + tm.id;
    const int64_t q0 = g * quads / teams, q1 = (g + 1) * quads / teams;
    tm.row0 = 4 * q0;
    tm.rows = (int)(min(4 * q1, n) - tm.row0);
#endif
  }
  float* base = smem + tm.id * (team_smem_bytes_g<G>(A) / sizeof(float));
  TeamSmem<G>& ts = *reinterpret_cast<TeamSmem<G>*>(base);
  float* s_obs = base + (sizeof(TeamSmem<G>) + 15) / 16 * 4;  // team_obs_bufs x 32 x O
  float* s_act = s_obs + team_obs_bufs<G>() * kTeamEnvs * O;  // 2 x (32 x A + 4)
  if (P.p.ended_clear && blockIdx.x == 0 && threadIdx.x == 0) {
    *P.p.ended_clear = 0;
    if (P.p.sat_clear) *P.p.sat_clear = 0;
  }
#ifdef SG_TIME_PROBE
  if (threadIdx.x == 0) atomicMin(&g_tprobe[0], globaltimer_ns());
#endif
  if (tm.rows > 0)
    team_dispatch<CH, G, TASK, MODE, SUB, GEN, TPC>(P, k_steps, s_obs, s_act, ts, tm, role,
                                                    std::make_integer_sequence<int, G>{});
#ifdef SG_TIME_PROBE
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMax(&g_tprobe[5], globaltimer_ns());
    __threadfence();
    if (atomicAdd(&g_tprobe_ticket, 1u) == gridDim.x - 1) {
      __threadfence();
      volatile unsigned long long* t = g_tprobe;
      if (k_steps > 1)
        printf("tprobe K=%d: loads %.2f us, step0 %.2f us, loop %.2f..%.2f us, end %.2f us (from first CTA start)\n",
               k_steps, (t[1] - t[0]) * 1e-3, (t[2] - t[0]) * 1e-3, (t[3] - t[0]) * 1e-3, (t[4] - t[0]) * 1e-3,
               (t[5] - t[0]) * 1e-3);
      t[0] = t[1] = t[3] = ~0ull;
      t[2] = t[4] = t[5] = 0;
      g_tprobe_ticket = 0;
    }
  }
#endif
  if (P.p.h_status) {  // host step: the last CTA to finish publishes the counters
    // every thread's zero-copy result rows are ordered before the CTA's ticket,
    // so the host may read them as soon as it sees h_status[3] == h_seq
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && P.p.chunk_flag) {  // this team's rows are in HBM: count it into its chunk
      const unsigned c = blockIdx.x / P.p.chunk_teams;
      const unsigned in_chunk = min((unsigned)P.p.chunk_teams, gridDim.x - c * P.p.chunk_teams);
      if (atomicAdd(&P.p.chunk_count[c], 1u) == in_chunk - 1) {
        P.p.chunk_count[c] = 0;
        __threadfence_system();
        atomicExch(&P.p.chunk_flag[c], (unsigned)P.p.h_seq);
      }
    }
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(P.p.ticket, 1u) == gridDim.x - 1) {
        __threadfence();
        volatile unsigned long long* hs = P.p.h_status;
        hs[0] = *reinterpret_cast<volatile unsigned long long*>(P.p.sat_step ? P.p.sat_step : P.p.sat_total);
        hs[1] = *reinterpret_cast<volatile unsigned long long*>(P.p.ended_total);
        hs[2] = static_cast<unsigned long long>(static_cast<uint32_t>(*reinterpret_cast<volatile int32_t*>(P.p.err)));
        __threadfence_system();
        hs[3] = P.p.h_seq;
        *P.p.ticket = 0;
        if (P.p.read_gate) *P.p.read_gate = 0;
      }
    }
  }
}


// reset() (envs.cpp:425-435): every row through reset_row, episode_count := 0,
// observe, clear flags and rewards.
template <class CH, int TASK>
__global__ void __launch_bounds__(128) env_reset_kernel(const __grid_constant__ StepParams P) {
  constexpr int D = CH::kDof;
  extern __shared__ __align__(16) float smem[];
  const RobotTable& R = P.robot;
  const TaskParams& T = P.task;
  const int A = CH::dof(R);
  const int O = 3 * A + 6;
  const int64_t n = T.n;
  const int64_t row0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t i = row0 + threadIdx.x;
  const int rows = (int)min((int64_t)blockDim.x, n - row0);
  if (i < n) {
    float q[D], qd[D], qt[D], goal[3], tip[3];
    int32_t wi = 0, wl = 0;
    const int e = reset_env<CH, TASK>(P, i);
    if (e) atomicOr(P.p.err, e);
    load_env<CH, TASK>(P, i, q, qd, qt, goal, tip, wi, wl);
    P.p.episode_count[i] = 0;
    P.p.terminated[i] = 0;
    P.p.timed_out[i] = 0;
    P.p.rewards[i] = 0.f;
    float* o = smem + threadIdx.x * O;
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (d < A) {
        o[d] = q[d];
        o[A + d] = qd[d];
        o[2 * A + 3 + d] = qt[d];
      }
    for (int k = 0; k < 3; ++k) {
      o[2 * A + k] = tip[k];
      o[3 * A + 3 + k] = goal[k];
    }
  }
  __syncthreads();
  block_store(P.p.obs + row0 * O, smem, rows * O);
}

// Host-side launch plumbing: one translation unit per chain instantiates its
// kernels (parallel compilation) and exposes a launcher.
constexpr int kResetBlock = 64;

// Team layout of a launch: one 32-env team per CTA (kLayoutAuto / Legacy), or
// the packed one-CTA-per-SM layout (TPC = 4 teams per CTA, env quads spread
// evenly, roles spread over the SM sub-partitions) when SG_TEAM_LAYOUT=packed.
// Packed balances issue across sub-partitions exactly but measured slower
// (PSM 16K: 192 vs 172 us per 250-step launch): the kernel is bound by the
// per-team step latency, not by issue.
enum TeamLayout : int { kLayoutAuto = 0, kLayoutLegacy = 1, kLayoutPacked = 2 };
constexpr int kPackedTeams = 4;

inline int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

template <class CH, int TASK, int MODE, int SUB, int G>
inline cudaError_t launch_team(const StepParams& P, int k_steps, bool gen, cudaStream_t st, int layout = kLayoutAuto) {
  if constexpr (CH::kExact && G == 2) {
    const int64_t sms = sm_count();
    const int64_t n = P.task.n;
    const bool fits = n <= sms * kTeamEnvs * kPackedTeams;
    if (fits && layout == kLayoutPacked) {
      constexpr int TPC = kPackedTeams;
      const size_t sm = TPC * team_smem_bytes<G>(P.robot.dof);
      cudaError_t e = cudaFuncSetAttribute(env_step_kernel<CH, G, TASK, MODE, SUB, true, 1, TPC>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(env_step_kernel<CH, G, TASK, MODE, SUB, false, 1, TPC>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      const unsigned grid = (unsigned)sms;
      if (gen) env_step_kernel<CH, G, TASK, MODE, SUB, true, 1, TPC><<<grid, 32 * G * TPC, sm, st>>>(P, k_steps);
      else env_step_kernel<CH, G, TASK, MODE, SUB, false, 1, TPC><<<grid, 32 * G * TPC, sm, st>>>(P, k_steps);
      return cudaGetLastError();
    }
  }
  const unsigned grid = (unsigned)((P.task.n + kTeamEnvs - 1) / kTeamEnvs);
  const size_t sm = team_smem_bytes<G>(P.robot.dof);
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(env_step_kernel<CH, G, TASK, MODE, SUB, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(env_step_kernel<CH, G, TASK, MODE, SUB, false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  if constexpr (CH::kExact && G == 2) {
    // more teams than resident slots at the uncapped register count: the
    // 8-CTAs-per-SM build (fewer, fuller waves)
    static int slots = -1;
    if (slots < 0) {
      int dev = 0, sms = 0, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, env_step_kernel<CH, G, TASK, MODE, SUB, true>, 32 * G,
                                                    sm);
      slots = sms * per_sm;
    }
    if ((int64_t)grid > slots) {
      if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(env_step_kernel<CH, G, TASK, MODE, SUB, true, 8>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(env_step_kernel<CH, G, TASK, MODE, SUB, false, 8>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
      }
      if (gen) env_step_kernel<CH, G, TASK, MODE, SUB, true, 8><<<grid, 32 * G, sm, st>>>(P, k_steps);
      else env_step_kernel<CH, G, TASK, MODE, SUB, false, 8><<<grid, 32 * G, sm, st>>>(P, k_steps);
      return cudaGetLastError();
    }
  }
  if (gen) env_step_kernel<CH, G, TASK, MODE, SUB, true><<<grid, 32 * G, sm, st>>>(P, k_steps);
  else env_step_kernel<CH, G, TASK, MODE, SUB, false><<<grid, 32 * G, sm, st>>>(P, k_steps);
  return cudaGetLastError();
}

template <class CH, int TASK>
inline cudaError_t launch_reset(const StepParams& P, cudaStream_t st) {
  const unsigned grid = (unsigned)((P.task.n + kResetBlock - 1) / kResetBlock);
  const size_t sm = (size_t)kResetBlock * (3 * P.robot.dof + 6) * sizeof(float);
  env_reset_kernel<CH, TASK><<<grid, kResetBlock, sm, st>>>(P);
  return cudaGetLastError();
}

// Positions the per-env bench action stream at draw (first_step*G + g)*A,
// g = row_offset + i (jump-ahead, O(log k) table of PCG32 powers).
struct JumpTable {
  uint64_t mult[64];
  uint64_t add[64];
};

static __global__ void bench_seed_kernel(uint64_t* act_state, int64_t n, uint64_t base_state, uint64_t first_draw,
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
  GenericChain<DMAX>::fk(R, q, tip);
  pos[i * 3 + 0] = tip[0];
  pos[i * 3 + 1] = tip[1];
  pos[i * 3 + 2] = tip[2];
}

}  // namespace sg
