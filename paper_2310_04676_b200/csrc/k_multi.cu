// MultiToolReaching step / reset kernels (multi.cuh). The step kernel is a
// team of T warps per 32 envs, warp t = tool t (lane = env): the tool's joint
// state (DoF-major SoA in HBM, one 128-byte line per DoF per warp) stays in
// registers for the whole fused launch, is integrated with the reference's
// per-DoF PD law (dynamics.cpp:127-185; position control on a specialised
// chain with dt / inertia folded into the gains like the single-tool
// kernels), and the tool FK (robot_model.cpp:371-395, on the tool's
// compile-time chain structure when it has one) is mapped through the tool's
// base pose. Warp 0 scores; observation rows are staged in shared memory and
// stored as one contiguous float4 run per team. The reset kernel stages one
// warp's 32 rows per warp (odd row stride Os: conflict-free).
#include "multi.cuh"
#include "launch.hpp"

namespace sg {
namespace {

// sample_goal (envs.cpp:230-239) around the tool's own workspace centre, z
// drawn first (g++ argument order), fp64 without FMA contraction.
__device__ __forceinline__ bool mt_sample_goal(uint64_t& s, uint64_t inc, double sigma, double radius,
                                               const double (&c)[3], double (&g)[3]) {
  for (int attempt = 0; attempt < kGoalRejectionLimit; ++attempt) {
    const double nz = __dmul_rn(sigma, pcg_normal(s, inc));
    const double ny = __dmul_rn(sigma, pcg_normal(s, inc));
    const double nx = __dmul_rn(sigma, pcg_normal(s, inc));
    g[0] = __dadd_rn(c[0], nx);
    g[1] = __dadd_rn(c[1], ny);
    g[2] = __dadd_rn(c[2], nz);
    if (norm3_rn(__dadd_rn(g[0], -c[0]), __dadd_rn(g[1], -c[1]), __dadd_rn(g[2], -c[2])) <= radius) return true;
  }
  return false;
}

// Tool FK: world tip = base_p + base_R * (p + m * tip); the camera axis
// (tips_[t].orientation * (0, 0, -1), envs.cpp:556-557) = base_R * (m * view).
// CH: the tool's compile-time chain structure (FixedChain: no runtime joint
// branches, no sin/cos range reduction) or GenericChain<kMaxToolDof>.
template <class CH = GenericChain<kMaxToolDof>>
__device__ __forceinline__ void tool_fk(const ToolEnc& E, const float (&q)[kMaxToolDof], float (&tip)[3],
                                        float (&axis)[3]) {
  const RobotTable& R = E.robot;
  float m[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
  float p[3] = {0.f, 0.f, 0.f};
  float t[3];
  if constexpr (CH::kExact) {
    CH::walk(R, reinterpret_cast<const float(&)[CH::kDof]>(q), m, p, std::make_integer_sequence<int, CH::kDof>{});
    fk_tip_offset(R, CH::kTipFlags, m, p, t);
  } else {
#pragma unroll
    for (int d = 0; d < kMaxToolDof; ++d) {
      if (d >= R.dof) break;
      const JointEnc& J = R.j[d];
      fk_joint(J, J.kind, J.axis_code, J.flags & 7, (J.flags >> 3) & 1, q[d], m, p);
    }
    fk_tip_offset(R, R.tip_flags, m, p, t);
  }
#pragma unroll
  for (int r = 0; r < 3; ++r)
    tip[r] = E.base_p[r] + E.base_R[r * 3 + 0] * t[0] + E.base_R[r * 3 + 1] * t[1] + E.base_R[r * 3 + 2] * t[2];
  if (E.camera) {
    float v[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) v[r] = m[r * 3 + 0] * E.view[0] + m[r * 3 + 1] * E.view[1] + m[r * 3 + 2] * E.view[2];
#pragma unroll
    for (int r = 0; r < 3; ++r)
      axis[r] = E.base_R[r * 3 + 0] * v[0] + E.base_R[r * 3 + 1] * v[1] + E.base_R[r * 3 + 2] * v[2];
  } else {
    axis[0] = axis[1] = axis[2] = 0.f;
  }
}

// Camera goal: midpoint of the other tools' tips (envs.cpp:339-348, 547-555):
// sum in tool order, then divide by the count.
template <int T>
__device__ __forceinline__ void camera_mid(const float (&tw)[T][3], int t, float (&mid)[3]) {
  mid[0] = mid[1] = mid[2] = 0.f;
#pragma unroll
  for (int u = 0; u < T; ++u) {
    if (u == t) continue;
#pragma unroll
    for (int k = 0; k < 3; ++k) mid[k] += tw[u][k];
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) mid[k] = mid[k] / (float)(T - 1);
}

// Observation row of env i from its HBM state (observe_rows, envs.cpp:362-408)
// into the lane's staging row.
template <int T>
__device__ __forceinline__ void stage_row_from_state(const MtParams& P, int64_t i, float* o) {
  const int64_t n = P.n;
  const int A = P.A;
  for (int c = 0; c < A; ++c) {
    o[c] = P.q[c * n + i];
    o[A + c] = P.qd[c * n + i];
    o[2 * A + 3 * T + c] = P.qt[c * n + i];
  }
#pragma unroll
  for (int k = 0; k < 3 * T; ++k) {
    o[2 * A + k] = P.tips[k * n + i];
    o[3 * A + 3 * T + k] = P.goals[k * n + i];
  }
}

// reset_row (envs.cpp:304-360) for one env, through HBM. Returns error bits.
template <int T>
__device__ __noinline__ int mt_reset_env(const MtParams& P, int64_t i) {
  const int64_t n = P.n;
  uint64_t s[T], inc[T];
  float tw[T][3];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const ToolEnc& E = P.tool[t];
    const RobotTable& R = E.robot;
    s[t] = P.rng_state[t * n + i];
    inc[t] = P.rng_inc[t * n + i];
    float q[kMaxToolDof];
#pragma unroll
    for (int d = 0; d < kMaxToolDof; ++d) {
      q[d] = 0.f;
      if (d < R.dof) {
        const double quarter = __dmul_rn(0.25, __dadd_rn(R.hi_d[d], -R.lo_d[d]));
        q[d] = (float)pcg_uniform(s[t], inc[t], __dadd_rn(R.lo_d[d], quarter), __dadd_rn(R.hi_d[d], -quarter));
        const int64_t c = E.off + d;
        P.q[c * n + i] = q[d];
        P.qd[c * n + i] = 0.f;
        P.qt[c * n + i] = q[d];
      }
    }
    float ax[3];
    tool_fk(E, q, tw[t], ax);
  }
  int err = 0;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const ToolEnc& E = P.tool[t];
    float g[3];
    if (E.camera) {
      camera_mid<T>(tw, t, g);
    } else {
      const double c[3] = {E.center[0], E.center[1], E.center[2]};
      double gd[3];
      if (!mt_sample_goal(s[t], inc[t], P.goal_sigma, P.radius, c, gd)) err |= kErrGoalSampling;
      g[0] = (float)gd[0];
      g[1] = (float)gd[1];
      g[2] = (float)gd[2];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      P.goals[(3 * t + k) * n + i] = g[k];
      P.tips[(3 * t + k) * n + i] = tw[t][k];
    }
    P.rng_state[t * n + i] = s[t];
  }
  P.step_count[i] = 0;
  P.hold_count[i] = 0;
  P.episode_count[i] += 1;
  return err;
}

// Warp store of `rows` staged rows (stride Os) to row-major global rows.
__device__ __forceinline__ void warp_store_rows(float* __restrict__ g, const float* __restrict__ s, int rows, int O,
                                                int Os, int lane) {
  for (int r = 0; r < rows; ++r)
    for (int c = lane; c < O; c += 32) g[(int64_t)r * O + c] = s[r * Os + c];
}

// Team shared memory (double-buffered by step parity where a buffer is read
// after the step's last barrier).
template <int T>
struct MtSmem {
  float tip[2][T][3][32];  // world tips, lane-contiguous
  float ax[2][T][3][32];   // camera axes
  uint32_t ended[2];
};

// One tool's step for the team's 32 envs (warp t = tool t). All tool warps
// run the SAME code with t a warp-uniform runtime index into the parameter
// block (per-tool code paths thrash the instruction cache: ncu showed
// `no_instructions` as the top stall with a compile-time tool index).
// State lives in registers for the whole launch.
struct ToolState {
  float q[kMaxToolDof], qd[kMaxToolDof], qt[kMaxToolDof];
  uint64_t act_s = 0;  // GEN: stream state at the env's row start
};

template <int T, bool GEN>
struct ToolWarp {

  __device__ __forceinline__ static void load(ToolState& S, const MtParams& P, const ToolEnc& E, int64_t i, bool active) {
    float (&q)[kMaxToolDof] = S.q;
    float (&qd)[kMaxToolDof] = S.qd;
    float (&qt)[kMaxToolDof] = S.qt;
    const int64_t n = P.n;
#pragma unroll
    for (int d = 0; d < kMaxToolDof; ++d) {
      q[d] = qd[d] = qt[d] = 0.f;
      if (d < E.robot.dof && active) {
        q[d] = P.q[(E.off + d) * n + i];
        qd[d] = P.qd[(E.off + d) * n + i];
        qt[d] = P.qt[(E.off + d) * n + i];
      }
    }
  }
  __device__ __forceinline__ static void store(const ToolState& S, const MtParams& P, const ToolEnc& E, int64_t i, bool active) {
    const float (&q)[kMaxToolDof] = S.q;
    const float (&qd)[kMaxToolDof] = S.qd;
    const float (&qt)[kMaxToolDof] = S.qt;
    const int64_t n = P.n;
    if (!active) return;
#pragma unroll
    for (int d = 0; d < kMaxToolDof; ++d) {
      if (d >= E.robot.dof) continue;
      P.q[(E.off + d) * n + i] = q[d];
      P.qd[(E.off + d) * n + i] = qd[d];
      P.qt[(E.off + d) * n + i] = qt[d];
    }
  }

  // dynamics (dynamics.cpp:127-185) + FK + staging of the tool's obs columns
  template <class CH>
  __device__ __forceinline__ static void step(ToolState& S, const MtParams& P, const ToolEnc& E, int t, const float* s_act_row,
                              float* s_act_out, float* o, int& sat, int& bad, float (&tip)[3], float (&axis)[3]) {
    float (&q)[kMaxToolDof] = S.q;
    float (&qd)[kMaxToolDof] = S.qd;
    float (&qt)[kMaxToolDof] = S.qt;
    uint64_t& act_s = S.act_s;
    const RobotTable& R = E.robot;
    // compile-time DoF count / jaw for the fixed chains
    const int dof = CH::kExact ? CH::kDof : R.dof;
    const int jaw = CH::kExact ? CH::jaw(R) : R.jaw;
    const int off = E.off, A = P.A;
    const int mode = P.control_mode;
    float kpqt[kMaxToolDof], vt[kMaxToolDof], tc[kMaxToolDof];
    uint64_t ds = GEN ? act_s * E.col_mult + E.col_add : 0;
#pragma unroll
    for (int d = 0; d < kMaxToolDof; ++d) {
      kpqt[d] = vt[d] = tc[d] = 0.f;
      if (d >= dof) continue;
      float ad;
      if (GEN) {
        // uniform(-1, 1) of bench.cpp:34 = (u - 2^31) * 2^-31, exact in fp64, rounded once
        const uint32_t u = pcg_next(ds, P.act_inc);
        ad = __int2float_rn((int32_t)(u ^ 0x80000000u)) * 0x1.0p-31f;
        s_act_out[off + d] = ad;
      } else {
        ad = s_act_row[off + d];
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
      if (mode == kModePosition) {
        qt[d] = (d == jaw) ? (ad > 0.f ? hi : lo) : rescale(ad, lo, hi);
        kpqt[d] = R.kp[d] * qt[d];
      } else if (mode == kModeVelocity) {
        vt[d] = rescale(ad, -R.vel[d], R.vel[d]);
      } else {
        tc[d] = rescale(ad, -R.eff[d], R.eff[d]);
      }
    }
    if (GEN) act_s = act_s * P.jump_mult + P.jump_add;
    const float dt = P.dt_sub;
    if (CH::kExact && mode == kModePosition) {
      // position control on a specialised chain: the PD law with dt / inertia
      // folded into the gains, read from shared memory once per step (not per
      // substep): u = clamp(gk qt - gk q - gd qd, +-ge), vv = clamp(gc qd + u,
      // +-vl) (fp32 rounding differs from the reference's operation order by a
      // few ulp, as in the single-tool specialised kernels)
      float gk[kMaxToolDof], gd[kMaxToolDof], gc[kMaxToolDof], ge[kMaxToolDof], vl[kMaxToolDof],
          lo[kMaxToolDof], hi[kMaxToolDof];
#pragma unroll
      for (int d = 0; d < kMaxToolDof; ++d) {
        gk[d] = gd[d] = gc[d] = ge[d] = vl[d] = lo[d] = hi[d] = 0.f;
        if (d >= dof) continue;
        const float dti = R.dt_over_inertia[d];
        gk[d] = R.kp[d] * dti;
        gd[d] = R.kd[d] * dti;
        gc[d] = 1.f - R.damping[d] * dti;
        ge[d] = R.eff[d] * dti;
        vl[d] = R.vel[d];
        lo[d] = R.lo[d];
        hi[d] = R.hi[d];
        kpqt[d] = gk[d] * qt[d];
      }
      for (int s = 0; s < P.substeps; ++s) {
#pragma unroll
        for (int d = 0; d < kMaxToolDof; ++d) {
          if (d >= dof) continue;
          const float u = fminf(fmaxf(fmaf(-gd[d], qd[d], fmaf(-gk[d], q[d], kpqt[d])), -ge[d]), ge[d]);
          const float vv = fminf(fmaxf(fmaf(qd[d], gc[d], u), -vl[d]), vl[d]);
          const float qq = fmaf(vv, dt, q[d]);
          const float qc = fminf(fmaxf(qq, lo[d]), hi[d]);  // limit projection
          qd[d] = qc != qq ? 0.f : vv;
          q[d] = qc;
        }
      }
    } else
    for (int s = 0; s < P.substeps; ++s) {
#pragma unroll
      for (int d = 0; d < kMaxToolDof; ++d) {
        if (d >= dof) continue;
        const float ef = R.eff[d], vl = R.vel[d];
        float tau;
        if (mode == kModePosition) tau = fmaf(-R.kd[d], qd[d], fmaf(-R.kp[d], q[d], kpqt[d]));
        else if (mode == kModeVelocity) tau = R.kd[d] * (vt[d] - qd[d]);
        else tau = tc[d];
        tau = fminf(fmaxf(tau, -ef), ef);
        float vv = qd[d] + (tau - R.damping[d] * qd[d]) * R.dt_over_inertia[d];
        vv = fminf(fmaxf(vv, -vl), vl);
        const float qq = q[d] + vv * dt;
        const float qc = fminf(fmaxf(qq, R.lo[d]), R.hi[d]);  // limit projection
        qd[d] = qc != qq ? 0.f : vv;
        q[d] = qc;
      }
    }
#pragma unroll
    for (int d = 0; d < kMaxToolDof; ++d) {
      if (d >= dof) continue;
      o[off + d] = q[d];
      o[A + off + d] = qd[d];
      o[2 * A + 3 * T + off + d] = qt[d];
    }
    tool_fk<CH>(E, q, tip, axis);  // refresh_tips (envs.cpp:456-463)
#pragma unroll
    for (int k = 0; k < 3; ++k) o[2 * A + 3 * t + k] = tip[k];
  }
};

// Fused multi-tool step: a CTA is a team of T warps for 32 envs; warp t runs
// tool t (dynamics, FK, its observation columns) with its state in registers
// for the whole launch, publishes the world tip / camera axis in shared
// memory, and after one barrier warp 0 scores the 32 envs (camera goals,
// view / collision penalties, hold, flags); after a second barrier all warps
// store the team's 32 observation rows (one contiguous run: float4 copy).
// Rows that ended are copied to terminal_observations, reset by warp 0
// (reset_row through HBM) and re-observed; the tool warps then reload them.
template <int T, bool GEN>
__global__ void __launch_bounds__(32 * T) mt_step_kernel(const __grid_constant__ MtParams P, int k_steps) {
  extern __shared__ __align__(16) float smem[];
  __shared__ MtSmem<T> ts;
  __shared__ __align__(16) ToolEnc s_tool[T];  // per-tool tables, dynamically indexed by warp (LDS, not param LD)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    static_assert(sizeof(ToolEnc) % 16 == 0, "ToolEnc copied as int4");
    const int4* src = reinterpret_cast<const int4*>(&P.tool[0]);
    int4* dst = reinterpret_cast<int4*>(s_tool);
    for (int k = threadIdx.x; k < (int)(T * sizeof(ToolEnc) / 16); k += 32 * T) dst[k] = src[k];
    __syncthreads();
  }
  const ToolEnc& E = s_tool[warp];
  const int64_t n = P.n;
  const int A = P.A, O = P.O;
  const int64_t row0 = (int64_t)blockIdx.x * 32;
  const int64_t i = row0 + lane;
  const bool active = i < n;
  const int rows = (int)min((int64_t)32, n - row0);
  float* s_obs = smem;              // [2][32][O]
  float* s_act = smem + 2 * 32 * O;  // [2][32][A]: GEN draws by step parity (caller actions: [32][A])
  const bool full = rows == 32;

  // one register state per thread; the warp's tool index selects the code
  // path (ToolWarp<..., t> adds no data, only compile-time offsets)
  ToolState st;
  using TW = ToolWarp<T, GEN>;
  TW::load(st, P, E, i, active);
  if (GEN && active) st.act_s = P.act_state[i];
  if (!GEN) {  // the team's caller action rows: one contiguous run
    const float* src = P.actions + row0 * A;
    const int cnt = rows * A;
    if (full && ((reinterpret_cast<uintptr_t>(src) & 15u) == 0)) {
      for (int k = threadIdx.x; k < cnt / 4; k += 32 * T)
        reinterpret_cast<float4*>(s_act)[k] = reinterpret_cast<const float4*>(src)[k];
      for (int k = (cnt / 4) * 4 + threadIdx.x; k < cnt; k += 32 * T) s_act[k] = src[k];
    } else {
      for (int k = threadIdx.x; k < cnt; k += 32 * T) s_act[k] = src[k];
    }
    __syncthreads();
  }
  // scorer (warp 0) task state
  int32_t sc = 0, hc = 0;
  float g[T][3];
  const auto load_task = [&]() {
#pragma unroll
    for (int u = 0; u < T; ++u)
#pragma unroll
      for (int k = 0; k < 3; ++k) g[u][k] = active ? P.goals[(3 * u + k) * n + i] : 0.f;
    sc = active ? P.step_count[i] : 0;
    hc = active ? P.hold_count[i] : 0;
  };
  const int scorer = P.scorer;  // the tool warp with the fewest DoFs scores (shortest own step)
  if (warp == scorer) load_task();

  for (int step = 0; step < k_steps; ++step) {
    const int b = step & 1;
    float* s_rows = s_obs + b * 32 * O;
    float* o = s_rows + lane * O;
    // a warp that finished storing step k-1's action rows may draw step k+1
    // while another still reads: the GEN draws alternate between two buffers
    float* sa = GEN ? s_act + b * 32 * A : s_act;
    int sat = 0, bad = 0;
    {
      float tip[3], axis[3];
      // one code path per chain structure (not per tool: both PSM warps of a
      // trimanual team share the PSM path)
      switch (E.chain) {
        case kChainPsm:
          TW::template step<PsmChain>(st, P, E, warp, sa + lane * A, sa + lane * A, o, sat, bad, tip, axis);
          break;
        case kChainEcm:
          TW::template step<EcmChain>(st, P, E, warp, sa + lane * A, sa + lane * A, o, sat, bad, tip, axis);
          break;
        case kChainStar:
          TW::template step<StarChain>(st, P, E, warp, sa + lane * A, sa + lane * A, o, sat, bad, tip, axis);
          break;
        default:
          TW::template step<GenericChain<kMaxToolDof>>(st, P, E, warp, sa + lane * A, sa + lane * A, o, sat,
                                                       bad, tip, axis);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        ts.tip[b][warp][k][lane] = tip[k];
        ts.ax[b][warp][k][lane] = axis[k];
      }
    }
    if (!GEN) {
      if (!active) sat = bad = 0;
      const unsigned wsat = __reduce_add_sync(0xffffffffu, (unsigned)sat);
      if (wsat && lane == 0) atomicAdd(P.sat_total, (unsigned long long)wsat);
      if (__any_sync(0xffffffffu, bad) && bad) atomicOr(P.err, kErrNonFiniteAction);
    }
    __syncthreads();  // B1: every tool published

    if (warp == scorer) {  // ---- scoring (envs.cpp:540-593)
      float tw[T][3];
#pragma unroll
      for (int u = 0; u < T; ++u)
#pragma unroll
        for (int k = 0; k < 3; ++k) tw[u][k] = ts.tip[b][u][k][lane];
      sc += 1;
      float reward = 0.f, err_sum = 0.f;
      int err_count = 0;
      bool all_in = true;
#pragma unroll
      for (int u = 0; u < T; ++u) {
        if (P.tool[u].camera) {
          float mid[3];
          camera_mid<T>(tw, u, mid);
          const float tm[3] = {mid[0] - tw[u][0], mid[1] - tw[u][1], mid[2] - tw[u][2]};
          const float nrm = sqrtf(tm[0] * tm[0] + tm[1] * tm[1] + tm[2] * tm[2]);
          if (nrm > 1e-12f) {
            // acos(clamp(axis . to_mid/|to_mid|, -1, 1)) evaluated as
            // atan2(|axis x u|, axis . u): the same angle (|axis| = 1)
            // without acos's loss of precision near 0 and pi in fp32
            const float uu[3] = {tm[0] / nrm, tm[1] / nrm, tm[2] / nrm};
            const float a0 = ts.ax[b][u][0][lane], a1 = ts.ax[b][u][1][lane], a2 = ts.ax[b][u][2][lane];
            const float cx = a1 * uu[2] - a2 * uu[1], cy = a2 * uu[0] - a0 * uu[2], cz = a0 * uu[1] - a1 * uu[0];
            reward += -P.view_penalty * atan2f(sqrtf(cx * cx + cy * cy + cz * cz), a0 * uu[0] + a1 * uu[1] + a2 * uu[2]);
          }
#pragma unroll
          for (int k = 0; k < 3; ++k) g[u][k] = mid[k];
        } else {
          const float dx = tw[u][0] - g[u][0], dy = tw[u][1] - g[u][1], dz = tw[u][2] - g[u][2];
          const float dist = sqrtf(dx * dx + dy * dy + dz * dz);
          reward += P.rho * dist;
          err_sum += dist;
          ++err_count;
          if (dist >= P.success_radius) all_in = false;
        }
      }
      float min_sep = __int_as_float(0x7f800000);
#pragma unroll
      for (int u = 0; u + 1 < T; ++u)
#pragma unroll
        for (int v = u + 1; v < T; ++v) {
          const float dx = tw[u][0] - tw[v][0], dy = tw[u][1] - tw[v][1], dz = tw[u][2] - tw[v][2];
          min_sep = fminf(min_sep, sqrtf(dx * dx + dy * dy + dz * dz));
        }
      if (min_sep < P.collision_threshold) reward += -P.collision_penalty;
      hc = all_in ? hc + 1 : 0;
      const bool term = hc >= P.success_hold;
      const bool tout = sc >= P.episode_len;
      if (active) {
        if (!isfinite(reward)) atomicOr(P.err, kErrNonFiniteReward);
        P.rewards[i] = reward;
        P.task_error[i] = err_count > 0 ? err_sum / (float)err_count : 0.f;
        P.terminated[i] = term ? 1 : 0;
        P.timed_out[i] = tout ? 1 : 0;
#pragma unroll
        for (int u = 0; u < T; ++u) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            P.tips[(3 * u + k) * n + i] = tw[u][k];
            if (P.tool[u].camera) P.goals[(3 * u + k) * n + i] = g[u][k];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < T; ++u)
#pragma unroll
        for (int k = 0; k < 3; ++k) o[3 * A + 3 * T + 3 * u + k] = g[u][k];
      const unsigned ended = __ballot_sync(0xffffffffu, active && (term || tout));
      if (lane == 0) {
        ts.ended[b] = ended;
        if (ended) atomicAdd(P.ended_total, (unsigned long long)__popc(ended));
      }
    }
    __syncthreads();  // B2: rows scored and staged

    // ---- team store of the 32 observation rows (and the generated actions)
    float* g_obs = P.obs + row0 * O;
    const int cnt = rows * O;
    if (full) {  // 32 * O floats from a 16-byte aligned row block
      const float4* s4 = reinterpret_cast<const float4*>(s_rows);
      float4* g4 = reinterpret_cast<float4*>(g_obs);
      for (int k = threadIdx.x; k < cnt / 4; k += 32 * T) g4[k] = s4[k];
      for (int k = (cnt / 4) * 4 + threadIdx.x; k < cnt; k += 32 * T) g_obs[k] = s_rows[k];
    } else {
      for (int k = threadIdx.x; k < cnt; k += 32 * T) g_obs[k] = s_rows[k];
    }
    if (GEN) {
      float* g_act = P.act_buf + row0 * A;
      for (int k = threadIdx.x; k < rows * A; k += 32 * T) g_act[k] = sa[k];
    }
    const unsigned ended = ts.ended[b];
    if (ended) {  // ---- terminal copy, reset_row, re-observe (envs.cpp:604-615)
      for (unsigned m = ended; m; m &= m - 1) {
        const int r = __ffs(m) - 1;
        for (int c = threadIdx.x; c < O; c += 32 * T) P.tobs[(row0 + r) * O + c] = s_rows[r * O + c];
      }
      __syncthreads();  // every terminal row copied before the scorer re-stages the reset rows
      if (warp == scorer) {
        if ((ended >> lane) & 1) {
          const int e = mt_reset_env<T>(P, i);
          if (e) atomicOr(P.err, e);
          stage_row_from_state<T>(P, i, o);
        }
        if ((ended >> lane) & 1) load_task();
      }
      __syncthreads();  // reset state in HBM, rows re-staged
      for (unsigned m = ended; m; m &= m - 1) {
        const int r = __ffs(m) - 1;
        for (int c = threadIdx.x; c < O; c += 32 * T) g_obs[(int64_t)r * O + c] = s_rows[r * O + c];
      }
      if ((ended >> lane) & 1) TW::load(st, P, E, i, active);
    }
  }
  if (warp == scorer && active) {
    P.step_count[i] = sc;
    P.hold_count[i] = hc;
  }
  TW::store(st, P, E, i, active);
  if (GEN && active && warp == 0) P.act_state[i] = st.act_s;
}

template <int T>
__global__ void __launch_bounds__(32 * kMtWarps) mt_reset_kernel(const __grid_constant__ MtParams P) {
  extern __shared__ __align__(16) float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = P.n;
  const int64_t row0 = ((int64_t)blockIdx.x * kMtWarps + warp) * 32;
  if (row0 >= n) return;
  const int64_t i = row0 + lane;
  const int rows = (int)min((int64_t)32, n - row0);
  float* s_obs = smem + warp * 32 * (P.Os + P.A);
  if (i < n) {  // VecTaskEnv::reset (envs.cpp:425-435)
    const int e = mt_reset_env<T>(P, i);
    if (e) atomicOr(P.err, e);
    P.episode_count[i] = 0;
    P.terminated[i] = 0;
    P.timed_out[i] = 0;
    P.rewards[i] = 0.f;
    stage_row_from_state<T>(P, i, s_obs + lane * P.Os);
  }
  __syncwarp();
  warp_store_rows(P.obs + row0 * P.O, s_obs, rows, P.O, P.Os, lane);
}

template <int T>
cudaError_t launch_t(const MtParams& P, int k_steps, bool gen, bool reset, cudaStream_t st) {
  const int64_t warps = (P.n + 31) / 32;
  const unsigned grid = (unsigned)((warps + kMtWarps - 1) / kMtWarps);
  const size_t sm = (size_t)kMtWarps * 32 * (P.Os + P.A) * sizeof(float);
  const auto prep = [&](const void* fn) {
    return sm > 48 * 1024 ? cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)
                          : cudaSuccess;
  };
  cudaError_t e;
  if (reset) {
    if ((e = prep((const void*)mt_reset_kernel<T>)) != cudaSuccess) return e;
    mt_reset_kernel<T><<<grid, 32 * kMtWarps, sm, st>>>(P);
  } else {
    const unsigned tgrid = (unsigned)((P.n + 31) / 32);
    const size_t tsm = (size_t)(2 * 32 * P.O + 2 * 32 * P.A) * sizeof(float);
    const void* fn = gen ? (const void*)mt_step_kernel<T, true> : (const void*)mt_step_kernel<T, false>;
    if (tsm > 40 * 1024 && (e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm)) !=
                               cudaSuccess)
      return e;
    if (gen) mt_step_kernel<T, true><<<tgrid, 32 * T, tsm, st>>>(P, k_steps);
    else mt_step_kernel<T, false><<<tgrid, 32 * T, tsm, st>>>(P, k_steps);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_multi(const MtParams& P, int k_steps, bool gen, bool reset, cudaStream_t st) {
  switch (P.T) {
    case 2: return launch_t<2>(P, k_steps, gen, reset, st);
    case 3: return launch_t<3>(P, k_steps, gen, reset, st);
    case 4: return launch_t<4>(P, k_steps, gen, reset, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sg
