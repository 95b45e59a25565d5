// MultiToolReaching step / reset kernels (multi.cuh). One thread owns one env
// and walks its T tools in order with the tool index a compile-time constant
// (T is a template parameter, so every ToolEnc field is a constant-bank load
// at a fixed offset). Per tool the joint state comes from the DoF-major SoA
// arrays (a warp's 32 envs read one 128-byte line per DoF), is integrated
// with the reference's per-DoF PD law (dynamics.cpp:127-185, the same fp32
// operation order as the single-tool generic kernel), written back, and the
// tool FK (robot_model.cpp:371-395) is mapped through the tool's base pose.
// Observation rows are staged per warp in shared memory (odd row stride: no
// bank conflicts) and stored row by row with coalesced warp stores.
#include "multi.cuh"

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
__device__ __forceinline__ void tool_fk(const ToolEnc& E, const float (&q)[kMaxToolDof], float (&tip)[3],
                                        float (&axis)[3]) {
  const RobotTable& R = E.robot;
  float m[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
  float p[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int d = 0; d < kMaxToolDof; ++d) {
    if (d >= R.dof) break;
    const JointEnc& J = R.j[d];
    fk_joint(J, J.kind, J.axis_code, J.flags & 7, (J.flags >> 3) & 1, q[d], m, p);
  }
  float t[3];
  fk_tip_offset(R, R.tip_flags, m, p, t);
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

template <int T, bool GEN>
__global__ void __launch_bounds__(32 * kMtWarps) mt_step_kernel(const __grid_constant__ MtParams P, int k_steps) {
  extern __shared__ __align__(16) float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n = P.n;
  const int A = P.A, O = P.O, Os = P.Os;
  const int64_t row0 = ((int64_t)blockIdx.x * kMtWarps + warp) * 32;
  if (row0 >= n) return;  // whole warp (no CTA-wide barriers below)
  const int64_t i = row0 + lane;
  const bool active = i < n;
  const int rows = (int)min((int64_t)32, n - row0);
  float* s_obs = smem + warp * 32 * (Os + A);
  float* s_act = s_obs + 32 * Os;
  float* o = s_obs + lane * Os;
  const int mode = P.control_mode;

  uint64_t act_s = 0;
  if (GEN) {
    if (active) act_s = P.act_state[i];
  } else {
    // the warp's caller action rows are one contiguous run: coalesced load
    const float* src = P.actions + row0 * A;
    for (int k = lane; k < rows * A; k += 32) s_act[k] = src[k];
    __syncwarp();
  }

  for (int step = 0; step < k_steps; ++step) {
    int sat = 0, bad = 0;
    float tw[T][3], ax[T][3];
    uint64_t ds = act_s;  // GEN: the row's draws are consecutive in column order
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const ToolEnc& E = P.tool[t];
      const RobotTable& R = E.robot;
      const int dof = R.dof, jaw = R.jaw, off = E.off;
      float q[kMaxToolDof], qd[kMaxToolDof], qt[kMaxToolDof], kpqt[kMaxToolDof], vt[kMaxToolDof],
          tc[kMaxToolDof];
#pragma unroll
      for (int d = 0; d < kMaxToolDof; ++d) {
        q[d] = qd[d] = qt[d] = kpqt[d] = vt[d] = tc[d] = 0.f;
        if (d >= dof) continue;
        const int64_t c = off + d;
        if (active) {
          q[d] = P.q[c * n + i];
          qd[d] = P.qd[c * n + i];
          qt[d] = P.qt[c * n + i];
        }
        float ad;
        if (GEN) {
          // uniform(-1, 1) of bench.cpp:34 = (u - 2^31) * 2^-31, exact in fp64, rounded once
          const uint32_t u = pcg_next(ds, P.act_inc);
          ad = __int2float_rn((int32_t)(u ^ 0x80000000u)) * 0x1.0p-31f;
          s_act[lane * A + c] = ad;
        } else {
          ad = s_act[lane * A + c];
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
      // dynamics.cpp:133-185, per-DoF operation order of the reference
      const float dt = P.dt_sub;
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
        const int64_t c = off + d;
        if (active) {
          P.q[c * n + i] = q[d];
          P.qd[c * n + i] = qd[d];
          P.qt[c * n + i] = qt[d];
        }
        o[c] = q[d];
        o[A + c] = qd[d];
        o[2 * A + 3 * T + c] = qt[d];
      }
      tool_fk(E, q, tw[t], ax[t]);  // refresh_tips (envs.cpp:456-463)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        o[2 * A + 3 * t + k] = tw[t][k];
        if (active) P.tips[(3 * t + k) * n + i] = tw[t][k];
      }
    }
    if (!GEN) {
      if (!active) sat = bad = 0;
      const unsigned wsat = __reduce_add_sync(0xffffffffu, (unsigned)sat);
      if (wsat && lane == 0) atomicAdd(P.sat_total, (unsigned long long)wsat);
      if (__any_sync(0xffffffffu, bad) && bad) atomicOr(P.err, kErrNonFiniteAction);
    }

    // ---- reward / camera goal / collision / hold / flags (envs.cpp:540-593)
    int32_t sc = 0, hc = 0;
    float g[T][3];
    if (active) {
      sc = P.step_count[i] + 1;
      hc = P.hold_count[i];
#pragma unroll
      for (int t = 0; t < T; ++t)
#pragma unroll
        for (int k = 0; k < 3; ++k) g[t][k] = P.goals[(3 * t + k) * n + i];
    } else {
#pragma unroll
      for (int t = 0; t < T; ++t) g[t][0] = g[t][1] = g[t][2] = 0.f;
    }
    float reward = 0.f, err_sum = 0.f;
    int err_count = 0;
    bool all_in = true;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      if (P.tool[t].camera) {
        float mid[3];
        camera_mid<T>(tw, t, mid);
        const float tm[3] = {mid[0] - tw[t][0], mid[1] - tw[t][1], mid[2] - tw[t][2]};
        const float nrm = sqrtf(tm[0] * tm[0] + tm[1] * tm[1] + tm[2] * tm[2]);
        if (nrm > 1e-12f) {
          // acos(clamp(axis . to_mid/|to_mid|, -1, 1)) evaluated as
          // atan2(|axis x u|, axis . u): the same angle (|axis| = 1) without
          // acos's loss of precision near 0 and pi in fp32
          const float u[3] = {tm[0] / nrm, tm[1] / nrm, tm[2] / nrm};
          const float* a = ax[t];
          const float cx = a[1] * u[2] - a[2] * u[1], cy = a[2] * u[0] - a[0] * u[2], cz = a[0] * u[1] - a[1] * u[0];
          const float ang = atan2f(sqrtf(cx * cx + cy * cy + cz * cz), a[0] * u[0] + a[1] * u[1] + a[2] * u[2]);
          reward += -P.view_penalty * ang;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) g[t][k] = mid[k];
        if (active)
#pragma unroll
          for (int k = 0; k < 3; ++k) P.goals[(3 * t + k) * n + i] = mid[k];
      } else {
        const float dx = tw[t][0] - g[t][0], dy = tw[t][1] - g[t][1], dz = tw[t][2] - g[t][2];
        const float dist = sqrtf(dx * dx + dy * dy + dz * dz);
        reward += P.rho * dist;
        err_sum += dist;
        ++err_count;
        if (dist >= P.success_radius) all_in = false;
      }
    }
    float min_sep = __int_as_float(0x7f800000);
#pragma unroll
    for (int t = 0; t + 1 < T; ++t)
#pragma unroll
      for (int u = t + 1; u < T; ++u) {
        const float dx = tw[t][0] - tw[u][0], dy = tw[t][1] - tw[u][1], dz = tw[t][2] - tw[u][2];
        min_sep = fminf(min_sep, sqrtf(dx * dx + dy * dy + dz * dz));
      }
    if (min_sep < P.collision_threshold) reward += -P.collision_penalty;
    const float terr = err_count > 0 ? err_sum / (float)err_count : 0.f;
    hc = all_in ? hc + 1 : 0;
    const bool term = hc >= P.success_hold;
    const bool tout = sc >= P.episode_len;
    if (active) {
      if (!isfinite(reward)) atomicOr(P.err, kErrNonFiniteReward);
      P.step_count[i] = sc;
      P.hold_count[i] = hc;
      P.rewards[i] = reward;
      P.task_error[i] = terr;
      P.terminated[i] = term ? 1 : 0;
      P.timed_out[i] = tout ? 1 : 0;
    }
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int k = 0; k < 3; ++k) o[3 * A + 3 * T + 3 * t + k] = g[t][k];
    __syncwarp();
    float* g_obs = P.obs + row0 * O;
    warp_store_rows(g_obs, s_obs, rows, O, Os, lane);
    if (GEN) {
      float* g_act = P.act_buf + row0 * A;
      for (int k = lane; k < rows * A; k += 32) g_act[k] = s_act[k];
      act_s = act_s * P.jump_mult + P.jump_add;
    }

    // ---- ended rows: terminal copy, reset_row, re-observe (envs.cpp:604-615)
    const unsigned ended = __ballot_sync(0xffffffffu, active && (term || tout));
    if (ended) {
      if (lane == 0) atomicAdd(P.ended_total, (unsigned long long)__popc(ended));
      for (unsigned m = ended; m; m &= m - 1) {
        const int r = __ffs(m) - 1;
        for (int c = lane; c < O; c += 32) P.tobs[(row0 + r) * O + c] = s_obs[r * Os + c];
      }
      __syncwarp();
      if ((ended >> lane) & 1) {
        const int e = mt_reset_env<T>(P, i);
        if (e) atomicOr(P.err, e);
        stage_row_from_state<T>(P, i, o);
      }
      __syncwarp();
      for (unsigned m = ended; m; m &= m - 1) {
        const int r = __ffs(m) - 1;
        for (int c = lane; c < O; c += 32) g_obs[(int64_t)r * O + c] = s_obs[r * Os + c];
      }
    }
    __syncwarp();
  }
  if (GEN && active) P.act_state[i] = act_s;
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
  } else if (gen) {
    if ((e = prep((const void*)mt_step_kernel<T, true>)) != cudaSuccess) return e;
    mt_step_kernel<T, true><<<grid, 32 * kMtWarps, sm, st>>>(P, k_steps);
  } else {
    if ((e = prep((const void*)mt_step_kernel<T, false>)) != cudaSuccess) return e;
    mt_step_kernel<T, false><<<grid, 32 * kMtWarps, sm, st>>>(P, k_steps);
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
