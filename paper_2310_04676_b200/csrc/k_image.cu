// ImageMatching step / reset kernels (image.cuh): one warp per env.
#include "image.cuh"
#include "launch.hpp"

namespace sg {
namespace {

constexpr unsigned kFull = 0xffffffffu;

#ifndef SG_IM_MINB
#define SG_IM_MINB 2  // CTAs per SM the step kernel is register-budgeted for (A/B: tools/ab.sh)
#endif

// fk_walk (robot_model.cpp:371-395) keeping the rotation: tip position and
// the camera rotation (last DoF frame x trailing rotation, Pose orientation
// as a matrix; the tool base of a single-robot env is the identity).
// CH: FixedChain (compile-time joint structure of PSM / ECM / STAR, no sin/cos
// range reduction: selected only when every revolute limit is within +-pi)
// or GenericChain<8|16> (runtime joint table).
template <class CH>
__device__ __forceinline__ void camera_pose(const ImParams& P, const float (&q)[CH::kDof], float (&Rc)[9],
                                            float (&pc)[3]) {
  const RobotTable& R = P.robot;
  float m[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
  float p[3] = {0.f, 0.f, 0.f};
  if constexpr (CH::kExact) {
    CH::walk(R, q, m, p, std::make_integer_sequence<int, CH::kDof>{});
    fk_tip_offset(R, CH::kTipFlags, m, p, pc);
  } else {
#pragma unroll
    for (int d = 0; d < CH::kDof; ++d) {
      if (d >= R.dof) break;
      const JointEnc& J = R.j[d];
      fk_joint(J, J.kind, J.axis_code, J.flags & 7, (J.flags >> 3) & 1, q[d], m, p);
    }
    fk_tip_offset(R, R.tip_flags, m, p, pc);
  }
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      Rc[r * 3 + c] = m[r * 3 + 0] * P.cam_R[0 * 3 + c] + m[r * 3 + 1] * P.cam_R[1 * 3 + c] +
                      m[r * 3 + 2] * P.cam_R[2 * 3 + c];
}

// Per-frame sphere constants: oc = camera - centre, c2 = |oc|^2 - r^2.
struct Frame {
  float R[9];
  float oc[3][3], c2[3], ka[3];  // ka = albedo / radius
};

__device__ __forceinline__ void make_frame(const float (&Rc)[9], const float (&pc)[3], const float (&sc)[15],
                                           Frame& F) {
#pragma unroll
  for (int k = 0; k < 9; ++k) F.R[k] = Rc[k];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const float o0 = pc[0] - sc[5 * s + 0], o1 = pc[1] - sc[5 * s + 1], o2 = pc[2] - sc[5 * s + 2];
    const float r = sc[5 * s + 3];
    F.oc[s][0] = o0;
    F.oc[s][1] = o1;
    F.oc[s][2] = o2;
    F.c2[s] = (o0 * o0 + o1 * o1 + o2 * o2) - r * r;
    F.ka[s] = sc[5 * s + 4] / r;
  }
}

// MUFU approximations without the IEEE / denormal fix-up sequences rsqrtf and
// sqrtf expand to (ncu: those fix-ups were 20 % of the kernel's instructions);
// ~2 ulp, far inside the fp32-vs-fp64 pixel tolerance.
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// One pixel of render.cpp:42-64 for the ray through camera coordinates
// (u, -v, -1). With the direction d normalised, the Lambert term
// n . (-d) = -(oc . d + t) / r = sqrt(disc) / r (t = -b - sqrt(disc)), so the
// nearest hit's shade needs no hit-point reconstruction; the three sphere
// tests are branch-free (selects) so the warp never diverges per pixel.
// Per-column constants of the camera rays. The unnormalised direction of
// pixel (u, v) is d = a - v R[:,1] with a = R (u, 0, -1) (top row looks up), so
// |d|^2 = A0 + v (A1 + v A2) and, per sphere, oc . d = ba + v bb: a pixel needs
// no direction vector, only these per-lane quadratics / lines in v.
struct Column {
  float A0, A1, A2;
  float ba[3], bb[3];
};
__device__ __forceinline__ Column column(const Frame& F, float u) {
  const float a0 = fmaf(F.R[0], u, -F.R[2]), a1 = fmaf(F.R[3], u, -F.R[5]), a2 = fmaf(F.R[6], u, -F.R[8]);
  const float r0 = F.R[1], r1 = F.R[4], r2 = F.R[7];
  Column C;
  C.A0 = fmaf(a0, a0, fmaf(a1, a1, a2 * a2));
  C.A1 = -2.f * fmaf(a0, r0, fmaf(a1, r1, a2 * r2));
  C.A2 = fmaf(r0, r0, fmaf(r1, r1, r2 * r2));
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    C.ba[s] = fmaf(F.oc[s][0], a0, fmaf(F.oc[s][1], a1, F.oc[s][2] * a2));
    C.bb[s] = -fmaf(F.oc[s][0], r0, fmaf(F.oc[s][1], r1, F.oc[s][2] * r2));
  }
  return C;
}

__device__ __forceinline__ float shade(const ImParams& P, const Frame& F, const Column& C, float v) {
  const float inv = rsqrt_approx(fmaf(v, fmaf(v, C.A2, C.A1), C.A0));  // 1 / |d|
  float best = P.far_, value = 0.f;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const float b = fmaf(v, C.bb[s], C.ba[s]) * inv;  // oc . d / |d|
    const float disc = fmaf(b, b, -F.c2[s]);
    const float sq = sqrt_approx(fmaxf(disc, 0.f));
    const float t = -b - sq;
    const bool hit = disc >= 0.f && t >= P.near_ && t < best;
    best = hit ? t : best;
    value = hit ? F.ka[s] * sq : value;  // albedo * lambert, lambert = sqrt(disc) / r
  }
  return value;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <int DMAX>
__device__ __forceinline__ void gather_q(float mine, float (&qa)[DMAX]) {
#pragma unroll
  for (int d = 0; d < DMAX; ++d) qa[d] = __shfl_sync(kFull, mine, d);
}

// reset_row for ImageMatching (envs.cpp:304-316, 269-295), warp-cooperative:
// every lane replays the env stream (q in the middle half, three spheres
// drawn z, y, x, radius, albedo -- g++ argument order --, target q in the
// middle quarter); the warp writes the new joint state, scene, target view
// and the post-reset observation row to HBM (the caller reloads its
// registers from there: no reference arguments, so the hot loop's state
// never lives on the stack).
template <class CH>
__device__ __noinline__ void im_reset_env(const ImParams& P, int64_t i, int lane) {
  float q, sc[15];
  constexpr int DMAX = CH::kDof;
  const RobotTable& R = P.robot;
  const int64_t n = P.n;
  const int A = R.dof;
  uint64_t s = P.rng_state[i];
  const uint64_t inc = P.rng_inc[i];
  float q0[DMAX], qT[DMAX];
#pragma unroll
  for (int d = 0; d < DMAX; ++d) {
    q0[d] = 0.f;
    if (d < A) {
      const double quarter = __dmul_rn(0.25, __dadd_rn(R.hi_d[d], -R.lo_d[d]));
      q0[d] = (float)pcg_uniform(s, inc, __dadd_rn(R.lo_d[d], quarter), __dadd_rn(R.hi_d[d], -quarter));
    }
  }
  const double s2 = __dmul_rn(2.0, P.sigma);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double z = -__dadd_rn(P.radius, pcg_uniform(s, inc, 0.1, 0.25));
    const double y = pcg_uniform(s, inc, -s2, s2);
    const double x = pcg_uniform(s, inc, -s2, s2);
    sc[5 * k + 0] = (float)__dadd_rn(P.center[0], x);
    sc[5 * k + 1] = (float)__dadd_rn(P.center[1], y);
    sc[5 * k + 2] = (float)__dadd_rn(P.center[2], z);
    sc[5 * k + 3] = (float)pcg_uniform(s, inc, 0.02, 0.05);
    sc[5 * k + 4] = (float)pcg_uniform(s, inc, 0.5, 1.0);
  }
#pragma unroll
  for (int d = 0; d < DMAX; ++d) {  // sample_q_fraction(rng, model, 0.25) (envs.cpp:31-39)
    qT[d] = 0.f;
    if (d < A) {
      const double margin = __dmul_rn(__dmul_rn(0.5, 0.75), __dadd_rn(R.hi_d[d], -R.lo_d[d]));
      qT[d] = (float)pcg_uniform(s, inc, __dadd_rn(R.lo_d[d], margin), __dadd_rn(R.hi_d[d], -margin));
    }
  }
  q = 0.f;
#pragma unroll
  for (int d = 0; d < DMAX; ++d)
    if (d == lane) q = q0[d];
  float RT[9], pT[3], R0[9], p0[3];
  camera_pose<CH>(P, qT, RT, pT);
  camera_pose<CH>(P, q0, R0, p0);
  if (lane == 0) P.rng_state[i] = s;
  if (lane < 15) {
    float v = 0.f;
#pragma unroll
    for (int k = 0; k < 15; ++k)
      if (k == lane) v = sc[k];
    P.scenes[i * 16 + lane] = v;
  }
  if (lane < 12) {
    float v = 0.f;
#pragma unroll
    for (int k = 0; k < 9; ++k)
      if (k == lane) v = RT[k];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (k + 9 == lane) v = pT[k];
    P.tcam[i * 12 + lane] = v;
  }
  if (lane < A) {
    P.q[lane * n + i] = q;
    P.qd[lane * n + i] = 0.f;
    P.qt[lane * n + i] = q;
  }
  if (lane < 3) P.tips[lane * n + i] = lane == 0 ? p0[0] : (lane == 1 ? p0[1] : p0[2]);
  if (lane == 0) {
    P.step_count[i] = 0;
    P.hold_count[i] = 0;
    P.episode_count[i] += 1;
  }
  // observation row: [q | qdot | tip | q_target | target image | current image]
  float* row = P.obs + i * P.O;
  if (lane < A) {
    row[lane] = q;
    row[A + lane] = 0.f;
    row[2 * A + 3 + lane] = q;
  }
  if (lane < 3) row[2 * A + lane] = lane == 0 ? p0[0] : (lane == 1 ? p0[1] : p0[2]);
  Frame FT, F0;
  make_frame(RT, pT, sc, FT);
  make_frame(R0, p0, sc, F0);
  const int head = 3 * A + 3, W = P.W, wh = P.wh;
  float* tgt = P.target + i * wh;
  for (int py = 0; py < P.H; ++py) {
    const float v = ((float)py + 0.5f - 0.5f * (float)P.H) * P.inv_f;
    for (int px = lane; px < W; px += 32) {
      const float u = ((float)px + 0.5f - 0.5f * (float)W) * P.inv_f;
      const int p = py * W + px;
      const float vt = shade(P, FT, column(FT, u), v);
      tgt[p] = vt;
      row[head + p] = vt;
      row[head + wh + p] = shade(P, F0, column(F0, u), v);
    }
  }
}

template <class CH, bool GEN>
__global__ void __launch_bounds__(32 * kImWarps, SG_IM_MINB) im_step_kernel(const __grid_constant__ ImParams P, int k_steps) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kImWarps + (threadIdx.x >> 5);
  const int64_t n = P.n;
  if (i >= n) return;  // whole warp
  const RobotTable& R = P.robot;
  const int A = R.dof, O = P.O, W = P.W, wh = P.wh;
  const int head = 3 * A + 3;
  const bool own = lane < A;
  const int dl = own ? lane : 0;
  // lane d's DoF constants in registers (per-lane indices would serialise
  // the constant cache inside the step loop)
  const float lo = R.lo[dl], hi = R.hi[dl], vl = R.vel[dl], ef = R.eff[dl], kp = R.kp[dl], kd = R.kd[dl],
              dmp = R.damping[dl], dti = R.dt_over_inertia[dl];
  const bool is_jaw = lane == R.jaw;
  const uint64_t pm = P.pow_mult[dl], pa = P.pow_add[dl];
  float q = own ? P.q[lane * n + i] : 0.f;
  float qd = own ? P.qd[lane * n + i] : 0.f;
  float qt = own ? P.qt[lane * n + i] : 0.f;
  float sc[15];
#pragma unroll
  for (int k = 0; k < 15; ++k) sc[k] = P.scenes[i * 16 + k];
  uint64_t act_s = GEN ? P.act_state[i] : 0;
  int32_t step_count = P.step_count[i];
  const int mode = P.control_mode;
  const float dt = P.dt_sub;

  for (int step = 0; step < k_steps; ++step) {
    // ---- dynamics of DoF `lane` (dynamics.cpp:127-185) ----------------------
    float ad = 0.f;
    int sat = 0, bad = 0;
    if (GEN) {
      const uint32_t u = pcg_output(act_s * pm + pa);
      ad = __int2float_rn((int32_t)(u ^ 0x80000000u)) * 0x1.0p-31f;
      if (own) P.act_buf[i * A + lane] = ad;
      act_s = act_s * P.jump_mult + P.jump_add;
    } else if (own) {
      ad = P.actions[i * A + lane];
      if (!isfinite(ad)) {
        bad = 1;
        ad = 0.f;
      }
      if (ad < -1.f || ad > 1.f) {
        ad = ad < -1.f ? -1.f : 1.f;
        sat = 1;
      }
    }
    float vt = 0.f, tc = 0.f, kpqt = 0.f;
    if (mode == kModePosition) {
      qt = is_jaw ? (ad > 0.f ? hi : lo) : rescale(ad, lo, hi);
      kpqt = kp * qt;
    } else if (mode == kModeVelocity) {
      vt = rescale(ad, -vl, vl);
    } else {
      tc = rescale(ad, -ef, ef);
    }
    for (int s = 0; s < P.substeps; ++s) {
      float tau;
      if (mode == kModePosition) tau = fmaf(-kd, qd, fmaf(-kp, q, kpqt));
      else if (mode == kModeVelocity) tau = kd * (vt - qd);
      else tau = tc;
      tau = fminf(fmaxf(tau, -ef), ef);
      float vv = qd + (tau - dmp * qd) * dti;
      vv = fminf(fmaxf(vv, -vl), vl);
      const float qq = q + vv * dt;
      const float qc = fminf(fmaxf(qq, lo), hi);  // limit projection
      qd = qc != qq ? 0.f : vv;
      q = qc;
    }
    if (!own) q = qd = qt = 0.f;
    if (!GEN) {
      const unsigned ns = __popc(__ballot_sync(kFull, sat));
      if (ns && lane == 0) atomicAdd(P.sat_total, (unsigned long long)ns);
      if (__any_sync(kFull, bad) && lane == 0) atomicOr(P.err, kErrNonFiniteAction);
    }
    // ---- camera FK (refresh_tips, envs.cpp:456-463) --------------------------
    constexpr int DMAX = CH::kDof;
    float qa[DMAX];
    gather_q<DMAX>(q, qa);
    float Rc[9], pc[3];
    camera_pose<CH>(P, qa, Rc, pc);
    if (lane < 3) P.tips[lane * n + i] = lane == 0 ? pc[0] : (lane == 1 ? pc[1] : pc[2]);
    step_count += 1;
    const bool ends = step_count >= P.episode_len;  // goal_met is never set for ImageMatching
    float* row = (ends ? P.tobs : P.obs) + i * O;
    if (own) {
      row[lane] = q;
      row[A + lane] = qd;
      row[2 * A + 3 + lane] = qt;
    }
    if (lane < 3) row[2 * A + lane] = lane == 0 ? pc[0] : (lane == 1 ? pc[1] : pc[2]);
    // ---- render (envs.cpp:464-473), L1 image error (envs.cpp:513-523) -------
    Frame F;
    make_frame(Rc, pc, sc, F);
    const float* tgt = P.target + i * wh;
    float* o_tgt = row + head;
    float* o_cur = row + head + wh;
    float acc = 0.f;
    if (W % 4 == 0 && 128 % W == 0 && wh % 128 == 0) {
      // 4 consecutive pixels per lane and 128 per warp iteration: the lane's
      // 4 columns are fixed (128 is a multiple of W), the target read is one
      // float4, the observation writes are float4 when the row is 16-byte
      // aligned (3A + 3 and O multiples of 4, e.g. PSM)
      const int px0 = (4 * lane) % W, prow = (4 * lane) / W, rows_it = 128 / W;
      Column C[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) C[j] = column(F, ((float)(px0 + j) + 0.5f - 0.5f * (float)W) * P.inv_f);
      const bool st4 = ((head | O) & 3) == 0;
      for (int it = 0; it < wh / 128; ++it) {
        const int p = 128 * it + 4 * lane;
        const float v = ((float)(it * rows_it + prow) + 0.5f - 0.5f * (float)P.H) * P.inv_f;
        const float4 t4 = *reinterpret_cast<const float4*>(tgt + p);
        const float c0 = shade(P, F, C[0], v), c1 = shade(P, F, C[1], v), c2 = shade(P, F, C[2], v),
                    c3 = shade(P, F, C[3], v);
        acc += (fabsf(c0 - t4.x) + fabsf(c1 - t4.y)) + (fabsf(c2 - t4.z) + fabsf(c3 - t4.w));
        if (st4) {
          *reinterpret_cast<float4*>(o_tgt + p) = t4;
          *reinterpret_cast<float4*>(o_cur + p) = make_float4(c0, c1, c2, c3);
        } else {
          o_tgt[p] = t4.x; o_tgt[p + 1] = t4.y; o_tgt[p + 2] = t4.z; o_tgt[p + 3] = t4.w;
          o_cur[p] = c0; o_cur[p + 1] = c1; o_cur[p + 2] = c2; o_cur[p + 3] = c3;
        }
      }
    } else {
      for (int px = lane; px < W; px += 32) {  // lane-fixed columns, rows in the inner loop
        const Column C = column(F, ((float)px + 0.5f - 0.5f * (float)W) * P.inv_f);
#pragma unroll 4
        for (int py = 0; py < P.H; ++py) {
          const float v = ((float)py + 0.5f - 0.5f * (float)P.H) * P.inv_f;
          const int p = py * W + px;
          const float c = shade(P, F, C, v);
          const float t = tgt[p];
          acc += fabsf(c - t);
          o_tgt[p] = t;
          o_cur[p] = c;
        }
      }
    }
    const float err = warp_sum(acc) / (float)wh;
    if (lane == 0) {
      const float reward = -err;
      if (!isfinite(reward)) atomicOr(P.err, kErrNonFiniteReward);
      P.rewards[i] = reward;
      P.task_error[i] = err;
      P.terminated[i] = 0;
      P.timed_out[i] = ends ? 1 : 0;
    }
    if (ends) {  // terminal row written above; reset_row + re-observe
      if (lane == 0) atomicAdd(P.ended_total, 1ull);
      __syncwarp();
      im_reset_env<CH>(P, i, lane);
      __syncwarp();
      q = own ? P.q[lane * n + i] : 0.f;
      qd = 0.f;
      qt = q;
#pragma unroll
      for (int k = 0; k < 15; ++k) sc[k] = P.scenes[i * 16 + k];
      step_count = 0;
    }
  }
  if (own) {
    P.q[lane * n + i] = q;
    P.qd[lane * n + i] = qd;
    P.qt[lane * n + i] = qt;
  }
  if (lane == 0) {
    P.step_count[i] = step_count;
    if (GEN) P.act_state[i] = act_s;
  }
}

template <class CH>
__global__ void __launch_bounds__(32 * kImWarps) im_reset_kernel(const __grid_constant__ ImParams P) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kImWarps + (threadIdx.x >> 5);
  if (i >= P.n) return;
  im_reset_env<CH>(P, i, lane);  // VecTaskEnv::reset (envs.cpp:425-435)
  if (lane == 0) {
    P.episode_count[i] = 0;
    P.terminated[i] = 0;
    P.timed_out[i] = 0;
    P.rewards[i] = 0.f;
  }
}

template <class CH>
cudaError_t launch_d(const ImParams& P, int k_steps, bool gen, bool reset, cudaStream_t st) {
  const unsigned grid = (unsigned)((P.n + kImWarps - 1) / kImWarps);
  if (reset) im_reset_kernel<CH><<<grid, 32 * kImWarps, 0, st>>>(P);
  else if (gen) im_step_kernel<CH, true><<<grid, 32 * kImWarps, 0, st>>>(P, k_steps);
  else im_step_kernel<CH, false><<<grid, 32 * kImWarps, 0, st>>>(P, k_steps);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_image(const ImParams& P, int k_steps, bool gen, bool reset, cudaStream_t st) {
  switch (P.chain) {
    case kChainPsm: return launch_d<PsmChain>(P, k_steps, gen, reset, st);
    case kChainEcm: return launch_d<EcmChain>(P, k_steps, gen, reset, st);
    case kChainStar: return launch_d<StarChain>(P, k_steps, gen, reset, st);
    case kChainGeneric16: return launch_d<GenericChain<16>>(P, k_steps, gen, reset, st);
    default: return launch_d<GenericChain<8>>(P, k_steps, gen, reset, st);
  }
}

}  // namespace sg
