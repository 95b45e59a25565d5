// Device kernels of the PPO update (config 5) around the library GEMMs:
//   * ELU forward / backward (Policy::trunk_forward's activation, policy.cpp:33,
//     and its derivative in Policy::backward, policy.cpp:163-218), fp32 or bf16,
//     16-byte vectors; the backward works from the OUTPUT h (d/dz expm1(z) =
//     exp(z) = h + 1 for z <= 0), so the forward keeps no pre-activation;
//   * the minibatch gather of ppo_update (ppo.cpp:173-190): one launch copies
//     the minibatch rows of obs (fp32 -> fp32 or bf16), actions, old log-probs,
//     advantages and returns by index.
// PyTorch's elementwise / index_select kernels were 30 % of the update
// (torch.profiler, tools/prof_ppo.py): ELU alone ran at ~5x its memory bound.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "sg_env.h"

namespace {

__device__ __forceinline__ float elu_f(float z, bool fast) {
  return z > 0.f ? z : (fast ? __expf(z) - 1.f : expm1f(z));
}

__global__ void elu_fwd_f32(const float4* __restrict__ z, float4* __restrict__ h, int64_t n4) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n4; k += (int64_t)gridDim.x * blockDim.x) {
    float4 v = z[k];
    v.x = elu_f(v.x, false);
    v.y = elu_f(v.y, false);
    v.z = elu_f(v.z, false);
    v.w = elu_f(v.w, false);
    h[k] = v;
  }
}

__global__ void elu_bwd_f32(const float4* __restrict__ h, const float4* __restrict__ dh, float4* __restrict__ dz,
                            int64_t n4) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n4; k += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = h[k], g = dh[k];
    dz[k] = make_float4(a.x > 0.f ? g.x : g.x * (a.x + 1.f), a.y > 0.f ? g.y : g.y * (a.y + 1.f),
                        a.z > 0.f ? g.z : g.z * (a.z + 1.f), a.w > 0.f ? g.w : g.w * (a.w + 1.f));
  }
}

// bf16: 8 values per 16-byte vector, fp32 math, one rounding
union Bf8 {
  uint4 u;
  __nv_bfloat162 h[4];
};

// bf16 kernels: kVec independent 16-byte vectors per thread per iteration
// (loads issued before any use: more bytes in flight per SM)
constexpr int kVec = 4;

__global__ void elu_fwd_bf16(const uint4* __restrict__ z, uint4* __restrict__ h, int64_t n8) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < n8; k0 += stride * kVec) {
    Bf8 v[kVec];
#pragma unroll
    for (int u = 0; u < kVec; ++u)
      if (k0 + u * stride < n8) v[u].u = z[k0 + u * stride];
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      if (k0 + u * stride >= n8) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(v[u].h[j]);
        v[u].h[j] = __floats2bfloat162_rn(elu_f(f.x, true), elu_f(f.y, true));
      }
      h[k0 + u * stride] = v[u].u;
    }
  }
}

__global__ void elu_bwd_bf16(const uint4* __restrict__ h, const uint4* __restrict__ dh, uint4* __restrict__ dz,
                             int64_t n8) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < n8; k0 += stride * kVec) {
    Bf8 a[kVec], g[kVec];
#pragma unroll
    for (int u = 0; u < kVec; ++u)
      if (k0 + u * stride < n8) {
        a[u].u = h[k0 + u * stride];
        g[u].u = dh[k0 + u * stride];
      }
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      if (k0 + u * stride >= n8) continue;
      Bf8 o;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 fa = __bfloat1622float2(a[u].h[j]), fg = __bfloat1622float2(g[u].h[j]);
        o.h[j] = __floats2bfloat162_rn(fa.x > 0.f ? fg.x : fg.x * (fa.x + 1.f),
                                       fa.y > 0.f ? fg.y : fg.y * (fa.y + 1.f));
      }
      dz[k0 + u * stride] = o.u;
    }
  }
}

// ELU backward + the bias gradient of the layer below in one pass
// (Policy::backward, policy.cpp:163-218): dz = dh * ELU'(h) over a row-major
// bf16 [m x n] activation, and colsum[c] += sum over rows of dz[., c] (the
// next-lower layer's db = 1^T dZ, which otherwise is an M = 1 split-K GEMM
// plus its reduction). h == null: dz = dh (a plain column sum of dh, the
// last layer's db); dz == null: no dz output. A thread owns 8 columns (one
// 16-byte vector) of rows t / (n/8), t / (n/8) + 256 / (n/8), ... and keeps
// fp32 column sums in registers; the block folds them in shared memory and
// adds one fp32 atomic per column.
__global__ void elu_bwd_colsum_bf16(const uint4* __restrict__ h, const uint4* __restrict__ dh, uint4* __restrict__ dz,
                                    int64_t m, int n, float* __restrict__ colsum) {
  extern __shared__ float sred[];  // [256 / tpr][n]
  const int tpr = n / 8, rpb = blockDim.x / tpr;  // threads per row, rows per block pass
  const int c8 = threadIdx.x % tpr, r0 = threadIdx.x / tpr;
  float acc[8] = {};
  if (r0 < rpb) {
    for (int64_t r = (int64_t)blockIdx.x * rpb + r0; r < m; r += (int64_t)gridDim.x * rpb) {
      const int64_t k = r * tpr + c8;
      Bf8 g, o;
      g.u = dh[k];
      if (h) {
        Bf8 a;
        a.u = h[k];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 fa = __bfloat1622float2(a.h[j]), fg = __bfloat1622float2(g.h[j]);
          o.h[j] = __floats2bfloat162_rn(fa.x > 0.f ? fg.x : fg.x * (fa.x + 1.f),
                                         fa.y > 0.f ? fg.y : fg.y * (fa.y + 1.f));
        }
      } else {
        o.u = g.u;
      }
      if (dz) dz[k] = o.u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(o.h[j]);
        acc[2 * j] += f.x;
        acc[2 * j + 1] += f.y;
      }
    }
  }
  if (r0 < rpb) {
#pragma unroll
    for (int j = 0; j < 8; ++j) sred[r0 * n + c8 * 8 + j] = acc[j];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    float t = 0.f;
    for (int q = 0; q < rpb; ++q) t += sred[q * n + c];
    atomicAdd(&colsum[c], t);
  }
}

// 8 threads per minibatch row: thread k copies float4 k of the obs row
// (coalesced 128-byte rows); thread 0 also copies the row's action, log-prob,
// advantage and return.
__global__ void ppo_gather_kernel(const int64_t* __restrict__ idx, int64_t m, const float* __restrict__ obs,
                                  int32_t obs_w, void* __restrict__ obs_out, int32_t out_w, int32_t obs_bf16,
                                  const float* __restrict__ act, int32_t A, float* __restrict__ act_out,
                                  const float* __restrict__ logp, float* __restrict__ logp_out,
                                  const float* __restrict__ adv, float* __restrict__ adv_out,
                                  const float* __restrict__ ret, float* __restrict__ ret_out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = t >> 3;
  const int k = (int)(t & 7);
  if (r >= m) return;
  const int64_t src = idx[r];
  if ((obs_w & 3) == 0 && obs_w == out_w) {  // aligned rows: 16-byte vectors
    const int n4 = obs_w >> 2;
    const float4* so = reinterpret_cast<const float4*>(obs + src * obs_w);
    for (int c = k; c < n4; c += 8) {
      const float4 v = so[c];
      if (obs_bf16) {
        __nv_bfloat162* d = reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(obs_out) + r * out_w + 4 * c);
        d[0] = __floats2bfloat162_rn(v.x, v.y);
        d[1] = __floats2bfloat162_rn(v.z, v.w);
      } else {
        reinterpret_cast<float4*>(static_cast<float*>(obs_out) + r * out_w)[c] = v;
      }
    }
  } else {  // unpadded rows (the env writes obs_dim-wide rows): element-wise, zero padding
    const float* so = obs + src * obs_w;
    for (int c = k; c < out_w; c += 8) {
      const float v = c < obs_w ? so[c] : 0.f;
      if (obs_bf16) static_cast<__nv_bfloat16*>(obs_out)[r * out_w + c] = __float2bfloat16_rn(v);
      else static_cast<float*>(obs_out)[r * out_w + c] = v;
    }
  }
  if (k == 0) {
    for (int a = 0; a < A; ++a) act_out[r * A + a] = act[src * A + a];
    logp_out[r] = logp[src];
    adv_out[r] = adv[src];
    ret_out[r] = ret[src];
  }
}

unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;  // grid-stride beyond 32 CTAs per SM
  return (unsigned)(g > 0 ? g : 1);
}

}  // namespace

extern "C" {

int sg_elu_forward(const void* z, void* h, int64_t count, int32_t dtype, void* stream) {
  const cudaStream_t st = (cudaStream_t)stream;
  if (dtype == 1) {
    if (count % 8) return SG_ERR_CONFIG;
    elu_fwd_bf16<<<grid_for((count / 8 + kVec - 1) / kVec, 256), 256, 0, st>>>((const uint4*)z, (uint4*)h, count / 8);
  } else {
    if (count % 4) return SG_ERR_CONFIG;
    elu_fwd_f32<<<grid_for(count / 4, 256), 256, 0, st>>>((const float4*)z, (float4*)h, count / 4);
  }
  return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_SIM;
}

int sg_elu_backward_colsum(const void* h, const void* dh, void* dz, int64_t m, int32_t n, float* colsum,
                           void* stream) {
  if (n % 8 || n < 8 || n > 2048 || !dh || !colsum) return SG_ERR_CONFIG;
  const int tpr = n / 8, rpb = 256 / tpr > 0 ? 256 / tpr : 1;
  const unsigned grid = grid_for((m + rpb - 1) / rpb, 1);
  const size_t smem = (size_t)rpb * n * sizeof(float);
  elu_bwd_colsum_bf16<<<grid < 592u ? grid : 592u, 256, smem, (cudaStream_t)stream>>>(
      (const uint4*)h, (const uint4*)dh, (uint4*)dz, m, n, colsum);
  return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_SIM;
}

int sg_elu_backward(const void* h, const void* dh, void* dz, int64_t count, int32_t dtype, void* stream) {
  const cudaStream_t st = (cudaStream_t)stream;
  if (dtype == 1) {
    if (count % 8) return SG_ERR_CONFIG;
    elu_bwd_bf16<<<grid_for((count / 8 + kVec - 1) / kVec, 256), 256, 0, st>>>((const uint4*)h, (const uint4*)dh,
                                                                              (uint4*)dz, count / 8);
  } else {
    if (count % 4) return SG_ERR_CONFIG;
    elu_bwd_f32<<<grid_for(count / 4, 256), 256, 0, st>>>((const float4*)h, (const float4*)dh, (float4*)dz,
                                                           count / 4);
  }
  return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_SIM;
}

int sg_ppo_gather(const int64_t* idx, int64_t m, const float* obs, int32_t obs_w, void* obs_out, int32_t obs_out_w,
                  int32_t obs_bf16, const float* act, int32_t A, float* act_out, const float* logp, float* logp_out,
                  const float* adv, float* adv_out, const float* ret, float* ret_out, void* stream) {
  if (obs_out_w < obs_w || obs_w < 1) return SG_ERR_CONFIG;
  const int64_t threads = m * 8;
  ppo_gather_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      idx, m, obs, obs_w, obs_out, obs_out_w, obs_bf16, act, A, act_out, logp, logp_out, adv, adv_out, ret, ret_out);
  return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_SIM;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// ppo_loss_and_grad's data part (ppo.cpp:90-154) in one pass: per sample the
// Gaussian log-prob of the taken action, ratio, clipped surrogate, value
// error, and the analytic gradients the reference forms (dmean, dvalue, and
// the log-std gradient summed over the minibatch); block partial sums of
// {surr, kl, value_sq, clipped, dlog_std[A]} go to acc by atomics, and a
// one-warp finalize forms the loss, metrics and the projected log-std gradient.
namespace {

template <typename T>
__device__ __forceinline__ float ld(const T* p) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
  else return *p;
}
template <typename T>
__device__ __forceinline__ void st(T* p, float v) {
  if constexpr (sizeof(T) == 2) *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
  else *p = v;
}

constexpr int kLossThreads = 256;
constexpr int kMaxLossA = 16;

template <typename T>
__global__ void __launch_bounds__(kLossThreads) ppo_loss_kernel(
    const T* __restrict__ mean, int32_t mstride, const T* __restrict__ value, int32_t vstride,
    const float* __restrict__ log_std_raw, const float* __restrict__ act, const float* __restrict__ old_logp,
    const float* __restrict__ adv, const float* __restrict__ ret, int64_t B, int32_t A, float clip_eps,
    float value_coef, float ls_min, float ls_max, T* __restrict__ dmean, T* __restrict__ dvalue,
    float* __restrict__ acc) {
  constexpr float kHalfLog2Pi = 0.9189385332046727f;  // ppo.cpp:28
  __shared__ float s_red[kLossThreads / 32][4 + kMaxLossA];
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const float inv_n = 1.f / (float)B;
  float part[4 + kMaxLossA];
#pragma unroll
  for (int k = 0; k < 4 + kMaxLossA; ++k) part[k] = 0.f;
  if (j < B) {
    float logp = 0.f;
    for (int i = 0; i < A; ++i) {
      const float ls = fminf(fmaxf(log_std_raw[i], ls_min), ls_max);
      const float inv_var = __expf(-2.f * ls);
      const float diff = act[j * A + i] - ld(mean + j * mstride + i);
      logp += -0.5f * diff * diff * inv_var - ls - kHalfLog2Pi;
    }
    const float ratio = __expf(logp - old_logp[j]);
    const float a = adv[j];
    const float unclipped = ratio * a;
    const float clipped_obj = fminf(fmaxf(ratio, 1.f - clip_eps), 1.f + clip_eps) * a;
    part[0] = fminf(unclipped, clipped_obj);
    part[1] = old_logp[j] - logp;
    part[3] = fabsf(ratio - 1.f) > clip_eps ? 1.f : 0.f;
    // d(-surr)/dlogp; zero when the clipped branch is active (ties: unclipped)
    const float dl_dlogp = -inv_n * (unclipped <= clipped_obj ? unclipped : 0.f);
    for (int i = 0; i < A; ++i) {
      const float ls = fminf(fmaxf(log_std_raw[i], ls_min), ls_max);
      const float inv_var = __expf(-2.f * ls);
      const float diff = act[j * A + i] - ld(mean + j * mstride + i);
      st(dmean + j * mstride + i, dl_dlogp * diff * inv_var);
      if (i < kMaxLossA) part[4 + i] = dl_dlogp * (diff * diff * inv_var - 1.f);
    }
    for (int i = A; i < mstride; ++i) st(dmean + j * mstride + i, 0.f);  // padded columns
    const float verr = ld(value + j * vstride) - ret[j];
    part[2] = verr * verr;
    st(dvalue + j * vstride, value_coef * verr * inv_n);
    for (int i = 1; i < vstride; ++i) st(dvalue + j * vstride + i, 0.f);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 4 + kMaxLossA; ++k) {
    float v = part[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_red[w][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4 + A) {
    float v = 0.f;
    for (int k = 0; k < kLossThreads / 32; ++k) v += s_red[k][threadIdx.x];
    atomicAdd(acc + threadIdx.x, v);
  }
}

// out[0] loss, out[1..5] metrics {policy_loss, value_loss, entropy, kl,
// clip_fraction}; dls[A] = projected log-std gradient (ppo.cpp:140-149).
__global__ void ppo_loss_finalize(const float* __restrict__ acc, const float* __restrict__ log_std_raw, int64_t B,
                                  int32_t A, float value_coef, float entropy_coef, float ls_min, float ls_max,
                                  float* __restrict__ out, float* __restrict__ dls) {
  constexpr float kHalfLog2Pi = 0.9189385332046727f;
  const int i = threadIdx.x;
  float ent = 0.f;
  if (i < A) {
    const float raw = log_std_raw[i];
    const float ls = fminf(fmaxf(raw, ls_min), ls_max);
    ent = ls + 0.5f + kHalfLog2Pi;
    const float g = acc[4 + i] - entropy_coef;
    dls[i] = (raw < ls_min || raw > ls_max) ? 0.f : g;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ent += __shfl_xor_sync(0xffffffffu, ent, o);
  if (i == 0) {
    const float inv_n = 1.f / (float)B;
    const float policy_loss = -acc[0] * inv_n, value_loss = 0.5f * acc[2] * inv_n;
    out[0] = policy_loss + value_coef * value_loss - entropy_coef * ent;
    out[1] = policy_loss;
    out[2] = value_loss;
    out[3] = ent;
    out[4] = acc[1] * inv_n;
    out[5] = acc[3] * inv_n;
  }
}

}  // namespace

extern "C" int sg_ppo_loss(const void* d_mean, int32_t mstride, const void* d_value, int32_t vstride, int32_t dtype,
                           const float* d_log_std_raw, const float* d_act, const float* d_old_logp,
                           const float* d_adv, const float* d_ret, int64_t B, int32_t A, double clip_eps,
                           double value_coef, double entropy_coef, double ls_min, double ls_max, void* d_dmean,
                           void* d_dvalue, float* d_dlog_std, float* d_acc, float* d_out, void* stream) {
  if (A < 1 || A > kMaxLossA || A > mstride || vstride < 1) return SG_ERR_CONFIG;
  const cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(d_acc, 0, (4 + A) * sizeof(float), s);
  const unsigned grid = (unsigned)((B + kLossThreads - 1) / kLossThreads);
  if (dtype == 1)
    ppo_loss_kernel<__nv_bfloat16><<<grid, kLossThreads, 0, s>>>(
        (const __nv_bfloat16*)d_mean, mstride, (const __nv_bfloat16*)d_value, vstride, d_log_std_raw, d_act,
        d_old_logp, d_adv, d_ret, B, A, (float)clip_eps, (float)value_coef, (float)ls_min, (float)ls_max,
        (__nv_bfloat16*)d_dmean, (__nv_bfloat16*)d_dvalue, d_acc);
  else
    ppo_loss_kernel<float><<<grid, kLossThreads, 0, s>>>(
        (const float*)d_mean, mstride, (const float*)d_value, vstride, d_log_std_raw, d_act, d_old_logp, d_adv,
        d_ret, B, A, (float)clip_eps, (float)value_coef, (float)ls_min, (float)ls_max, (float*)d_dmean,
        (float*)d_dvalue, d_acc);
  ppo_loss_finalize<<<1, 32, 0, s>>>(d_acc, d_log_std_raw, B, A, (float)value_coef, (float)entropy_coef,
                                     (float)ls_min, (float)ls_max, d_out, d_dlog_std);
  return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_SIM;
}
