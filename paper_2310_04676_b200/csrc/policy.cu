// Policy MLP forward on the 5th-generation tensor cores (tcgen05 / TMEM).
//
// Reference: Policy::forward / trunk_forward (proj/src/policy.cpp:110-161):
// actor  obs -> 256 -> 128 -> 64 -> A  (ELU on hidden layers, policy.cpp:33)
// critic obs -> 256 -> 128 -> 64 -> 1
// flat fp64 parameter vector laid out actor (W_l [out x in] row-major, b_l)
// for l = 0..3, then critic, then log_std (policy.cpp:42-63).
//
// Device design (one CTA = one 128-row tile, 16 warps, 1 CTA per SM):
//  * weights are packed once per parameter update into bf16 images in the
//    UMMA K-major no-swizzle canonical layout; every CTA bulk-copies all of
//    them into shared memory at launch (cp.async.bulk -> UBLKCP, mbarrier
//    complete_tx; 200 KB, L2-resident across CTAs);
//  * every layer is tcgen05.mma.cta_group::1.kind::f16 (BF16 x BF16 -> FP32)
//    issued by one thread, M = 128, accumulators in TMEM (512 columns);
//  * activations never leave tensor memory: the epilogue reads its TMEM lane
//    (tcgen05.ld 32x32b), adds the bias, applies ELU, packs bf16 pairs and
//    writes them back with tcgen05.st as the next layer's A operand
//    (tcgen05.mma with A in TMEM); only the last layer's fp32 mean / value
//    leave the SM;
//  * L1 of actor and critic is issued together; then the actor (warps 0-7)
//    and the critic (warps 8-15) run as two pipelines with their own MMA
//    issuer, commit barrier and named barrier, the critic one epilogue
//    behind, so one trunk's MUFU-bound ELU overlaps the other's MMAs;
//  * fused rollout sampling: the fp64 Box-Muller draws run while layer 2 is
//    on the tensor cores; the actions / log-probs are formed from the mean
//    row in the kernel's tail.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sg_env.h"

namespace sgp {

constexpr int kRows = 128;  // UMMA M
constexpr int kK0 = 32;     // padded obs width
constexpr int kH1 = 256, kH2 = 128, kH3 = 64, kNOut = 16;  // kNOut: padded output width

// Shared-memory plan (bytes): every weight image stays resident (bulk-copied
// once per launch, L2-resident across CTAs); activations never touch shared
// memory -- they live in TMEM as the next layer's A operand. The X / W1 region
// is free once layer 1 has run and holds the fused sampling's scratch.
constexpr uint32_t kX0 = 0;                  // 128 x 32 bf16 obs tile
constexpr uint32_t kW1 = 8192;               // 512 x 32 bf16 (actor rows | critic rows)
constexpr uint32_t kW2a = 40960;             // 128 x 256 bf16
constexpr uint32_t kW2c = kW2a + 65536;      // 128 x 256 bf16
constexpr uint32_t kW34 = kW2c + 65536;      // W3a | W3c (64 x 128) | W4a | W4c (16 x 64)
constexpr uint32_t kW3a = kW34, kW3c = kW34 + 16384, kW4a = kW34 + 32768, kW4c = kW34 + 34816;
constexpr uint32_t kBar = kW34 + 36864;      // mbarriers + TMEM slot
constexpr uint32_t kBias = kBar + 128;       // 928 fp32 biases
constexpr uint32_t kSmem = kBias + 928 * 4;  // 212,736 B
constexpr int kThreads = 512;  // 16 warps: 2 trunks x 2 column halves x 4 TMEM lane quarters
constexpr int kGroups = kThreads / kRows;

// Packed parameter image (global): same byte layout as the smem regions.
struct PolicyImage {
  const uint8_t* w1;    // 32768 B
  const uint8_t* w2a;   // 65536 B
  const uint8_t* w2c;
  const uint8_t* w34;   // W3a | W3c | W4a | W4c, 36864 B
  const float* b1;      // 512 (actor | critic)
  const float* b2a;     // 128
  const float* b2c;
  const float* b3a;     // 64
  const float* b3c;
  const float* b4a;     // 16 (padded)
  const float* b4c;     // 16 (padded)
};

// Byte offset of element (r, k) in a K-major, no-swizzle UMMA tile with R
// rows: 8x(16 B) core matrices, 8-row groups contiguous (SBO = 128 B), K
// chunks of 8 elements R*16 B apart (LBO).
__host__ __device__ constexpr uint32_t kmajor_off(uint32_t r, uint32_t k, uint32_t R) {
  return (k >> 3) * (R * 16u) + (r >> 3) * 128u + (r & 7u) * 16u + (k & 7u) * 2u;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// kind::f16 instruction descriptor: BF16 x BF16 -> F32, both K-major.
__host__ __device__ constexpr uint32_t make_idesc(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(mbar),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void async_proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 16 consecutive fp32 accumulator columns of this thread's TMEM lane, issued
// without waiting (tcgen05.ld is asynchronous until tcgen05.wait::ld, which
// covers every load the thread issued before it).
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  tmem_ld16_async(taddr, r);
  tmem_wait_ld();
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(r[k]);
}

__device__ __forceinline__ float elu(float x) { return x > 0.f ? x : __expf(x) - 1.f; }  // policy.cpp:33

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ELU(acc + bias) (policy.cpp:33) of two adjacent columns -> one bf16x2 word:
// max(x, 2^min(x log2 e, 0) - 1) == (x > 0 ? x : e^x - 1) (e^x - 1 >= x), the
// column pair in packed fp32 ops (FADD2 / FMUL2), one MUFU.EX2 per value.
__device__ __forceinline__ uint32_t elu_pair(uint32_t a0, uint32_t a1, float2 b) {
  const float2 x = __fadd2_rn(make_float2(__uint_as_float(a0), __uint_as_float(a1)), b);
  const float2 t = __fmul2_rn(x, make_float2(1.4426950408889634f, 1.4426950408889634f));
  const float2 e =
      __fadd2_rn(make_float2(ex2_approx(fminf(t.x, 0.f)), ex2_approx(fminf(t.y, 0.f))), make_float2(-1.f, -1.f));
  return pack_bf16(fmaxf(x.x, e.x), fmaxf(x.y, e.y));
}

// The same on the FMA pipe: 2^t for t in [-127, 0] as 2^round(t) * p(t - round(t)),
// round by the 1.5 * 2^23 magic add, p a degree-5 fit of 2^f on [-0.5, 0.5]
// (max rel. error 1.9e-7 in fp32 Horner, like MUFU.EX2's ~2 ulp), the
// exponent added in the integer domain. Meant to move every kPolyEvery-th
// column pair off the MUFU pipe; measured slower (forward in a CUDA graph:
// all MUFU 10.11 us, every 8th pair 10.23, 4th 10.66, 3rd 10.87): the
// epilogues are issue / latency bound, not MUFU bound. Off by default.
#ifndef SG_ELU_POLY_EVERY
#define SG_ELU_POLY_EVERY 0
#endif
constexpr int kPolyEvery = SG_ELU_POLY_EVERY;  // 0: all MUFU
__device__ __forceinline__ uint32_t elu_pair_poly(uint32_t a0, uint32_t a1, float2 b) {
  const float2 x = __fadd2_rn(make_float2(__uint_as_float(a0), __uint_as_float(a1)), b);
  const float2 tl = __fmul2_rn(x, make_float2(1.4426950408889634f, 1.4426950408889634f));
  const float2 t = make_float2(fmaxf(fminf(tl.x, 0.f), -127.f), fmaxf(fminf(tl.y, 0.f), -127.f));
  const float2 y = __fadd2_rn(t, make_float2(12582912.f, 12582912.f));
  const float2 fi = __fadd2_rn(y, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(t, make_float2(-fi.x, -fi.y));
  float2 p = __ffma2_rn(f, make_float2(0.0013264729641377926f, 0.0013264729641377926f),
                        make_float2(0.009671512991189957f, 0.009671512991189957f));
  p = __ffma2_rn(p, f, make_float2(0.05550733581185341f, 0.05550733581185341f));
  p = __ffma2_rn(p, f, make_float2(0.24022242426872253f, 0.24022242426872253f));
  p = __ffma2_rn(p, f, make_float2(0.6931470036506653f, 0.6931470036506653f));
  p = __ffma2_rn(p, f, make_float2(1.f, 1.f));
  const float ex = __int_as_float(__float_as_int(p.x) + ((__float_as_int(y.x) - 0x4B400000) << 23));
  const float ey = __int_as_float(__float_as_int(p.y) + ((__float_as_int(y.y) - 0x4B400000) << 23));
  const float2 e = __fadd2_rn(make_float2(ex, ey), make_float2(-1.f, -1.f));
  return pack_bf16(fmaxf(x.x, e.x), fmaxf(x.y, e.y));
}

// Hidden-layer epilogue in tensor memory: this thread's NC accumulator
// columns [src, src + NC) of its TMEM lane -> ELU(acc + bias) -> bf16 pairs
// written to columns [dst, dst + NC/2) of the same lane, where the next
// layer's MMA reads them as its A operand (row = lane, two K elements per
// 32-bit column). Batches of 32 columns (REV: last batch first), the next
// batch's TMEM loads in flight while the current one is converted; a batch
// only overwrites columns that this thread has already read (packing in
// place: dst == src forward, or dst == src + NC/2 in reverse) or a disjoint
// range.
template <int NC, bool REV = false, bool STORE = false>
__device__ __forceinline__ void epi_tmem(uint32_t trow, uint32_t src, uint32_t dst, const float* __restrict__ bias,
                                         __nv_bfloat16* __restrict__ g = nullptr) {
  constexpr int NB = NC / 32;
  const auto bat = [](int j) { return REV ? NB - 1 - j : j; };
  uint32_t r[2][2][16];
  tmem_ld16_async(trow + src + 32 * bat(0), r[0][0]);
  tmem_ld16_async(trow + src + 32 * bat(0) + 16, r[0][1]);
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    tmem_wait_ld();
    if (j + 1 < NB) {
      tmem_ld16_async(trow + src + 32 * bat(j + 1), r[(j + 1) & 1][0]);
      tmem_ld16_async(trow + src + 32 * bat(j + 1) + 16, r[(j + 1) & 1][1]);
    }
    const int c = 32 * bat(j);
    uint32_t p[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      p[k] = (kPolyEvery > 0 && k % kPolyEvery == kPolyEvery - 1)
                 ? elu_pair_poly(r[j & 1][k >> 3][2 * (k & 7)], r[j & 1][k >> 3][2 * (k & 7) + 1],
                                 *reinterpret_cast<const float2*>(bias + c + 2 * k))
                 : elu_pair(r[j & 1][k >> 3][2 * (k & 7)], r[j & 1][k >> 3][2 * (k & 7) + 1],
                            *reinterpret_cast<const float2*>(bias + c + 2 * k));
    tmem_st16(trow + dst + c / 2, p);
    if constexpr (STORE) {  // the activations the backward pass needs: bf16 row segment of this thread
      if (g) {
#ifndef SG_STORE_V4
        // 32-byte stores (STG.E.ENL2.256): one full sector of the row per
        // instruction, half the L1 wavefronts of 16-byte stores
#pragma unroll
        for (int q = 0; q < 16; q += 8)
          asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(g + c + 2 * q), "r"(p[q]),
                       "r"(p[q + 1]), "r"(p[q + 2]), "r"(p[q + 3]), "r"(p[q + 4]), "r"(p[q + 5]), "r"(p[q + 6]),
                       "r"(p[q + 7])
                       : "memory");
#else
        uint4* gv = reinterpret_cast<uint4*>(g + c);
        gv[0] = make_uint4(p[0], p[1], p[2], p[3]);
        gv[1] = make_uint4(p[4], p[5], p[6], p[7]);
        gv[2] = make_uint4(p[8], p[9], p[10], p[11]);
        gv[3] = make_uint4(p[12], p[13], p[14], p[15]);
#endif
      }
    }
  }
}

// Issue one layer with A in shared memory: D[128 x N] (+)= A[128 x K] * B[N x K]^T, K in steps of 16.
__device__ __forceinline__ void issue_layer(uint32_t d_tmem, uint32_t a_addr, uint32_t a_rows, uint32_t b_addr,
                                            uint32_t b_rows, int K, int N) {
  const uint32_t idesc = make_idesc(kRows, N);
  const uint32_t lbo_a = a_rows * 16u, lbo_b = b_rows * 16u;
  for (int s = 0; s < K / 16; ++s) {
    const uint64_t a = make_desc(a_addr + 2u * s * lbo_a, lbo_a, 128u);
    const uint64_t b = make_desc(b_addr + 2u * s * lbo_b, lbo_b, 128u);
    mma_bf16(d_tmem, a, b, idesc, s > 0 ? 1u : 0u);
  }
}

// tcgen05.mma with the A operand in tensor memory (.kind::f16, BF16 x BF16 -> FP32).
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

// Issue one layer with A in TMEM: K-step s (16 elements = 8 packed columns)
// reads A at column a0 + 8 s for s < split, a1 + 8 (s - split) after (the
// epilogue's two column halves); B = N rows of a K-major image with row
// stride lbo (bytes between K chunks).
__device__ __forceinline__ void issue_layer_ts(uint32_t d_tmem, uint32_t a0, uint32_t a1, int split, uint32_t b_addr,
                                               uint32_t lbo, int K, int N) {
  const uint32_t idesc = make_idesc(kRows, N);
  for (int s = 0; s < K / 16; ++s) {
    const uint32_t a = s < split ? a0 + 8u * s : a1 + 8u * (s - split);
    mma_bf16_ts(d_tmem, a, make_desc(b_addr + 2u * s * lbo, lbo, 128u), idesc, s > 0 ? 1u : 0u);
  }
}

// ---- rollout sampling (ppo.cpp:262-277) ------------------------------------
// The reference draws z for (env e, dim i) from ONE trainer stream
// make_stream(seed, 0x7261696e) in row-major order, 2 u32 per Box-Muller
// normal. Each thread jumps its copy of that stream to draw
// pos + step_off + 2*(e*A + i) (O(log k) PCG32 jump table) so the device
// consumes exactly the reference's u32 sequence.
struct Jump64 {
  uint64_t mult[64];
  uint64_t add[64];
};

__device__ __forceinline__ uint32_t pcg32_next(uint64_t& s, uint64_t inc) {
  const uint64_t old = s;
  s = old * 6364136223846793005ULL + inc;
  const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u), rot = (uint32_t)(old >> 59u);
  return (xs >> rot) | (xs << ((32u - rot) & 31u));
}

// One (env, dim) draw of the rollout sampling at PCG32 state s (consumes 2
// u32), fp64 throughout like the reference: the standard normal z (Box-Muller,
// rng.hpp:53-57), the dim's log-prob term -z^2/2 - ls - log(2 pi)/2, and the
// action mean + exp(ls) z rounded once to fp32. z and the term depend on the
// stream and log-std only, so the fused kernel draws them before the MLP.
__device__ __forceinline__ double clamp_log_std(float log_std_raw) {
  const double ls = (double)log_std_raw;
  return ls < -5.0 ? -5.0 : (ls > 2.0 ? 2.0 : ls);  // Policy::log_std clamp (policy.hpp:28-29)
}
__device__ __forceinline__ double draw_normal(uint64_t& s, uint64_t inc) {
  const double u1 = __dmul_rn(__dadd_rn((double)pcg32_next(s, inc), 0.5), 0x1.0p-32);
  const double u2 = (double)pcg32_next(s, inc) * 0x1.0p-32;
  return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(6.283185307179586477, u2)));
}
__device__ __forceinline__ double logp_term(double z, double ls) {
  return __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(-0.5, z), z), -ls), -0.9189385332046727);
}
__device__ __forceinline__ float action_of(float mean, double z, double ls) {
  return (float)__dadd_rn((double)mean, __dmul_rn(exp(ls), z));
}
__device__ __forceinline__ float draw_action(uint64_t& s, uint64_t inc, float mean, float log_std_raw, double& term) {
  const double ls = clamp_log_std(log_std_raw);
  const double z = draw_normal(s, inc);
  term = logp_term(z, ls);
  return action_of(mean, z, ls);
}

// s0 advanced by k draws (J[b] = 2^b-step advance).
__device__ __forceinline__ uint64_t jump(uint64_t s0, uint64_t k, const Jump64& J) {
  uint64_t s = s0;
  for (int b = 0; k; ++b, k >>= 1)
    if (k & 1) s = s * J.mult[b] + J.add[b];
  return s;
}

// PCG32 state s0 advanced by k draws, computed by a whole warp: lane l takes
// the jumps of bits l and l + 32 of k, and the (commuting) affine maps are
// combined by a 5-round butterfly. Every lane returns the result.
__device__ __forceinline__ uint64_t jump_warp(uint64_t s0, uint64_t k, const Jump64& J) {
  const int lane = threadIdx.x & 31;
  uint64_t m = 1, a = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int b = lane + 32 * h;
    if ((k >> b) & 1) {
      const uint64_t M = J.mult[b], Ad = J.add[b];
      a = a * M + Ad;
      m *= M;
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const uint64_t m2 = __shfl_xor_sync(0xffffffffu, m, off), a2 = __shfl_xor_sync(0xffffffffu, a, off);
    a = a * m2 + a2;
    m *= m2;
  }
  return s0 * m + a;
}

struct FwdArgs {
  const float* obs;  // n x obs_stride fp32 (first obs_dim columns used)
  int64_t n;
  int32_t obs_dim;
  int32_t obs_stride;
  int32_t act_dim;
  float* mean;   // n x act_dim (may be null: value only)
  float* value;  // n
  // bootstrap mode (ppo.cpp:304-313): when set, only rows with
  // timed_out && !terminated get V(terminal obs); other rows get 0 and tiles
  // without such rows exit before any tensor-core work.
  const uint8_t* timed_out;
  const uint8_t* terminated;
  // fused rollout sampling (ppo.cpp:262-277), when actions != null: the
  // trainer-stream draws of every (row, dim) at pos + step_off + 2 (row A + dim)
  const float* log_std_raw;
  uint64_t s0, inc;
  const uint64_t* pos;
  uint64_t step_off;
  float* actions;
  float* logp;
  // precomputed sampling (sg_policy_noise), when non-null: actions =
  // (float)(mean + noise[row A + dim]); logp was written by the noise kernel
  const double* noise;
  // folded bootstrap of the PREVIOUS rollout step (ppo.cpp:304-313), when
  // boot_obs != null: boot_value[r] = V(boot_obs row r) for rows with
  // boot_timed_out && !boot_terminated, 0 elsewhere (what sg_policy_bootstrap
  // computes, without its own launch; tiles with no such row only write zeros)
  const float* boot_obs;
  int32_t boot_stride;
  const uint8_t* boot_timed_out;
  const uint8_t* boot_terminated;
  float* boot_value;
};

#ifdef SG_POLICY_PROBE
// Phase probe (A/B builds only): clock64 at each phase of CTA 0, printed by
// lane 0 of warps 0 / 4 / 8 / 12 (actor halves, critic halves).
#define PPROBE(k) (probe_t[k] = clock64())
#else
#define PPROBE(k) ((void)0)
#endif

// One CTA = one 128-row tile. Layer 1 of both trunks is issued together;
// then the actor (warps 0-7) and the critic (warps 8-15) run as two
// independent pipelines, each with its own MMA issuer (lane 0 of its first
// warp), commit mbarrier and named barrier, so one trunk's epilogue (TMEM ->
// ELU -> TMEM, MUFU / FMA pipes) overlaps the other trunk's MMAs. Warp w of
// a trunk reads TMEM lane quarter w % 4 and column half (w / 4) % 2.
//
// TMEM columns of trunk t (T = 256 t), fp32 accumulators / packed bf16 A:
//   L1 acc        [T, T+256)                     (N = 256)
//   A2 (h1)       [T, T+64) | [T+192, T+256)     (half 0 packs forward in place, half 1 backwards
//                                                 into the top of its range)
//   L2 acc        [T+64, T+192)                  (N = 128)
//   A3 (h2)       [T, T+64)
//   L3 acc        [T+64, T+128)                  (N = 64)
//   A4 (h3)       [T+128, T+160)
//   L4 acc        [T, T+16)                      (N = 16)
// The critic's first epilogue starts when the actor's is done: from then on
// one trunk's epilogue (MUFU-bound ELU) runs while the other trunk's MMAs do.
__global__ void __launch_bounds__(kThreads, 1) policy_fwd_kernel(const __grid_constant__ PolicyImage W,
                                                                 const __grid_constant__ FwdArgs args,
                                                                 const __grid_constant__ Jump64 J) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t row0 = (int64_t)blockIdx.x * kRows;
  const int row = tid & (kRows - 1);  // TMEM lane == tile row (lane quarter = warp % 4)
  const int group = tid / kRows;      // warp / 4: trunk * 2 + column half
  const int trunk = warp >> 3, half = (warp >> 2) & 1;
#ifdef SG_POLICY_PROBE
  long long probe_t[14] = {};
#endif
  PPROBE(0);
  bool boot_row = true;
  if (args.timed_out) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t r = row0 + row;
    boot_row = r < args.n && args.timed_out[r] && !args.terminated[r];
    if (!__syncthreads_or(group == 0 && boot_row)) {
      if (group == 0 && r < args.n) args.value[r] = 0.f;
      return;
    }
  }
  float* sbias = reinterpret_cast<float*>(smem + kBias);  // the 7 bias vectors, bulk-copied (contiguous)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kBar + 64);
  const uint32_t bar_bias = smem_u32(&bars[0]), bar_w1 = smem_u32(&bars[1]);
  const uint32_t bar_w2 = smem_u32(&bars[2 + trunk]), bar_w34 = smem_u32(&bars[4]);
  const uint32_t bar_mma = smem_u32(&bars[5 + trunk]);
  const uint32_t sbase = smem_u32(smem);

  if (tid == 0) {
    for (int b = 0; b < 7; ++b) mbar_init(smem_u32(&bars[b]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // TMEM: all 512 columns (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  PPROBE(11);
  if (tid == 0) {  // every weight image, in the order the layers need them, while the obs tile is converted
    bulk_load(sbase + kBias, W.b1, 928 * 4, smem_u32(&bars[0]));
    bulk_load(sbase + kW1, W.w1, 32768, smem_u32(&bars[1]));
    bulk_load(sbase + kW2a, W.w2a, 65536, smem_u32(&bars[2]));
    bulk_load(sbase + kW2c, W.w2c, 65536, smem_u32(&bars[3]));
    bulk_load(sbase + kW34, W.w34, 36864, smem_u32(&bars[4]));
  }
  // Launched with programmatic stream serialization (sg_policy_act* after an
  // env step): the set-up above (barriers, TMEM, the weight images -- written
  // by the trainer long before the rollout's env step) overlaps the env
  // step's last CTAs; everything below reads what the previous kernels wrote.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (warp == 1 && args.actions && !args.noise) {  // the trainer-stream state of this tile's first draw (row0, dim 0)
    const uint64_t s = jump_warp(args.s0, *args.pos + args.step_off + 2ull * (uint64_t)row0 * (uint64_t)args.act_dim, J);
    if ((tid & 31) == 0) *reinterpret_cast<uint64_t*>(smem + kBar + 72) = s;
  }
  // obs tile -> bf16 K-major [128 x 32] (zero padded rows / columns); thread
  // (row, group) converts the 8 columns of K chunk `group`
  {
    float x[8];
    const int c0 = group * 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = 0.f;
    if (row0 + row < args.n) {
      const float* src = args.obs + (row0 + row) * args.obs_stride;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (c0 + k < args.obs_dim) x[k] = __ldg(src + c0 + k);
    }
    uint4* d = reinterpret_cast<uint4*>(smem + kX0 + kmajor_off(row, c0, kRows));
    *d = make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]), pack_bf16(x[6], x[7]));
  }
  PPROBE(12);
  async_proxy_fence();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  PPROBE(1);
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t T = 256u * trunk;
  const bool issuer = (tid & 255) == 0;

  // ---- layer 1 of both trunks: [128 x 32] x [256 x 32]^T -> cols 0..255 | 256..511
  if (tid == 0) {
    mbar_wait(bar_w1, 0);
    tc_fence_after();
    issue_layer(tmem + 0, sbase + kX0, kRows, sbase + kW1, 512, kK0, 256);
    issue_layer(tmem + 256, sbase + kX0, kRows, sbase + kW1 + kmajor_off(256, 0, 512), 512, kK0, 256);
    mma_commit(smem_u32(&bars[5]));
    mma_commit(smem_u32(&bars[6]));
  }
  constexpr int kDraws = kNOut / kGroups;
  double zs[kDraws], terms[kDraws];
  const int64_t srow = row0 + row;
  const bool sampling = args.actions != nullptr && !args.noise && srow < args.n && group < args.act_dim;
  mbar_wait(bar_bias, 0);  // bulk-copied biases visible to this thread
  const float* b1 = sbias + 256 * trunk;
  const float* b2 = sbias + 512 + 128 * trunk;
  const float* b3 = sbias + 768 + 64 * trunk;
  const float* b4 = sbias + 896 + 16 * trunk;
  const auto trunk_sync = [&]() {  // named barrier of this trunk's 8 warps
    asm volatile("bar.sync %0, 256;" ::"r"(1 + trunk) : "memory");
  };
  const auto handoff = [&]() {  // this thread's TMEM stores -> the trunk's next MMA
    tmem_wait_st();
    tc_fence_before();
    trunk_sync();
  };

  // h1 = ELU(L1 + b1) -> A2
  mbar_wait(bar_mma, 0);
  tc_fence_after();
  PPROBE(2);
#ifndef SG_POLICY_NO_STAGGER
  if (trunk == 1) asm volatile("bar.sync 3, 512;" ::: "memory");
#endif
  if (half == 0)
    epi_tmem<128>(trow, T, T, b1);
  else
    epi_tmem<128, true>(trow, T + 128, T + 192, b1 + 128);
  handoff();
#ifndef SG_POLICY_NO_STAGGER
  if (trunk == 0) asm volatile("bar.arrive 3, 512;" ::: "memory");
#endif
  PPROBE(3);
  if (issuer) {  // layer 2: N = 128, K = 256 (A2 halves at T and T + 192)
    tc_fence_after();
    mbar_wait(bar_w2, 0);
    issue_layer_ts(tmem + T + 64, tmem + T, tmem + T + 192, 8, sbase + (trunk ? kW2c : kW2a), kH2 * 16, kH1, kH2);
    mma_commit(bar_mma);
  }
  // Fused sampling, stream part: the normals and log-prob terms of this
  // thread's (row, dim) draws depend on the trainer stream and the log-std
  // only, so they are drawn while layer 2 -- the longest MMA -- runs (dims
  // group, group + 4, ...: a <= 13-bit jump from the tile's first draw, then
  // + 8 draws per dim; fp64 Box-Muller like the reference).
  if (sampling) {
    const int A = args.act_dim;
    uint64_t st = jump(*reinterpret_cast<const uint64_t*>(smem + kBar + 72),
                       2ull * ((uint64_t)row * (uint64_t)A + (uint64_t)group), J);
#pragma unroll
    for (int j = 0; j < kDraws; ++j) {
      const int d = group + j * kGroups;
      zs[j] = terms[j] = 0.0;
      if (d < A) {
        uint64_t t = st;
        zs[j] = draw_normal(t, args.inc);
        terms[j] = logp_term(zs[j], clamp_log_std(args.log_std_raw[d]));
        st = st * J.mult[3] + J.add[3];
      }
    }
  }
  // h2 = ELU(L2 + b2) -> A3
  PPROBE(4);
  mbar_wait(bar_mma, 1);
  tc_fence_after();
  PPROBE(5);
  epi_tmem<64>(trow, T + 64 + 64 * half, T + 32 * half, b2 + 64 * half);
  handoff();
  PPROBE(6);
  if (issuer) {  // layer 3: N = 64, K = 128
    tc_fence_after();
    mbar_wait(bar_w34, 0);
    issue_layer_ts(tmem + T + 64, tmem + T, tmem + T, 8, sbase + (trunk ? kW3c : kW3a), kH3 * 16, kH2, kH3);
    mma_commit(bar_mma);
  }
  // h3 = ELU(L3 + b3) -> A4
  mbar_wait(bar_mma, 0);
  tc_fence_after();
  PPROBE(7);
  epi_tmem<32>(trow, T + 64 + 32 * half, T + 128 + 16 * half, b3 + 32 * half);
  handoff();
  if (issuer) {  // layer 4: N = 16, K = 64
    tc_fence_after();
    issue_layer_ts(tmem + T, tmem + T + 128, tmem + T + 128, 4, sbase + (trunk ? kW4c : kW4a), kNOut * 16, kH3, kNOut);
    mma_commit(bar_mma);
  }
  mbar_wait(bar_mma, 1);
  tc_fence_after();
  PPROBE(8);
  float mv[kNOut];  // the actor's output row (trunk 0, half 0), kept for the fused sampling
  if (half == 0) {
    float v[16];
    tmem_ld16(trow + T, v);
    if (trunk == 0) {
#pragma unroll
      for (int k = 0; k < kNOut; ++k) mv[k] = v[k] + b4[k];
      if (row0 + row < args.n && args.mean) {
        float* dst = args.mean + (row0 + row) * args.act_dim;
        for (int k = 0; k < args.act_dim; ++k) dst[k] = mv[k];
      }
    } else if (row0 + row < args.n) {
      args.value[row0 + row] = boot_row ? v[0] + b4[0] : 0.f;
    }
  }
  if (args.noise) {
    // precomputed sampling: the actor's output rows plus the scaled noise
    if (group == 0 && srow < args.n) {
      const int A = args.act_dim;
      const double* nz = args.noise + srow * A;
#pragma unroll
      for (int d = 0; d < kNOut; ++d)
        if (d < A) args.actions[srow * A + d] = (float)__dadd_rn((double)mv[d], nz[d]);
    }
  } else if (args.actions) {
    // Fused sampling, action part: the mean rows go to the (idle since layer 1)
    // X / W1 region, each thread forms the actions of its draws, the per-dim
    // log-prob terms meet there too and group 0 sums them in dim order -- the
    // same arithmetic as policy_sample_kernel.
    float* smean = reinterpret_cast<float*>(smem + kX0);           // 128 x 16 fp32
    double* sterm = reinterpret_cast<double*>(smem + kX0 + 8192);  // 128 x 16 fp64
    if (group == 0) {
#pragma unroll
      for (int k = 0; k < kNOut; ++k) smean[row * kNOut + k] = mv[k];
    }
    __syncthreads();
    const int A = args.act_dim;
    if (sampling) {
#pragma unroll
      for (int j = 0; j < kDraws; ++j) {
        const int d = group + j * kGroups;
        if (d < A) {
          args.actions[srow * A + d] = action_of(smean[row * kNOut + d], zs[j], clamp_log_std(args.log_std_raw[d]));
          sterm[row * kNOut + d] = terms[j];
        }
      }
    }
    __syncthreads();
    if (group == 0 && srow < args.n) {
      double lp = 0.0;
      for (int d = 0; d < A; ++d) lp = __dadd_rn(lp, sterm[row * kNOut + d]);
      args.logp[srow] = (float)lp;
    }
  }
  if (args.boot_obs) {
    // ---- folded bootstrap: the critic trunk again, on the previous step's
    // terminal rows (only in tiles that have a timed-out, non-terminated row)
    const int64_t r = row0 + row;
    const bool need = r < args.n && args.boot_timed_out[r] && !args.boot_terminated[r];
    tc_fence_before();
    if (!__syncthreads_or(group == 0 && need)) {
      if (group == 0 && r < args.n) args.boot_value[r] = 0.f;
    } else {
      // W1's smem was the sampling scratch: bulk-copy it again (phase 1 of its barrier)
      if (tid == 0) {
        async_proxy_fence();
        bulk_load(sbase + kW1, W.w1, 32768, bar_w1);
      }
      {
        float x[8];
        const int c0 = group * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = 0.f;
        if (r < args.n) {
          const float* src = args.boot_obs + r * args.boot_stride;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (c0 + k < args.obs_dim) x[k] = __ldg(src + c0 + k);
        }
        uint4* d = reinterpret_cast<uint4*>(smem + kX0 + kmajor_off(row, c0, kRows));
        *d = make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]), pack_bf16(x[6], x[7]));
      }
      async_proxy_fence();
      tc_fence_before();
      __syncthreads();
      tc_fence_after();
      if (trunk == 1) {
        if (issuer) {
          mbar_wait(bar_w1, 1);
          tc_fence_after();
          issue_layer(tmem + 256, sbase + kX0, kRows, sbase + kW1 + kmajor_off(256, 0, 512), 512, kK0, 256);
          mma_commit(bar_mma);
        }
        mbar_wait(bar_mma, 0);
        tc_fence_after();
        if (half == 0)
          epi_tmem<128>(trow, T, T, b1);
        else
          epi_tmem<128, true>(trow, T + 128, T + 192, b1 + 128);
        handoff();
        if (issuer) {
          tc_fence_after();
          issue_layer_ts(tmem + T + 64, tmem + T, tmem + T + 192, 8, sbase + kW2c, kH2 * 16, kH1, kH2);
          mma_commit(bar_mma);
        }
        mbar_wait(bar_mma, 1);
        tc_fence_after();
        epi_tmem<64>(trow, T + 64 + 64 * half, T + 32 * half, b2 + 64 * half);
        handoff();
        if (issuer) {
          tc_fence_after();
          issue_layer_ts(tmem + T + 64, tmem + T, tmem + T, 8, sbase + kW3c, kH3 * 16, kH2, kH3);
          mma_commit(bar_mma);
        }
        mbar_wait(bar_mma, 0);
        tc_fence_after();
        epi_tmem<32>(trow, T + 64 + 32 * half, T + 128 + 16 * half, b3 + 32 * half);
        handoff();
        if (issuer) {
          tc_fence_after();
          issue_layer_ts(tmem + T, tmem + T + 128, tmem + T + 128, 4, sbase + kW4c, kNOut * 16, kH3, kNOut);
          mma_commit(bar_mma);
        }
        mbar_wait(bar_mma, 1);
        tc_fence_after();
        if (half == 0) {
          float v[16];
          tmem_ld16(trow + T, v);
          if (r < args.n) args.boot_value[r] = need ? v[0] + b4[0] : 0.f;
        }
      }
    }
  }
  PPROBE(9);
  tc_fence_before();
  __syncthreads();
  PPROBE(10);
#ifdef SG_POLICY_PROBE
  if (blockIdx.x == 0 && (tid & 127) == 0)
    printf("pprobe warp %2d: init %lld obsld %lld sync %lld | obs %lld L1 %lld epi1 %lld draws %lld L2 %lld epi2 %lld L3 %lld epi3+L4 %lld out %lld end %lld\n",
           warp, probe_t[11] - probe_t[0], probe_t[12] - probe_t[11], probe_t[1] - probe_t[12],
           probe_t[1] - probe_t[0], probe_t[2] - probe_t[1], probe_t[3] - probe_t[2], probe_t[4] - probe_t[3],
           probe_t[5] - probe_t[4], probe_t[6] - probe_t[5], probe_t[7] - probe_t[6], probe_t[8] - probe_t[7],
           probe_t[9] - probe_t[8], probe_t[10] - probe_t[0]);
#endif
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---- training forward: the PPO update's minibatch forward ---------------------
// The update (ppo.cpp:157-224) runs Policy::forward on 131,072-row minibatches
// and backpropagates through it. This kernel is the rollout forward made
// persistent (one CTA per SM loops over 128-row tiles; weights, barriers and
// TMEM set up once) with bf16 observation rows in, and every hidden
// activation the backward pass needs stored as it is packed for the next
// layer: h1 / h2 / h3 of both trunks (bf16, row-major [trunk][n][width]) and
// the padded last-layer outputs (bf16 [trunk][n][8]: actor mean, critic
// value in column 0). Same arithmetic as the library path it replaces (bf16
// operands, fp32 accumulation, bias + ELU in fp32, one rounding to bf16).
struct TrainFwdArgs {
  const __nv_bfloat16* obs;  // n x obs_stride bf16 (the first 32 columns, zero padded)
  int64_t n;
  int32_t obs_stride;
  __nv_bfloat16* h1;   // [2][n][256]
  __nv_bfloat16* h2;   // [2][n][128]
  __nv_bfloat16* h3;   // [2][n][64]
  __nv_bfloat16* out;  // [2][n][8]
};

__global__ void __launch_bounds__(kThreads, 1) policy_train_fwd_kernel(const __grid_constant__ PolicyImage W,
                                                                       const __grid_constant__ TrainFwdArgs args) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & (kRows - 1);
  const int group = tid / kRows;
  const int trunk = warp >> 3, half = (warp >> 2) & 1;
  float* sbias = reinterpret_cast<float*>(smem + kBias);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kBar + 64);
  const uint32_t bar_bias = smem_u32(&bars[0]), bar_w1 = smem_u32(&bars[1]);
  const uint32_t bar_w2 = smem_u32(&bars[2 + trunk]), bar_w34 = smem_u32(&bars[4]);
  const uint32_t bar_mma = smem_u32(&bars[5 + trunk]);
  const uint32_t sbase = smem_u32(smem);
  if (tid == 0) {
    for (int b = 0; b < 7; ++b) mbar_init(smem_u32(&bars[b]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (tid == 0) {
    bulk_load(sbase + kBias, W.b1, 928 * 4, smem_u32(&bars[0]));
    bulk_load(sbase + kW1, W.w1, 32768, smem_u32(&bars[1]));
    bulk_load(sbase + kW2a, W.w2a, 65536, smem_u32(&bars[2]));
    bulk_load(sbase + kW2c, W.w2c, 65536, smem_u32(&bars[3]));
    bulk_load(sbase + kW34, W.w34, 36864, smem_u32(&bars[4]));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t T = 256u * trunk;
  const bool issuer = (tid & 255) == 0;
  const float* b1 = sbias + 256 * trunk;
  const float* b2 = sbias + 512 + 128 * trunk;
  const float* b3 = sbias + 768 + 64 * trunk;
  const float* b4 = sbias + 896 + 16 * trunk;
  const int64_t n = args.n;
  const auto trunk_sync = [&]() { asm volatile("bar.sync %0, 256;" ::"r"(1 + trunk) : "memory"); };
  const auto handoff = [&]() {
    tmem_wait_st();
    tc_fence_before();
    trunk_sync();
  };
  const int64_t tiles = (n + kRows - 1) / kRows;
  // obs tile: thread (row, group) copies K chunk `group` (8 bf16 = 16 B); the
  // next tile's chunk is loaded into registers while this tile computes
  const auto load_obs = [&](int64_t tile) {
    const int64_t rr = tile * kRows + row;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (tile < tiles && rr < n) v = *reinterpret_cast<const uint4*>(args.obs + rr * args.obs_stride + 8 * group);
    return v;
  };
  uint4 obs_next = load_obs(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t row0 = tile * kRows, r = row0 + row;
    const bool valid = r < n;
    *reinterpret_cast<uint4*>(smem + kX0 + kmajor_off(row, 8 * group, kRows)) = obs_next;
    obs_next = load_obs(tile + gridDim.x);
    async_proxy_fence();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      mbar_wait(bar_w1, 0);
      tc_fence_after();
      issue_layer(tmem + 0, sbase + kX0, kRows, sbase + kW1, 512, kK0, 256);
      issue_layer(tmem + 256, sbase + kX0, kRows, sbase + kW1 + kmajor_off(256, 0, 512), 512, kK0, 256);
      mma_commit(smem_u32(&bars[5]));
      mma_commit(smem_u32(&bars[6]));
    }
    mbar_wait(bar_bias, 0);
    const int64_t tr = trunk * n + r;  // activation row of this thread
    // h1 -> A2 (+ global)
    mbar_wait(bar_mma, 0);
    tc_fence_after();
#ifndef SG_TRAIN_NO_STAGGER
    if (trunk == 1) asm volatile("bar.sync 3, 512;" ::: "memory");
#endif
    if (half == 0)
      epi_tmem<128, false, true>(trow, T, T, b1, valid ? args.h1 + tr * 256 : nullptr);
    else
      epi_tmem<128, true, true>(trow, T + 128, T + 192, b1 + 128, valid ? args.h1 + tr * 256 + 128 : nullptr);
    handoff();
#ifndef SG_TRAIN_NO_STAGGER
    if (trunk == 0) asm volatile("bar.arrive 3, 512;" ::: "memory");
#endif
    if (issuer) {
      tc_fence_after();
      mbar_wait(bar_w2, 0);
      issue_layer_ts(tmem + T + 64, tmem + T, tmem + T + 192, 8, sbase + (trunk ? kW2c : kW2a), kH2 * 16, kH1, kH2);
      mma_commit(bar_mma);
    }
    // h2 -> A3 (+ global)
    mbar_wait(bar_mma, 1);
    tc_fence_after();
    epi_tmem<64, false, true>(trow, T + 64 + 64 * half, T + 32 * half, b2 + 64 * half,
                              valid ? args.h2 + tr * 128 + 64 * half : nullptr);
    handoff();
    if (issuer) {
      tc_fence_after();
      mbar_wait(bar_w34, 0);
      issue_layer_ts(tmem + T + 64, tmem + T, tmem + T, 8, sbase + (trunk ? kW3c : kW3a), kH3 * 16, kH2, kH3);
      mma_commit(bar_mma);
    }
    // h3 -> A4 (+ global)
    mbar_wait(bar_mma, 0);
    tc_fence_after();
    epi_tmem<32, false, true>(trow, T + 64 + 32 * half, T + 128 + 16 * half, b3 + 32 * half,
                              valid ? args.h3 + tr * 64 + 32 * half : nullptr);
    handoff();
    if (issuer) {
      tc_fence_after();
      issue_layer_ts(tmem + T, tmem + T + 128, tmem + T + 128, 4, sbase + (trunk ? kW4c : kW4a), kNOut * 16, kH3,
                     kNOut);
      mma_commit(bar_mma);
    }
    mbar_wait(bar_mma, 1);
    tc_fence_after();
    if (half == 0) {  // padded last-layer outputs (8 columns)
      float v[16];
      tmem_ld16(trow + T, v);
      if (valid) {
        uint4 o;
        o.x = pack_bf16(v[0] + b4[0], v[1] + b4[1]);
        o.y = pack_bf16(v[2] + b4[2], v[3] + b4[3]);
        o.z = pack_bf16(v[4] + b4[4], v[5] + b4[5]);
        o.w = pack_bf16(v[6] + b4[6], v[7] + b4[7]);
        *reinterpret_cast<uint4*>(args.out + tr * 8) = o;
      }
    }
    tc_fence_before();
    __syncthreads();  // every TMEM read of this tile is done before the next tile's layer 1
    tc_fence_after();
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---- fused data gradient + ELU derivative (the update's backward) ---------
// Policy::backward (policy.cpp:163-218) through one hidden layer of the PPO
// update's minibatch: dZ = (dY W) * ELU'(h), ELU'(h) = h > 0 ? 1 : h + 1 (from
// the stored output h), as one persistent tensor-core kernel instead of a
// library GEMM that writes dY W in bf16 plus an elementwise pass that reads it
// back: D[128 x N] = dY_tile [128 x KP] x (W^T)[N x KP]^T in TMEM (fp32),
// multiplied by ELU'(h) in the epilogue and rounded once to bf16.
// W^T is packed per minibatch into a K-major image (policy_pack_wt_kernel).
struct DgradArgs {
  const __nv_bfloat16* dy;  // [m x k], row stride dy_stride
  int32_t dy_stride;
  int32_t k;
  const uint8_t* wt;        // W^T image [N x KP] bf16, K-major canonical
  const __nv_bfloat16* h;   // [m x N]
  __nv_bfloat16* dz;        // [m x N]
  int64_t m;
};

#ifndef SG_DGRAD_CTAS
#define SG_DGRAD_CTAS 2
#endif
constexpr int kDgradCtas = SG_DGRAD_CTAS;  // CTAs per SM (one's epilogue overlaps the other's loads / MMA)

template <int N, int KP>
__global__ void __launch_bounds__(256, kDgradCtas) policy_dgrad_elu_kernel(const __grid_constant__ DgradArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr uint32_t kBBytes = N * KP * 2, kABytes = kRows * KP * 2;
  constexpr uint32_t kA = kBBytes, kBarOff = kA + kABytes;
  constexpr int kChunks = kRows * KP / 8 / 256;  // 16-byte A chunks per thread per tile
  constexpr uint32_t kCols = N < 32 ? 32 : N;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + kBarOff + 16);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_b = smem_u32(&bars[0]), bar_mma = smem_u32(&bars[1]);
  if (tid == 0) {
    mbar_init(bar_b, 1);
    mbar_init(bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (tid == 0) bulk_load(sbase, a.wt, kBBytes, bar_b);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const int half = warp >> 2;
  const int64_t tiles = (a.m + kRows - 1) / kRows;
  const auto load_a = [&](int64_t tile, uint4 (&v)[kChunks]) {
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      const int c = tid + 256 * j, row = c % kRows, kc = c / kRows;
      const int64_t r = tile * kRows + row;
      v[j] = make_uint4(0u, 0u, 0u, 0u);
      if (tile < tiles && r < a.m && kc * 8 < a.k)
        v[j] = *reinterpret_cast<const uint4*>(a.dy + r * a.dy_stride + kc * 8);
    }
  };
  uint4 nxt[kChunks];
  load_a(blockIdx.x, nxt);
  uint32_t phase = 0;
  bool first = true;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      const int c = tid + 256 * j, row = c % kRows, kc = c / kRows;
      *reinterpret_cast<uint4*>(smem + kA + kmajor_off(row, kc * 8, kRows)) = nxt[j];
    }
    load_a(tile + gridDim.x, nxt);  // the next tile's rows are in flight during this tile
    async_proxy_fence();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      if (first) mbar_wait(bar_b, 0);
      tc_fence_after();
      issue_layer(tmem, sbase + kA, kRows, sbase, N, KP, N);
      mma_commit(bar_mma);
    }
    first = false;
    mbar_wait(bar_mma, phase);
    phase ^= 1;
    tc_fence_after();
    const int64_t r = tile * kRows + (warp & 3) * 32 + lane;
#pragma unroll
    for (int cb = 0; cb < N / 2; cb += 16) {
      const int c = half * (N / 2) + cb;
      uint32_t d[16];
      tmem_ld16_async(trow + c, d);
      uint4 hv[2] = {};
      if (r < a.m) {
        const uint4* hp = reinterpret_cast<const uint4*>(a.h + r * N + c);
        hv[0] = hp[0];
        hv[1] = hp[1];
      }
      tmem_wait_ld();
      if (r < a.m) {
        uint4 o[2];
        uint32_t* ow = reinterpret_cast<uint32_t*>(o);
        const uint32_t* hw = reinterpret_cast<const uint32_t*>(hv);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hw[q]));
          const float gx = hf.x > 0.f ? 1.f : hf.x + 1.f, gy = hf.y > 0.f ? 1.f : hf.y + 1.f;
          ow[q] = pack_bf16(__uint_as_float(d[2 * q]) * gx, __uint_as_float(d[2 * q + 1]) * gy);
        }
        uint4* zp = reinterpret_cast<uint4*>(a.dz + r * N + c);
        zp[0] = o[0];
        zp[1] = o[1];
      }
    }
    tc_fence_before();
    __syncthreads();  // A smem and the TMEM accumulator are reused by the next tile
    tc_fence_after();
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
}

struct WtTable {
  int64_t w_off[6];   // flat offset of W [K x N] row-major (trunk * 3 + layer 1..3)
  int32_t k[6], n[6], kp[6];
  int64_t img_off[6];  // byte offset of the image
  int64_t total;       // elements over all images
};

// W^T images for policy_dgrad_elu_kernel: element (n, k) = W[k][n] (0 for
// k >= K), bf16, K-major canonical over KP columns.
__global__ void policy_pack_wt_kernel(const float* __restrict__ flat, const __grid_constant__ WtTable t,
                                      uint8_t* __restrict__ out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= t.total) return;
  int i = 0;
  while (e >= (int64_t)t.n[i] * t.kp[i]) {
    e -= (int64_t)t.n[i] * t.kp[i];
    ++i;
  }
  const int nn = (int)(e / t.kp[i]), kk = (int)(e % t.kp[i]);
  const float v = kk < t.k[i] ? flat[t.w_off[i] + (int64_t)kk * t.n[i] + nn] : 0.f;
  *reinterpret_cast<__nv_bfloat16*>(out + t.img_off[i] + kmajor_off(nn, kk, t.n[i])) = __float2bfloat16_rn(v);
}

// ---- weight gradients of the update (dW = dY^T X over the minibatch) --------
// Policy::backward's dW (policy.cpp:163-218) reduces over all 131,072 rows of
// a minibatch; as library GEMMs that is a split-K GEMM + reduction per layer
// and trunk at ~25-30 us each whatever the shape. Here: each CTA takes a
// contiguous slice of rows, streams 64-row stages of dY [rows x out] and X
// [rows x in] into shared memory with cp.async -- 16-byte pieces of rows are
// exactly the rows of the UMMA *MN-major* canonical layout (8 MN elements x 8
// K rows per core matrix), so no transpose -- and accumulates
// dW[out x in] = dY^T X with tcgen05.mma (A = dY^T, B = X^T, both MN-major) in
// TMEM over its slice; the per-CTA partials are summed by a second kernel.
// out is padded to 128 (or 256) MMA rows with zero A rows.
__host__ __device__ constexpr uint32_t mnmajor_off(uint32_t mn, uint32_t k, uint32_t MN) {
  return (k >> 3) * (MN * 16u) + (mn >> 3) * 128u + (k & 7u) * 16u + (mn & 7u) * 2u;
}
__host__ __device__ constexpr uint32_t make_idesc_mn(uint32_t M, uint32_t N) {  // BF16 x BF16 -> F32, A and B MN-major
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}

struct WgradArgs {
  const __nv_bfloat16* dy;  // [m x out] row-major
  const __nv_bfloat16* x;   // [m x in] row-major
  int64_t m;
  int64_t rows_per_cta;     // multiple of the 64-row stage
  float* partial;           // [gridDim.x][out][in]
};

#ifndef SG_WGRAD_STAGES
#define SG_WGRAD_STAGES 4
#endif
constexpr int kWgradStages = SG_WGRAD_STAGES;

template <int OUT, int IN>
__global__ void __launch_bounds__(128, 1) policy_wgrad_kernel(const __grid_constant__ WgradArgs a) {
  constexpr int MP = OUT <= 128 ? 128 : 256, MT = MP / 128;  // padded MMA rows, M tiles
  constexpr int S = 64;                                      // rows per stage (4 K-steps)
  constexpr int NS = kWgradStages;                           // stages in flight
  constexpr uint32_t kA = MP * S * 2, kB = IN * S * 2, kStage = kA + kB;
  constexpr uint32_t kCols = MT * IN < 32 ? 32 : (MT * IN <= 64 ? 64 : (MT * IN <= 128 ? 128 : (MT * IN <= 256 ? 256 : 512)));
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * kStage);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + NS * kStage + 8 * NS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem);
  if (tid == 0) {
    for (int b = 0; b < NS; ++b) mbar_init(smem_u32(&bars[b]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // zero both stages once: the padded A rows (out..MP) are never written again
  for (uint32_t o = tid * 16; o < NS * kStage; o += 128 * 16) *reinterpret_cast<uint4*>(smem + o) = make_uint4(0, 0, 0, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int64_t r_begin = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t r_end = min(a.m, r_begin + a.rows_per_cta);
  const int stages = r_begin < r_end ? (int)((r_end - r_begin + S - 1) / S) : 0;
  // stage loader: dY rows -> A (MN = out), X rows -> B (MN = in); 16-byte
  // pieces (8 consecutive out / in values of one row) are MN-major core rows
  const auto load = [&](int st, int buf) {
    const int64_t r0 = r_begin + (int64_t)st * S;
    const uint32_t base = sbase + buf * kStage;
    constexpr int kPa = S * OUT / 8, kPb = S * IN / 8;  // 16-byte pieces per stage
    // piece p -> row (p / (8 * W8)) * 8 + p % 8, column block (p / 8) % W8:
    // consecutive threads fill consecutive 16-byte rows of one core matrix
    // (conflict-free shared stores; 8 rows x 64 bytes per warp from global)
    for (int p = tid; p < kPa; p += 128) {
      constexpr int W8 = OUT / 8;
      const int r = (p / (8 * W8)) * 8 + (p & 7), o8 = (p >> 3) % W8;
      const int64_t gr = r0 + r;
      const bool ok = gr < r_end;
      cp_async16(base + mnmajor_off(o8 * 8, r, MP), a.dy + (ok ? gr : 0) * OUT + o8 * 8, ok);
    }
    for (int p = tid; p < kPb; p += 128) {
      constexpr int W8 = IN / 8;
      const int r = (p / (8 * W8)) * 8 + (p & 7), i8 = (p >> 3) % W8;
      const int64_t gr = r0 + r;
      const bool ok = gr < r_end;
      cp_async16(base + kA + mnmajor_off(i8 * 8, r, IN), a.x + (ok ? gr : 0) * IN + i8 * 8, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  uint32_t phase[NS] = {};
  for (int st = 0; st < NS && st < stages; ++st) load(st, st);
  for (int st = 0; st < stages; ++st) {
    const int buf = st % NS;
    // stage st has landed once at most (issued after it) groups are pending:
    // stages issued so far = min(stages, NS + max(st - 1, 0))
    const int issued = min(stages, NS + (st > 0 ? st - 1 : 0));
    const int after = issued - st - 1;
    if (after >= 3) asm volatile("cp.async.wait_group 3;" ::: "memory");
    else if (after == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else if (after == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    async_proxy_fence();  // this thread's cp.async data -> the tensor core's (async proxy) reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      const uint32_t A = sbase + buf * kStage, B = A + kA;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int ks = 0; ks < S / 16; ++ks) {
          const uint64_t da = make_desc(A + mt * 16 * 128 + 2u * ks * (MP * 16), MP * 16, 128);
          const uint64_t db = make_desc(B + 2u * ks * (IN * 16), IN * 16, 128);
          mma_bf16(tmem + mt * IN, da, db, make_idesc_mn(128, IN), (st > 0 || ks > 0) ? 1u : 0u);
        }
      mma_commit(smem_u32(&bars[buf]));
    }
    // refill the PREVIOUS stage's buffer (its MMAs were issued an iteration
    // ago) with stage st - 1 + NS; this stage's MMAs run meanwhile
    if (st >= 1 && st - 1 + NS < stages) {
      const int pb = (st - 1) % NS;
      mbar_wait(smem_u32(&bars[pb]), phase[pb]);
      phase[pb] ^= 1;
      load(st - 1 + NS, pb);
    }
  }
  if (stages > 0) {  // the last stage's commit covers every MMA of this CTA
    const int last = (stages - 1) % NS;
    mbar_wait(smem_u32(&bars[last]), phase[last]);
  }
  tc_fence_after();
  // epilogue: this CTA's partial dW (zero for an empty slice)
  float* dst = a.partial + (int64_t)blockIdx.x * OUT * IN;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int o = mt * 128 + warp * 32 + lane;
#pragma unroll
    for (int c = 0; c < IN; c += 16) {
      float v[16];
      tmem_ld16(trow + mt * IN + c, v);
      if (o < OUT) {
        float4* d4 = reinterpret_cast<float4*>(dst + (int64_t)o * IN + c);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          d4[q] = stages > 0 ? make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3])
                             : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
  }
}

// The same reduction fed by TMA for the wide layers (OUT, IN multiples of 64):
// one 2-D tensor-map box per 64-column block and 64-row stage, written by
// the TMA unit with the 128-byte swizzle, which is the UMMA MN-major
// SWIZZLE_128B canonical layout (64 MN elements per 128-byte row, 8-row
// groups 1 KB apart: SBO = 1 KB; the next 64-column block = the next box,
// LBO = 8 KB). One thread issues the TMA boxes and the MMAs (a 4-stage
// full / empty mbarrier ring); all warps drain TMEM at the end.
// swizzled UMMA smem descriptor; layout type 2 = SWIZZLE_128B, 4 = SWIZZLE_64B
__device__ __forceinline__ uint64_t make_desc_sw(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t type) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  d |= (uint64_t)type << 61;
  return d;
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}

template <int OUT, int IN, bool ATOMIC>
__global__ void __launch_bounds__(128, 1) policy_wgrad_tma_kernel(const __grid_constant__ CUtensorMap mdy,
                                                                  const __grid_constant__ CUtensorMap mx,
                                                                  const __grid_constant__ WgradArgs a) {
  constexpr int MP = OUT <= 128 ? 128 : 256, MT = MP / 128;
  constexpr int S = 64, NS = 4;
  constexpr uint32_t kBox = S * 128;  // one 64-column x 64-row box (128-byte swizzle)
  constexpr int BW = IN >= 64 ? 64 : IN;  // B box width: 64 (SWIZZLE_128B) or 32 (SWIZZLE_64B)
  constexpr uint32_t kBoxB = S * BW * 2, kRowB = BW * 2;
  constexpr uint32_t kSwB = BW == 64 ? 2u : 4u;
  constexpr uint32_t kA = (OUT / 64) * kBox, kB = (IN / BW) * kBoxB, kStage = kA + kB;
  static_assert(OUT % 64 == 0 && (IN % 64 == 0 || IN == 32), "TMA path: 64-column blocks (or one 32-column B)");
  constexpr uint32_t kCols = MT * IN <= 64 ? 64 : (MT * IN <= 128 ? 128 : (MT * IN <= 256 ? 256 : 512));
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // 1 KB alignment for the swizzle
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * kStage);  // full[NS] | empty[NS]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + NS * kStage + 16 * NS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem);
  if (tid == 0) {
    for (int b = 0; b < 2 * NS; ++b) mbar_init(smem_u32(&bars[b]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mdy)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mx)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int64_t r_begin = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t r_end = min(a.m, r_begin + a.rows_per_cta);
  const int stages = r_begin < r_end ? (int)((r_end - r_begin + S - 1) / S) : 0;
  if (tid == 0 && stages > 0) {
    const auto issue = [&](int st, int buf) {  // rows beyond m are zero-filled by the TMA unit
      const uint32_t base = sbase + buf * kStage, full = smem_u32(&bars[buf]);
      const int row = (int)(r_begin + (int64_t)st * S);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full), "r"(kStage) : "memory");
#pragma unroll
      for (int b = 0; b < OUT / 64; ++b) tma_load_2d(base + b * kBox, &mdy, b * 64, row, full);
#pragma unroll
      for (int b = 0; b < IN / BW; ++b) tma_load_2d(base + kA + b * kBoxB, &mx, b * BW, row, full);
    };
    uint32_t fph[NS] = {}, eph[NS] = {};
    for (int st = 0; st < NS && st < stages; ++st) issue(st, st);
    for (int st = 0; st < stages; ++st) {
      const int buf = st % NS;
      mbar_wait(smem_u32(&bars[buf]), fph[buf]);
      fph[buf] ^= 1;
      tc_fence_after();
      const uint32_t A = sbase + buf * kStage, B = A + kA;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int ks = 0; ks < S / 16; ++ks)
          mma_bf16(tmem + mt * IN, make_desc_sw(A + mt * 2 * kBox + ks * 2048, kBox, 1024, 2),
                   make_desc_sw(B + ks * 16 * kRowB, kBoxB, 8 * kRowB, kSwB), make_idesc_mn(128, IN),
                   (st > 0 || ks > 0) ? 1u : 0u);
      mma_commit(smem_u32(&bars[NS + buf]));
      if (st >= 1 && st - 1 + NS < stages) {  // refill the previous stage's buffer
        const int pb = (st - 1) % NS;
        mbar_wait(smem_u32(&bars[NS + pb]), eph[pb]);
        eph[pb] ^= 1;
        issue(st - 1 + NS, pb);
      }
    }
    const int last = (stages - 1) % NS;  // its commit covers every MMA
    mbar_wait(smem_u32(&bars[NS + last]), eph[last]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // ATOMIC: add this CTA's slice sum straight into the (zeroed) gradient
  // with vector reductions; else write the partial for the reduction pass
  float* dst = ATOMIC ? a.partial : a.partial + (int64_t)blockIdx.x * OUT * IN;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int o = mt * 128 + warp * 32 + lane;
#pragma unroll 4
    for (int c = 0; c < IN; c += 16) {
      float v[16];
      tmem_ld16(trow + mt * IN + c, v);
      if (o < OUT) {
        float* row = dst + (int64_t)o * IN + c;
        if constexpr (ATOMIC) {
          if (stages > 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + 4 * q), "f"(v[4 * q]),
                           "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3])
                           : "memory");
          }
        } else {
          float4* d4 = reinterpret_cast<float4*>(row);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            d4[q] = stages > 0 ? make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3])
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
  }
}

// The whole backward through one hidden layer l in one launch
// (Policy::backward, policy.cpp:163-218), per 128-row tile:
//   dZ_{l-1} = (dY_l W_l) * ELU'(h)        (MMA 1: A = dY tile, B = W^T image)
//   dW_l^T  += h^T dY_l                     (MMA 2, accumulated in TMEM over the CTA's tiles)
//   db_{l-1} += 1^T dZ_{l-1}                (column sums, per CTA in registers)
// h = x_l is both the ELU' argument and the weight-gradient operand. Its
// rows arrive as 128-row x 64-column TMA boxes with the 128-byte swizzle --
// the UMMA MN-major SWIZZLE_128B layout, so MMA 2 reads h^T straight from
// them (SBO = 1 KB per 8 rows, LBO = one box) -- and MMA 2's B operand is
// the dY tile as staged for MMA 1: its 8 x 16-byte core matrices hold 8
// rows x 8 dY columns, which read as N-contiguous (MN-major, no swizzle)
// core matrices with K (row) blocks 128 B apart and N blocks 2 KB apart.
// The epilogue turns each thread's (row's) TMEM accumulators and the h
// values it reads back from shared memory into dZ in place, and one thread
// stores the boxes with TMA -- coalesced both ways, where the per-row 16-byte
// global accesses of policy_dgrad_elu_kernel touch 32 rows per instruction.
// At the end the CTA adds its dW_l^T (lane = input column, TMEM column =
// output row) into the fp32 gradient with coalesced reductions (lanes =
// consecutive inputs). colsum / wgrad nullable.
__device__ __forceinline__ uint32_t sw128_off(uint32_t r, uint32_t c) {  // (row, column) in a 128 x 64 bf16 box
  return r * 128u + ((((c >> 3) ^ (r & 7u)) & 7u) << 4) + (c & 7u) * 2u;
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
}

//
// L0 (the 256-wide layer 1 only): the input layer's weight gradient too --
// dW_0 += dZ_0^T x_0 with dZ_0 read back from the boxes it was written into
// (MN-major SWIZZLE_128B) and the tile's x_0 (obs, 32 columns) as one more
// TMA box (SWIZZLE_64B) -- so dZ_0 never goes to HBM. TMEM then holds
// dW_1^T (256 columns) and dW_0 (64) besides the per-tile accumulator,
// which shrinks to 128 columns: the tile's two column halves of dY W run
// one after the other.
// Column sums of an N-column bf16 tile held as 128-row x 64-column SW128
// boxes: thread tid owns 8 consecutive columns (one 16-byte piece per row)
// of every (256 / (N / 8))-th row, so a warp's load covers whole 128-byte box
// rows (conflict-free) and each thread adds 8 columns per load; acc carries
// the partial sums across tiles (one atomic per column per thread at the end).
template <int N>
__device__ __forceinline__ void boxes_colsum8(const uint8_t* boxes, int tid, float (&acc)[8]) {
  constexpr int CG = N / 8, RG = 256 / CG, RPT = kRows / RG;
  const int cg = tid % CG, rg = tid / CG, g = cg & 7;
  const uint8_t* box = boxes + (cg >> 3) * (kRows * 128);
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int r = rg + RG * j;
    const uint4 v = *reinterpret_cast<const uint4*>(box + r * 128 + ((g ^ (r & 7)) << 4));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      acc[2 * q] += __uint_as_float(w[q] << 16);
      acc[2 * q + 1] += __uint_as_float(w[q] & 0xffff0000u);
    }
  }
}
// the CTA's column sums: the row groups' partials through shared memory
// (red: 256 x 8 floats, free by now), then one atomic per column. Call with
// every thread of the CTA.
template <int N>
__device__ __forceinline__ void colsum8_flush(float* colsum, float* red, int tid, const float (&acc)[8]) {
  constexpr int CG = N / 8, RG = 256 / CG;
#pragma unroll
  for (int q = 0; q < 8; ++q) red[(tid / CG) * N + (tid % CG) * 8 + q] = acc[q];
  __syncthreads();
  if (tid < N) {
    float t = 0.f;
#pragma unroll 8
    for (int g = 0; g < RG; ++g) t += red[g * N + tid];
    atomicAdd(&colsum[tid], t);
  }
  __syncthreads();
}

template <int N, int KP, bool L0>
__global__ void __launch_bounds__(256, 1) policy_dgrad_tma_kernel(const __grid_constant__ CUtensorMap mh,
                                                                  const __grid_constant__ CUtensorMap mdz,
                                                                  const __grid_constant__ CUtensorMap mx0,
                                                                  const __grid_constant__ DgradArgs a,
                                                                  float* __restrict__ colsum,
                                                                  float* __restrict__ wgrad,
                                                                  float* __restrict__ wgrad0) {
  static_assert(!L0 || N == 256, "L0: the 256-wide first hidden layer");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  constexpr uint32_t kBBytes = N * KP * 2, kABytes = kRows * KP * 2, kBox = kRows * 128;
  constexpr int MT = N < 128 ? 1 : N / 128;  // MMA 2 row blocks (N = 64 reads a 2nd, ignored box)
  constexpr uint32_t kHBoxes = N < 128 ? 2 : N / 64;
  constexpr uint32_t kA = kBBytes, kH = (kA + kABytes + 1023) / 1024 * 1024, kX0 = kH + kHBoxes * kBox;
  constexpr uint32_t kX0Bytes = L0 ? kRows * 64 : 0, kBarOff = kX0 + kX0Bytes;
  constexpr int kChunks = kRows * KP / 8 / 256;
  constexpr int kSc = L0 ? 128 : N, kRounds = N / kSc;  // per-tile accumulator columns, column rounds
  constexpr uint32_t kWCol = kSc;                         // dW^T accumulator columns [kSc, kSc + MT * KP)
  constexpr uint32_t kW0Col = kSc + MT * KP;              // L0: dW_0 [256 x 32] as 2 x 32 columns
  constexpr uint32_t kUsed = kW0Col + (L0 ? 64 : 0);
  constexpr uint32_t kCols = kUsed <= 128 ? 128 : (kUsed <= 256 ? 256 : 512);
  static_assert(kUsed <= 512, "TMEM columns");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);  // B, MMA, H, L0
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + kBarOff + 32);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_b = smem_u32(&bars[0]), bar_mma = smem_u32(&bars[1]), bar_h = smem_u32(&bars[2]);
  const uint32_t bar_l0 = smem_u32(&bars[3]);
  if (tid == 0) {
    mbar_init(bar_b, 1);
    mbar_init(bar_mma, 1);
    mbar_init(bar_h, 1);
    mbar_init(bar_l0, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mh)) : "memory");
    if (L0)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mx0)) : "memory");
    else
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mdz)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (tid == 0) bulk_load(sbase, a.wt, kBBytes, bar_b);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const int half = warp >> 2;
  const int64_t tiles = (a.m + kRows - 1) / kRows;
  const auto load_a = [&](int64_t tile, uint4 (&v)[kChunks]) {
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      const int c = tid + 256 * j, row = c % kRows, kc = c / kRows;
      const int64_t r = tile * kRows + row;
      v[j] = make_uint4(0u, 0u, 0u, 0u);
      if (tile < tiles && r < a.m && kc * 8 < a.k)
        v[j] = *reinterpret_cast<const uint4*>(a.dy + r * a.dy_stride + kc * 8);
    }
  };
  uint4 nxt[kChunks];
  load_a(blockIdx.x, nxt);
  uint32_t ph = 0, pm = 0;
  int it = 0;
  bool first = true;
  float csum[8] = {};  // partial column sums of dZ over this CTA's tiles
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
    const int row0 = (int)(tile * kRows);
    if (tid == 0) {  // this tile's h boxes (the previous tile's dZ stores / dW_0 MMAs have read the buffers)
      if constexpr (L0) {
        if (it > 0) mbar_wait(bar_l0, (uint32_t)(it - 1) & 1u);
      } else {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_h),
                   "r"((N / 64) * kBox + kX0Bytes)
                   : "memory");
#pragma unroll
      for (int b = 0; b < N / 64; ++b) tma_load_2d(sbase + kH + b * kBox, &mh, b * 64, row0, bar_h);
      if constexpr (L0) tma_load_2d(sbase + kX0, &mx0, 0, row0, bar_h);
    }
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      const int c = tid + 256 * j, row = c % kRows, kc = c / kRows;
      *reinterpret_cast<uint4*>(smem + kA + kmajor_off(row, kc * 8, kRows)) = nxt[j];
    }
    load_a(tile + gridDim.x, nxt);
    async_proxy_fence();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      if (first) mbar_wait(bar_b, 0);
      tc_fence_after();
      issue_layer(tmem, sbase + kA, kRows, sbase, N, KP, kSc);  // (L0: the first column half)
      if (wgrad) {  // dW^T += h^T dY, once this tile's h boxes have landed
        mbar_wait(bar_h, ph);
        tc_fence_after();
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int ks = 0; ks < kRows / 16; ++ks)
            mma_bf16(tmem + kWCol + mt * KP, make_desc_sw(sbase + kH + mt * 2 * kBox + ks * 2048, kBox, 1024, 2),
                     make_desc(sbase + kA + ks * 256, 128, kRows * 16), make_idesc_mn(128, KP),
                     (!first || ks > 0) ? 1u : 0u);
      }
      mma_commit(bar_mma);
    }
    first = false;
    mbar_wait(bar_mma, pm);
    pm ^= 1;
    mbar_wait(bar_h, ph);
    ph ^= 1;
    tc_fence_after();
    const uint32_t r = (uint32_t)((warp & 3) * 32 + lane);
#pragma unroll
    for (int round = 0; round < kRounds; ++round) {
    if (round > 0) {  // L0: the second column half into the same accumulator columns
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        issue_layer(tmem, sbase + kA, kRows, sbase + round * (kSc / 8) * 128, N, KP, kSc);
        mma_commit(bar_mma);
      }
      mbar_wait(bar_mma, pm);
      pm ^= 1;
      tc_fence_after();
    }
#pragma unroll
    for (int cb = 0; cb < kSc / 2; cb += 16) {  // this warp half's columns, 16 at a time
      const int c = round * kSc + half * (kSc / 2) + cb;
      uint32_t d[16];
      tmem_ld16_async(trow + (c - round * kSc), d);      uint8_t* box = smem + kH + (c >> 6) * kBox;
      const uint32_t o0 = sw128_off(r, c & 63), o1 = sw128_off(r, (c & 63) + 8);
      uint4 hv[2] = {*reinterpret_cast<const uint4*>(box + o0), *reinterpret_cast<const uint4*>(box + o1)};
      tmem_wait_ld();
      uint4 ov[2];
      const uint32_t* hw = reinterpret_cast<const uint32_t*>(hv);
      uint32_t* ow = reinterpret_cast<uint32_t*>(ov);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hw[q]));
        const float gx = hf.x > 0.f ? 1.f : hf.x + 1.f, gy = hf.y > 0.f ? 1.f : hf.y + 1.f;
        ow[q] = pack_bf16(__uint_as_float(d[2 * q]) * gx, __uint_as_float(d[2 * q + 1]) * gy);
      }
      *reinterpret_cast<uint4*>(box + o0) = ov[0];
      *reinterpret_cast<uint4*>(box + o1) = ov[1];
    }
    }
    async_proxy_fence();
    tc_fence_before();
    __syncthreads();  // dZ complete in shared memory
    tc_fence_after();
    if (tid == 0) {
      if constexpr (L0) {  // dW_0 [256 x 32] += dZ_0^T x_0: A = dZ_0^T (MN-major SW128), B = x_0^T (MN-major SW64)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int ks = 0; ks < kRows / 16; ++ks)
            mma_bf16(tmem + kW0Col + mt * 32, make_desc_sw(sbase + kH + mt * 2 * kBox + ks * 2048, kBox, 1024, 2),
                     make_desc_sw(sbase + kX0 + ks * 1024, 8192, 512, 4), make_idesc_mn(128, 32),
                     (it > 0 || ks > 0) ? 1u : 0u);
        mma_commit(bar_l0);
      } else {
#pragma unroll
        for (int b = 0; b < N / 64; ++b) tma_store_2d(&mdz, b * 64, row0, sbase + kH + b * kBox);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (colsum) boxes_colsum8<N>(smem + kH, tid, csum);  // (rows past m: zero dY rows -> zero dZ rows)
    __syncthreads();  // the column sums have read the tile before the next tile's h lands
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // dZ stores done
  if constexpr (L0) {
    if (it > 0) {  // this CTA's dW_0: lane = output row, 32 input columns -> vector reductions
      mbar_wait(bar_l0, (uint32_t)(it - 1) & 1u);
      tc_fence_after();
      const int o = half * 128 + (warp & 3) * 32 + lane;
#pragma unroll
      for (int c = 0; c < 32; c += 16) {
        float v[16];
        tmem_ld16(trow + kW0Col + half * 32 + c, v);
        float* row = wgrad0 + (int64_t)o * 32 + c;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + 4 * q), "f"(v[4 * q]),
                       "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3])
                       : "memory");
      }
    }
  }
  __syncthreads();  // the dZ stores and the dW_0 MMAs have read the boxes: they hold the column-sum partials now
  if (colsum && it > 0) colsum8_flush<N>(colsum, reinterpret_cast<float*>(smem + kH), tid, csum);
  if (wgrad && tiles > blockIdx.x) {  // this CTA's dW^T -> dW[o][i] += (lane i, column o)
    tc_fence_after();
    constexpr int kHalf = MT == 1 && KP >= 32 ? KP / 2 : KP;  // MT = 1: warps 4-7 take the upper columns
    const int mt = MT == 1 ? 0 : half, c0 = MT == 1 ? half * kHalf : 0;
    const int i = mt * 128 + (warp & 3) * 32 + lane;
    if (MT > 1 || KP >= 32 || half == 0) {
#pragma unroll 2
      for (int c = c0; c < c0 + kHalf; c += 16) {
        float v[16];
        tmem_ld16(trow + kWCol + mt * KP + c, v);
        if (i < N) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (c + q < a.k)
              asm volatile("red.global.add.f32 [%0], %1;" ::"l"(wgrad + (int64_t)(c + q) * N + i), "f"(v[q])
                           : "memory");
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
  }
}

// The update backward's head -- layer 1 (256 wide) and the first layer's
// weight gradient -- pipelined across tiles (policy_dgrad_tma_kernel<256,
// 128, true> does the same work one tile at a time). Per tile, with the
// tile's h_1 boxes split into the column halves A (0-127) and B (128-255):
//   MMA  dY W (half A columns) + dW_1^T (rows of half A)   -> epilogue A (dZ_0 half A in place)
//   MMA  dW_0 (half A) | dY W (half B) + dW_1^T (half B)  -> column sums A, epilogue B
//   the NEXT tile's half-A boxes and x_0 (double-buffered) load now,
//   MMA  dW_0 (half B)                                     -> column sums B
//   and the next tile's half-B boxes load at its start, behind its first MMAs.
// So every h_1 load is in flight while the previous half's MMAs / epilogue
// run, where the one-tile kernel waits for all four boxes after the last
// dW_0 MMA of the tile before.
__global__ void __launch_bounds__(256, 1) policy_bwd_head_kernel(const __grid_constant__ CUtensorMap mh,
                                                                 const __grid_constant__ CUtensorMap mx0,
                                                                 const __grid_constant__ DgradArgs a,
                                                                 float* __restrict__ colsum,
                                                                 float* __restrict__ wgrad,
                                                                 float* __restrict__ wgrad0) {
  constexpr int N = 256, KP = 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  constexpr uint32_t kBBytes = N * KP * 2, kABytes = kRows * KP * 2, kBox = kRows * 128;
  constexpr uint32_t kSlot = 2 * kBox;  // one column half of an h_1 tile (two boxes)
  constexpr uint32_t kA = kBBytes, kH = kA + kABytes, kX0 = kH + 2 * kSlot, kX0Bytes = kRows * 64;
  constexpr uint32_t kBarOff = kX0 + 2 * kX0Bytes;
  constexpr int kChunks = kRows * KP / 8 / 256;
  constexpr uint32_t kWCol = 128, kW0Col = 384;  // [0, 128) tile accumulator, dW_1^T, dW_0
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, half = warp >> 2;
  // B, MMA, H0 (even tiles), H1, L0A, L0B, H0 (odd tiles)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + kBarOff + 64);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_b = smem_u32(&bars[0]), bar_mma = smem_u32(&bars[1]), bar_ha = smem_u32(&bars[2]),
                 bar_hb = smem_u32(&bars[3]), bar_l0a = smem_u32(&bars[4]), bar_l0b = smem_u32(&bars[5]);
  if (tid == 0) {
    for (int b = 0; b < 7; ++b) mbar_init(smem_u32(&bars[b]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mx0)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  const int64_t tiles = (a.m + kRows - 1) / kRows;
  // column half h of every tile in slot h (measured: a ring of three slots that loads each half a
  // half-tile earlier was slower, 52.1 vs 47.8 us)
  const auto slot = [&](int i, int h) { return kH + (uint32_t)h * kSlot + 0u * (uint32_t)i; };
  const auto load_half = [&](int64_t tile, int i, int h) {  // half 0 brings x_0 along (buffer i & 1)
    const int row0 = (int)(tile * kRows);
    const uint32_t bar = h ? bar_hb : smem_u32(&bars[(i & 1) ? 6 : 2]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kSlot + (h ? 0 : kX0Bytes))
                 : "memory");
    tma_load_2d(sbase + slot(i, h), &mh, 128 * h, row0, bar);
    tma_load_2d(sbase + slot(i, h) + kBox, &mh, 128 * h + 64, row0, bar);
    if (!h) tma_load_2d(sbase + kX0 + (i & 1) * kX0Bytes, &mx0, 0, row0, bar);
  };
  if (tid == 0) {
    bulk_load(sbase, a.wt, kBBytes, bar_b);
    if (blockIdx.x < tiles) load_half(blockIdx.x, 0, 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t r = (uint32_t)((warp & 3) * 32 + lane);
  const auto load_a = [&](int64_t tile, uint4 (&v)[kChunks]) {
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      const int c = tid + 256 * j, row = c % kRows, kc = c / kRows;
      const int64_t rr = tile * kRows + row;
      v[j] = make_uint4(0u, 0u, 0u, 0u);
      if (tile < tiles && rr < a.m && kc * 8 < a.k)
        v[j] = *reinterpret_cast<const uint4*>(a.dy + rr * a.dy_stride + kc * 8);
    }
  };
  // dZ = acc * ELU'(h) for this warp half's 64 columns of a column half (in place in the boxes)
  const auto epilogue = [&](uint32_t base) {  // base: the column half's ring slot
#pragma unroll
    for (int cb = 0; cb < 64; cb += 16) {
      const int c = half * 64 + cb;  // column within the half
      uint32_t d[16];
      tmem_ld16_async(trow + c, d);
      uint8_t* box = smem + base + (c >> 6) * kBox;
      const uint32_t o0 = sw128_off(r, c & 63), o1 = sw128_off(r, (c & 63) + 8);
      uint4 hv[2] = {*reinterpret_cast<const uint4*>(box + o0), *reinterpret_cast<const uint4*>(box + o1)};
      tmem_wait_ld();
      uint4 ov[2];
      const uint32_t* hw = reinterpret_cast<const uint32_t*>(hv);
      uint32_t* ow = reinterpret_cast<uint32_t*>(ov);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hw[q]));
        const float gx = hf.x > 0.f ? 1.f : hf.x + 1.f, gy = hf.y > 0.f ? 1.f : hf.y + 1.f;
        ow[q] = pack_bf16(__uint_as_float(d[2 * q]) * gx, __uint_as_float(d[2 * q + 1]) * gy);
      }
      *reinterpret_cast<uint4*>(box + o0) = ov[0];
      *reinterpret_cast<uint4*>(box + o1) = ov[1];
    }
  };
  const auto mma_w1t = [&](int mt, uint32_t base, bool acc0) {  // dW_1^T rows of column half mt += h^T dY
#pragma unroll
    for (int ks = 0; ks < kRows / 16; ++ks)
      mma_bf16(tmem + kWCol + mt * KP, make_desc_sw(sbase + base + ks * 2048, kBox, 1024, 2),
               make_desc(sbase + kA + ks * 256, 128, kRows * 16), make_idesc_mn(128, KP), (acc0 || ks > 0) ? 1u : 0u);
  };
  const auto mma_w0 = [&](int mt, uint32_t base, int buf, bool acc0) {  // dW_0 rows of column half mt += dZ_0^T x_0
#pragma unroll
    for (int ks = 0; ks < kRows / 16; ++ks)
      mma_bf16(tmem + kW0Col + mt * 32, make_desc_sw(sbase + base + ks * 2048, kBox, 1024, 2),
               make_desc_sw(sbase + kX0 + buf * kX0Bytes + ks * 1024, 8192, 512, 4), make_idesc_mn(128, 32),
               (acc0 || ks > 0) ? 1u : 0u);
  };
  uint4 nxt[kChunks];
  load_a(blockIdx.x, nxt);
  uint32_t pm = 0;
  int it = 0;
  float csum[8] = {};  // partial column sums of dZ_0 (colsum_boxes layout over the 4 boxes)
  float csa[8] = {}, csb[8] = {};
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
    const uint32_t ph = (uint32_t)it & 1u;
    const int buf = it & 1;
    const uint32_t bar_h0 = smem_u32(&bars[buf ? 6 : 2]), ph0 = (uint32_t)(it >> 1) & 1u;
    const uint32_t s0 = slot(it, 0), s1 = slot(it, 1);
    const bool more = tile + gridDim.x < tiles;
    if (tid == 0) {  // this tile's half 1 (the previous tile's half-1 dW_0 MMAs have read the slot)
      if (it > 0) mbar_wait(bar_l0b, ph ^ 1u);
      load_half(tile, it, 1);
    }
#pragma unroll
    for (int j = 0; j < kChunks; ++j) {
      const int c = tid + 256 * j, row = c % kRows, kc = c / kRows;
      *reinterpret_cast<uint4*>(smem + kA + kmajor_off(row, kc * 8, kRows)) = nxt[j];
    }
    load_a(tile + gridDim.x, nxt);
    async_proxy_fence();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      if (it == 0) mbar_wait(bar_b, 0);
      tc_fence_after();
      issue_layer(tmem, sbase + kA, kRows, sbase, N, KP, 128);  // dY W, half 0 columns
      mbar_wait(bar_h0, ph0);
      tc_fence_after();
      if (wgrad) mma_w1t(0, s0, it > 0);
      mma_commit(bar_mma);
    }
    mbar_wait(bar_mma, pm);
    pm ^= 1;
    mbar_wait(bar_h0, ph0);
    tc_fence_after();
    epilogue(s0);
    async_proxy_fence();
    tc_fence_before();
    __syncthreads();  // dZ_0 half 0 complete
    tc_fence_after();
    if (tid == 0) {
      mma_w0(0, s0, buf, it > 0);
      mma_commit(bar_l0a);
      issue_layer(tmem, sbase + kA, kRows, sbase + 2048, N, KP, 128);  // dY W, half 1 columns
      mbar_wait(bar_hb, ph);
      tc_fence_after();
      if (wgrad) mma_w1t(1, s1, it > 0);
      mma_commit(bar_mma);
    }
    if (colsum) boxes_colsum8<128>(smem + s0, tid, csa);
    mbar_wait(bar_mma, pm);
    pm ^= 1;
    mbar_wait(bar_hb, ph);
    tc_fence_after();
    epilogue(s1);
    async_proxy_fence();
    tc_fence_before();
    __syncthreads();  // dZ_0 half 1 complete; the half-0 column sums have read their slot
    tc_fence_after();
    if (tid == 0) {
      mbar_wait(bar_l0a, ph);  // the half-0 dW_0 MMAs have read their slot
      if (more) load_half(tile + gridDim.x, it + 1, 0);  // the next tile's half 0 (+ x_0) into it
      tc_fence_after();
      mma_w0(1, s1, buf, it > 0);
      mma_commit(bar_l0b);
    }
    if (colsum) boxes_colsum8<128>(smem + s1, tid, csb);
    __syncthreads();  // the half-1 column sums have read their slot before it is reloaded
  }
  (void)csum;
  if (it > 0) {  // this CTA's dW_0: lane = output row, 32 input columns -> vector reductions
    mbar_wait(bar_l0b, (uint32_t)(it - 1) & 1u);
    tc_fence_after();
    const int o = half * 128 + (warp & 3) * 32 + lane;
#pragma unroll
    for (int c = 0; c < 32; c += 16) {
      float v[16];
      tmem_ld16(trow + kW0Col + half * 32 + c, v);
      float* row = wgrad0 + (int64_t)o * 32 + c;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + 4 * q), "f"(v[4 * q]),
                     "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3])
                     : "memory");
    }
  }
  __syncthreads();  // every MMA has read the boxes: they hold the column-sum partials now
  if (colsum && it > 0) {
    colsum8_flush<128>(colsum, reinterpret_cast<float*>(smem + kH), tid, csa);
    colsum8_flush<128>(colsum + 128, reinterpret_cast<float*>(smem + kH), tid, csb);
  }
  if (wgrad && it > 0) {  // this CTA's dW_1^T -> dW_1[o][i] += (lane i, column o)
    tc_fence_after();
    const int i = half * 128 + (warp & 3) * 32 + lane;
#pragma unroll 2
    for (int c = 0; c < KP; c += 16) {
      float v[16];
      tmem_ld16(trow + kWCol + half * KP + c, v);
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (c + q < a.k)
          asm volatile("red.global.add.f32 [%0], %1;" ::"l"(wgrad + (int64_t)(c + q) * N + i), "f"(v[q]) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

// The update backward's tail -- the last two layers of one trunk -- in one
// launch (Policy::backward, policy.cpp:163-218), per 128-row tile:
//   db_3 += 1^T dY_3                          (per-thread row sums, no reduction per tile)
//   dZ_2  = (dY_3 W_3) * ELU'(h_3)            (MMA: A = dY_3 tile, B = W_3^T image)
//   dW_3^T += h_3^T dY_3                      (MMA, TMEM-resident over the CTA's tiles)
//   dZ_1  = (dZ_2 W_2) * ELU'(h_2)            (MMA: A = dZ_2 read back as K-major SWIZZLE_128B)
//   dW_2^T += h_2^T dZ_2                      (MMA: B = dZ_2 read back as MN-major SWIZZLE_128B)
//   db_2 += 1^T dZ_2, db_1 += 1^T dZ_1        (column sums from shared memory)
// dZ_2 is written in place into the h_3 box it was computed from -- a
// 128-row x 64-column box with 128-byte rows is both the K-major and the
// MN-major SWIZZLE_128B canonical layout, so it feeds the next layer's data
// gradient (A, K steps of 32 bytes) and this layer's weight gradient (B)
// without a copy -- and dZ_1 likewise into the h_2 boxes, which one thread
// stores with TMA; dZ_2 never reaches HBM. 71 KB of shared memory and 256
// TMEM columns: two CTAs per SM overlap one tile's MMAs with the other's
// epilogue. TMEM: [0, 128) the tile's accumulator (dY_3 W_3 in [0, 64),
// then dZ_2 W_2), [128, 144) dW_3^T, [144, 208) dW_2^T.
struct TailArgs {
  const __nv_bfloat16* dy;  // dY_3 [m x k3], row stride dy_stride
  int32_t dy_stride;
  int32_t k3;               // valid dY_3 columns (<= 16)
  const uint8_t* wt3;       // W_3^T image [64 x 16]
  const uint8_t* wt2;       // W_2^T image [128 x 64]
  int64_t m;
  float* db3;               // [k3]
  float* dw3;               // [k3 x 64]
  float* db2;               // [64]
  float* dw2;               // [64 x 128]
  float* db1;               // [128]
};

__global__ void __launch_bounds__(256, 2) policy_bwd_tail_kernel(const __grid_constant__ CUtensorMap mh3,
                                                                 const __grid_constant__ CUtensorMap mh2,
                                                                 const __grid_constant__ CUtensorMap mdz1,
                                                                 const __grid_constant__ TailArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  constexpr uint32_t kBox = kRows * 128;
  constexpr uint32_t kW3 = 0, kW2 = 64 * 16 * 2, kA = kW2 + 128 * 64 * 2, kH3 = (kA + kRows * 16 * 2 + 1023) / 1024 * 1024;
  constexpr uint32_t kH2 = kH3 + kBox, kBarOff = kH2 + 2 * kBox;
  constexpr uint32_t kDW3 = 128, kDW2 = 144, kCols = 256;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, half = warp >> 2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);  // W, MMA, H3, H2
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + kBarOff + 32);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_w = smem_u32(&bars[0]), bar_mma = smem_u32(&bars[1]), bar_h3 = smem_u32(&bars[2]),
                 bar_h2 = smem_u32(&bars[3]);
  if (tid == 0) {
    mbar_init(bar_w, 1);
    mbar_init(bar_mma, 1);
    mbar_init(bar_h3, 1);
    mbar_init(bar_h2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mh3)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mh2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mdz1)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_w), "r"(kA) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sbase + kW3),
                 "l"(a.wt3), "r"(kW2), "r"(bar_w)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sbase + kW2),
                 "l"(a.wt2), "r"(kA - kW2), "r"(bar_w)
                 : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t r = (uint32_t)((warp & 3) * 32 + lane);
  const int64_t tiles = (a.m + kRows - 1) / kRows;
  const auto load_a = [&](int64_t tile) {  // one 16-byte piece per thread: row tid % 128, columns 8 (tid / 128) ..
    const int row = tid % kRows, kc = tid / kRows;
    const int64_t rr = tile * kRows + row;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (tile < tiles && rr < a.m && kc * 8 < a.k3) v = *reinterpret_cast<const uint4*>(a.dy + rr * a.dy_stride + kc * 8);
    return v;
  };
  uint4 nxt = load_a(blockIdx.x);
  uint32_t pm = 0, ph = 0;
  int it = 0;
  float cs3[8] = {}, cs2[8] = {}, cs1[8] = {};
  // ELU'(h) * acc for 16 accumulator columns of row r, in place in a 128 x 64 SW128 box
  const auto elu_bwd16 = [&](uint8_t* box, int c, const uint32_t (&d)[16]) {
    const uint32_t o0 = sw128_off(r, c), o1 = sw128_off(r, c + 8);
    uint4 hv[2] = {*reinterpret_cast<const uint4*>(box + o0), *reinterpret_cast<const uint4*>(box + o1)};
    uint4 ov[2];
    const uint32_t* hw = reinterpret_cast<const uint32_t*>(hv);
    uint32_t* ow = reinterpret_cast<uint32_t*>(ov);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hw[q]));
      const float gx = hf.x > 0.f ? 1.f : hf.x + 1.f, gy = hf.y > 0.f ? 1.f : hf.y + 1.f;
      ow[q] = pack_bf16(__uint_as_float(d[2 * q]) * gx, __uint_as_float(d[2 * q + 1]) * gy);
    }
    *reinterpret_cast<uint4*>(box + o0) = ov[0];
    *reinterpret_cast<uint4*>(box + o1) = ov[1];
  };
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
    const int row0 = (int)(tile * kRows);
    if (tid == 0) {  // the tile's h_3 and h_2 boxes (the previous tile's dZ_1 stores have read the h_2 boxes)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_h3), "r"(kBox) : "memory");
      tma_load_2d(sbase + kH3, &mh3, 0, row0, bar_h3);
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_h2), "r"(2 * kBox) : "memory");
      tma_load_2d(sbase + kH2, &mh2, 0, row0, bar_h2);
      tma_load_2d(sbase + kH2 + kBox, &mh2, 64, row0, bar_h2);
    }
    *reinterpret_cast<uint4*>(smem + kA + kmajor_off(tid % kRows, (tid / kRows) * 8, kRows)) = nxt;
    if (tid < kRows) {  // db_3: this thread's row of dY_3 (columns 0-7; k3 <= 8 on the trunk)
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&nxt);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[q]));
        cs3[2 * q] += f.x;
        cs3[2 * q + 1] += f.y;
      }
    }
    nxt = load_a(tile + gridDim.x);
    async_proxy_fence();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      if (it == 0) mbar_wait(bar_w, 0);
      tc_fence_after();
      issue_layer(tmem, sbase + kA, kRows, sbase + kW3, 64, 16, 64);  // dY_3 W_3 -> [0, 64)
      mbar_wait(bar_h3, ph);
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < kRows / 16; ++ks)  // dW_3^T += h_3^T dY_3 (M = 128: lanes 64-127 read the h_2 box, unused)
        mma_bf16(tmem + kDW3, make_desc_sw(sbase + kH3 + ks * 2048, kBox, 1024, 2),
                 make_desc(sbase + kA + ks * 256, 128, kRows * 16), make_idesc_mn(128, 16), (it > 0 || ks > 0) ? 1u : 0u);
      mma_commit(bar_mma);
    }
    mbar_wait(bar_mma, pm);
    pm ^= 1;
    mbar_wait(bar_h3, ph);
    tc_fence_after();
#pragma unroll
    for (int cb = 0; cb < 32; cb += 16) {  // dZ_2 = (dY_3 W_3) * ELU'(h_3): warps 4-7 take columns 32-63
      const int c = half * 32 + cb;
      uint32_t d[16];
      tmem_ld16_async(trow + c, d);
      tmem_wait_ld();
      elu_bwd16(smem + kH3, c, d);
    }
    async_proxy_fence();
    tc_fence_before();
    __syncthreads();  // dZ_2 complete in the h_3 box
    tc_fence_after();
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < 64 / 16; ++ks)  // dZ_2 W_2 -> [0, 128): A = dZ_2 K-major SW128, K steps of 32 bytes
        mma_bf16(tmem, make_desc_sw(sbase + kH3 + ks * 32, 16, 1024, 2),
                 make_desc(sbase + kW2 + 2u * ks * (128 * 16), 128 * 16, 128), make_idesc(kRows, 128), ks > 0 ? 1u : 0u);
      mbar_wait(bar_h2, ph);
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < kRows / 16; ++ks)  // dW_2^T += h_2^T dZ_2: B = dZ_2 MN-major SW128
        mma_bf16(tmem + kDW2, make_desc_sw(sbase + kH2 + ks * 2048, kBox, 1024, 2),
                 make_desc_sw(sbase + kH3 + ks * 2048, kBox, 1024, 2), make_idesc_mn(128, 64),
                 (it > 0 || ks > 0) ? 1u : 0u);
      mma_commit(bar_mma);
    }
    boxes_colsum8<64>(smem + kH3, tid, cs2);  // db_2 (reads only, beside the MMAs)
    mbar_wait(bar_mma, pm);
    pm ^= 1;
    mbar_wait(bar_h2, ph);
    ph ^= 1;
    tc_fence_after();
#pragma unroll
    for (int cb = 0; cb < 64; cb += 16) {  // dZ_1 = (dZ_2 W_2) * ELU'(h_2): warps 4-7 take columns 64-127
      const int c = half * 64 + cb;
      uint32_t d[16];
      tmem_ld16_async(trow + c, d);
      tmem_wait_ld();
      elu_bwd16(smem + kH2 + (c >> 6) * kBox, c & 63, d);
    }
    async_proxy_fence();
    tc_fence_before();
    __syncthreads();  // dZ_1 complete in the h_2 boxes
    tc_fence_after();
    if (tid == 0) {
      tma_store_2d(&mdz1, 0, row0, sbase + kH2);
      tma_store_2d(&mdz1, 64, row0, sbase + kH2 + kBox);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    boxes_colsum8<128>(smem + kH2, tid, cs1);
    __syncthreads();  // the column sums have read the boxes before the next tile's loads land
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  if (it > 0) {  // (the h boxes are free: the last dZ_1 stores have read them)
    colsum8_flush<64>(a.db2, reinterpret_cast<float*>(smem + kH2), tid, cs2);
    colsum8_flush<128>(a.db1, reinterpret_cast<float*>(smem + kH2), tid, cs1);
  }
  if (warp < 4) {  // db_3: warp sums of the per-row partials
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float v = cs3[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && q < a.k3) atomicAdd(&a.db3[q], v);
    }
  }
  if (it > 0) {
    tc_fence_after();
    if (half == 0) {  // dW_3^T (lanes 0-63 = inputs, 16 columns = outputs) and dW_2^T columns 0-31
      float v[16];
      tmem_ld16(trow + kDW3, v);
      if (r < 64) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (q < a.k3)
            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(a.dw3 + q * 64 + r), "f"(v[q]) : "memory");
      }
    }
#pragma unroll
    for (int cb = 0; cb < 32; cb += 16) {  // dW_2^T: lane = input (128), column = output (64); warps 4-7 the upper 32
      const int c = half * 32 + cb;
      float v[16];
      tmem_ld16(trow + kDW2 + c, v);
#pragma unroll
      for (int q = 0; q < 16; ++q)
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(a.dw2 + (int64_t)(c + q) * 128 + r), "f"(v[q]) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
  }
}

// sum of the per-CTA partials -> the weight gradient (fp32, written). A block
// owns 32 consecutive float4s; its 8 warps split the partials (coalesced
// 512-byte rows, ~19 independent loads per lane in flight), then fold.
__global__ void __launch_bounds__(256) policy_wgrad_reduce_kernel(const float4* __restrict__ partial, int parts,
                                                                  int64_t n4, float4* __restrict__ out) {
  __shared__ float4 red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t k = (int64_t)blockIdx.x * 32 + lane;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (k < n4) {
#pragma unroll 4
    for (int p = warp; p < parts; p += 8) {
      const float4 v = partial[(int64_t)p * n4 + k];
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && k < n4) {
    float4 t = red[0][lane];
    for (int w = 1; w < 8; ++w) {
      t.x += red[w][lane].x;
      t.y += red[w][lane].y;
      t.z += red[w][lane].z;
      t.w += red[w][lane].w;
    }
    out[k] = t;
  }
}

// ---- packing: flat fp32 params (reference layout) -> bf16 UMMA images -----
struct PackTable {
  int64_t w_off[2][4];  // flat offsets of W_l [out x in] per trunk
  int64_t b_off[2][4];
  int32_t in_dim[4];
  int32_t out_dim[2][4];
};

__global__ void policy_pack_kernel(const float* __restrict__ flat, const __grid_constant__ PackTable t, uint8_t* w1,
                                   uint8_t* w2a, uint8_t* w2c, uint8_t* w34, float* bias) {
  // one thread per destination bf16 element of every image, then biases
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // image element counts: W1 512x32, W2 128x256 (x2), W3 64x128 (x2), W4 16x64 (x2)
  const int64_t n1 = 512 * 32, n2 = 128 * 256, n3 = 64 * 128, n4 = 16 * 64;
  int64_t k = i;
  auto emit = [&](uint8_t* base, int trunk, int layer, int R, int K, int64_t e) {
    const int r = (int)(e / K), c = (int)(e % K);
    float v = 0.f;
    if (r < t.out_dim[trunk][layer] && c < t.in_dim[layer])
      v = flat[t.w_off[trunk][layer] + (int64_t)r * t.in_dim[layer] + c];
    *reinterpret_cast<__nv_bfloat16*>(base + kmajor_off(r, c, R)) = __float2bfloat16_rn(v);
  };
  if (k < n1) {  // W1: actor rows 0..255, critic rows 256..511
    const int r = (int)(k / 32), c = (int)(k % 32), trunk = r >= 256;
    const int rr = r - 256 * trunk;
    float v = 0.f;
    if (c < t.in_dim[0]) v = flat[t.w_off[trunk][0] + (int64_t)rr * t.in_dim[0] + c];
    *reinterpret_cast<__nv_bfloat16*>(w1 + kmajor_off(r, c, 512)) = __float2bfloat16_rn(v);
    return;
  }
  k -= n1;
  if (k < n2) return emit(w2a, 0, 1, 128, 256, k);
  k -= n2;
  if (k < n2) return emit(w2c, 1, 1, 128, 256, k);
  k -= n2;
  if (k < n3) return emit(w34 + 0, 0, 2, 64, 128, k);
  k -= n3;
  if (k < n3) return emit(w34 + 16384, 1, 2, 64, 128, k);
  k -= n3;
  if (k < n4) return emit(w34 + 32768, 0, 3, 16, 64, k);
  k -= n4;
  if (k < n4) return emit(w34 + 34816, 1, 3, 16, 64, k);
  k -= n4;
  // biases: b1 (512) | b2a b2c (128+128) | b3a b3c (64+64) | b4a b4c (16+16)
  if (k < 512) {
    const int trunk = k >= 256, r = (int)k - 256 * trunk;
    bias[k] = flat[t.b_off[trunk][0] + r];
    return;
  }
  k -= 512;
  if (k < 256) {
    const int trunk = k >= 128, r = (int)k - 128 * trunk;
    bias[512 + k] = flat[t.b_off[trunk][1] + r];
    return;
  }
  k -= 256;
  if (k < 128) {
    const int trunk = k >= 64, r = (int)k - 64 * trunk;
    bias[768 + k] = flat[t.b_off[trunk][2] + r];
    return;
  }
  k -= 128;
  if (k < 32) {
    const int trunk = k >= 16, r = (int)k - 16 * trunk;
    bias[896 + k] = r < t.out_dim[trunk][3] ? flat[t.b_off[trunk][3] + r] : 0.f;
  }
}

__global__ void policy_sample_kernel(const float* __restrict__ mean, int64_t n, int A,
                                     const float* __restrict__ log_std_raw, uint64_t s0, uint64_t inc,
                                     const uint64_t* __restrict__ pos, uint64_t step_off,
                                     const __grid_constant__ Jump64 J, float* __restrict__ actions,
                                     float* __restrict__ logp) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  uint64_t s = jump(s0, *pos + step_off + 2ull * (uint64_t)e * (uint64_t)A, J);
  double lp = 0.0;
  for (int i = 0; i < A; ++i) {
    double term;
    actions[e * A + i] = draw_action(s, inc, mean[e * A + i], log_std_raw[i], term);
    lp = __dadd_rn(lp, term);
  }
  logp[e] = (float)lp;
}

// The stream part of the rollout sampling (ppo.cpp:262-277) ahead of the
// forward: block = 32 envs x A dims, one (env, dim) draw per thread at
// pos + step_off + 2 (e A + dim) (warp-parallel jump to the block's first
// draw, then <= 10 bits), sz = exp(clamp(ls)) z in fp64 and the env's log-prob
// (terms summed in dim order, as policy_sample_kernel). Runs on the fp64 pipe
// while the env step (SIMT fp32, a few warps per SM) produces the
// observations the forward consumes.
__global__ void policy_noise_kernel(int64_t n, int A, const float* __restrict__ log_std_raw, uint64_t s0,
                                    uint64_t inc, const uint64_t* __restrict__ pos, uint64_t step_off,
                                    const __grid_constant__ Jump64 J, double* __restrict__ sz, float* __restrict__ logp) {
  __shared__ double sterm[32 * kNOut];
  __shared__ uint64_t sbase;
  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * 32;
  if (tid < 32) {
    const uint64_t b = jump_warp(s0, *pos + step_off + 2ull * (uint64_t)e0 * (uint64_t)A, J);
    if (tid == 0) sbase = b;
  }
  __syncthreads();
  const int64_t e = e0 + tid / A;
  const int d = tid % A;
  double term = 0.0;
  if (e < n) {
    uint64_t st = jump(sbase, 2ull * (uint64_t)tid, J);
    const double ls = clamp_log_std(log_std_raw[d]);
    const double z = draw_normal(st, inc);
    term = logp_term(z, ls);
    sz[e * A + d] = __dmul_rn(exp(ls), z);
  }
  sterm[tid] = term;
  __syncthreads();
  if (tid < 32 && e0 + tid < n) {
    double lp = 0.0;
    for (int k = 0; k < A; ++k) lp = __dadd_rn(lp, sterm[tid * A + k]);
    logp[e0 + tid] = (float)lp;
  }
}

// ---- GAE (rollout.cpp:42-66) + episode statistics (ppo.cpp:286-303) --------
// Time-major buffers [T][n]. One thread per env: backward GAE recursion with
// terminated masking and timeout bootstrap, then a forward pass accumulating
// per-env episode returns (carried across iterations in ep_acc).
__global__ void gae_kernel(const float* __restrict__ rewards, const float* __restrict__ values,
                           const uint8_t* __restrict__ term, const uint8_t* __restrict__ tout,
                           const float* __restrict__ boot, const float* __restrict__ last_values,
                           const float* __restrict__ task_error, int T, int64_t n, float gamma, float lam,
                           float* __restrict__ adv, float* __restrict__ ret, float* __restrict__ ep_acc,
                           double* __restrict__ stats) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double reward_sum = 0.0, ep_reward = 0.0, ep_err = 0.0, episodes = 0.0;
  if (e < n) {
    float running = 0.f;
    for (int t = T - 1; t >= 0; --t) {
      const int64_t k = (int64_t)t * n + e;
      const bool te = term[k] != 0, to = tout[k] != 0;
      float delta;
      if (te) delta = rewards[k] - values[k];
      else if (to) delta = rewards[k] + gamma * boot[k] - values[k];
      else {
        const float v_next = t == T - 1 ? last_values[e] : values[k + n];
        delta = rewards[k] + gamma * v_next - values[k];
      }
      running = (te || to) ? delta : delta + gamma * lam * running;
      adv[k] = running;
      ret[k] = running + values[k];
    }
    float acc = ep_acc[e];
    for (int t = 0; t < T; ++t) {
      const int64_t k = (int64_t)t * n + e;
      reward_sum += rewards[k];
      acc += rewards[k];
      if (term[k] || tout[k]) {
        ep_reward += acc;
        ep_err += task_error[k];
        episodes += 1.0;
        acc = 0.f;
      }
    }
    ep_acc[e] = acc;
  }
  // warp reduce, one atomic per warp
  for (int o = 16; o; o >>= 1) {
    reward_sum += __shfl_down_sync(0xffffffffu, reward_sum, o);
    ep_reward += __shfl_down_sync(0xffffffffu, ep_reward, o);
    ep_err += __shfl_down_sync(0xffffffffu, ep_err, o);
    episodes += __shfl_down_sync(0xffffffffu, episodes, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(stats + 0, reward_sum);
    atomicAdd(stats + 1, ep_reward);
    atomicAdd(stats + 2, ep_err);
    atomicAdd(stats + 3, episodes);
  }
}

}  // namespace sgp

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
struct sg_policy {
  int obs_dim = 0, act_dim = 0, device = 0;
  int64_t param_count = 0, log_std_offset = 0;
  uint8_t* img = nullptr;  // w1 | w2a | w2c | w34
  float* bias = nullptr;   // 928
  sgp::PackTable table{};
  std::string err;
};

namespace {
thread_local std::string g_policy_err;

int fail(int code, const std::string& m) {
  g_policy_err = m;
  return code;
}
}  // namespace

namespace sgp {

// ---- ppo_update's optimizer step (ppo.cpp:199-207, Adam::step :56-64) -------
// grad_sq: global sum of squared gradients; the Adam kernel applies the clip
// scale max_norm / norm (when norm > max_norm), the reference's Adam with
// bias correction, the log-std box projection, and refreshes the bf16 mirror
// of the parameters the next minibatch's GEMMs read.
__global__ void grad_sq_kernel(const float* __restrict__ g, int64_t n, float* __restrict__ out, int32_t* step) {
  float acc = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc = fmaf(g[i], g[i], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ float part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) atomicAdd(out, acc);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(step, 1);  // Adam::step ++t_
}

struct AdamArgs {
  float lr, beta1, beta2, eps, max_norm;
  int64_t ls_off;
  int32_t ls_n;
  float ls_min, ls_max;
};

__global__ void adam_kernel(float* __restrict__ p, float* __restrict__ g, float* __restrict__ m, float* __restrict__ v,
                            __nv_bfloat16* __restrict__ mirror, int64_t n, const float* __restrict__ grad_sq,
                            const int32_t* __restrict__ step, const __grid_constant__ AdamArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float norm = sqrtf(grad_sq[0]);
  if (!isfinite(norm)) {  // ppo.cpp:193-199 throws here: leave the parameters, flag it (sticky)
    if (i == 0) const_cast<float*>(grad_sq)[1] = 1.f;
    g[i] = 0.f;
    return;
  }
  const float scale = (a.max_norm > 0.f && norm > a.max_norm) ? a.max_norm / norm : 1.f;
  const int t = *step;
  const float bc1 = 1.f - powf(a.beta1, (float)t), bc2 = 1.f - powf(a.beta2, (float)t);
  const float gi = g[i] * scale;
  const float mi = fmaf(a.beta1, m[i], (1.f - a.beta1) * gi);
  const float vi = fmaf(a.beta2, v[i], (1.f - a.beta2) * gi * gi);
  m[i] = mi;
  v[i] = vi;
  float pi = p[i] - a.lr * (mi / bc1) / (sqrtf(vi / bc2) + a.eps);
  if (i >= a.ls_off && i < a.ls_off + a.ls_n) pi = fminf(fmaxf(pi, a.ls_min), a.ls_max);
  p[i] = pi;
  g[i] = 0.f;  // ready for the next minibatch's accumulation
  if (mirror) mirror[i] = __float2bfloat16_rn(pi);
}

}  // namespace sgp

// cudaFuncSetAttribute is per device: remember which devices a kernel's
// shared-memory opt-in was made for (one bit per device, up to 64).
static bool smem_opt_in(const void* fn, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load() & bit) return true;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  done.fetch_or(bit);
  return true;
}

template <int N, int KP>
static int launch_dgrad(const sgp::DgradArgs& a, cudaStream_t st) {
  constexpr size_t smem = (size_t)N * KP * 2 + (size_t)sgp::kRows * KP * 2 + 64;
  static std::atomic<unsigned long long> done{0};
  if (!smem_opt_in(reinterpret_cast<const void*>(sgp::policy_dgrad_elu_kernel<N, KP>), (int)smem, done))
    return fail(SG_ERR_SIM, "policy: cannot reserve shared memory");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (a.m + sgp::kRows - 1) / sgp::kRows;
  const int64_t slots = (int64_t)sms * sgp::kDgradCtas;
  sgp::policy_dgrad_elu_kernel<N, KP><<<(unsigned)(tiles < slots ? tiles : slots), 256, smem, st>>>(a);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

using TensorMapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TensorMapEncodeFn tensor_map_encode() {
  static TensorMapEncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<TensorMapEncodeFn>(nullptr);
    return reinterpret_cast<TensorMapEncodeFn>(p);
  }();
  return fn;
}
// 2-D bf16 row-major [rows x cols] map, boxes of min(cols, 64) columns x 64
// rows, 128-byte (64-column) or 64-byte (32-column) swizzle
static bool encode_rows(CUtensorMap* map, const void* base, int cols, int64_t rows) {
  const TensorMapEncodeFn enc = tensor_map_encode();
  if (!enc) return false;
  const int bw = cols >= 64 ? 64 : cols;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  const cuuint32_t box[2] = {(cuuint32_t)bw, 64};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, bw == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int OUT, int IN, bool ATOMIC = false>
static int launch_wgrad_tma(const void* dy, const void* x, int64_t m, float* partial, int parts, float* out,
                            cudaStream_t st) {
  constexpr size_t smem = 4 * ((size_t)(OUT / 64) * 64 * 128 + (size_t)IN * 64 * 2) + 1024 + 256;
  static std::atomic<unsigned long long> done{0};
  if (!smem_opt_in(reinterpret_cast<const void*>(sgp::policy_wgrad_tma_kernel<OUT, IN, ATOMIC>), (int)smem, done))
    return fail(SG_ERR_SIM, "policy: cannot reserve shared memory");
  CUtensorMap mdy, mx;
  if (!encode_rows(&mdy, dy, OUT, m) || !encode_rows(&mx, x, IN, m))
    return fail(SG_ERR_SIM, "sg_policy_wgrad: cuTensorMapEncodeTiled failed");
  const int64_t per = ((m + parts - 1) / parts + 63) / 64 * 64;
  if constexpr (ATOMIC) {  // vector reductions into the zeroed gradient
    const sgp::WgradArgs a{static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x), m, per, out};
    if (cudaMemsetAsync(out, 0, (size_t)OUT * IN * sizeof(float), st) != cudaSuccess)
      return fail(SG_ERR_SIM, "sg_policy_wgrad: memset failed");
    sgp::policy_wgrad_tma_kernel<OUT, IN, true><<<parts, 128, smem, st>>>(mdy, mx, a);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
  }
  const sgp::WgradArgs a{static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x), m, per, partial};
  sgp::policy_wgrad_tma_kernel<OUT, IN, false><<<parts, 128, smem, st>>>(mdy, mx, a);
  const int64_t n4 = (int64_t)OUT * IN / 4;
  sgp::policy_wgrad_reduce_kernel<<<(unsigned)((n4 + 31) / 32), 256, 0, st>>>(
      reinterpret_cast<const float4*>(partial), parts, n4, reinterpret_cast<float4*>(out));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

template <int OUT, int IN>
static int launch_wgrad(const void* dy, const void* x, int64_t m, float* partial, int parts, float* out,
                        cudaStream_t st) {
  constexpr int MP = OUT <= 128 ? 128 : 256;
  constexpr size_t smem = sgp::kWgradStages * ((size_t)MP * 64 * 2 + (size_t)IN * 64 * 2) + 128;
  static std::atomic<unsigned long long> done{0};
  if (!smem_opt_in(reinterpret_cast<const void*>(sgp::policy_wgrad_kernel<OUT, IN>), (int)smem, done))
    return fail(SG_ERR_SIM, "policy: cannot reserve shared memory");
  const int64_t per = ((m + parts - 1) / parts + 63) / 64 * 64;
  const sgp::WgradArgs a{static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x), m, per, partial};
  sgp::policy_wgrad_kernel<OUT, IN><<<parts, 128, smem, st>>>(a);
  const int64_t n4 = (int64_t)OUT * IN / 4;
  sgp::policy_wgrad_reduce_kernel<<<(unsigned)((n4 + 31) / 32), 256, 0, st>>>(
      reinterpret_cast<const float4*>(partial), parts, n4, reinterpret_cast<float4*>(out));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

// 2-D bf16 row-major [rows x cols] map with 64-column x 128-row boxes, 128-byte swizzle
static bool encode_rows128(CUtensorMap* map, const void* base, int cols, int64_t rows) {
  const TensorMapEncodeFn enc = tensor_map_encode();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int N, int KP, bool L0>
static int launch_dgrad_tma(const sgp::DgradArgs& a, float* colsum, float* wgrad, const void* x0, float* wgrad0,
                            cudaStream_t st) {
  constexpr size_t kH = ((size_t)N * KP * 2 + (size_t)sgp::kRows * KP * 2 + 1023) / 1024 * 1024;
  constexpr size_t smem = kH + (size_t)(N < 128 ? 2 : N / 64) * sgp::kRows * 128 + (L0 ? sgp::kRows * 64 : 0) + 64 +
                          1024;
  static std::atomic<unsigned long long> done{0};
  if (!smem_opt_in(reinterpret_cast<const void*>(sgp::policy_dgrad_tma_kernel<N, KP, L0>), (int)smem, done))
    return fail(SG_ERR_SIM, "policy: cannot reserve shared memory");
  CUtensorMap mh, mdz, mx0;
  bool ok = encode_rows128(&mh, a.h, N, a.m);
  if (L0) {  // x_0: [m x 32] bf16, one 32-column x 128-row box, 64-byte swizzle
    const TensorMapEncodeFn enc = tensor_map_encode();
    const cuuint64_t dims[2] = {32, (cuuint64_t)a.m};
    const cuuint64_t strides[1] = {64};
    const cuuint32_t box[2] = {32, 128};
    const cuuint32_t estr[2] = {1, 1};
    ok = ok && enc &&
         enc(&mx0, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x0), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    mdz = mh;
  } else {
    ok = ok && encode_rows128(&mdz, a.dz, N, a.m);
    mx0 = mh;
  }
  if (!ok) return fail(SG_ERR_SIM, "sg_policy_layer_backward: cuTensorMapEncodeTiled failed");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (a.m + sgp::kRows - 1) / sgp::kRows;
  if constexpr (L0) {
    static const bool one_tile = getenv("SG_BWD_HEAD_ONETILE") != nullptr;  // A/B: the one-tile kernel
    if (!one_tile) {
      constexpr size_t hsmem = ((size_t)N * KP * 2 + (size_t)sgp::kRows * KP * 2) + 4 * (size_t)sgp::kRows * 128 +
                               2 * (size_t)sgp::kRows * 64 + 128 + 1024;
      static std::atomic<unsigned long long> hdone{0};
      if (!smem_opt_in(reinterpret_cast<const void*>(sgp::policy_bwd_head_kernel), (int)hsmem, hdone))
        return fail(SG_ERR_SIM, "policy: cannot reserve shared memory");
      sgp::policy_bwd_head_kernel<<<(unsigned)(tiles < sms ? tiles : sms), 256, hsmem, st>>>(mh, mx0, a, colsum,
                                                                                               wgrad, wgrad0);
      const cudaError_t e = cudaGetLastError();
      return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
    }
  }
  sgp::policy_dgrad_tma_kernel<N, KP, L0>
      <<<(unsigned)(tiles < sms ? tiles : sms), 256, smem, st>>>(mh, mdz, mx0, a, colsum, wgrad, wgrad0);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

static int launch_bwd_tail(const sgp::TailArgs& a, const void* h3, const void* h2, void* dz1, cudaStream_t st) {
  constexpr size_t smem = 71 * 1024 + 64 + 1024;
  static std::atomic<unsigned long long> done{0};
  if (!smem_opt_in(reinterpret_cast<const void*>(sgp::policy_bwd_tail_kernel), (int)smem, done))
    return fail(SG_ERR_SIM, "policy: cannot reserve shared memory");
  CUtensorMap mh3, mh2, mdz1;
  if (!encode_rows128(&mh3, h3, 64, a.m) || !encode_rows128(&mh2, h2, 128, a.m) ||
      !encode_rows128(&mdz1, dz1, 128, a.m))
    return fail(SG_ERR_SIM, "sg_policy_backward_tail: cuTensorMapEncodeTiled failed");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (a.m + sgp::kRows - 1) / sgp::kRows;
  const int64_t grid = tiles < 2 * sms ? tiles : 2 * sms;
  sgp::policy_bwd_tail_kernel<<<(unsigned)grid, 256, smem, st>>>(mh3, mh2, mdz1, a);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

extern "C" {

int sg_adam_step(float* d_params, float* d_grad, float* d_m, float* d_v, void* d_bf16_mirror, int64_t n,
                 float* d_grad_sq, int32_t* d_step, double lr, double beta1, double beta2, double eps,
                 double max_grad_norm, int64_t log_std_offset, int32_t log_std_n, double log_std_min,
                 double log_std_max, void* stream) {
  const cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(d_grad_sq, 0, sizeof(float), st);
  sgp::grad_sq_kernel<<<148, 512, 0, st>>>(d_grad, n, d_grad_sq, d_step);
  const sgp::AdamArgs a{(float)lr, (float)beta1, (float)beta2, (float)eps, (float)max_grad_norm, log_std_offset,
                        log_std_n, (float)log_std_min, (float)log_std_max};
  const int b = 256;
  sgp::adam_kernel<<<(unsigned)((n + b - 1) / b), b, 0, st>>>(d_params, d_grad, d_m, d_v,
                                                               (__nv_bfloat16*)d_bf16_mirror, n, d_grad_sq, d_step, a);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}


const char* sg_policy_last_error(void) { return g_policy_err.c_str(); }

int sg_policy_create(int32_t obs_dim, int32_t action_dim, const int32_t* hidden, int32_t n_hidden, int32_t device,
                     sg_policy** out) {
  // Policy::Policy (policy.cpp:42-63); the tensor-core kernel is built for the
  // reference's default trunk 256/128/64 and obs_dim <= 32, action_dim <= 16.
  if (obs_dim < 1 || action_dim < 1) return fail(SG_ERR_CONFIG, "policy: bad dimensions");
  if (n_hidden != 3 || hidden[0] != 256 || hidden[1] != 128 || hidden[2] != 64)
    return fail(SG_ERR_CONFIG, "policy: the sm_100a kernel implements hidden = {256, 128, 64}");
  if (obs_dim > sgp::kK0 || action_dim > sgp::kNOut)
    return fail(SG_ERR_CONFIG, "policy: obs_dim <= 32 and action_dim <= 16 required");
  if (cudaSetDevice(device) != cudaSuccess) return fail(SG_ERR_SIM, "policy: cudaSetDevice failed");
  auto* p = new sg_policy;
  p->obs_dim = obs_dim;
  p->act_dim = action_dim;
  p->device = device;
  int64_t off = 0;
  const int dims[5] = {obs_dim, 256, 128, 64, 0};
  for (int trunk = 0; trunk < 2; ++trunk) {
    const int out_last = trunk == 0 ? action_dim : 1;
    for (int l = 0; l < 4; ++l) {
      const int in = dims[l], o = l < 3 ? dims[l + 1] : out_last;
      p->table.w_off[trunk][l] = off;
      off += (int64_t)o * in;
      p->table.b_off[trunk][l] = off;
      off += o;
      p->table.in_dim[l] = in;
      p->table.out_dim[trunk][l] = o;
    }
  }
  p->log_std_offset = off;
  p->param_count = off + action_dim;
  if (cudaMalloc(&p->img, 32768 + 65536 * 2 + 36864) != cudaSuccess ||
      cudaMalloc(&p->bias, 928 * sizeof(float)) != cudaSuccess) {
    delete p;
    return fail(SG_ERR_SIM, "policy: cudaMalloc failed");
  }
  cudaMemset(p->img, 0, 32768 + 65536 * 2 + 36864);
  cudaMemset(p->bias, 0, 928 * sizeof(float));
  if (cudaFuncSetAttribute(sgp::policy_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sgp::kSmem) !=
      cudaSuccess) {
    delete p;
    return fail(SG_ERR_SIM, "policy: cannot reserve shared memory");
  }
  *out = p;
  return SG_OK;
}

void sg_policy_destroy(sg_policy* p) {
  if (!p) return;
  cudaFree(p->img);
  cudaFree(p->bias);
  delete p;
}

int sg_policy_param_count(const sg_policy* p, int64_t* count, int64_t* log_std_offset) {
  *count = p->param_count;
  *log_std_offset = p->log_std_offset;
  return SG_OK;
}

// Policy::init_params (policy.cpp:87-102): weights N(0, 2/fan_in) from
// make_stream(seed, 0x9019) in (trunk, layer, row, col) order, last layer
// scaled by 0.01, biases 0, log-std = init_log_std. Host fp64, then fp32.
int sg_policy_init_params(const sg_policy* p, uint64_t seed, double init_log_std, float* h_flat) {
  uint64_t x = seed ^ (0x2545f4914f6cdd1dULL * (0x9019ULL + 1));
  auto splitmix = [&]() {
    x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  const uint64_t initstate = splitmix(), initseq = splitmix();
  uint64_t st = 0, inc = (initseq << 1u) | 1u;
  auto next = [&]() {
    const uint64_t old = st;
    st = old * 6364136223846793005ULL + inc;
    const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u), rot = (uint32_t)(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  };
  next();
  st += initstate;
  next();
  auto normal = [&]() {
    const double u1 = (next() + 0.5) * 0x1.0p-32;
    const double u2 = next() * 0x1.0p-32;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586477 * u2);
  };
  for (int64_t k = 0; k < p->param_count; ++k) h_flat[k] = 0.f;
  for (int trunk = 0; trunk < 2; ++trunk)
    for (int l = 0; l < 4; ++l) {
      const int rows = p->table.out_dim[trunk][l], cols = p->table.in_dim[l];
      const double scale = std::sqrt(2.0 / cols);
      for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
          double w = scale * normal();
          if (l == 3) w *= 0.01;
          h_flat[p->table.w_off[trunk][l] + (int64_t)r * cols + c] = (float)w;
        }
    }
  for (int a = 0; a < p->act_dim; ++a) h_flat[p->log_std_offset + a] = (float)init_log_std;
  return SG_OK;
}

int sg_policy_load_params(sg_policy* p, const float* d_flat, void* stream) {
  const int64_t total = 512 * 32 + 2 * 128 * 256 + 2 * 64 * 128 + 2 * 16 * 64 + 928;
  const int b = 256;
  sgp::policy_pack_kernel<<<(unsigned)((total + b - 1) / b), b, 0, (cudaStream_t)stream>>>(
      d_flat, p->table, p->img, p->img + 32768, p->img + 32768 + 65536, p->img + 32768 + 131072, p->bias);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

static sgp::Jump64 jump_table(uint64_t inc) {  // J[b] = 2^b PCG32 advances of the stream
  sgp::Jump64 J;
  uint64_t cm = 6364136223846793005ULL, ca = inc;
  for (int b = 0; b < 64; ++b) {
    J.mult[b] = cm;
    J.add[b] = ca;
    ca = (cm + 1) * ca;
    cm *= cm;
  }
  return J;
}

struct SampleArgs {
  const float* log_std_raw = nullptr;
  uint64_t s0 = 0, inc = 0;
  const uint64_t* pos = nullptr;
  uint64_t step_off = 0;
  float* actions = nullptr;
  float* logp = nullptr;
  const double* noise = nullptr;
  // folded bootstrap of the previous step
  const float* boot_obs = nullptr;
  int32_t boot_stride = 0;
  const uint8_t* boot_timed_out = nullptr;
  const uint8_t* boot_terminated = nullptr;
  float* boot_value = nullptr;
};

static int policy_forward(const sg_policy* p, const float* d_obs, int64_t n, int32_t obs_stride, float* d_mean,
                          float* d_value, const uint8_t* d_timed_out, const uint8_t* d_terminated, void* stream,
                          const SampleArgs& smp = SampleArgs()) {
  if (n <= 0) return SG_OK;
  sgp::PolicyImage W;
  W.w1 = p->img;
  W.w2a = p->img + 32768;
  W.w2c = p->img + 32768 + 65536;
  W.w34 = p->img + 32768 + 131072;
  W.b1 = p->bias;
  W.b2a = p->bias + 512;
  W.b2c = p->bias + 640;
  W.b3a = p->bias + 768;
  W.b3c = p->bias + 832;
  W.b4a = p->bias + 896;
  W.b4c = p->bias + 912;
  sgp::FwdArgs a{d_obs, n, p->obs_dim, obs_stride > 0 ? obs_stride : p->obs_dim, p->act_dim, d_mean, d_value,
                 d_timed_out, d_terminated, smp.log_std_raw, smp.s0, smp.inc, smp.pos, smp.step_off, smp.actions,
                 smp.logp, smp.noise, smp.boot_obs, smp.boot_stride, smp.boot_timed_out, smp.boot_terminated,
                 smp.boot_value};
  static const sgp::Jump64 kNone{};
  const sgp::Jump64 J = smp.actions && !smp.noise ? jump_table(smp.inc) : kNone;
  const unsigned grid = (unsigned)((n + sgp::kRows - 1) / sgp::kRows);
  static const bool no_pdl = getenv("SG_NO_PDL") != nullptr;  // A/B: plain stream-ordered launch
  if (no_pdl) {
    sgp::policy_fwd_kernel<<<grid, sgp::kThreads, sgp::kSmem, (cudaStream_t)stream>>>(W, a, J);
  } else {  // programmatic dependent launch: the prologue may start while the previous kernel drains
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(sgp::kThreads);
    cfg.dynamicSmemBytes = sgp::kSmem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, sgp::policy_fwd_kernel, W, a, J);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

int sg_policy_forward(const sg_policy* p, const float* d_obs, int64_t n, int32_t obs_stride, float* d_mean,
                      float* d_value, void* stream) {
  return policy_forward(p, d_obs, n, obs_stride, d_mean, d_value, nullptr, nullptr, stream);
}

int sg_policy_bootstrap(const sg_policy* p, const float* d_terminal_obs, int64_t n, int32_t obs_stride,
                        const uint8_t* d_timed_out, const uint8_t* d_terminated, float* d_value, void* stream) {
  return policy_forward(p, d_terminal_obs, n, obs_stride, nullptr, d_value, d_timed_out, d_terminated, stream);
}

int sg_policy_act(const sg_policy* p, const float* d_obs, int64_t n, int32_t obs_stride, const float* d_log_std_raw,
                  uint64_t stream_state, uint64_t stream_inc, const uint64_t* d_draw_pos, uint64_t step_offset,
                  float* d_actions, float* d_logp, float* d_mean, float* d_value, void* stream) {
  if (!d_actions || !d_logp || !d_log_std_raw || !d_draw_pos || !d_value)
    return fail(SG_ERR_CONFIG, "sg_policy_act: null argument");
  if (p->act_dim > sgp::kNOut) return fail(SG_ERR_CONFIG, "sg_policy_act: action_dim > 16");
  SampleArgs smp;
  smp.log_std_raw = d_log_std_raw;
  smp.s0 = stream_state;
  smp.inc = stream_inc;
  smp.pos = d_draw_pos;
  smp.step_off = step_offset;
  smp.actions = d_actions;
  smp.logp = d_logp;
  return policy_forward(p, d_obs, n, obs_stride, d_mean, d_value, nullptr, nullptr, stream, smp);
}

int sg_policy_act_bootstrap(const sg_policy* p, const float* d_obs, int64_t n, int32_t obs_stride,
                            const float* d_log_std_raw, uint64_t stream_state, uint64_t stream_inc,
                            const uint64_t* d_draw_pos, uint64_t step_offset, float* d_actions, float* d_logp,
                            float* d_mean, float* d_value, const float* d_boot_obs, int32_t boot_stride,
                            const uint8_t* d_timed_out, const uint8_t* d_terminated, float* d_boot_value,
                            void* stream) {
  if (!d_actions || !d_logp || !d_log_std_raw || !d_draw_pos || !d_value)
    return fail(SG_ERR_CONFIG, "sg_policy_act_bootstrap: null argument");
  if (!d_boot_obs || !d_timed_out || !d_terminated || !d_boot_value)
    return fail(SG_ERR_CONFIG, "sg_policy_act_bootstrap: null bootstrap argument");
  if (p->act_dim > sgp::kNOut) return fail(SG_ERR_CONFIG, "sg_policy_act_bootstrap: action_dim > 16");
  SampleArgs smp;
  smp.log_std_raw = d_log_std_raw;
  smp.s0 = stream_state;
  smp.inc = stream_inc;
  smp.pos = d_draw_pos;
  smp.step_off = step_offset;
  smp.actions = d_actions;
  smp.logp = d_logp;
  smp.boot_obs = d_boot_obs;
  smp.boot_stride = boot_stride > 0 ? boot_stride : p->obs_dim;
  smp.boot_timed_out = d_timed_out;
  smp.boot_terminated = d_terminated;
  smp.boot_value = d_boot_value;
  return policy_forward(p, d_obs, n, obs_stride, d_mean, d_value, nullptr, nullptr, stream, smp);
}

int sg_policy_noise(const sg_policy* p, int64_t n, const float* d_log_std_raw, uint64_t stream_state,
                    uint64_t stream_inc, const uint64_t* d_draw_pos, uint64_t step_offset, double* d_scaled_noise,
                    float* d_logp, void* stream) {
  if (n <= 0) return SG_OK;
  if (!d_log_std_raw || !d_draw_pos || !d_scaled_noise || !d_logp)
    return fail(SG_ERR_CONFIG, "sg_policy_noise: null argument");
  if (p->act_dim > sgp::kNOut) return fail(SG_ERR_CONFIG, "sg_policy_noise: action_dim > 16");
  const sgp::Jump64 J = jump_table(stream_inc);
  const int A = p->act_dim;
  sgp::policy_noise_kernel<<<(unsigned)((n + 31) / 32), 32 * A, 0, (cudaStream_t)stream>>>(
      n, A, d_log_std_raw, stream_state, stream_inc, d_draw_pos, step_offset, J, d_scaled_noise, d_logp);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

int sg_policy_act_noise(const sg_policy* p, const float* d_obs, int64_t n, int32_t obs_stride,
                        const double* d_scaled_noise, float* d_actions, float* d_mean, float* d_value, void* stream) {
  if (!d_actions || !d_scaled_noise || !d_value) return fail(SG_ERR_CONFIG, "sg_policy_act_noise: null argument");
  if (p->act_dim > sgp::kNOut) return fail(SG_ERR_CONFIG, "sg_policy_act_noise: action_dim > 16");
  SampleArgs smp;
  smp.actions = d_actions;
  smp.noise = d_scaled_noise;
  return policy_forward(p, d_obs, n, obs_stride, d_mean, d_value, nullptr, nullptr, stream, smp);
}

int sg_policy_train_forward(const sg_policy* p, const void* d_obs_bf16, int64_t n, int32_t obs_stride, void* d_h1,
                            void* d_h2, void* d_h3, void* d_out, void* stream) {
  if (n <= 0) return SG_OK;
  if (!d_obs_bf16 || !d_h1 || !d_h2 || !d_h3 || !d_out)
    return fail(SG_ERR_CONFIG, "sg_policy_train_forward: null argument");
  if (obs_stride < sgp::kK0 || obs_stride % 8 != 0)
    return fail(SG_ERR_CONFIG, "sg_policy_train_forward: obs_stride must be >= 32 and a multiple of 8");
  static std::atomic<unsigned long long> done{0};
  if (!smem_opt_in(reinterpret_cast<const void*>(sgp::policy_train_fwd_kernel), (int)sgp::kSmem, done))
    return fail(SG_ERR_SIM, "policy: cannot reserve shared memory");
  sgp::PolicyImage W;
  W.w1 = p->img;
  W.w2a = p->img + 32768;
  W.w2c = p->img + 32768 + 65536;
  W.w34 = p->img + 32768 + 131072;
  W.b1 = p->bias;
  W.b2a = p->bias + 512;
  W.b2c = p->bias + 640;
  W.b3a = p->bias + 768;
  W.b3c = p->bias + 832;
  W.b4a = p->bias + 896;
  W.b4c = p->bias + 912;
  const sgp::TrainFwdArgs a{static_cast<const __nv_bfloat16*>(d_obs_bf16), n, obs_stride,
                            static_cast<__nv_bfloat16*>(d_h1), static_cast<__nv_bfloat16*>(d_h2),
                            static_cast<__nv_bfloat16*>(d_h3), static_cast<__nv_bfloat16*>(d_out)};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (n + sgp::kRows - 1) / sgp::kRows;
  const unsigned grid = (unsigned)(tiles < sms ? tiles : sms);
  sgp::policy_train_fwd_kernel<<<grid, sgp::kThreads, sgp::kSmem, (cudaStream_t)stream>>>(W, a);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

int sg_policy_pack_wt(const float* d_flat, const int64_t* w_off, const int32_t* out_dim, const int32_t* in_dim,
                      uint8_t* d_images, void* stream) {
  sgp::WtTable t{};
  int64_t off = 0, total = 0;
  for (int i = 0; i < 6; ++i) {
    t.w_off[i] = w_off[i];
    t.k[i] = out_dim[i];
    t.n[i] = in_dim[i];
    t.kp[i] = (out_dim[i] + 15) / 16 * 16;
    t.img_off[i] = off;
    off += (int64_t)t.n[i] * t.kp[i] * 2;
    total += (int64_t)t.n[i] * t.kp[i];
  }
  t.total = total;
  const int b = 256;
  sgp::policy_pack_wt_kernel<<<(unsigned)((total + b - 1) / b), b, 0, (cudaStream_t)stream>>>(d_flat, t, d_images);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

int sg_policy_wgrad(const void* d_dy, int32_t out_dim, const void* d_x, int32_t in_dim, int64_t m,
                    float* d_partial, int32_t parts, float* d_grad, void* stream) {
  if (m <= 0) return SG_OK;
  if (!d_dy || !d_x || !d_partial || !d_grad || parts < 1) return fail(SG_ERR_CONFIG, "sg_policy_wgrad: bad argument");
  const cudaStream_t st = (cudaStream_t)stream;
  const bool tma = std::getenv("SG_WGRAD_CPASYNC") == nullptr;  // A/B: the cp.async ring
  const bool red = std::getenv("SG_WGRAD_PARTIALS") == nullptr;   // A/B: partials + reduction pass
  if (out_dim == 256 && in_dim == 32) {
    if (!tma) return launch_wgrad<256, 32>(d_dy, d_x, m, d_partial, parts, d_grad, st);
    return red ? launch_wgrad_tma<256, 32, true>(d_dy, d_x, m, d_partial, parts, d_grad, st)
               : launch_wgrad_tma<256, 32, false>(d_dy, d_x, m, d_partial, parts, d_grad, st);
  }
  if (out_dim == 128 && in_dim == 256) {
    if (!tma) return launch_wgrad<128, 256>(d_dy, d_x, m, d_partial, parts, d_grad, st);
    return red ? launch_wgrad_tma<128, 256, true>(d_dy, d_x, m, d_partial, parts, d_grad, st)
               : launch_wgrad_tma<128, 256, false>(d_dy, d_x, m, d_partial, parts, d_grad, st);
  }
  if (out_dim == 64 && in_dim == 128) {
    if (!tma) return launch_wgrad<64, 128>(d_dy, d_x, m, d_partial, parts, d_grad, st);
    return red ? launch_wgrad_tma<64, 128, true>(d_dy, d_x, m, d_partial, parts, d_grad, st)
               : launch_wgrad_tma<64, 128, false>(d_dy, d_x, m, d_partial, parts, d_grad, st);
  }
  if (out_dim == 8 && in_dim == 64) return launch_wgrad<8, 64>(d_dy, d_x, m, d_partial, parts, d_grad, st);
  return fail(SG_ERR_CONFIG, "sg_policy_wgrad: layer shape not instantiated (256/128/64 trunk, padded obs / outputs)");
}

int sg_policy_dgrad_elu(const void* d_dy, int32_t dy_stride, int32_t k, const void* d_wt_image, int32_t n_in,
                        const void* d_h, void* d_dz, int64_t m, void* stream) {
  if (m <= 0) return SG_OK;
  if (!d_dy || !d_wt_image || !d_h || !d_dz) return fail(SG_ERR_CONFIG, "sg_policy_dgrad_elu: null argument");
  const sgp::DgradArgs a{static_cast<const __nv_bfloat16*>(d_dy), dy_stride, k,
                         static_cast<const uint8_t*>(d_wt_image), static_cast<const __nv_bfloat16*>(d_h),
                         static_cast<__nv_bfloat16*>(d_dz), m};
  const cudaStream_t st = (cudaStream_t)stream;
  const int kp = (k + 15) / 16 * 16;
  if (n_in == 64 && kp == 16) return launch_dgrad<64, 16>(a, st);
  if (n_in == 128 && kp == 64) return launch_dgrad<128, 64>(a, st);
  if (n_in == 256 && kp == 128) return launch_dgrad<256, 128>(a, st);
  return fail(SG_ERR_CONFIG, "sg_policy_dgrad_elu: layer shape not instantiated (256/128/64 trunk)");
}

int sg_policy_layer_backward(const void* d_dy, int32_t dy_stride, int32_t k, const void* d_wt_image, int32_t n_in,
                             const void* d_h, void* d_dz, int64_t m, float* d_colsum, float* d_wgrad,
                             const void* d_x0, int32_t x0_width, float* d_wgrad0, void* stream) {
  if (m <= 0) return SG_OK;
  if (!d_dy || !d_wt_image || !d_h) return fail(SG_ERR_CONFIG, "sg_policy_layer_backward: null argument");
  if (d_x0) {
    if (n_in != 256 || (k + 15) / 16 * 16 != 128 || x0_width != 32 || !d_wgrad0)
      return fail(SG_ERR_CONFIG, "sg_policy_layer_backward: x0 needs the 256-wide layer, x0_width 32 and d_wgrad0");
  } else if (!d_dz) {
    return fail(SG_ERR_CONFIG, "sg_policy_layer_backward: null d_dz");
  }
  const sgp::DgradArgs a{static_cast<const __nv_bfloat16*>(d_dy), dy_stride, k,
                         static_cast<const uint8_t*>(d_wt_image), static_cast<const __nv_bfloat16*>(d_h),
                         static_cast<__nv_bfloat16*>(d_dz), m};
  const cudaStream_t st = (cudaStream_t)stream;
  const int kp = (k + 15) / 16 * 16;
  if (n_in == 64 && kp == 16) return launch_dgrad_tma<64, 16, false>(a, d_colsum, d_wgrad, nullptr, nullptr, st);
  if (n_in == 128 && kp == 64) return launch_dgrad_tma<128, 64, false>(a, d_colsum, d_wgrad, nullptr, nullptr, st);
  if (n_in == 256 && kp == 128)
    return d_x0 ? launch_dgrad_tma<256, 128, true>(a, d_colsum, d_wgrad, d_x0, d_wgrad0, st)
                : launch_dgrad_tma<256, 128, false>(a, d_colsum, d_wgrad, nullptr, nullptr, st);
  return fail(SG_ERR_CONFIG, "sg_policy_layer_backward: layer shape not instantiated (256/128/64 trunk)");
}

int sg_policy_backward_tail(const void* d_dy3, int32_t dy3_stride, int32_t k3, const void* d_wt3_image,
                            const void* d_wt2_image, const void* d_h3, const void* d_h2, void* d_dz1, int64_t m,
                            float* d_db3, float* d_dw3, float* d_db2, float* d_dw2, float* d_db1, void* stream) {
  if (m <= 0) return SG_OK;
  if (!d_dy3 || !d_wt3_image || !d_wt2_image || !d_h3 || !d_h2 || !d_dz1 || !d_db3 || !d_dw3 || !d_db2 || !d_dw2 ||
      !d_db1)
    return fail(SG_ERR_CONFIG, "sg_policy_backward_tail: null argument");
  if (k3 < 1 || k3 > 8 || dy3_stride < 8 || dy3_stride % 8 != 0)
    return fail(SG_ERR_CONFIG, "sg_policy_backward_tail: k3 in 1..8 and a 16-byte row stride");
  const sgp::TailArgs a{static_cast<const __nv_bfloat16*>(d_dy3), dy3_stride, k3,
                        static_cast<const uint8_t*>(d_wt3_image), static_cast<const uint8_t*>(d_wt2_image), m,
                        d_db3, d_dw3, d_db2, d_dw2, d_db1};
  return launch_bwd_tail(a, d_h3, d_h2, d_dz1, (cudaStream_t)stream);
}

int sg_policy_set_param_layout(sg_policy* p, const int64_t* w_off, const int64_t* b_off, const int32_t* in_dim,
                               const int32_t* out_dim) {
  for (int t = 0; t < 2; ++t)
    for (int l = 0; l < 4; ++l) {
      p->table.w_off[t][l] = w_off[4 * t + l];
      p->table.b_off[t][l] = b_off[4 * t + l];
      p->table.out_dim[t][l] = out_dim[4 * t + l];
    }
  for (int l = 0; l < 4; ++l) p->table.in_dim[l] = in_dim[l];
  return SG_OK;
}

int sg_policy_sample(const float* d_mean, int64_t n, int32_t action_dim, const float* d_log_std_raw,
                     uint64_t stream_state, uint64_t stream_inc, const uint64_t* d_draw_pos, uint64_t step_offset,
                     float* d_actions, float* d_logp, void* stream) {
  if (n <= 0) return SG_OK;
  const sgp::Jump64 J = jump_table(stream_inc);
  const int b = 128;
  sgp::policy_sample_kernel<<<(unsigned)((n + b - 1) / b), b, 0, (cudaStream_t)stream>>>(
      d_mean, n, action_dim, d_log_std_raw, stream_state, stream_inc, d_draw_pos, step_offset, J, d_actions, d_logp);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

// ---- checkpoints (save_checkpoint / load_checkpoint, policy.cpp:220-295) ---
// Byte layout of the reference: "SCLPCKP1", u32 version 1, u32 obs_dim,
// u32 action_dim, u32 n_hidden, n_hidden x u32, u32-length-prefixed robot and
// task strings, u64 param count, param_count little-endian fp64.
namespace {
constexpr char kCkptMagic[8] = {'S', 'C', 'L', 'P', 'C', 'K', 'P', '1'};
constexpr uint32_t kCkptVersion = 1;

int64_t trunk_param_count(int obs_dim, int act_dim, const int32_t* hidden, int n_hidden) {
  int64_t total = 0;
  for (int trunk = 0; trunk < 2; ++trunk) {  // Policy::Policy (policy.cpp:42-63)
    int in = obs_dim;
    for (int l = 0; l <= n_hidden; ++l) {
      const int out = l < n_hidden ? hidden[l] : (trunk == 0 ? act_dim : 1);
      total += (int64_t)out * in + out;
      in = out;
    }
  }
  return total + act_dim;  // log_std
}
}  // namespace

int sg_checkpoint_save(const char* path, int32_t obs_dim, int32_t action_dim, const int32_t* hidden,
                       int32_t n_hidden, const char* robot, const char* task, const double* h_params,
                       int64_t param_count) {
  if (param_count != trunk_param_count(obs_dim, action_dim, hidden, n_hidden))
    return fail(SG_ERR_CONFIG, "checkpoint: parameter count does not match the shape");
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(SG_ERR_SIM, std::string("cannot write checkpoint '") + path + "'");
  bool ok = std::fwrite(kCkptMagic, 1, 8, f) == 8;
  const auto u32 = [&](uint32_t v) { ok = ok && std::fwrite(&v, 4, 1, f) == 1; };
  const auto str = [&](const char* c) {
    const std::string v = c ? c : "";
    u32(static_cast<uint32_t>(v.size()));
    ok = ok && std::fwrite(v.data(), 1, v.size(), f) == v.size();
  };
  u32(kCkptVersion);
  u32(static_cast<uint32_t>(obs_dim));
  u32(static_cast<uint32_t>(action_dim));
  u32(static_cast<uint32_t>(n_hidden));
  for (int i = 0; i < n_hidden; ++i) u32(static_cast<uint32_t>(hidden[i]));
  str(robot);
  str(task);
  const uint64_t cnt = static_cast<uint64_t>(param_count);
  ok = ok && std::fwrite(&cnt, 8, 1, f) == 1;
  ok = ok && std::fwrite(h_params, sizeof(double), param_count, f) == static_cast<size_t>(param_count);
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return fail(SG_ERR_SIM, std::string("short write on checkpoint '") + path + "'");
  return SG_OK;
}

int sg_checkpoint_load(const char* path, int32_t* obs_dim, int32_t* action_dim, int32_t* hidden, int32_t* n_hidden,
                       char* robot, int32_t robot_cap, char* task, int32_t task_cap, double* h_params,
                       int64_t params_cap, int64_t* param_count) {
  FILE* f = std::fopen(path, "rb");
  const std::string p = path;
  if (!f) return fail(SG_ERR_CONFIG, "cannot open checkpoint '" + p + "'");
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  bool ok = true;
  const auto u32 = [&]() {
    uint32_t v = 0;
    ok = ok && std::fread(&v, 4, 1, f) == 1;
    return v;
  };
  char magic[8];
  if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kCkptMagic, 8) != 0)
    return fail(SG_ERR_CONFIG, "'" + p + "' is not a scalpel checkpoint");
  const uint32_t version = u32();
  if (version != kCkptVersion)
    return fail(SG_ERR_CONFIG, "checkpoint '" + p + "' has unsupported version " + std::to_string(version));
  const int od = static_cast<int>(u32()), ad = static_cast<int>(u32());
  const uint32_t nh = u32();
  if (!ok || nh > 64) return fail(SG_ERR_CONFIG, "corrupt checkpoint '" + p + "'");
  std::vector<int32_t> hid(nh);
  for (auto& h : hid) h = static_cast<int32_t>(u32());
  std::string strs[2];
  for (auto& s : strs) {
    const uint32_t len = u32();
    if (!ok || len > (1u << 20)) return fail(SG_ERR_CONFIG, "corrupt checkpoint '" + p + "'");
    s.resize(len);
    ok = ok && std::fread(s.data(), 1, len, f) == len;
  }
  uint64_t cnt = 0;
  ok = ok && std::fread(&cnt, 8, 1, f) == 1;
  if (!ok) return fail(SG_ERR_CONFIG, "checkpoint '" + p + "' is truncated");
  if (static_cast<int64_t>(cnt) != trunk_param_count(od, ad, hid.data(), static_cast<int>(nh)))
    return fail(SG_ERR_CONFIG, "checkpoint '" + p + "' parameter count does not match its shape header");
  if (obs_dim) *obs_dim = od;
  if (action_dim) *action_dim = ad;
  if (n_hidden) *n_hidden = static_cast<int32_t>(nh);
  if (hidden)
    for (uint32_t i = 0; i < nh && i < 64; ++i) hidden[i] = hid[i];
  const auto put = [](char* dst, int32_t cap, const std::string& v) {
    if (!dst || cap <= 0) return;
    const size_t k = std::min(v.size(), static_cast<size_t>(cap - 1));
    std::memcpy(dst, v.data(), k);
    dst[k] = '\0';
  };
  put(robot, robot_cap, strs[0]);
  put(task, task_cap, strs[1]);
  if (param_count) *param_count = static_cast<int64_t>(cnt);
  if (h_params) {
    if (params_cap < static_cast<int64_t>(cnt)) return fail(SG_ERR_CONFIG, "checkpoint: parameter buffer too small");
    if (std::fread(h_params, sizeof(double), cnt, f) != cnt)
      return fail(SG_ERR_CONFIG, "checkpoint '" + p + "' is truncated");
  }
  return SG_OK;
}

int sg_compute_gae(const float* d_rewards, const float* d_values, const uint8_t* d_terminated,
                   const uint8_t* d_timed_out, const float* d_bootstrap, const float* d_last_values,
                   const float* d_task_error, int32_t n_steps, int64_t n_envs, double gamma, double lambda,
                   float* d_advantages, float* d_returns, float* d_ep_acc, double* d_stats4, void* stream) {
  const int b = 128;
  sgp::gae_kernel<<<(unsigned)((n_envs + b - 1) / b), b, 0, (cudaStream_t)stream>>>(
      d_rewards, d_values, d_terminated, d_timed_out, d_bootstrap, d_last_values, d_task_error, n_steps, n_envs,
      (float)gamma, (float)lambda, d_advantages, d_returns, d_ep_acc, d_stats4);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : fail(SG_ERR_SIM, cudaGetErrorString(e));
}

}  // extern "C"
