// fp64 issue-rate / latency probe on one GPU:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_probe tools/fp64_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

template <int ILP>
__global__ void dadd_chains(double* out, int iters, double a) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x + k;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), a);
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP>
void run(int blocks, int threads, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  dadd_chains<ILP><<<blocks, threads>>>(out, 16, 1.0000001);
  cudaEventRecord(e0);
  dadd_chains<ILP><<<blocks, threads>>>(out, iters, 1.0000001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * iters * ILP * (double)blocks * threads;  // DMUL + DADD lane-ops
  printf("ILP %2d blocks %5d threads %4d: %8.3f ms  %7.2f T DP lane-ops/s  (%.1f ns per dependent op pair)\n", ILP,
         blocks, threads, ms, ops / ms / 1e9, ms * 1e6 / iters);
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 26);
  for (int warps : {1, 4, 8, 16}) {
    run<1>(148, 32 * warps, out);
    run<4>(148, 32 * warps, out);
    run<16>(148, 32 * warps, out);
  }
  return 0;
}
