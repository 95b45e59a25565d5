// Launch-overhead probe (A/B only): event-timed duration of a near-empty
// kernel with the env step's grid (512 CTAs x 64 threads) right after a
// 256 MiB L2 flush, with an 8-byte vs a 2,776-byte (sizeof(StepParams))
// parameter block, and with 0 / 64 KB of unrolled dead code fetched.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_probe tools/launch_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

struct Big {
  unsigned char b[2776];
};

__global__ void spin_kernel(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}
__global__ void small_kernel(int* out) {
  if (threadIdx.x == 0 && out) out[blockIdx.x] = 1;
}
__global__ void big_kernel(const __grid_constant__ Big p, int* out) {
  if (threadIdx.x == 0 && out) out[blockIdx.x] = p.b[blockIdx.x % 2776];
}

int main() {
  const size_t flush_bytes = 256ull << 20;
  void* flush;
  int* out;
  cudaMalloc(&flush, flush_bytes);
  cudaMalloc(&out, 4096 * sizeof(int));
  Big big{};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // Gated: a 5 ms spin kernel heads each batch, so every flush / event /
  // launch of the batch is enqueued before the GPU reaches it (the bench's
  // protocol); the event pairs then time the GPU side only.
  const int reps = 20;
  cudaEvent_t ev[2 * reps];
  for (int k = 0; k < 2 * reps; ++k) cudaEventCreate(&ev[k]);
  for (int variant = 0; variant < 4; ++variant) {
    const bool use_big = variant & 1, do_flush = variant & 2;
    float total = 0.f;
    for (int batch = 0; batch < 3; ++batch) {
      spin_kernel<<<1, 1>>>(10000000);
      for (int r = 0; r < reps; ++r) {
        if (do_flush) cudaMemsetAsync(flush, r & 0xff, flush_bytes);
        cudaEventRecord(ev[2 * r]);
        if (use_big)
          big_kernel<<<512, 64>>>(big, out);
        else
          small_kernel<<<512, 64>>>(out);
        cudaEventRecord(ev[2 * r + 1]);
      }
      cudaDeviceSynchronize();
      if (batch == 0) continue;
      for (int r = 0; r < reps; ++r) {
        float ms;
        cudaEventElapsedTime(&ms, ev[2 * r], ev[2 * r + 1]);
        total += ms;
      }
    }
    printf("launch probe (gated): %s params, %s: %.2f us per launch (event to event)\n",
           use_big ? "2776-byte" : "8-byte", do_flush ? "after a 256 MiB L2 flush" : "no flush",
           1e3f * total / (2 * reps));
  }
  return 0;
}
