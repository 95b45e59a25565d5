// Launch-path probe (experiments only): event-to-event device time of empty
// launches of several shapes, gated behind a spin kernel like bench.py, after
// a 256 MiB L2 flush. Separates the event pair, the launch, and the grid size.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void spin_kernel(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}
__global__ void empty_kernel(int* out) {
  if (threadIdx.x == 0 && out) out[blockIdx.x & 4095] = 1;
}
__global__ void smem_kernel(int* out) {
  extern __shared__ int s[];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && out) out[blockIdx.x & 4095] = s[5];
}

int main() {
  const size_t flush_bytes = 256ull << 20;
  void* flush;
  int* out;
  cudaMalloc(&flush, flush_bytes);
  cudaMalloc(&out, 4096 * sizeof(int));
  cudaFuncSetAttribute(smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int reps = 20;
  cudaEvent_t ev[2 * reps];
  for (int k = 0; k < 2 * reps; ++k) cudaEventCreate(&ev[k]);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const char* names[] = {"events only", "empty 1x32", "empty 148x64", "empty 512x64", "2x empty 512x64",
                         "empty 512x64 + 10 KB smem", "empty 4096x64", "memset 4 B", "empty 512x64 no flush", "graph: empty 512x64", "graph: 2x empty 512x64"};
  cudaGraph_t g1, g2;
  cudaGraphExec_t x1, x2;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  empty_kernel<<<512, 64, 0, st>>>(out);
  cudaStreamEndCapture(st, &g1);
  cudaGraphInstantiate(&x1, g1, 0);
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  empty_kernel<<<512, 64, 0, st>>>(out);
  empty_kernel<<<512, 64, 0, st>>>(out);
  cudaStreamEndCapture(st, &g2);
  cudaGraphInstantiate(&x2, g2, 0);
  cudaGraphUpload(x1, st);
  cudaGraphUpload(x2, st);
  for (int variant = 0; variant < 11; ++variant) {
    float total = 0.f;
    for (int batch = 0; batch < 3; ++batch) {
      spin_kernel<<<1, 1, 0, st>>>(20000000);
      for (int r = 0; r < reps; ++r) {
        if (variant != 8) cudaMemsetAsync(flush, r & 0xff, flush_bytes, st);
        cudaEventRecord(ev[2 * r], st);
        switch (variant) {
          case 0: break;
          case 1: empty_kernel<<<1, 32, 0, st>>>(out); break;
          case 2: empty_kernel<<<148, 64, 0, st>>>(out); break;
          case 3: case 8: empty_kernel<<<512, 64, 0, st>>>(out); break;
          case 4: empty_kernel<<<512, 64, 0, st>>>(out); empty_kernel<<<512, 64, 0, st>>>(out); break;
          case 5: smem_kernel<<<512, 64, 10 * 1024, st>>>(out); break;
          case 6: empty_kernel<<<4096, 64, 0, st>>>(out); break;
          case 7: cudaMemsetAsync(out, 0, 4, st); break;
          case 9: cudaGraphLaunch(x1, st); break;
          case 10: cudaGraphLaunch(x2, st); break;
        }
        cudaEventRecord(ev[2 * r + 1], st);
      }
      cudaStreamSynchronize(st);
      if (batch == 0) continue;
      for (int r = 0; r < reps; ++r) {
        float ms;
        cudaEventElapsedTime(&ms, ev[2 * r], ev[2 * r + 1]);
        total += ms;
      }
    }
    printf("launch probe 2: %-28s %.2f us (event to event, mean of %d)\n", names[variant], 1e3f * total / (2 * reps),
           2 * reps);
  }
  return 0;
}
