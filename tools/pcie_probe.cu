// PCIe transfer probe for the e2e (host-buffer) step path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/pcie_probe tools/pcie_probe.cu
// Measures, for the PSM config-2 StepResult sizes (16,384 envs):
//   copy-engine H2D / D2H alone and overlapped, zero-copy kernel writes to
//   pinned host memory and zero-copy reads, and the host cost of one
//   cudaMemcpyAsync / cudaLaunchKernel / cudaGraphLaunch call.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));                \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

__global__ void zc_write(float4* __restrict__ dst, const float4* __restrict__ src, size_t n4) {
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n4; k += (size_t)gridDim.x * blockDim.x)
    dst[k] = src[k];
}
__global__ void noop() {}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const size_t n = 16384, A = 7, O = 27;
  const size_t h2d = n * A * 4, d2h = n * O * 4 + n * 10;
  char *hi, *ho, *di, *dout;
  CK(cudaMallocHost(&hi, 64 << 20));
  CK(cudaMallocHost(&ho, 64 << 20));
  CK(cudaMalloc(&di, 64 << 20));
  CK(cudaMalloc(&dout, 64 << 20));
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int R = 200;
  auto timed = [&](auto&& body) -> float {
    for (int w = 0; w < 10; ++w) body();
    cudaDeviceSynchronize();
    cudaEventRecord(e0, s0);
    for (int r = 0; r < R; ++r) body();
    cudaStreamWaitEvent(s0, e0, 0);
    cudaEvent_t j;
    cudaEventCreate(&j);
    cudaEventRecord(j, s1);
    cudaStreamWaitEvent(s0, j, 0);
    cudaEventRecord(e1, s0);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(j);
    return ms * 1000.f / R;
  };
  for (size_t bytes : {h2d, d2h, (size_t)(8 << 20), (size_t)(32 << 20)}) {
    float t1 = timed([&] { cudaMemcpyAsync(di, hi, bytes, cudaMemcpyHostToDevice, s0); });
    float t2 = timed([&] { cudaMemcpyAsync(ho, dout, bytes, cudaMemcpyDeviceToHost, s0); });
    float t3 = timed([&] {
      cudaMemcpyAsync(di, hi, bytes, cudaMemcpyHostToDevice, s0);
      cudaMemcpyAsync(ho, dout, bytes, cudaMemcpyDeviceToHost, s1);
    });
    printf("bytes %9zu  H2D %8.2f us (%6.1f GB/s)  D2H %8.2f us (%6.1f GB/s)  both %8.2f us\n", bytes, t1,
           bytes / t1 / 1e3, t2, bytes / t2 / 1e3, t3);
  }
  for (int grid : {148, 296, 592, 1184}) {
    for (size_t bytes : {d2h, (size_t)(32 << 20)}) {
      float tw = timed([&] { zc_write<<<grid, 256, 0, s0>>>((float4*)ho, (const float4*)dout, bytes / 16); });
      float tr = timed([&] { zc_write<<<grid, 256, 0, s0>>>((float4*)di, (const float4*)hi, bytes / 16); });
      printf("zero-copy grid %5d bytes %9zu  write %8.2f us (%6.1f GB/s)  read %8.2f us (%6.1f GB/s)\n", grid, bytes,
             tw, bytes / tw / 1e3, tr, bytes / tr / 1e3);
    }
  }
  // host cost per API call
  {
    cudaDeviceSynchronize();
    double t = now_us();
    for (int r = 0; r < 1000; ++r) cudaMemcpyAsync(di, hi, 4096, cudaMemcpyHostToDevice, s0);
    double tm = (now_us() - t) / 1000;
    cudaDeviceSynchronize();
    t = now_us();
    for (int r = 0; r < 1000; ++r) noop<<<1, 32, 0, s0>>>();
    double tl = (now_us() - t) / 1000;
    cudaDeviceSynchronize();
    t = now_us();
    for (int r = 0; r < 1000; ++r) {
      noop<<<1, 32, 0, s0>>>();
      cudaStreamSynchronize(s0);
    }
    double ts = (now_us() - t) / 1000;
    cudaPointerAttributes pa;
    t = now_us();
    for (int r = 0; r < 1000; ++r) cudaPointerGetAttributes(&pa, hi + (r & 63) * 64);
    double tp = (now_us() - t) / 1000;
    cudaDeviceSynchronize();
    t = now_us();
    for (int r = 0; r < 1000; ++r) {
      cudaMemsetAsync(di, 0, 8, s0);
      noop<<<1, 32, 0, s0>>>();
      cudaMemcpyAsync(ho, di, 24, cudaMemcpyDeviceToHost, s0);
      cudaStreamSynchronize(s0);
    }
    double tc = (now_us() - t) / 1000;
    t = now_us();
    for (int r = 0; r < 1000; ++r) {
      noop<<<1, 32, 0, s0>>>();
      cudaStreamSynchronize(s0);
    }
    double tk = (now_us() - t) / 1000;
    printf("host per call: memcpyAsync %.2f us, launch %.2f us, launch+sync round trip %.2f us, "
           "cudaPointerGetAttributes %.2f us, memset+launch+memcpy+sync %.2f us, launch+sync %.2f us\n",
           tm, tl, ts, tp, tc, tk);
  }
  // step mimic: H2D actions, kernel, D2H results, sync — per step wall time
  {
    const int S = 300;
    auto wall = [&](auto&& body) {
      for (int w = 0; w < 10; ++w) body();
      double t = now_us();
      for (int r = 0; r < S; ++r) body();
      return (now_us() - t) / S;
    };
    double a = wall([&] {
      cudaMemcpyAsync(di, hi, h2d, cudaMemcpyHostToDevice, s0);
      noop<<<512, 64, 0, s0>>>();
      cudaMemcpyAsync(ho, dout, d2h, cudaMemcpyDeviceToHost, s0);
      cudaStreamSynchronize(s0);
    });
    double b = wall([&] {
      zc_write<<<592, 256, 0, s0>>>((float4*)di, (const float4*)hi, h2d / 16);
      zc_write<<<592, 256, 0, s0>>>((float4*)ho, (const float4*)dout, d2h / 16);
      cudaStreamSynchronize(s0);
    });
    printf("step mimic wall: copy-engine serial %.2f us, zero-copy %.2f us\n", a, b);
    for (int C : {2, 4, 8}) {
      double c = wall([&] {
        for (int k = 0; k < C; ++k) {
          cudaStream_t s = (k & 1) ? s1 : s0;
          cudaMemcpyAsync(di + k * h2d / C, hi + k * h2d / C, h2d / C, cudaMemcpyHostToDevice, s);
          noop<<<512 / C, 64, 0, s>>>();
          cudaMemcpyAsync(ho + k * d2h / C, dout + k * d2h / C, d2h / C, cudaMemcpyDeviceToHost, s);
        }
        cudaStreamSynchronize(s0);
        cudaStreamSynchronize(s1);
      });
      printf("step mimic wall: %d chunks on 2 streams %.2f us\n", C, c);
    }
  }
  return 0;
}
