// mbar_lat.cu — cost of an mbarrier wait whose phase has ALREADY completed, per wait form:
// try_wait.parity with the suspend-time hint (the kernel's mbar_wait), try_wait without a hint,
// test_wait; one warp, 32 lanes waiting (like a softmax warp) and one lane (like an issuer).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/mbar_lat.cu -o tools/mbar_lat
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2511_02749_b200/csrc/kernels/sm100.cuh"

using namespace spq;

__global__ void lat(long long* out) {
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&bar);  // completes phase 0
  __syncthreads();
  constexpr int N = 64;
  for (int mode = 0; mode < 3; ++mode) {
    for (int lanes = 32; lanes >= 1; lanes -= 31) {
      if (threadIdx.x < lanes) {
        const long long t0 = clock64();
        for (int i = 0; i < N; ++i) {
          if (mode == 0)
            while (!mbar_try_wait_sleep(&bar, 0)) {
            }
          else if (mode == 1)
            while (!mbar_try_wait(&bar, 0)) {
            }
          else
            while (!mbar_test_wait(&bar, 0)) {
            }
        }
        const long long t1 = clock64();
        if (threadIdx.x == 0) out[mode * 2 + (lanes == 1)] = (t1 - t0) / N;
      }
      __syncwarp();
    }
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 6 * 8);
  lat<<<1, 32>>>(d);
  cudaDeviceSynchronize();
  long long h[6];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[3] = {"try_wait + suspend hint", "try_wait (no hint)", "test_wait"};
  for (int m = 0; m < 3; ++m)
    printf("%-26s completed phase: %lld cycles per wait (32 lanes), %lld (1 lane)\n", names[m], h[2 * m], h[2 * m + 1]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
