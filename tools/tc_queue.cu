// tc_queue.cu — does a tcgen05.mma issue block? One thread per CTA (one CTA per SM) issues 64
// SS MMAs (M=128, N=64, K=16: the S sub-tile form of span_attn_tc) back to back and records the
// SM clock after each; a flat slope then a step means the issue queue filled. Also: the same with
// a commit every 8 MMAs, and the completion time of the whole batch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tc_queue.cu -o tools/tc_queue
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2511_02749_b200/csrc/kernels/sm100.cuh"

using namespace spq;

struct Sm {
  alignas(1024) uint8_t a[32768];
  alignas(1024) uint8_t b[32768];
  uint64_t bar;
  uint32_t tmem;
};

__global__ void __launch_bounds__(128, 1) q(int mode, long long* out) {
  extern __shared__ uint8_t raw[];
  Sm& s = *reinterpret_cast<Sm*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int t = threadIdx.x, warp = t / 32;
  for (int i = t; i < 32768 / 4; i += 128) {
    reinterpret_cast<uint32_t*>(s.a)[i] = 0x3c003c00u;
    reinterpret_cast<uint32_t*>(s.b)[i] = 0x3c003c00u;
  }
  if (t == 0) {
    mbar_init(&s.bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&s.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = s.tmem;
  constexpr uint32_t idS = idesc_bf16_f32(128, 64, false, false);
  constexpr int N = 64;
  if (t == 32) {
    long long ts[N + 1];
    const uint64_t ad0 = desc_sw128(smem_u32(s.a), 16, 1024), bd0 = desc_sw128(smem_u32(s.b), 16, 1024);
    const long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int kk = i & 7;
      mma_ss(tm + 64 * ((i >> 3) & 3), desc_add(ad0, (kk / 4) * 16384 + (kk % 4) * 32),
             desc_add(bd0, (kk / 4) * 8192 + (kk % 4) * 32), idS, kk > 0 ? 1u : 0u);
      if (mode == 1 && kk == 7) mma_commit(&s.bar);
      ts[i] = clock64();
    }
    mma_commit(&s.bar);
    mbar_wait(&s.bar, mode == 1 ? 0 : 0);
    if (mode == 1) {  // 8 earlier commits + 1: 9 phases; wait for the last (parity of phase 8)
      while (!mbar_try_wait(&s.bar, 0)) {
      }
    }
    ts[N] = clock64();
    if (blockIdx.x == 0)
      for (int i = 0; i <= N; ++i) out[i] = ts[i] - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

int main() {
  long long* d;
  cudaMalloc(&d, 65 * 8);
  const int smem = sizeof(Sm) + 1024;
  cudaFuncSetAttribute(q, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      q<<<148, 128, smem>>>(mode, d);
      cudaDeviceSynchronize();
    }
    long long h[65];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mode %d (%s): issue clock after MMA i:", mode, mode ? "commit every 8" : "no commits");
    for (int i = 0; i < 64; ++i) printf(" %lld", h[i]);
    printf("\n  all complete: %lld cycles (64 x N=64 SS: ideal ~%d at 32 cycles each)\n", h[64], 64 * 32);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
