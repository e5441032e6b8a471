// tc_rate.cu — microbenchmark of the tcgen05 forms used by span_attn_tc (one CTA per SM):
//   SS  : D[128x128] += A[smem,K-major] B[smem,K-major]^T      (S = Q K^T), K=16 per instr
//   TS  : D[128x128] += A[tmem] B[smem,MN-major]              (O += P V)
//   and the round trip commit -> mbarrier -> other warp arrive -> issuing thread wakes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tc_rate.cu -o tools/tc_rate
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2511_02749_b200/csrc/kernels/sm100.cuh"

using namespace spq;

struct Sm {
  alignas(1024) uint8_t a[32768];
  alignas(1024) uint8_t b[32768];
  uint64_t bar, bar2;
  uint32_t tmem;
};

__global__ void __launch_bounds__(128, 1) rate(int mode, int iters, long long* out) {
  extern __shared__ uint8_t raw[];
  Sm& s = *reinterpret_cast<Sm*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int t = threadIdx.x, warp = t / 32;
  for (int i = t; i < 32768 / 4; i += 128) {
    reinterpret_cast<uint32_t*>(s.a)[i] = 0x3c003c00u;
    reinterpret_cast<uint32_t*>(s.b)[i] = 0x3c003c00u;
  }
  if (t == 0) {
    mbar_init(&s.bar, 1);
    mbar_init(&s.bar2, 32);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&s.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = s.tmem;
  constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false);
  constexpr uint32_t idO = idesc_bf16_f32(128, 128, false, true);
  long long t0 = clock64();
  if (mode >= 4) {
    // one span_attn period: S_A, S_B (M128 N64 K128 SS: 8 instr each), PV_A, PV_B (M128 N128 K64 TS)
    constexpr uint32_t idS64 = idesc_bf16_f32(128, 64, false, false);
    if (t == 0) {
      for (int it = 0; it < iters; ++it) {
        for (int x = 0; x < 2; ++x)
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
            if (mode == 4 || mode == 5)
              mma_ss(tm + 64 * x, desc_sw128(smem_u32(s.a) + off, 16, 1024),
                     desc_sw128(smem_u32(s.b) + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024), idS64, 1u);
          }
        for (int x = 0; x < 2; ++x)
          for (int kk = 0; kk < 4; ++kk)
            if (mode == 4 || mode == 6)
              mma_ts(tm + 256 + 128 * x, tm + 128 + kk * 8, desc_sw128(smem_u32(s.b) + kk * 2048, 8192, 1024), idO, 1u);
      }
      mma_commit(&s.bar);
      mbar_wait(&s.bar, 0);
    }
  } else if (mode < 3) {
    if (t == 0) {
      for (int it = 0; it < iters; ++it) {
        for (int kk = 0; kk < 8; ++kk) {
          if (mode == 0 || mode == 2) {
            const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
            mma_ss(tm + 0, desc_sw128(smem_u32(s.a) + off, 16, 1024), desc_sw128(smem_u32(s.b) + off, 16, 1024), idS,
                   1u);
          }
          if (mode == 1 || mode == 2) {
            mma_ts(tm + 256, tm + 128 + kk * 8, desc_sw128(smem_u32(s.b) + kk * 2048, 16384, 1024), idO, 1u);
          }
        }
      }
      mma_commit(&s.bar);
      mbar_wait(&s.bar, 0);
    }
  } else {
    // mode 3: ping-pong latency: thread 0 commits (empty), warp 1 waits and arrives, thread 0 waits
    for (int it = 0; it < iters; ++it) {
      if (t == 0) {
        mma_ss(tm + 0, desc_sw128(smem_u32(s.a), 16, 1024), desc_sw128(smem_u32(s.b), 16, 1024), idS, 1u);
        mma_commit(&s.bar);
        mbar_wait(&s.bar2, it & 1);
      } else if (warp == 1) {
        mbar_wait(&s.bar, it & 1);
        mbar_arrive(&s.bar2);
      }
    }
  }
  long long t1 = clock64();
  if (t == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = sizeof(Sm) + 1024;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"SS S=QK^T (8 x 128x128x16)", "TS O+=PV (8 x 128x128x16, B MN-major)", "SS+TS interleaved",
                         "commit->wait->arrive->wait round trip", "period: 2x(8 SS N64) + 2x(4 TS N128)",
                         "period SS part only (16 SS N64)", "period TS part only (8 TS N128)"};
  for (int mode = 0; mode < 7; ++mode) {
    const int iters = mode == 3 ? 1000 : 2000;
    for (int grid : {1, 148}) {
      rate<<<grid, 128, smem>>>(mode, iters, d);
      cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      const double per = mx / iters;
      if (mode >= 4) {
        const double flops = (mode == 4 ? 2.0 : 1.0) * 16 * 2.0 * 128 * 64 * 16 * (mode == 6 ? 1 : 1);
        printf("%-40s grid %3d: %8.1f cycles per period, %6.0f flop/cycle/SM (%.0f%% of 8192)\n", names[mode], grid, per,
               flops / per, 100.0 * flops / per / 8192);
      } else if (mode < 3) {
        const double flops = (mode == 2 ? 2 : 1) * 8.0 * 2 * 128 * 128 * 16;
        printf("%-40s grid %3d: %8.1f cycles per 8-MMA group, %6.0f flop/cycle/SM (%.0f%% of 8192)\n", names[mode], grid,
               per, flops / per, 100.0 * flops / per / 8192);
      } else {
        printf("%-40s grid %3d: %8.1f cycles per round trip\n", names[mode], grid, per);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
