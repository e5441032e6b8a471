// sm_rate.cu — microbenchmark of the span_attn_tc softmax step in isolation (one CTA per SM,
// 512 threads like the kernel): warps 4-7 / 8-11 run the single-pass 64-key softmax on TMEM
// sub-tiles of heads A / B; optionally warp 1 keeps the tensor core busy with the kernel's MMA
// period (S SS N=64 + PV TS N=128) on other TMEM columns. Reports cycles per 64-key sub-tile.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/sm_rate.cu -o tools/sm_rate
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>

#include "../paper_2511_02749_b200/csrc/kernels/sm100.cuh"

using namespace spq;

struct Sm {
  alignas(1024) uint8_t a[32768];
  alignas(1024) uint8_t b[32768];
  uint64_t bar;
  uint32_t tmem;
  int stop;
};

template <bool kPoly>
__device__ __forceinline__ float softmax_sub(uint32_t scol, float sl2, float thr, float& m, float& alpha) {
  uint32_t v[64];
  tmem_ld64(scol, v);
  tmem_wait_ld();
  float mx4[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) mx4[k] = fmaxf(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
#pragma unroll
  for (int i = 4; i < 32; ++i) mx4[i & 3] = fmax3(mx4[i & 3], __uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
  const float mx = fmax3(fmaxf(mx4[0], mx4[1]), mx4[2], mx4[3]) * sl2;
  const float m_new = fmaxf(m, mx);
  const bool resc = m_new > m + thr;
  const float m_use = resc ? m_new : m;
  alpha = resc ? ex2_approx(m - m_new) : 1.f;
  m = m_use;
  const float msub = (m_use == -INFINITY) ? 0.f : m_use;
  float sum8[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) sum8[i] = 0.f;
  uint32_t pk[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float x0 = fmaf(__uint_as_float(v[2 * i]), sl2, -msub);
    const float x1 = fmaf(__uint_as_float(v[2 * i + 1]), sl2, -msub);
    const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
    sum8[(2 * i) & 7] += p0;
    sum8[(2 * i + 1) & 7] += p1;
    pk[i] = pack_bf16x2(p0, p1);
  }
  tmem_st32(scol, pk);
  tmem_wait_st();
  return ((sum8[0] + sum8[1]) + (sum8[2] + sum8[3])) + ((sum8[4] + sum8[5]) + (sum8[6] + sum8[7]));
}

__global__ void __launch_bounds__(512, 1) rate(int mode, int iters, long long* out, float* sink) {
  extern __shared__ uint8_t raw[];
  Sm& s = *reinterpret_cast<Sm*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int t = threadIdx.x, warp = t / 32;
  for (int i = t; i < 32768 / 4; i += 512) {
    reinterpret_cast<uint32_t*>(s.a)[i] = 0x3c003c00u;
    reinterpret_cast<uint32_t*>(s.b)[i] = 0x3c003c00u;
  }
  if (t == 0) {
    mbar_init(&s.bar, 1);
    s.stop = 0;
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  if (warp == 2) tmem_alloc<512>(&s.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = s.tmem;
  long long t0 = clock64();
  if (mode >= 16 && warp >= 4 && warp < ((mode & 1) ? 12 : 8)) {
    // raw ex2 throughput: 16 independent chains per thread, 64 ex2 per iteration
    float r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = -0.001f * (t + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = -ex2_approx(r[i]);
    }
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) acc += r[i];
    sink[blockIdx.x * 512 + t] = acc;
    long long t1 = clock64();
    if ((t & 127) == 0) out[blockIdx.x * 4 + (warp < 8 ? 0 : 1)] = t1 - t0;
  }
  if (mode < 16 && warp >= 4 && warp < ((mode & 4) ? 8 : 12) && (mode & 1)) {
    const int x = warp < 8 ? 0 : 1;
    const uint32_t lane_base = static_cast<uint32_t>(((t & 127) / 32) * 32) << 16;
    float m = -INFINITY, l = 0.f;
    for (int it = 0; it < iters; ++it) {
      const uint32_t scol = tm + lane_base + 128 * x + 64 * (it & 1);
      float alpha;
      l = l * 1.0f + softmax_sub<false>(scol, 0.09f, 8.f, m, alpha);
    }
    sink[blockIdx.x * 512 + t] = l;
    long long t1 = clock64();
    if ((t & 127) == 0) out[blockIdx.x * 4 + x] = t1 - t0;
  }
  if (warp == 1 && (mode & 2) && elect_one()) {
    // MMA period on columns [256, 512): S_A, S_B into 256/320 (N=64), PV into 384 (N=128)
    constexpr uint32_t idS64 = idesc_bf16_f32(128, 64, false, false);
    constexpr uint32_t idO = idesc_bf16_f32(128, 128, false, true);
    for (int it = 0; it < iters; ++it) {
      for (int x = 0; x < 2; ++x)
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
          mma_ss(tm + 256 + 64 * x, desc_sw128(smem_u32(s.a) + off, 16, 1024),
                 desc_sw128(smem_u32(s.b) + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024), idS64, 1u);
        }
      for (int x = 0; x < 2; ++x)
        for (int kk = 0; kk < 4; ++kk)
          mma_ts(tm + 384, tm + 256 + kk * 8, desc_sw128(smem_u32(s.b) + kk * 2048, 8192, 1024), idO, 1u);
    }
    mma_commit(&s.bar);
    mbar_wait(&s.bar, 0);
    long long t1 = clock64();
    out[blockIdx.x * 4 + 2] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tm);
}

int main() {
  long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 4 * 8);
  cudaMalloc(&sink, 148 * 512 * 4);
  const int smem = sizeof(Sm) + 1024;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  for (int mode : {1, 2, 3, 5, 7, 16, 17}) {
    cudaMemset(d, 0, 148 * 4 * 8);
    rate<<<148, 512, smem>>>(mode, iters, d, sink);
    cudaDeviceSynchronize();
    long long h[148 * 4];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mode %d (%s): softmax A %.1f B %.1f cycles/sub-tile, MMA %.1f cycles/period\n", mode,
           mode == 1 ? "softmax only" : mode == 2 ? "MMA only" : mode == 3 ? "both" : mode == 5 ? "softmax A only" : mode == 7 ? "softmax A + MMA" : mode == 16 ? "ex2 x64, warps 4-7" : "ex2 x64, warps 4-11", h[0] / double(iters), h[1] / double(iters),
           h[2] / double(iters));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
