// tc2_probe.cu — bring-up probe for the CTA-pair (cta_group::2) primitives of the paired
// span-attention kernel, validated against a host reference on the B200:
//   A. S = Q K^T, M = 256 (Q rows 0-127 in CTA 0's smem, 128-255 in CTA 1's), N = 64 keys split
//      across the pair (CTA r holds keys [32r, 32r+32), K-major SWIZZLE_128B), K = 128: SS form,
//      issued by the leader CTA only; D rows 128r.. land in CTA r's TMEM
//   B. O = P V, M = 256 (P in each CTA's TMEM), N = 128 head-dim columns split across the pair (CTA r
//      holds V columns [64r, 64r+64) for all 64 keys, MN-major SWIZZLE_128B), K = 64 keys: TS form
//   Both CTAs' TMA loads complete_tx on the leader's mbarrier (.cta_group::2); commits multicast to
//   both CTAs' barriers; TMEM allocated with cta_group::2 by one warp of each CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tc2_probe.cu -o tools/tc2_probe
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2511_02749_b200/csrc/kernels/sm100.cuh"

using namespace spq;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = reinterpret_cast<EncodeFn>(fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, uint32_t bar_cluster, int32_t x,
                                                 int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

struct Smem {
  alignas(1024) uint8_t q[2][16384];  // this CTA's 128 Q rows, two 64-column chunks
  alignas(1024) uint8_t k[2][4096];   // this CTA's 32 keys, two 64-column chunks
  alignas(1024) uint8_t v[8192];      // all 64 keys, this CTA's 64 V columns
  uint64_t bar_tma, bar_mma;
  uint32_t tmem_base;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
          const __grid_constant__ CUtensorMap mv, const __nv_bfloat16* P, float* outS, float* outO) {
  extern __shared__ uint8_t raw[];
  Smem& s = *reinterpret_cast<Smem*>(raw);
  const int t = threadIdx.x, warp = t / 32;
  const uint32_t rank = cluster_rank();
  if (t == 0) {
    mbar_init(&s.bar_tma, 1);
    mbar_init(&s.bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  const uint32_t bar_leader = mapa_u32(smem_u32(&s.bar_tma), 0);
  if (t == 0) {
    if (rank == 0) mbar_arrive_expect_tx(&s.bar_tma, 2 * (32768 + 8192 + 8192));
    for (int c = 0; c < 2; ++c) {
      tma_load_2d_pair(s.q[c], &mq, bar_leader, c * 64, 128 * rank);
      tma_load_2d_pair(s.k[c], &mk, bar_leader, c * 64, 32 * rank);
    }
    tma_load_2d_pair(s.v, &mv, bar_leader, 64 * rank, 0);
  }
  // ---- A: S = Q K^T into cols [0, 64)
  if (rank == 0 && t == 0) {
    mbar_wait(&s.bar_tma, 0);
    tc_fence_after();
    const uint32_t id = idesc_bf16_f32(256, 64, false, false);
    for (int k = 0; k < 8; ++k) {
      const int c = k / 4, kk = k % 4;
      mma2_ss(tmem, desc_sw128(smem_u32(s.q[c] + kk * 32), 16, 1024), desc_sw128(smem_u32(s.k[c] + kk * 32), 16, 1024),
              id, k > 0);
    }
    commit2(&s.bar_mma);
  }
  mbar_wait(&s.bar_mma, 0);
  tc_fence_after();
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  const int row = 128 * rank + t;
  for (int c0 = 0; c0 < 64; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + lane_off + c0, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) outS[row * 64 + c0 + i] = __uint_as_float(r[i]);
  }
  // ---- B: P (this CTA's rows) -> TMEM cols [128, 160) packed bf16x2; O = P V into cols [256, 384)
  {
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) {
      const __nv_bfloat16 lo = P[row * 64 + 2 * i], hi = P[row * 64 + 2 * i + 1];
      r[i] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
    }
    tmem_st32(tmem + lane_off + 128, r);
    tmem_wait_st();
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (rank == 0 && t == 0) {
    const uint32_t id = idesc_bf16_f32(256, 128, false, true);
    for (int k = 0; k < 4; ++k)
      mma2_ts(tmem + 256, tmem + 128 + k * 8, desc_sw128(smem_u32(s.v + k * 2048), 8192, 1024), id, k > 0);
    commit2(&s.bar_mma);
  }
  mbar_wait(&s.bar_mma, 1);
  tc_fence_after();
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + lane_off + 256 + c0, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) outO[row * 128 + c0 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static float bf(const __nv_bfloat16& x) { return __bfloat162float(x); }

int main() {
  std::vector<__nv_bfloat16> hQ(256 * 128), hK(64 * 128), hV(64 * 128), hP(256 * 64);
  srand(1);
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
  for (auto& x : hQ) x = __float2bfloat16(rnd());
  for (auto& x : hK) x = __float2bfloat16(rnd());
  for (auto& x : hV) x = __float2bfloat16(rnd());
  for (auto& x : hP) x = __float2bfloat16(rnd());
  __nv_bfloat16 *dQ, *dK, *dV, *dP;
  float *oS, *oO;
  CK(cudaMalloc(&dQ, hQ.size() * 2));
  CK(cudaMalloc(&dK, hK.size() * 2));
  CK(cudaMalloc(&dV, hV.size() * 2));
  CK(cudaMalloc(&dP, hP.size() * 2));
  CK(cudaMalloc(&oS, 256 * 64 * 4));
  CK(cudaMalloc(&oO, 256 * 128 * 4));
  CK(cudaMemcpy(dQ, hQ.data(), hQ.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dK, hK.data(), hK.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dV, hV.data(), hV.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dP, hP.data(), hP.size() * 2, cudaMemcpyHostToDevice));
  CUtensorMap mq = make_map(dQ, 256, 128, 128), mk = make_map(dK, 64, 128, 32), mv = make_map(dV, 64, 128, 64);
  const int smem = sizeof(Smem);
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<<<2, 128, smem>>>(mq, mk, mv, dP, oS, oO);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> hS(256 * 64), hO(256 * 128);
  CK(cudaMemcpy(hS.data(), oS, hS.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hO.data(), oO, hO.size() * 4, cudaMemcpyDeviceToHost));
  double eS = 0, eO = 0;
  for (int m = 0; m < 256; ++m) {
    for (int j = 0; j < 64; ++j) {
      double acc = 0;
      for (int k = 0; k < 128; ++k) acc += (double)bf(hQ[m * 128 + k]) * bf(hK[j * 128 + k]);
      eS = fmax(eS, fabs(acc - hS[m * 64 + j]));
    }
    for (int j = 0; j < 128; ++j) {
      double acc = 0;
      for (int k = 0; k < 64; ++k) acc += (double)bf(hP[m * 64 + k]) * bf(hV[k * 128 + j]);
      eO = fmax(eO, fabs(acc - hO[m * 128 + j]));
    }
  }
  printf("A  SS M=256 N=64 (K split over the pair)  max_err %.3e %s\n", eS, eS < 1e-2 ? "PASS" : "FAIL");
  printf("B  TS M=256 N=128 (V split over the pair)  max_err %.3e %s\n", eO, eO < 1e-2 ? "PASS" : "FAIL");
  printf("S[0][0..2] %f %f %f  S[200][5] %f\n", hS[0], hS[1], hS[2], hS[200 * 64 + 5]);
  return 0;
}
