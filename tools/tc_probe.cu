// tc_probe.cu — bring-up probe for the sm_100a primitives used by the span-attention kernel.
// Validates on the GPU, against a host fp32 reference:
//   1. TMA SWIZZLE_128B loads + K-major SS tcgen05.mma (S = Q K^T, M=N=K=128)
//   2. thread-written manual SWIZZLE_128B Q tile (the Q-prep layout) gives the same S
//   3. P staged in TMEM via tcgen05.st + TS tcgen05.mma with MN-major V (O = P V)
//   4. same as 3 at N = 64 (head_dim 64)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/tc_probe.cu -o /tmp/tc_probe
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
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return reinterpret_cast<EncodeFn>(fn);
}

static CUtensorMap make_map(void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

struct Smem {
  alignas(1024) uint8_t a[32768];
  alignas(1024) uint8_t a2[32768];
  alignas(1024) uint8_t b[32768];
  alignas(1024) uint8_t v[32768];
  uint64_t bar_tma;
  uint64_t bar_mma;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(128, 1)
    probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
          const __grid_constant__ CUtensorMap mv, const __nv_bfloat16* A, const __nv_bfloat16* P,
          float* out1, float* out2, float* out3, float* out4) {
  extern __shared__ uint8_t raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int t = threadIdx.x;
  const int warp = t / 32;
  if (t == 0) {
    mbar_init(&s.bar_tma, 1);
    mbar_init(&s.bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&s.tmem_base);
  // thread-written manual swizzle of A into a2 (row t)
  for (int c = 0; c < 2; ++c)
    for (int u = 0; u < 8; ++u) {
      const uint4 val = *reinterpret_cast<const uint4*>(A + t * 128 + c * 64 + u * 8);
      *reinterpret_cast<uint4*>(s.a2 + c * 16384 + t * 128 + ((u ^ (t & 7)) * 16)) = val;
    }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  if (t == 0) {
    mbar_arrive_expect_tx(&s.bar_tma, 3 * 32768);
    for (int c = 0; c < 2; ++c) {
      tma_load_2d(s.a + c * 16384, &ma, &s.bar_tma, c * 64, 0);
      tma_load_2d(s.b + c * 16384, &mb, &s.bar_tma, c * 64, 0);
      tma_load_2d(s.v + c * 16384, &mv, &s.bar_tma, c * 64, 0);
    }
  }
  mbar_wait(&s.bar_tma, 0);
  // ---- test 1 & 2: S = A B^T into cols [0,128) and A2 B^T into [128,256)
  if (t == 0) {
    tc_fence_after();
    const uint32_t id = idesc_bf16_f32(128, 128, false, false);
    for (int k = 0; k < 8; ++k) {
      const int c = k / 4, kk = k % 4;
      uint64_t ad = desc_sw128(smem_u32(s.a + c * 16384 + kk * 32), 16, 1024);
      uint64_t a2 = desc_sw128(smem_u32(s.a2 + c * 16384 + kk * 32), 16, 1024);
      uint64_t bd = desc_sw128(smem_u32(s.b + c * 16384 + kk * 32), 16, 1024);
      mma_ss(tmem + 0, ad, bd, id, k > 0);
      mma_ss(tmem + 128, a2, bd, id, k > 0);
    }
    mma_commit(&s.bar_mma);
  }
  mbar_wait(&s.bar_mma, 0);
  tc_fence_after();
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + lane_off + c0, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) out1[t * 128 + c0 + i] = __uint_as_float(r[i]);
    tmem_ld32(tmem + lane_off + 128 + c0, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) out2[t * 128 + c0 + i] = __uint_as_float(r[i]);
  }
  // ---- test 3: P (row t) -> TMEM cols [256, 320) packed bf16x2; O = P V into cols [320, 448)
  {
    uint32_t r[32];
    for (int h = 0; h < 2; ++h) {
      for (int i = 0; i < 32; ++i) {
        const __nv_bfloat16 lo = P[t * 128 + h * 64 + 2 * i];
        const __nv_bfloat16 hi = P[t * 128 + h * 64 + 2 * i + 1];
        r[i] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
      }
      tmem_st32(tmem + lane_off + 256 + h * 32, r);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  if (t == 0) {
    tc_fence_after();
    const uint32_t id = idesc_bf16_f32(128, 128, false, true);
    const uint32_t id64 = idesc_bf16_f32(128, 64, false, true);
    for (int k = 0; k < 8; ++k) {
      uint64_t vd = desc_sw128(smem_u32(s.v + k * 2048), 16384, 1024);
      mma_ts(tmem + 320, tmem + 256 + k * 8, vd, id, k > 0);
    }
    mma_commit(&s.bar_mma);
    // test 4: N = 64 (only first d-chunk) into cols [448, 512)
    for (int k = 0; k < 8; ++k) {
      uint64_t vd = desc_sw128(smem_u32(s.v + k * 2048), 16384, 1024);
      mma_ts(tmem + 448, tmem + 256 + k * 8, vd, id64, k > 0);
    }
    mma_commit(&s.bar_mma);
  }
  mbar_wait(&s.bar_mma, 1);
  mbar_wait(&s.bar_mma, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + lane_off + 320 + c0, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) out3[t * 128 + c0 + i] = __uint_as_float(r[i]);
  }
  for (int c0 = 0; c0 < 64; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + lane_off + 448 + c0, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) out4[t * 64 + c0 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

static float bf(const __nv_bfloat16& x) { return __bfloat162float(x); }

int main() {
  const int n = 128 * 128;
  std::vector<__nv_bfloat16> hA(n), hB(n), hV(n), hP(n);
  srand(1);
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
  for (int i = 0; i < n; ++i) {
    hA[i] = __float2bfloat16(rnd());
    hB[i] = __float2bfloat16(rnd());
    hV[i] = __float2bfloat16(rnd());
    hP[i] = __float2bfloat16(rnd());
  }
  __nv_bfloat16 *dA, *dB, *dV, *dP;
  float *o1, *o2, *o3, *o4;
  CK(cudaMalloc(&dA, n * 2));
  CK(cudaMalloc(&dB, n * 2));
  CK(cudaMalloc(&dV, n * 2));
  CK(cudaMalloc(&dP, n * 2));
  CK(cudaMalloc(&o1, n * 4));
  CK(cudaMalloc(&o2, n * 4));
  CK(cudaMalloc(&o3, n * 4));
  CK(cudaMalloc(&o4, n * 4));
  CK(cudaMemcpy(dA, hA.data(), n * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), n * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dV, hV.data(), n * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dP, hP.data(), n * 2, cudaMemcpyHostToDevice));
  CUtensorMap ma = make_map(dA, 128, 128, 128), mb = make_map(dB, 128, 128, 128),
              mv = make_map(dV, 128, 128, 128);
  const int smem = sizeof(Smem) + 1024;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<<<1, 128, smem>>>(ma, mb, mv, dA, dP, o1, o2, o3, o4);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> h1(n), h2(n), h3(n), h4(128 * 64);
  CK(cudaMemcpy(h1.data(), o1, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2.data(), o2, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h3.data(), o3, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h4.data(), o4, 128 * 64 * 4, cudaMemcpyDeviceToHost));
  double e1 = 0, e2 = 0, e3 = 0, e4 = 0;
  for (int m = 0; m < 128; ++m)
    for (int j = 0; j < 128; ++j) {
      double s = 0, o = 0;
      for (int k = 0; k < 128; ++k) {
        s += (double)bf(hA[m * 128 + k]) * bf(hB[j * 128 + k]);
        o += (double)bf(hP[m * 128 + k]) * bf(hV[k * 128 + j]);
      }
      e1 = fmax(e1, fabs(s - h1[m * 128 + j]));
      e2 = fmax(e2, fabs(s - h2[m * 128 + j]));
      e3 = fmax(e3, fabs(o - h3[m * 128 + j]));
      if (j < 64) e4 = fmax(e4, fabs(o - h4[m * 64 + j]));
    }
  printf("test1 SS TMA K-major      max_err %.3e %s\n", e1, e1 < 1e-2 ? "PASS" : "FAIL");
  printf("test2 SS manual swizzle   max_err %.3e %s\n", e2, e2 < 1e-2 ? "PASS" : "FAIL");
  printf("test3 TS P(tmem) V MN-maj max_err %.3e %s\n", e3, e3 < 1e-2 ? "PASS" : "FAIL");
  printf("test4 TS N=64             max_err %.3e %s\n", e4, e4 < 1e-2 ? "PASS" : "FAIL");
  printf("sample S[0][0..3] gpu %f %f %f %f\n", h1[0], h1[1], h1[2], h1[3]);
  return 0;
}
