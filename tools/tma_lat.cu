// tma_lat.cu — TMA load latency / throughput probe for the span-attention K/V ring (profiling aid).
// One CTA per SM; warp 0 lane 0 streams 16 KB sub-tiles (two {64 col, 64 row} bf16 boxes,
// SWIZZLE_128B — the K/V pool layout) into an R-slot ring, warp 1 lane 0 consumes each after a
// fixed "compute" delay and frees the slot. Reports issue->landed latency and cycles per sub-tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_lat tools/tma_lat.cu
//   tools/tma_lat <slots> <delay cycles> <region MB> [extra streaming TMA KB per sub-tile]
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(par)
        : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(su32(bar)), "r"(x), "r"(y)
      : "memory");
}

constexpr int kMaxSlots = 8;
constexpr int kN = 512;  // sub-tiles per CTA

__global__ void __launch_bounds__(64, 1) lat_kernel(const __grid_constant__ CUtensorMap m, int slots, int delay,
                                                    int rows_region, int extra_boxes, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[kMaxSlots], empty[kMaxSlots], xbar;
  __shared__ long long t_issue[kN];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kMaxSlots; ++i) {
      bar_init(&full[i], 1);
      bar_init(&empty[i], 1);
    }
    bar_init(&xbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint8_t* ring = smem;
  uint8_t* xbuf = smem + kMaxSlots * 16384;  // extra traffic target (Q-like loads)
  uint32_t seed = 12345u + blockIdx.x * 7919u;
  if (warp == 0 && lane == 0) {
    uint32_t xph = 0;
    for (int n = 0; n < kN; ++n) {
      const int s = n % slots;
      bar_wait(&empty[s], ((n / slots) & 1) ^ 1);
      seed = seed * 1664525u + 1013904223u;
      const int row = static_cast<int>((seed >> 8) % static_cast<uint32_t>(rows_region / 64)) * 64;
      long long t;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
      t_issue[n] = t;
      bar_expect(&full[s], 16384);
      tma2d(ring + s * 16384, &m, &full[s], 0, row);
      tma2d(ring + s * 16384 + 8192, &m, &full[s], 64, row);
      if (extra_boxes > 0 && (n % 2) == 0) {  // interleaved streaming loads (8 KB boxes), waited at once
        bar_expect(&xbar, extra_boxes * 8192 * 2);
        for (int e = 0; e < 2 * extra_boxes; ++e) {
          seed = seed * 1664525u + 1013904223u;
          const int r2 = static_cast<int>((seed >> 8) % static_cast<uint32_t>(rows_region / 64)) * 64;
          tma2d(xbuf + (e % 4) * 8192, &m, &xbar, (e & 1) * 64, r2);
        }
        bar_wait(&xbar, xph);
        xph ^= 1;
      }
    }
  } else if (warp == 1 && lane == 0) {
    long long lat_sum = 0, t0 = 0, t1 = 0;
    std::int64_t lats[64];
    int nl = 0;
    for (int n = 0; n < kN; ++n) {
      const int s = n % slots;
      bar_wait(&full[s], (n / slots) & 1);
      long long t;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
      if (n == 16) t0 = t;
      t1 = t;
      if (n >= 16) lat_sum += t - t_issue[n];
      if (n >= 16 && nl < 64) lats[nl++] = t - t_issue[n];
      long long ts = t;
      while (t - ts < delay) asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
      bar_arrive(&empty[s]);
    }
    out[blockIdx.x * 2] = lat_sum / (kN - 16);
    out[blockIdx.x * 2 + 1] = (t1 - t0) / (kN - 17);
  }
}

int main(int argc, char** argv) {
  const int slots = argc > 1 ? atoi(argv[1]) : 3;
  const int delay = argc > 2 ? atoi(argv[2]) : 0;
  const int region_mb = argc > 3 ? atoi(argv[3]) : 32;
  const int extra = argc > 4 ? atoi(argv[4]) : 0;
  const size_t bytes = static_cast<size_t>(512) << 20;
  void* buf = nullptr;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  const int total_rows = static_cast<int>(bytes / 256);
  const int rows_region = std::min<long long>(total_rows, static_cast<long long>(region_mb) << 20 >> 8);
  CUtensorMap m{};
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(total_rows)}, strides[1] = {256};
  cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
  reinterpret_cast<Fn>(fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* out;
  cudaMalloc(&out, sms * 2 * sizeof(long long));
  const int smem = kMaxSlots * 16384 + 4 * 8192;
  cudaFuncSetAttribute(lat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) lat_kernel<<<sms, 64, smem>>>(m, slots, delay, rows_region, extra, out);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(sms * 2);
  cudaMemcpy(h.data(), out, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
  std::vector<long long> lat, per;
  for (int i = 0; i < sms; ++i) {
    lat.push_back(h[2 * i]);
    per.push_back(h[2 * i + 1]);
  }
  std::sort(lat.begin(), lat.end());
  std::sort(per.begin(), per.end());
  const double gbs = 16384.0 * sms / (per[sms / 2] / 1.9e9) / 1e9;
  printf("%s slots %d delay %d region %d MB extra %d: latency med %lld p90 %lld cyc | cycles/subtile med %lld (%.0f GB/s chip @1.9GHz)\n",
         e == cudaSuccess ? "ok" : cudaGetErrorString(e), slots, delay, region_mb, extra, lat[sms / 2], lat[sms * 9 / 10],
         per[sms / 2], gbs);
  return 0;
}
