// split_join.cu — the HBM-side kernels of the owner-side split join (§4.3
// the sub-trees of a span query are independent and run in parallel, map-reduce style).
//
// With W ranks the fragments of a home query q live on their owner ranks. Instead of moving their
// KV to q's home (K6, 2·Hkv·d·elt bytes per key), the home sends q's cross Q rows to each owner
// (Hq·d·elt bytes per row), the owner attends them over its fragments (the join kernel, Q
// counter-rotated by Δ_f) and returns one partial (O normalized fp32, LSE) per (row, head); the home
// merges its local part with the owners' partials:
//   lse = log(exp(lse_local) + Σ_w exp(lse_w)),  O = exp(lse_local - lse)·O_local + Σ_w exp(lse_w - lse)·O_w
// in a fixed order (local, then owners by rank) — the same LSE merge as K4 (combine.cu).
//
//   K10 gather_rows:   packed q rows (join row space) -> the Q send buffer, owner-major
//   K11 merge_split:   local fp32 (O, LSE) + received partials -> o (out dtype), lse
// Both are HBM-bound: 16-byte vectors (gather) / one warp per (row, head) with d/32 columns per
// lane (merge), grids a multiple of the SM count.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "launch.h"

namespace spq {
namespace {

__global__ void __launch_bounds__(256) gather_rows_kernel(const int32_t* __restrict__ rows, int64_t n,
                                                          const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                          int64_t words_per_row) {
  const int64_t total = n * words_per_row;
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < total;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = w / words_per_row, off = w - i * words_per_row;
    dst[w] = __ldg(src + static_cast<int64_t>(__ldg(rows + i)) * words_per_row + off);
  }
}

__device__ __forceinline__ void store2(__nv_bfloat16* p, float a, float b) {
  *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
}
__device__ __forceinline__ void store2(float* p, float a, float b) { *reinterpret_cast<float2*>(p) = make_float2(a, b); }

// one warp per (join row r, head h); the row's sources: merge_src[merge_off[q] ..) + (r - row0(q))
template <int D, typename TO>
__global__ void __launch_bounds__(256) merge_split_kernel(const SplitMergeDesc* __restrict__ desc, int32_t n_desc,
                                                          const int64_t* __restrict__ src, const float* __restrict__ o_loc,
                                                          const float* __restrict__ lse_loc,
                                                          const float* __restrict__ o_rem,
                                                          const float* __restrict__ lse_rem, TO* __restrict__ o,
                                                          float* __restrict__ lse, int hq, int64_t total_rows) {
  constexpr int E = D / 32;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * blockDim.x / 32;
  for (int64_t item = gw; item < total_rows * hq; item += nw) {
    const int64_t r = item / hq;
    const int h = static_cast<int>(item % hq);
    // the query of row r (descs are in row order: binary search)
    int lo = 0, hi = n_desc - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (desc[mid].row0 <= r) lo = mid; else hi = mid - 1;
    }
    const SplitMergeDesc d = desc[lo];
    const int64_t i = r - d.row0;
    float m = lse_loc[r * hq + h];
    float acc[E];
    const float* ol = o_loc + (r * hq + h) * D + lane * E;
#pragma unroll
    for (int e = 0; e < E; e += 2) {
      const float2 v = *reinterpret_cast<const float2*>(ol + e);
      acc[e] = v.x;
      acc[e + 1] = v.y;
    }
    // running (m, tot): the local part has weight 1 at m = lse_local
    float tot = m == -INFINITY ? 0.f : 1.f;
    if (m == -INFINITY) {
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = 0.f;
    }
    for (int s = d.src_begin; s < d.src_end; ++s) {
      const int64_t rr = src[s] + i;  // row of the received partial buffer
      const float ls = lse_rem[rr * hq + h];
      if (ls == -INFINITY) continue;
      const float mn = fmaxf(m, ls);
      const float c_old = m == -INFINITY ? 0.f : __expf(m - mn), c_new = __expf(ls - mn);
      const float* orr = o_rem + (rr * hq + h) * D + lane * E;
      tot = tot * c_old + c_new;
#pragma unroll
      for (int e = 0; e < E; e += 2) {
        const float2 v = *reinterpret_cast<const float2*>(orr + e);
        acc[e] = acc[e] * c_old + c_new * v.x;
        acc[e + 1] = acc[e + 1] * c_old + c_new * v.y;
      }
      m = mn;
    }
    const float inv = tot > 0.f ? 1.f / tot : 0.f;
    TO* dst = o + (r * hq + h) * D + lane * E;
#pragma unroll
    for (int e = 0; e < E; e += 2) store2(dst + e, acc[e] * inv, acc[e + 1] * inv);
    if (lse != nullptr && lane == 0) lse[r * hq + h] = tot > 0.f ? m + logf(tot) : -INFINITY;
  }
}

template <int D, typename TO>
cudaError_t launch_merge_t(const SplitMergeArgs& a, cudaStream_t st) {
  const int64_t warps = a.total_rows * a.hq;
  const int grid = static_cast<int>(std::min<int64_t>((warps * 32 + 255) / 256, static_cast<int64_t>(a.num_sms) * 8));
  merge_split_kernel<D, TO><<<std::max(grid, 1), 256, 0, st>>>(a.desc, a.n_desc, a.src, a.o_loc, a.lse_loc, a.o_rem,
                                                              a.lse_rem, static_cast<TO*>(a.o), a.lse, a.hq, a.total_rows);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gather_rows(const int32_t* rows, int64_t n, const void* src, void* dst, int64_t row_bytes,
                               int num_sms, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (row_bytes % 16 != 0) return cudaErrorInvalidValue;
  const int64_t wpr = row_bytes / 16, total = n * wpr;
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, static_cast<int64_t>(num_sms) * 8));
  gather_rows_kernel<<<grid, 256, 0, st>>>(rows, n, static_cast<const uint4*>(src), static_cast<uint4*>(dst), wpr);
  return cudaGetLastError();
}

cudaError_t launch_merge_split(const SplitMergeArgs& a, cudaStream_t st) {
  if (a.total_rows <= 0) return cudaSuccess;
  if (a.d == 64) return a.out_fp32 ? launch_merge_t<64, float>(a, st) : launch_merge_t<64, __nv_bfloat16>(a, st);
  if (a.d == 128) return a.out_fp32 ? launch_merge_t<128, float>(a, st) : launch_merge_t<128, __nv_bfloat16>(a, st);
  return cudaErrorInvalidValue;
}

}  // namespace spq
