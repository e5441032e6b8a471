// combine.cu — K4: merge split-KV partial attention results.
//
//   lse = log Σ_s exp(lse_s),   O = Σ_s exp(lse_s - lse) · O_s
// over the splits s of one (row, head), in a fixed order (deterministic, no atomics). Partials
// hold normalized O_s (fp32) and natural-log lse_s (-inf when the split saw no visible key).
// One warp per (row, head); each lane owns d/32 consecutive columns (float2 loads).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "launch.h"

namespace spq {
namespace {

__device__ __forceinline__ void store2(__nv_bfloat16* p, float a, float b) {
  *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
}
__device__ __forceinline__ void store2(float* p, float a, float b) {
  *reinterpret_cast<float2*>(p) = make_float2(a, b);
}

template <int D, typename TO>
__global__ void __launch_bounds__(256) combine_kernel(const CombineDesc* __restrict__ desc,
                                                      const float* __restrict__ opart,
                                                      const float* __restrict__ lsepart,
                                                      TO* __restrict__ o,
                                                      float* __restrict__ lse, int hq, int rpp) {
  constexpr int E = D / 32;  // columns per lane
  // launched as a programmatic dependent of the join it merges (when nothing sits between them):
  // the partials are read only once that grid has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const CombineDesc cd = desc[blockIdx.x];
  if (static_cast<int>(blockIdx.y) >= cd.n_heads) return;
  const int h = cd.head0 + blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // grid.z splits the rows of a tile into groups of blockDim/32 rows: one warp per row. A partial
  // slot holds rpp rows per head (kTileRows for joins, 1 for decode)
  for (int r = blockIdx.z * (blockDim.x / 32) + warp; r < cd.n_rows; r += gridDim.z * (blockDim.x / 32)) {
    const int64_t pstride = static_cast<int64_t>(cd.n_heads) * rpp;  // next split, same (head, row)
    const int64_t base = (static_cast<int64_t>(cd.part_base) * cd.n_heads + blockIdx.y) * rpp + r;
    const int64_t base2 = (static_cast<int64_t>(cd.part_base2) * cd.n_heads + blockIdx.y) * rpp + r;
    const int n_all = cd.n_split + cd.n_split2;
    float m = -INFINITY;
    float acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = 0.f;
    float tot = 0.f;
    // up to 8 splits with every load issued before the arithmetic (latency-bound otherwise)
    constexpr int kU = 8;
    for (int s0 = 0; s0 < n_all; s0 += kU) {
      float ls[kU];
      float2 ov[kU][E / 2];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int si = s0 + u;
        const bool ok = si < n_all;
        const int64_t pidx = si < cd.n_split ? base + si * pstride : base2 + (si - cd.n_split) * pstride;
        ls[u] = ok ? lsepart[pidx] : -INFINITY;
#pragma unroll
        for (int e = 0; e < E; e += 2)
          ov[u][e / 2] = ok ? *reinterpret_cast<const float2*>(opart + pidx * D + lane * E + e) : make_float2(0.f, 0.f);
      }
      float mb = m;
#pragma unroll
      for (int u = 0; u < kU; ++u) mb = fmaxf(mb, ls[u]);
      // rescale what was accumulated under the previous max (only when n_split > 8)
      const float c = (m == -INFINITY) ? 0.f : __expf(m - mb);
      tot *= c;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] *= c;
      m = mb;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const float w = (ls[u] == -INFINITY) ? 0.f : __expf(ls[u] - m);
        tot += w;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
          acc[e] = fmaf(w, ov[u][e / 2].x, acc[e]);
          acc[e + 1] = fmaf(w, ov[u][e / 2].y, acc[e + 1]);
        }
      }
    }
    const float inv = 1.f / tot;
    const int64_t row = cd.row0 + r;
    TO* dst = o + (row * hq + h) * D + lane * E;
#pragma unroll
    for (int e = 0; e < E; e += 2) store2(dst + e, acc[e] * inv, acc[e + 1] * inv);
    if (lse != nullptr && lane == 0) lse[row * hq + h] = m + logf(tot);
  }
}

}  // namespace

template <int D, typename TO>
void launch_dt(const CombineArgs& a, cudaStream_t st) {
  const int rpp = a.rows_per_part > 0 ? a.rows_per_part : kTileRows;
  dim3 grid(a.n_desc, a.heads_per_desc, (rpp + 7) / 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, combine_kernel<D, TO>, a.desc, a.opart, a.lsepart, static_cast<TO*>(a.o), a.lse, a.hq, rpp);
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t st) {
  if (a.n_desc == 0) return cudaSuccess;
  if (a.d == 64)
    a.out_fp32 ? launch_dt<64, float>(a, st) : launch_dt<64, __nv_bfloat16>(a, st);
  else if (a.d == 128)
    a.out_fp32 ? launch_dt<128, float>(a, st) : launch_dt<128, __nv_bfloat16>(a, st);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace spq
