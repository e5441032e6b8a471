// span_attn_f32.cu — K5: the fp32 span-attention path (SURVEY §8(a) a6/a7, fp32 tolerance 1e-5).
//
// Same semantics as the tcgen05 kernel (work.h): per (work item, q head), each query row r
// streams the item's KV tiles; for every tile it uses q rotated to pos[r] - rot_delta (so cached
// fragment KV at span-local positions is attended at its new position without being touched,
// P:610), masks t >= n_valid and, in causal tiles, key_pos0 + t > pos[r], and keeps an online
// softmax in fp32. tcgen05 has no true-fp32 MMA kind (tf32 would miss 1e-5), so this path is
// SIMT: one warp per query row, lane l owns elements l + 32k (k < d/32) so both halves of a
// rotate-half pair (e, e + d/2) are in the same lane; dot products reduce with warp shuffles.
#include <cuda_runtime.h>

#include <cmath>

#include "launch.h"

namespace spq {
namespace {

template <int D>
__global__ void __launch_bounds__(128) span_attn_f32_kernel(AttnArgs a) {
  constexpr int NE = D / 32;
  const WorkItem it = a.items[blockIdx.x];
  const int h = blockIdx.y;
  const int kvh = h / (a.hq / a.hkv);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const float* q = static_cast<const float*>(a.q);
  const float* kp = static_cast<const float*>(a.k_pool);
  const float* vp = static_cast<const float*>(a.v_pool);
  const float scale = rsqrtf(static_cast<float>(D));
  const int bpt = kTileKeys / a.bs;
  const int64_t layer_rows = static_cast<int64_t>(a.layer) * a.nblk * a.hkv * a.bs;
  for (int r = warp; r < it.n_rows; r += blockDim.x / 32) {
    const int64_t row = it.row0 + r;
    const int p = a.pos[row];
    float qraw[NE], qr[NE], acc[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
      qraw[k] = q[(row * a.hq + h) * D + lane + 32 * k];
      acc[k] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    int cur_rot = INT_MIN;
    for (int t = it.tile_begin; t < it.tile_end; ++t) {
      const KvTile tl = a.tiles[t];
      if (tl.rot_delta != cur_rot) {
        cur_rot = tl.rot_delta;
        const float2* cs = a.rope + static_cast<int64_t>(p - cur_rot) * (D / 2);
#pragma unroll
        for (int k = 0; k < NE / 2; ++k) {
          const float2 c = cs[lane + 32 * k];
          const float x1 = qraw[k], x2 = qraw[k + NE / 2];
          qr[k] = x1 * c.x - x2 * c.y;
          qr[k + NE / 2] = x2 * c.x + x1 * c.y;
        }
      }
      for (int i = 0; i < tl.n_valid; ++i) {
        if (tl.causal && tl.key_pos0 + i > p) break;
        const int blk = a.tile_blocks[tl.blk_off + i / a.bs];
        const int64_t krow = layer_rows + (static_cast<int64_t>(blk) * a.hkv + kvh) * a.bs + i % a.bs;
        const float* kr = kp + krow * D;
        float dot = 0.f;
#pragma unroll
        for (int k = 0; k < NE; ++k) dot = fmaf(qr[k], kr[lane + 32 * k], dot);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
        const float s = dot * scale;
        const float m_new = fmaxf(m, s);
        const float alpha = expf(m - m_new);  // m = -inf -> 0
        const float pe = expf(s - m_new);
        l = l * alpha + pe;
        const float* vr = vp + krow * D;
#pragma unroll
        for (int k = 0; k < NE; ++k) acc[k] = fmaf(acc[k], alpha, pe * vr[lane + 32 * k]);
        m = m_new;
      }
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    float* o = static_cast<float*>(a.o);
#pragma unroll
    for (int k = 0; k < NE; ++k) o[(row * a.hq + h) * D + lane + 32 * k] = acc[k] * inv;
    if (a.lse != nullptr && lane == 0) a.lse[row * a.hq + h] = l > 0.f ? m + logf(l) : -INFINITY;
  }
}

}  // namespace

cudaError_t launch_span_attn_f32(const AttnArgs& a, cudaStream_t st) {
  if (a.n_items == 0) return cudaSuccess;
  dim3 grid(a.n_items, a.hq);
  switch (a.d) {
    case 32: span_attn_f32_kernel<32><<<grid, 128, 0, st>>>(a); break;
    case 64: span_attn_f32_kernel<64><<<grid, 128, 0, st>>>(a); break;
    case 128: span_attn_f32_kernel<128><<<grid, 128, 0, st>>>(a); break;
    case 256: span_attn_f32_kernel<256><<<grid, 128, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace spq
