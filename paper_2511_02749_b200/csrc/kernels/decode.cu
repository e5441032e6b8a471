// decode.cu — K9: decode attention after the join (§4.1 "G" token
// generation over a span query, and nested generation P:461-462).
//
// One new query row per home query (generated token t at position N_q + t, N_q = P + S + C)
// attends over [prefix | every fragment at Δ_f | cross + generated tokens 0..t] in the paged
// pool. Fragment KV stays at span-local positions: the row's q is counter-rotated by Δ_f per
// fragment segment, exactly as in the join. Keys of the cross+gen segment are causal by
// position, so unwritten slots of the reserved generation blocks are never read.
//
// B200 design: HBM-bound (one row per query: per key, g dot products of length d against
// 2·d·elt bytes of K and V), so CUDA cores, not tensor cores. Split-KV: a CTA = (query, kv head,
// chunk of <= T KV tiles of 128 keys), 128 threads; the g = Hq/Hkv q heads of the kv head share
// every K/V tile (loaded once into shared memory with 16-byte vector loads). Per tile: thread =
// key for the scores (g fp32 accumulators, q rotated once per segment in fp32 from the fp64-built
// table), one warp per head for the online-softmax max/sum, thread = (head, column slice) for
// P·V. Chunks write fp32 partials (normalized O, natural-log LSE) merged by K4 (combine.cu) in a
// fixed order; an unsplit (query, kv head) writes O / LSE directly.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "launch.h"

namespace spq {
namespace {

constexpr int kThreads = 128;
constexpr int kTileK = 128;  // keys per KV tile (work.h kTileKeys)
constexpr int kMaxG = 8;     // q heads per kv head

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f(__nv_bfloat16 x) {
  return __bfloat162float(x);
}
template <>
__device__ __forceinline__ float to_f(float x) {
  return x;
}

template <typename T>
__device__ __forceinline__ void store_out(T* p, float x);
template <>
__device__ __forceinline__ void store_out(__nv_bfloat16* p, float x) {
  *p = __float2bfloat16_rn(x);
}
template <>
__device__ __forceinline__ void store_out(float* p, float x) {
  *p = x;
}

// T: pool / q dtype; TO: output dtype. D: head dim; G: q heads per kv head.
template <typename T, typename TO, int D, int G>
__global__ void __launch_bounds__(kThreads) decode_kernel(const DecodeArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  constexpr int KP = D + 16 / static_cast<int>(sizeof(T));  // padded K row (bank spread)
  T* Ks = reinterpret_cast<T*>(smem_raw);                     // [kTileK][KP]
  T* Vs = Ks + kTileK * KP;                                   // [kTileK][D]
  float* qr = reinterpret_cast<float*>(Vs + kTileK * D);      // [G][D] rotated q (fp32)
  float* ps = qr + G * D;                                     // [G][kTileK] scores / P
  float* st = ps + G * kTileK;                                // [G][3] m, l, alpha
  const DecodeItem it = a.items[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pos = a.pos_base[it.row] + a.step;
  const int h0 = it.kvh * G;
  constexpr int VEC = 16 / sizeof(T);  // elements per 16-byte vector
  constexpr int OUT = (G * D + kThreads - 1) / kThreads;  // P·V outputs per thread
  float acc[OUT];
#pragma unroll
  for (int e = 0; e < OUT; ++e) acc[e] = 0.f;
  if (tid < G) {
    st[tid * 3 + 0] = -INFINITY;
    st[tid * 3 + 1] = 0.f;
  }
  const T* qg = static_cast<const T*>(a.q) + (static_cast<int64_t>(it.row) * a.hq + h0) * D;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  int cur_rot = INT32_MIN;
  const int64_t layer_rows = static_cast<int64_t>(a.layer) * a.nblk * a.hkv * a.bs;
  for (int t = it.tile_begin; t < it.tile_end; ++t) {
    const KvTile tl = a.tiles[t];
    const int n_vis = tl.causal ? min(tl.n_valid, pos - tl.key_pos0 + 1) : tl.n_valid;
    if (n_vis <= 0) continue;  // uniform across the CTA
    __syncthreads();           // the previous tile's smem is no longer read
    if (tl.rot_delta != cur_rot) {  // a new segment: q rotated to pos - Δ (rotate-half pairs)
      cur_rot = tl.rot_delta;
      const int rp = min(max(pos - cur_rot, 0), a.max_pos - 1);
      for (int i = tid; i < G * (D / 2); i += kThreads) {
        const int h = i / (D / 2), c = i % (D / 2);
        const float x = to_f(qg[h * D + c]), y = to_f(qg[h * D + c + D / 2]);
        const float2 cs = a.rope[static_cast<int64_t>(rp) * (D / 2) + c];
        qr[h * D + c] = x * cs.x - y * cs.y;
        qr[h * D + c + D / 2] = y * cs.x + x * cs.y;
      }
    }
    // K / V rows [0, n_vis) of the tile -> smem (16-byte vectors, a warp covers whole rows)
    for (int i = tid; i < n_vis * (D / VEC); i += kThreads) {
      const int key = i / (D / VEC), u = i % (D / VEC);
      const int32_t blk = a.tile_blocks[tl.blk_off + key / a.bs];
      const int64_t row = layer_rows + (static_cast<int64_t>(blk) * a.hkv + it.kvh) * a.bs + key % a.bs;
      *reinterpret_cast<uint4*>(Ks + key * KP + u * VEC) =
          *reinterpret_cast<const uint4*>(static_cast<const T*>(a.k_pool) + row * D + u * VEC);
      *reinterpret_cast<uint4*>(Vs + key * D + u * VEC) =
          *reinterpret_cast<const uint4*>(static_cast<const T*>(a.v_pool) + row * D + u * VEC);
    }
    __syncthreads();
    // scores: thread = key
    if (tid < n_vis) {
      float s[G];
#pragma unroll
      for (int h = 0; h < G; ++h) s[h] = 0.f;
#pragma unroll 4
      for (int c = 0; c < D; c += VEC) {
        const uint4 kv = *reinterpret_cast<const uint4*>(Ks + tid * KP + c);
        const T* ke = reinterpret_cast<const T*>(&kv);
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const float kf = to_f(ke[e]);
#pragma unroll
          for (int h = 0; h < G; ++h) s[h] = fmaf(qr[h * D + c + e], kf, s[h]);
        }
      }
#pragma unroll
      for (int h = 0; h < G; ++h) ps[h * kTileK + tid] = s[h] * scale_log2;
    }
    __syncthreads();
    // online softmax: one warp per head (heads h, h + 4, ...)
    for (int h = warp; h < G; h += kThreads / 32) {
      float mx = -INFINITY;
      for (int i = lane; i < n_vis; i += 32) mx = fmaxf(mx, ps[h * kTileK + i]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float m_old = st[h * 3 + 0];
      const float m_new = fmaxf(m_old, mx);
      float sum = 0.f;
      for (int i = lane; i < n_vis; i += 32) {
        const float p = exp2f(ps[h * kTileK + i] - m_new);
        ps[h * kTileK + i] = p;
        sum += p;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      __syncwarp();
      if (lane == 0) {
        const float alpha = m_old == -INFINITY ? 0.f : exp2f(m_old - m_new);
        st[h * 3 + 0] = m_new;
        st[h * 3 + 1] = st[h * 3 + 1] * alpha + sum;
        st[h * 3 + 2] = alpha;
      }
    }
    __syncthreads();
    // O = O * alpha + P V: thread = (head, OUT consecutive columns)
#pragma unroll
    for (int e = 0; e < OUT; ++e) {
      const int f = tid * OUT + e;
      if (f < G * D) {
        const int h = f / D, c = f % D;
        float o = acc[e] * st[h * 3 + 2];
        const float* pr = ps + h * kTileK;
        for (int i = 0; i < n_vis; ++i) o = fmaf(pr[i], to_f(Vs[i * D + c]), o);
        acc[e] = o;
      }
    }
  }
  __syncthreads();
  // normalized O and natural-log LSE: final, or a split partial merged by combine
#pragma unroll
  for (int e = 0; e < OUT; ++e) {
    const int f = tid * OUT + e;
    if (f >= G * D) continue;
    const int h = f / D, c = f % D;
    const float l = st[h * 3 + 1];
    const float v = l > 0.f ? acc[e] / l : 0.f;
    if (it.part >= 0)
      a.opart[(static_cast<int64_t>(it.part) * G + h) * D + c] = v;
    else
      store_out(static_cast<TO*>(a.o) + (static_cast<int64_t>(it.row) * a.hq + h0 + h) * D + c, v);
  }
  if (tid < G) {
    const float l = st[tid * 3 + 1];
    const float lse = l > 0.f ? (st[tid * 3 + 0] + log2f(l)) * 0.69314718055994531f : -INFINITY;
    if (it.part >= 0)
      a.lsepart[static_cast<int64_t>(it.part) * G + tid] = lse;
    else if (a.lse != nullptr)
      a.lse[static_cast<int64_t>(it.row) * a.hq + h0 + tid] = lse;
  }
}

template <typename T, typename TO, int D, int G>
cudaError_t launch_g(const DecodeArgs& a, cudaStream_t st) {
  constexpr int KP = D + 16 / static_cast<int>(sizeof(T));
  const size_t smem = sizeof(T) * (kTileK * KP + kTileK * D) + sizeof(float) * (G * D + G * kTileK + G * 3);
  static_assert(sizeof(T) * (kTileK * (D + 16 / sizeof(T)) + kTileK * D) + sizeof(float) * (G * D + G * kTileK + G * 3) <= 232448,
                "decode smem");
  cudaError_t e = cudaFuncSetAttribute(decode_kernel<T, TO, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  decode_kernel<T, TO, D, G><<<a.n_items, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename T, typename TO, int D>
cudaError_t launch_d(const DecodeArgs& a, cudaStream_t st) {
  switch (a.hq / a.hkv) {
    case 1: return launch_g<T, TO, D, 1>(a, st);
    case 2: return launch_g<T, TO, D, 2>(a, st);
    case 4: return launch_g<T, TO, D, 4>(a, st);
    case 8: return launch_g<T, TO, D, 8>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T, typename TO>
cudaError_t launch_t(const DecodeArgs& a, cudaStream_t st) {
  switch (a.d) {
    case 64: return launch_d<T, TO, 64>(a, st);
    case 128: return launch_d<T, TO, 128>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_decode(const DecodeArgs& a, cudaStream_t st) {
  if (a.n_items == 0) return cudaSuccess;
  if (a.fp32) return launch_t<float, float>(a, st);
  return a.out_fp32 ? launch_t<__nv_bfloat16, float>(a, st) : launch_t<__nv_bfloat16, __nv_bfloat16>(a, st);
}

}  // namespace spq
