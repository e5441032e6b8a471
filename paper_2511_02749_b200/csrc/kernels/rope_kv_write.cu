// rope_kv_write.cu — K1: fused RoPE + paged KV-cache write.
//
// For every packed row r with slot[r] >= 0 and every kv head h:
//   k_pool[layer][slot/bs][h][slot%bs][:] = RoPE(k[r,h,:], pos[r])      (R15 rotate-half)
//   v_pool[layer][slot/bs][h][slot%bs][:] = v[r,h,:]
// plus zero-fill of the plan's pad slots (partial blocks, reading R8).
// RoPE positions: span-local for fragments (reading R2), global for prefix/cross (§5.5
// P:610). cos/sin come from the fp64-built table [max_pos][d/2] (float2).
//
// HBM-bound, no reuse: one thread moves a 16-byte vector of k and of v from each half of d —
// a rotate-half pair (element i <-> i + d/2) — so the (cos, sin) row is read once per pair and
// no shuffle is needed. Loads/stores are 128-bit; a warp covers whole rows contiguously.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "launch.h"

namespace spq {
namespace {

template <typename T>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void unpack(const uint4& u, float (&f)[8]) {
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 t = __bfloat1622float2(p[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  __device__ static uint4 pack(const float (&f)[8]) {
    uint4 u;
    __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return u;
  }
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ static void unpack(const uint4& u, float (&f)[4]) {
    f[0] = __uint_as_float(u.x);
    f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z);
    f[3] = __uint_as_float(u.w);
  }
  __device__ static uint4 pack(const float (&f)[4]) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
  }
};

// G = d / N vectors per (row, head). A thread owns vector u < G/2 of the first half of d and its
// rotate-half partner u + G/2 (the same (cos, sin) pairs), so the table row is read once per
// pair and no shuffle is needed; the lanes of one (row, head) are G/2 consecutive lanes.
template <typename T, int D>
__global__ void __launch_bounds__(256) rope_kv_write_kernel(
    const T* __restrict__ k, const T* __restrict__ v, const int32_t* __restrict__ pos,
    const int64_t* __restrict__ slot, int64_t rows, const int64_t* __restrict__ pad_slots,
    int64_t n_pad, T* __restrict__ k_pool, T* __restrict__ v_pool, int hkv, int bs, int64_t nblk,
    int layer, const float2* __restrict__ rope) {
  constexpr int N = Vec<T>::N;
  constexpr int G = D / N;
  constexpr int H = G / 2;  // threads per (row, head)
  static_assert(G <= 32 && (G & (G - 1)) == 0 && G >= 2, "d/N must be a power of two in [2, 32]");
  // the attention launch that reads these pages may start its prologue now (it waits for this
  // grid's completion before touching the pool: griddepcontrol.wait in span_attn_tc)
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per_row = static_cast<int64_t>(hkv) * H;
  const int64_t total = rows * per_row;
  const int64_t layer_off = static_cast<int64_t>(layer) * nblk * hkv * bs * D;
  if (gid < total) {
    const int64_t r = gid / per_row;
    const int rem = static_cast<int>(gid - r * per_row);
    const int h = rem / H, u = rem % H;
    const int64_t src = (r * hkv + h) * D + u * N;
    // every load issued up front, independent of the others (rows with slot -1 — resident
    // blocks — load for nothing)
    const int64_t s = slot[r];
    const int p = pos[r];
    const uint4 k0 = __ldg(reinterpret_cast<const uint4*>(k + src));
    const uint4 k1 = __ldg(reinterpret_cast<const uint4*>(k + src + D / 2));
    const uint4 v0 = __ldg(reinterpret_cast<const uint4*>(v + src));
    const uint4 v1 = __ldg(reinterpret_cast<const uint4*>(v + src + D / 2));
    if (s < 0) return;
    const float4* cs = reinterpret_cast<const float4*>(rope + static_cast<int64_t>(p) * (D / 2) + u * N);
    float x[N], y[N], ox[N], oy[N];
    Vec<T>::unpack(k0, x);
    Vec<T>::unpack(k1, y);
#pragma unroll
    for (int e = 0; e < N; e += 2) {
      const float4 c = __ldg(cs + e / 2);  // (cos, sin) of pairs u*N+e, u*N+e+1
      // first half: x cos - y sin ; second half: y cos + x sin
      ox[e] = fmaf(x[e], c.x, -y[e] * c.y);
      oy[e] = fmaf(y[e], c.x, x[e] * c.y);
      ox[e + 1] = fmaf(x[e + 1], c.z, -y[e + 1] * c.w);
      oy[e + 1] = fmaf(y[e + 1], c.z, x[e + 1] * c.w);
    }
    const int64_t blk = s / bs, off = s % bs;
    const int64_t dst = layer_off + ((blk * hkv + h) * bs + off) * D + u * N;
    *reinterpret_cast<uint4*>(k_pool + dst) = Vec<T>::pack(ox);
    *reinterpret_cast<uint4*>(k_pool + dst + D / 2) = Vec<T>::pack(oy);
    *reinterpret_cast<uint4*>(v_pool + dst) = v0;
    *reinterpret_cast<uint4*>(v_pool + dst + D / 2) = v1;
    return;
  }
  // pad slots: zero K and V of every head
  const int64_t pid = gid - total;
  if (pid >= n_pad * per_row) return;
  const int64_t pr = pid / per_row;
  const int prem = static_cast<int>(pid - pr * per_row);
  const int ph = prem / H, pu = prem % H;
  const int64_t ps = pad_slots[pr];
  const int64_t pblk = ps / bs, poff = ps % bs;
  const int64_t dst = layer_off + ((pblk * hkv + ph) * bs + poff) * D + pu * N;
  const uint4 z = make_uint4(0, 0, 0, 0);
  *reinterpret_cast<uint4*>(k_pool + dst) = z;
  *reinterpret_cast<uint4*>(k_pool + dst + D / 2) = z;
  *reinterpret_cast<uint4*>(v_pool + dst) = z;
  *reinterpret_cast<uint4*>(v_pool + dst + D / 2) = z;
}

template <typename T, int D>
cudaError_t launch_t(const KvWriteArgs& a, cudaStream_t st) {
  constexpr int H = D / Vec<T>::N / 2;
  const int64_t threads = (a.rows + a.n_pad) * static_cast<int64_t>(a.hkv) * H;
  if (threads == 0) return cudaSuccess;
  const int64_t blocks = (threads + 255) / 256;
  rope_kv_write_kernel<T, D><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
      static_cast<const T*>(a.k), static_cast<const T*>(a.v), a.pos, a.slot, a.rows, a.pad_slots,
      a.n_pad, static_cast<T*>(a.k_pool), static_cast<T*>(a.v_pool), a.hkv, a.bs, a.nblk, a.layer,
      a.rope);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_rope_kv_write(const KvWriteArgs& a, cudaStream_t st) {
  if (a.fp32) {
    switch (a.d) {
      case 32: return launch_t<float, 32>(a, st);
      case 64: return launch_t<float, 64>(a, st);
      case 128: return launch_t<float, 128>(a, st);
    }
  } else {
    switch (a.d) {
      case 64: return launch_t<__nv_bfloat16, 64>(a, st);
      case 128: return launch_t<__nv_bfloat16, 128>(a, st);
      case 256: return launch_t<__nv_bfloat16, 256>(a, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace spq
