// cidra.cu — K8: CIDRA in-place block repositioning (§5.5.1).
//
// Executes the host schedule (host/cidra.h): per component, a sequence of ops
//   mode 0: block dst <- R(block src, delta)    mode 1: tmp <- block src    mode 2: dst <- R(tmp, delta)
// where R rotates K by delta positions (ReRoPE P:610: k' = rope(k, +delta), rotate-half pairs
// (i, i + d/2), reading R15) and copies V. The order inside a component is what makes the
// update safe in place; components are independent.
//
// B200 design: HBM-bound element-parallel work, no shared memory and no block-level sync.
// Every element of a (block, layer, kv head) tile is touched by the same thread in every op of
// its component (the same row t and columns in each block), so the in-place dependencies are
// plain program order inside one thread — the "scratch block" of a cycle is a few registers.
// CTA (component, layer x kv head, slice of rows); a thread owns rows t and a 16-byte unit u of
// the first half of d plus its rotate-half partner unit in the second half (8 pairs for bf16, 4
// for fp32): 128-bit loads/stores, a warp covers whole rows contiguously. Rows are split over
// grid.z when components x layers x heads alone would not fill the GPU (one long cycle at L = 1
// is 8 CTAs otherwise); small grids also use 4-byte units (one rotate-half pair per thread: 4x
// the threads in flight) and load the next op's source while the current op is rotated and
// stored (legal: the schedule reads every block before any op writes it — only the scratch of
// mode 2 comes from an earlier op — so a thread's chain of ops is latency-bound, not
// order-bound). cos/sin of delta * theta_i come from the ctx's fp64-built table at |delta| (sin
// negated for delta < 0).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "launch.h"

namespace spq {
namespace {

template <typename T>
struct V16;
template <>
struct V16<__nv_bfloat16> {
  static constexpr int N = 8;  // elements per 16-byte unit
  using raw = uint4;
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
struct V16<float> {
  static constexpr int N = 4;
  using raw = uint4;
  __device__ static void unpack(const uint4& u, float (&f)[4]) {
    f[0] = __uint_as_float(u.x);
    f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z);
    f[3] = __uint_as_float(u.w);
  }
  __device__ static uint4 pack(const float (&f)[4]) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  }
};

// 8-byte units
template <typename T>
struct V8;
template <>
struct V8<__nv_bfloat16> {
  static constexpr int N = 4;
  using raw = uint2;
  __device__ static void unpack(const uint2& u, float (&f)[4]) {
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float2 t = __bfloat1622float2(p[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  __device__ static uint2 pack(const float (&f)[4]) {
    uint2 u;
    __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 2; ++i) p[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return u;
  }
};
template <>
struct V8<float> {
  static constexpr int N = 2;
  using raw = uint2;
  __device__ static void unpack(const uint2& u, float (&f)[2]) {
    f[0] = __uint_as_float(u.x);
    f[1] = __uint_as_float(u.y);
  }
  __device__ static uint2 pack(const float (&f)[2]) { return make_uint2(__float_as_uint(f[0]), __float_as_uint(f[1])); }
};

// 4-byte units
template <typename T>
struct V4;
template <>
struct V4<__nv_bfloat16> {
  static constexpr int N = 2;
  using raw = uint32_t;
  __device__ static void unpack(const uint32_t& u, float (&f)[2]) {
    const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
    f[0] = t.x;
    f[1] = t.y;
  }
  __device__ static uint32_t pack(const float (&f)[2]) {
    const __nv_bfloat162 p = __floats2bfloat162_rn(f[0], f[1]);
    return *reinterpret_cast<const uint32_t*>(&p);
  }
};
template <>
struct V4<float> {
  static constexpr int N = 1;
  using raw = uint32_t;
  __device__ static void unpack(const uint32_t& u, float (&f)[1]) { f[0] = __uint_as_float(u); }
  __device__ static uint32_t pack(const float (&f)[1]) { return __float_as_uint(f[0]); }
};
// small grids: 4-byte units (one rotate-half pair of bf16 per thread and half row), 4x the
// threads of the 16-byte form, so 4x the loads in flight on the latency-bound op chains
// (C2's 268 random moves at one layer: 0.249 -> 0.190 ms per call; 8-byte units 0.228, 2-byte
// units 0.29; the 40-layer case keeps 16-byte units)
template <typename T>
using VSmall = V4<T>;

template <typename T, int D, bool AHEAD, typename VT>
__global__ void __launch_bounds__(256) cidra_kernel(const int4* __restrict__ ops, const int32_t* __restrict__ comp_off,
                                                    T* k_pool, T* v_pool, const float2* __restrict__ rope, int hkv,
                                                    int bs, int64_t nblk, int layer0, int units_per_cta) {
  constexpr int N = VT::N;
  using R = typename VT::raw;
  constexpr int U = D / 2 / N;  // units per half row
  const int comp = blockIdx.x;
  const int layer = layer0 + static_cast<int>(blockIdx.y) / hkv;
  const int h = static_cast<int>(blockIdx.y) % hkv;
  const int o0 = comp_off[comp], o1 = comp_off[comp + 1];
  // element offset of (block b, this layer/head, row t, column c): ((layer*nblk + b)*hkv + h)*bs*D + t*D + c
  const int64_t lh = static_cast<int64_t>(layer) * nblk;
  auto tile = [&](int32_t b) { return ((lh + b) * hkv + h) * static_cast<int64_t>(bs) * D; };
  const int i0 = static_cast<int>(blockIdx.z) * units_per_cta, i1 = min(bs * U, i0 + units_per_cta);
  for (int idx = i0 + threadIdx.x; idx < i1; idx += blockDim.x) {
    const int t = idx / U, u = idx % U;
    const int c0 = t * D + u * N;  // first-half unit; partner at + D/2
    R tk0 = R{}, tk1 = tk0, tv0 = tk0, tv1 = tk0;  // the cycle's scratch
    // AHEAD: the source units of op o are loaded during op o - 1
    R nk0 = tk0, nk1 = tk0, nv0 = tk0, nv1 = tk0;
    auto load_src = [&](const int4& op, R& k0, R& k1, R& v0, R& v1) {
      const int64_t s = tile(op.y) + c0;
      k0 = *reinterpret_cast<const R*>(k_pool + s);
      k1 = *reinterpret_cast<const R*>(k_pool + s + D / 2);
      v0 = *reinterpret_cast<const R*>(v_pool + s);
      v1 = *reinterpret_cast<const R*>(v_pool + s + D / 2);
    };
    int4 nop = o0 < o1 ? ops[o0] : make_int4(0, 0, 0, 2);
    if (AHEAD && nop.w != 2) load_src(nop, nk0, nk1, nv0, nv1);
    for (int o = o0; o < o1; ++o) {
      const int4 op = nop;  // {dst, src, delta, mode}
      R k0, k1, v0, v1;
      if (AHEAD) {
        k0 = nk0, k1 = nk1, v0 = nv0, v1 = nv1;
        if (o + 1 < o1) {
          nop = ops[o + 1];
          if (nop.w != 2) load_src(nop, nk0, nk1, nv0, nv1);
        }
      } else if (o + 1 < o1) {
        nop = ops[o + 1];
      }
      if (op.w == 2) {
        k0 = tk0, k1 = tk1, v0 = tv0, v1 = tv1;
      } else {
        if (!AHEAD) load_src(op, k0, k1, v0, v1);
        if (op.w == 1) {
          tk0 = k0, tk1 = k1, tv0 = v0, tv1 = v1;
          continue;
        }
      }
      float x[N], y[N];
      VT::unpack(k0, x);
      VT::unpack(k1, y);
      const int ad = op.z < 0 ? -op.z : op.z;
      const float sg = op.z < 0 ? -1.f : 1.f;
      const float2* cs = rope + static_cast<int64_t>(ad) * (D / 2) + u * N;
#pragma unroll
      for (int e = 0; e < N; ++e) {
        const float2 a = __ldg(cs + e);
        const float sn = sg * a.y;
        const float xr = x[e] * a.x - y[e] * sn;  // first half: x cos - y sin
        const float yr = y[e] * a.x + x[e] * sn;  // second half: y cos + x sin
        x[e] = xr;
        y[e] = yr;
      }
      const int64_t d = tile(op.x) + c0;
      *reinterpret_cast<R*>(k_pool + d) = VT::pack(x);
      *reinterpret_cast<R*>(k_pool + d + D / 2) = VT::pack(y);
      *reinterpret_cast<R*>(v_pool + d) = v0;
      *reinterpret_cast<R*>(v_pool + d + D / 2) = v1;
    }
  }
}

template <typename T, int D>
cudaError_t launch_t(const CidraArgs& a, cudaStream_t st) {
  const int64_t tiles = static_cast<int64_t>(a.n_comp) * (a.layer_end - a.layer_begin) * a.hkv;
  // rows split over grid.z until the grid holds ~2 CTAs per SM (slices of >= 64 units); small
  // grids also use narrower units (VSmall): more threads, so more loads in flight on the
  // latency-bound op chains
  const int64_t want = 2LL * (a.num_sms > 0 ? a.num_sms : 148);
  const bool small = tiles < want;
  const int units = a.bs * (D / 2 / (small ? VSmall<T>::N : V16<T>::N));
  int splits = static_cast<int>(std::min<int64_t>(std::max<int64_t>(1, (want + tiles - 1) / tiles), std::max(1, units / 64)));
  const int per = ((units + splits - 1) / splits + 31) / 32 * 32;
  splits = (units + per - 1) / per;
  const dim3 grid(static_cast<unsigned>(a.n_comp), static_cast<unsigned>((a.layer_end - a.layer_begin) * a.hkv),
                  static_cast<unsigned>(splits));
  const int threads = per >= 256 ? 256 : per;
  // small grids are latency-bound on each thread's chain of ops: load one op ahead there (with
  // 40 layers of work the look-ahead measured slower: 1.22 vs 1.11 ms)
  if (small)
    cidra_kernel<T, D, true, VSmall<T>><<<grid, threads, 0, st>>>(a.ops, a.comp_off, static_cast<T*>(a.k_pool),
                                                              static_cast<T*>(a.v_pool), a.rope, a.hkv, a.bs,
                                                              a.nblk, a.layer_begin, per);
  else
    cidra_kernel<T, D, false, V16<T>><<<grid, threads, 0, st>>>(a.ops, a.comp_off, static_cast<T*>(a.k_pool),
                                                                static_cast<T*>(a.v_pool), a.rope, a.hkv, a.bs,
                                                                a.nblk, a.layer_begin, per);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_cidra(const CidraArgs& a, cudaStream_t st) {
  if (a.n_comp == 0 || a.layer_end <= a.layer_begin) return cudaSuccess;
  if (a.fp32) {
    switch (a.d) {
      case 64: return launch_t<float, 64>(a, st);
      case 128: return launch_t<float, 128>(a, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (a.d) {
    case 64: return launch_t<__nv_bfloat16, 64>(a, st);
    case 128: return launch_t<__nv_bfloat16, 128>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace spq
