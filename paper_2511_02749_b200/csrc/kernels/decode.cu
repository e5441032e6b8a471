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
// every K/V sub-tile of 64 keys, double-buffered in shared memory by cp.async (16-byte, no
// register round trip). Per sub-tile: thread = (key, half of the heads) for the scores (fp32
// accumulators, q rotated once per segment in fp32 from the fp64-built table, float4 broadcast
// reads), one warp per head for the online-softmax max/sum, thread = (head, 4 consecutive
// columns) for P·V. Chunks write fp32 partials (normalized O, natural-log LSE) merged by K4 (combine.cu) in a
// fixed order; an unsplit (query, kv head) writes O / LSE directly.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "launch.h"
#include "sm100.cuh"

namespace spq {
namespace {

constexpr int kThreads = 128;
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

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int kSub = 64;  // keys per pipelined sub-tile (half a KV tile)

// T: pool / q dtype; TO: output dtype. D: head dim; G: q heads per kv head.
// Sub-tiles of 64 keys are double-buffered: cp.async (16-byte, no register round trip) loads
// sub-tile s+1 while s is scored, so a CTA keeps ~34 KB (d = 128, bf16) of K/V in flight.
template <typename T, typename TO, int D, int G>
__global__ void __launch_bounds__(kThreads) decode_kernel(const DecodeArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  constexpr int KP = D + 16 / static_cast<int>(sizeof(T));  // padded K row (bank spread)
  constexpr int kBufElems = kSub * KP + kSub * D;             // K then V of one sub-tile
  T* bufs = reinterpret_cast<T*>(smem_raw);                   // [2][kBufElems]
  float* qr = reinterpret_cast<float*>(bufs + 2 * kBufElems);  // [G][D] rotated q (fp32)
  float* ps = qr + G * D;                                      // [G][kSub] scores / P
  float* st = ps + G * kSub;                                   // [G][3] m, l, alpha
  const DecodeItem it = a.items[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pos = a.pos_base[it.row] + a.step;
  const int h0 = it.kvh * G;
  constexpr int VEC = 16 / sizeof(T);  // elements per 16-byte vector
  constexpr int OUT = (G * D + kThreads - 1) / kThreads;  // P·V outputs per thread
  constexpr int HPT = (G + 1) / 2;                         // score heads per thread (2 threads per key)
  float acc[OUT];
#pragma unroll
  for (int e = 0; e < OUT; ++e) acc[e] = 0.f;
  if (tid < G) {
    st[tid * 3 + 0] = -INFINITY;
    st[tid * 3 + 1] = 0.f;
  }
  const T* qg = static_cast<const T*>(a.q) + (static_cast<int64_t>(it.row) * a.hq + h0) * D;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  const int64_t layer_rows = static_cast<int64_t>(a.layer) * a.nblk * a.hkv * a.bs;
  // the item's sub-tiles in order: (tile, half); causal tiles of the cross+gen segment end the
  // list at the row's position (later keys are not generated yet)
  auto n_vis_of = [&](int t) {
    const KvTile tl = a.tiles[t];
    return tl.causal ? min(tl.n_valid, pos - tl.key_pos0 + 1) : tl.n_valid;
  };
  auto issue = [&](int t, int hh, int buf) {  // cp.async of sub-tile (t, hh) into buffer buf
    const KvTile tl = a.tiles[t];
    const int nk = min(kSub, n_vis_of(t) - hh * kSub);
    T* Kb = bufs + buf * kBufElems;
    T* Vb = Kb + kSub * KP;
    for (int i = tid; i < nk * (D / VEC); i += kThreads) {
      const int key = i / (D / VEC), u = i % (D / VEC);
      const int kk = hh * kSub + key;
      const int32_t blk = a.tile_blocks[tl.blk_off + kk / a.bs];
      const int64_t row = layer_rows + (static_cast<int64_t>(blk) * a.hkv + it.kvh) * a.bs + kk % a.bs;
      cp_async16(Kb + key * KP + u * VEC, static_cast<const T*>(a.k_pool) + row * D + u * VEC);
      cp_async16(Vb + key * D + u * VEC, static_cast<const T*>(a.v_pool) + row * D + u * VEC);
    }
    cp_async_commit();
  };
  auto next_sub = [&](int& t, int& hh) {  // advance (t, hh); t = tile_end when done
    if (hh == 0 && n_vis_of(t) > kSub) {
      hh = 1;
      return;
    }
    hh = 0;
    ++t;
    if (t < it.tile_end && n_vis_of(t) <= 0) t = it.tile_end;
  };
  int t = it.tile_begin, hh = 0;
  if (t < it.tile_end && n_vis_of(t) <= 0) t = it.tile_end;
  if (t < it.tile_end) issue(t, hh, 0);
  int cur_rot = INT32_MIN;
  for (int buf = 0; t < it.tile_end; buf ^= 1) {
    int t2 = t, hh2 = hh;
    next_sub(t2, hh2);
    if (t2 < it.tile_end) {
      issue(t2, hh2, buf ^ 1);  // the other buffer was released by the previous sub-tile's end sync
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    const KvTile tl = a.tiles[t];
    const int nk = min(kSub, n_vis_of(t) - hh * kSub);
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
    __syncthreads();  // this sub-tile's K/V (every thread's cp.async) and q are in smem
    const T* Kb = bufs + buf * kBufElems;
    const T* Vb = Kb + kSub * KP;
    // scores: thread = (key, half of the heads)
    {
      const int key = tid % kSub, hs = (tid / kSub) * HPT;
      if (key < nk && hs < G) {
        float s[HPT];
#pragma unroll
        for (int j = 0; j < HPT; ++j) s[j] = 0.f;
#pragma unroll 2
        for (int c = 0; c < D; c += VEC) {
          const uint4 kv = *reinterpret_cast<const uint4*>(Kb + key * KP + c);
          const T* ke = reinterpret_cast<const T*>(&kv);
          float kf[VEC];
#pragma unroll
          for (int e = 0; e < VEC; ++e) kf[e] = to_f(ke[e]);
#pragma unroll
          for (int j = 0; j < HPT; ++j) {
            if (hs + j >= G) continue;
#pragma unroll
            for (int e = 0; e < VEC; e += 4) {  // q as float4 broadcasts
              const float4 q4 = *reinterpret_cast<const float4*>(qr + (hs + j) * D + c + e);
              s[j] = fmaf(q4.x, kf[e], s[j]);
              s[j] = fmaf(q4.y, kf[e + 1], s[j]);
              s[j] = fmaf(q4.z, kf[e + 2], s[j]);
              s[j] = fmaf(q4.w, kf[e + 3], s[j]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < HPT; ++j)
          if (hs + j < G) ps[(hs + j) * kSub + key] = s[j] * scale_log2;
      }
    }
    __syncthreads();
    // online softmax: one warp per head (heads h, h + 4, ...)
    for (int h = warp; h < G; h += kThreads / 32) {
      float mx = -INFINITY;
      for (int i = lane; i < nk; i += 32) mx = fmaxf(mx, ps[h * kSub + i]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float m_old = st[h * 3 + 0];
      const float m_new = fmaxf(m_old, mx);
      float sum = 0.f;
      for (int i = lane; i < nk; i += 32) {
        const float p = exp2f(ps[h * kSub + i] - m_new);
        ps[h * kSub + i] = p;
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
    if (tid * OUT < G * D) {  // OUT consecutive columns of one head (OUT divides D)
      const int f0 = tid * OUT, h = f0 / D, c0 = f0 % D;
      const float alpha = st[h * 3 + 2];
#pragma unroll
      for (int e = 0; e < OUT; ++e) acc[e] *= alpha;
      const float* pr = ps + h * kSub;
#pragma unroll 4
      for (int i = 0; i < nk; ++i) {
        const float p = pr[i];
        if constexpr (OUT % 4 == 0 && sizeof(T) == 2) {
#pragma unroll
          for (int e = 0; e < OUT; e += 4) {
            const uint2 u = *reinterpret_cast<const uint2*>(Vb + i * D + c0 + e);
            const float2 v01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
            const float2 v23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
            acc[e] = fmaf(p, v01.x, acc[e]);
            acc[e + 1] = fmaf(p, v01.y, acc[e + 1]);
            acc[e + 2] = fmaf(p, v23.x, acc[e + 2]);
            acc[e + 3] = fmaf(p, v23.y, acc[e + 3]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < OUT; ++e) acc[e] = fmaf(p, to_f(Vb[i * D + c0 + e]), acc[e]);
        }
      }
    }
    __syncthreads();  // buffer buf and ps are free for the next sub-tile
    t = t2;
    hh = hh2;
  }
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

// ---------------------------------------------------------------- bf16 pools: warp-split decode
// The bf16 path is HBM-bound by K and V (2·d·2 bytes per key and kv head), so what limits it is
// how many bytes each SM keeps in flight, and that is set by how long a warp spends on each group
// of keys between its loads. The CTA's chunk is split over its 4 warps: warp w takes the chunk's
// 16-key groups w, w+4, ... and runs its own pipeline — cp.async double-buffered K / V group in
// its smem region (rows XOR-swizzled by 16-byte unit), its own online softmax — with no CTA
// barrier until the four (m, l, O) partials are merged at the end. Per group the two products are
// warp-level tensor-core MMAs (mma.sync m16n8k16, bf16 in, fp32 accumulate) with the q heads as
// the N = 8 side: S^T[16 keys x 8 heads] = K · Q^T (K by ldmatrix, the counter-rotated Q^T held
// in registers per segment, rounded to bf16 like the join's tcgen05 operand), then
// O^T[d x 8 heads] += V^T · P^T (V^T by ldmatrix.trans, P^T bf16 through 256 bytes of smem).
// That is ~150 instructions per group where per-lane FMA dot products took ~1200, so a warp gets
// back to its next load ~8x sooner. Heads >= G are zero padding of the N side.
constexpr int kGrp = 16;   // keys per warp step
constexpr int kWarps = 4;
constexpr int kPadHeads = 8;  // MMA N

template <int D, int G>
struct DecSmem {
  static constexpr int kUnits = D / 8;                        // 16-byte units per bf16 row
  static constexpr int kStage = 2 * kGrp * D;                 // bf16 elements: K then V of a group
  __nv_bfloat16 kv[kWarps][kDecStages][kStage];               // per warp: ring of groups
  __nv_bfloat16 pt[kWarps][kPadHeads * kGrp];                 // per warp: P^T [head][key] (bf16)
  float ml[kWarps][2 * G];                                    // merge: m, l per warp and head
};

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
// D[16x8] += A[16x16] · B[16x8]: bf16 operands, fp32 accumulators (thread fragments as in PTX ISA
// "mma.m16n8k16": g = lane / 4, t = lane % 4; A rows g / g+8, cols 2t+{0,1} / +8; B rows
// (k) 2t+{0,1} / +8, col g; C rows g / g+8, cols 2t+{0,1})
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
               "{%0, %1, %2, %3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

template <typename TO, int D, int G>
__global__ void __launch_bounds__(kThreads) decode_bf16_kernel(const DecodeArgs a) {
  using T = __nv_bfloat16;
  using Sm = DecSmem<D, G>;
  constexpr int U = Sm::kUnits;
  constexpr int KS = D / 16;  // k-steps of the score MMA = m-tiles of the P·V MMA
  static_assert(G <= kPadHeads && D % 32 == 0, "q heads per kv head fill at most the MMA N side; d in 16-column k-steps, halves in whole k-steps");
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Sm& S = *reinterpret_cast<Sm*>(smem_raw);
  const DecodeItem it = a.items[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t = lane & 3;  // MMA fragment coordinates
  const int pos = a.pos_base[it.row] + a.step;
  const int h0 = it.kvh * G;
  const T* qg = static_cast<const T*>(a.q) + (static_cast<int64_t>(it.row) * a.hq + h0) * D;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  const int64_t layer_rows = static_cast<int64_t>(a.layer) * a.nblk * a.hkv * a.bs;
  __nv_bfloat16* pt = S.pt[w];
  // this warp's groups: the chunk's groups in (tile, group) order, every kWarps-th one
  struct Grp {
    int g, nk, blk_off, rot;  // group in its tile, valid keys, the tile's block-table offset and Δ
  };
  auto n_vis_of = [&](const KvTile& tl) {
    return tl.causal ? min(tl.n_valid, pos - tl.key_pos0 + 1) : tl.n_valid;
  };
  // iterator over this warp's groups: chunk-order group indices w, w + 4, ...; the current tile's
  // fields are read once per tile (not once per group scanned: a per-group reload of the tile
  // record was a dependent load on every step of the walk)
  int it_t = it.tile_begin, it_base = 0, my_gi = w;
  KvTile cur_tile{};
  int it_nv = 0;
  if (it_t < it.tile_end) {
    cur_tile = a.tiles[it_t];
    it_nv = n_vis_of(cur_tile);
  }
  auto next_mine = [&](Grp& out) -> bool {
    while (it_t < it.tile_end) {
      const int ng = it_nv > 0 ? (it_nv + kGrp - 1) / kGrp : 0;
      const int local = my_gi - it_base;
      if (local < ng) {
        out = Grp{local, min(kGrp, it_nv - local * kGrp), cur_tile.blk_off, cur_tile.rot_delta};
        my_gi += kWarps;
        return true;
      }
      it_base += ng;
      if (++it_t < it.tile_end) {
        cur_tile = a.tiles[it_t];
        it_nv = n_vis_of(cur_tile);
      }
    }
    return false;
  };
  auto issue = [&](const Grp& gr, int buf) {  // cp.async of the group's K and V rows
    // bf16 pools have bs >= 16 (a power of two), so a 16-key group lies in one block and its
    // K (and V) rows of this kv head are one contiguous run: one block-table read per group,
    // then lane i copies 16-byte unit i of the run. Rows past the valid keys are zero-filled
    // (P is 0 there, and 0 · V must not meet stale bits that decode as NaN).
    const int kk0 = gr.g * kGrp;
    const int32_t blk = a.tile_blocks[gr.blk_off + kk0 / a.bs];
    const int64_t row0 = layer_rows + (static_cast<int64_t>(blk) * a.hkv + it.kvh) * a.bs + (kk0 & (a.bs - 1));
    const T* ks = static_cast<const T*>(a.k_pool) + row0 * D;
    const T* vs = static_cast<const T*>(a.v_pool) + row0 * D;
    __nv_bfloat16* Kb = S.kv[w][buf];
    __nv_bfloat16* Vb = Kb + kGrp * D;
    const int n = gr.nk * U;
#pragma unroll
    for (int j = 0; j < kGrp * U / 32; ++j) {
      const int i = lane + 32 * j;
      const int key = i / U, u = i % U;
      const int so = (key * U + (u ^ (key & (U - 1)))) * 8;
      const bool ok = i < n;
      cp_async16_zfill(Kb + so, ks + (ok ? i * 8 : 0), ok);
      cp_async16_zfill(Vb + so, vs + (ok ? i * 8 : 0), ok);
    }
    cp_async_commit();
  };
  float m2[2] = {-INFINITY, -INFINITY}, l2[2] = {0.f, 0.f};  // heads 2t, 2t+1
  float oc[KS][4];  // O^T: d = mt*16 + g (+8), heads 2t, 2t+1
#pragma unroll
  for (int mt = 0; mt < KS; ++mt)
#pragma unroll
    for (int e = 0; e < 4; ++e) oc[mt][e] = 0.f;
  uint32_t qf[KS][2];  // Q^T B fragments: head g, d = ks*16 + 2t + {0,1} (and + 8)
  int cur_rot = INT32_MIN;
  // kDecStages-deep ring: groups pend[0..NS-2] are in flight, pend[0] in buffer `buf`; every
  // iteration commits one cp.async group (possibly empty) so wait_group<NS-1> means "pend[0] landed"
  constexpr int NS = kDecStages;
  Grp pend[NS - 1];
  bool hv[NS - 1];
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    hv[s] = (s == 0 || hv[s - 1]) && next_mine(pend[s]);
    if (hv[s]) issue(pend[s], s);
    else cp_async_commit();
  }
  for (int buf = 0; hv[0]; buf = buf + 1 == NS ? 0 : buf + 1) {
    Grp nxt;
    const bool more = hv[NS - 2] && next_mine(nxt);
    if (more) issue(nxt, buf + NS - 1 >= NS ? buf - 1 : buf + NS - 1);  // the slot freed last iteration
    else cp_async_commit();
    cp_async_wait<NS - 1>();
    const Grp cur = pend[0];
    const int rot = cur.rot;
    if (rot != cur_rot) {  // a new segment: q rotated to pos - Δ (rotate-half pairs), fp32 -> bf16
      cur_rot = rot;
      const int rp = min(max(pos - rot, 0), a.max_pos - 1);
      const float2* cs = a.rope + static_cast<int64_t>(rp) * (D / 2);
#pragma unroll
      for (int ks = 0; ks < KS / 2; ++ks)
#pragma unroll
        for (int hi = 0; hi < 2; ++hi) {
          const int c = ks * 16 + hi * 8 + 2 * t;  // c, c + 1 < D / 2; partners c + D / 2 in k-step ks + KS / 2
          if (g < G) {
            const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(qg + g * D + c));
            const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(qg + g * D + c + D / 2));
            const float2 c0 = cs[c], c1 = cs[c + 1];
            qf[ks][hi] = pack_bf16x2(x.x * c0.x - y.x * c0.y, x.y * c1.x - y.y * c1.y);
            qf[ks + KS / 2][hi] = pack_bf16x2(y.x * c0.x + x.x * c0.y, y.y * c1.x + x.y * c1.y);
          } else {
            qf[ks][hi] = 0u;
            qf[ks + KS / 2][hi] = 0u;
          }
        }
    }
    __syncwarp();  // every lane's cp.async of this group is visible
    const __nv_bfloat16* Kb = S.kv[w][buf];
    const __nv_bfloat16* Vb = Kb + kGrp * D;
    const int mi = lane >> 3, r8 = lane & 7;  // ldmatrix: this lane's matrix and row
    // S^T = K · Q^T: sc = S[key g][heads 2t, 2t+1], S[key g+8][heads 2t, 2t+1]
    float sc[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const int key = r8 + (mi & 1) * 8;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        uint32_t af[4];
        ldsm_x4(af, Kb + (key * U + ((ks * 2 + (mi >> 1)) ^ (key & (U - 1)))) * 8);
        mma_bf16(sc, af, qf[ks][0], qf[ks][1]);
      }
    }
    // online softmax per head over the group's 16 keys: a head's 16 scores sit in the 8 lanes
    // of equal t (2 rows each)
    float alpha[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float s0 = g < cur.nk ? sc[j] * scale_log2 : -INFINITY;
      const float s1 = g + 8 < cur.nk ? sc[j + 2] * scale_log2 : -INFINITY;
      float mx = fmaxf(s0, s1);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float m_new = fmaxf(m2[j], mx);
      const float p0 = exp2f(s0 - m_new), p1 = exp2f(s1 - m_new);
      float sum = p0 + p1;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      alpha[j] = m2[j] == -INFINITY ? 0.f : exp2f(m2[j] - m_new);
      l2[j] = l2[j] * alpha[j] + sum;
      m2[j] = m_new;
      pt[(2 * t + j) * kGrp + g] = __float2bfloat16_rn(p0);
      pt[(2 * t + j) * kGrp + g + 8] = __float2bfloat16_rn(p1);
    }
#pragma unroll
    for (int mt = 0; mt < KS; ++mt) {
      oc[mt][0] *= alpha[0];
      oc[mt][1] *= alpha[1];
      oc[mt][2] *= alpha[0];
      oc[mt][3] *= alpha[1];
    }
    __syncwarp();  // P^T visible
    const uint32_t pb0 = *reinterpret_cast<const uint32_t*>(pt + g * kGrp + 2 * t);
    const uint32_t pb1 = *reinterpret_cast<const uint32_t*>(pt + g * kGrp + 2 * t + 8);
    // O^T += V^T · P^T
    {
      const int key = r8 + (mi >> 1) * 8;
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        uint32_t af[4];
        ldsm_x4_t(af, Vb + (key * U + ((mt * 2 + (mi & 1)) ^ (key & (U - 1)))) * 8);
        mma_bf16(oc[mt], af, pb0, pb1);
      }
    }
    __syncwarp();  // the buffer and P^T are reused by the next group
#pragma unroll
    for (int s = 0; s < NS - 2; ++s) {
      pend[s] = pend[s + 1];
      hv[s] = hv[s + 1];
    }
    pend[NS - 2] = nxt;
    hv[NS - 2] = more;
  }
  // merge the four warps' partials (buffers reused: every warp is past its last cp.async)
  __syncthreads();
  float* om = reinterpret_cast<float*>(&S.kv[0][0][0]);  // [kWarps][G][D]
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int h = 2 * t + j;
    if (h < G) {
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        om[(w * G + h) * D + mt * 16 + g] = oc[mt][j];
        om[(w * G + h) * D + mt * 16 + g + 8] = oc[mt][j + 2];
      }
      if (g == 0) {
        S.ml[w][2 * h] = m2[j];
        S.ml[w][2 * h + 1] = l2[j];
      }
    }
  }
  __syncthreads();
  for (int f = tid; f < G * D; f += kThreads) {
    const int h = f / D, c = f % D;
    float M = -INFINITY;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) M = fmaxf(M, S.ml[ww][2 * h]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) {
      const float mw = S.ml[ww][2 * h];
      const float sc2 = mw == -INFINITY ? 0.f : exp2f(mw - M);
      L += S.ml[ww][2 * h + 1] * sc2;
      O += om[(ww * G + h) * D + c] * sc2;
    }
    const float v = L > 0.f ? O / L : 0.f;
    if (it.part >= 0)
      a.opart[(static_cast<int64_t>(it.part) * G + h) * D + c] = v;
    else
      store_out(static_cast<TO*>(a.o) + (static_cast<int64_t>(it.row) * a.hq + h0 + h) * D + c, v);
    if (c == 0) {
      const float lse = L > 0.f ? (M + log2f(L)) * 0.69314718055994531f : -INFINITY;
      if (it.part >= 0)
        a.lsepart[static_cast<int64_t>(it.part) * G + h] = lse;
      else if (a.lse != nullptr)
        a.lse[static_cast<int64_t>(it.row) * a.hq + h0 + h] = lse;
    }
  }
  if (it.part < 0) return;
  // split (row, kv head): the last of its chunks to finish merges every chunk's partial, in chunk
  // order (the same fixed-order LSE merge as K4, so the result does not depend on which CTA is
  // last), instead of a separate combine launch
  __shared__ int last;
  __threadfence();  // this chunk's partial is visible before its arrival is counted
  __syncthreads();
  if (tid == 0) {
    last = atomicAdd(a.done + it.pair, 1) == it.n_chunks - 1;
    if (last) a.done[it.pair] = 0;  // for the next step (no other chunk of this launch is left)
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // LSE weights of every chunk (per head) in shared memory, then one float4 of O per thread and
  // chunk, loads unrolled (the merge is latency-bound: n_chunks dependent reads otherwise)
  const int n = it.n_chunks;
  float* wts = reinterpret_cast<float*>(&S.kv[0][0][0]);  // [n][G] weights, then [G] M and L
  float* ML = wts + n * G;
  for (int i = tid; i < n * G; i += kThreads) wts[i] = __ldcg(a.lsepart + static_cast<int64_t>(it.part0) * G + i);
  __syncthreads();
  // M and L per head: warp w reduces heads w, w + 4, ... over the n chunks (lane-strided + shuffles)
  for (int h = w; h < G; h += kWarps) {
    float M = -INFINITY;
    for (int k = lane; k < n; k += 32) M = fmaxf(M, wts[k * G + h]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f;
    for (int k = lane; k < n; k += 32) {
      const float lk = wts[k * G + h];
      const float wk = lk == -INFINITY ? 0.f : __expf(lk - M);
      wts[k * G + h] = wk;
      L += wk;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (lane == 0) {
      ML[2 * h] = M;
      ML[2 * h + 1] = L;
    }
  }
  __syncthreads();
  for (int f4 = tid; f4 < G * D / 4; f4 += kThreads) {
    const int h = (f4 * 4) / D, c = (f4 * 4) % D;
    const float4* src = reinterpret_cast<const float4*>(a.opart + (static_cast<int64_t>(it.part0) * G + h) * D + c);
    const int64_t stride = static_cast<int64_t>(G) * D / 4;  // next chunk, same (head, columns)
    float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
    // batches of kMB predicated loads, all in flight before their FMAs: ceil(n / kMB) L2 round
    // trips (a runtime-n unrolled loop leaves a serial remainder of up to kMB - 1 dependent loads)
    constexpr int kMB = 16;
    for (int k0 = 0; k0 < n; k0 += kMB) {
      float4 v4[kMB];
#pragma unroll
      for (int j = 0; j < kMB; ++j) v4[j] = k0 + j < n ? __ldcg(src + (k0 + j) * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < kMB; ++j) {
        const float wk = k0 + j < n ? wts[(k0 + j) * G + h] : 0.f;
        acc4.x = fmaf(wk, v4[j].x, acc4.x);
        acc4.y = fmaf(wk, v4[j].y, acc4.y);
        acc4.z = fmaf(wk, v4[j].z, acc4.z);
        acc4.w = fmaf(wk, v4[j].w, acc4.w);
      }
    }
    const float inv = 1.f / ML[2 * h + 1];
    TO* dst = static_cast<TO*>(a.o) + (static_cast<int64_t>(it.row) * a.hq + h0 + h) * D + c;
    store_out(dst, acc4.x * inv);
    store_out(dst + 1, acc4.y * inv);
    store_out(dst + 2, acc4.z * inv);
    store_out(dst + 3, acc4.w * inv);
    if (c == 0 && a.lse != nullptr) a.lse[static_cast<int64_t>(it.row) * a.hq + h0 + h] = ML[2 * h] + logf(ML[2 * h + 1]);
  }
}

template <typename TO, int D, int G>
cudaError_t launch_bf16_g(const DecodeArgs& a, cudaStream_t st) {
  constexpr size_t smem = sizeof(DecSmem<D, G>);
  static_assert(sizeof(DecSmem<D, G>) <= 232448, "decode smem");
  static_assert(sizeof(DecSmem<D, G>) >= sizeof(float) * kWarps * G * D, "merge area");
  cudaError_t e = cudaFuncSetAttribute(decode_bf16_kernel<TO, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  decode_bf16_kernel<TO, D, G><<<a.n_items, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename T, typename TO, int D, int G>
cudaError_t launch_g(const DecodeArgs& a, cudaStream_t st) {
  constexpr int KP = D + 16 / static_cast<int>(sizeof(T));
  constexpr size_t smem = sizeof(T) * 2 * (kSub * KP + kSub * D) + sizeof(float) * (G * D + G * kSub + G * 3);
  static_assert(smem <= 232448, "decode smem");
  cudaError_t e = cudaFuncSetAttribute(decode_kernel<T, TO, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  decode_kernel<T, TO, D, G><<<a.n_items, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename T, typename TO, int D>
cudaError_t launch_d(const DecodeArgs& a, cudaStream_t st) {
  if constexpr (sizeof(T) == 2) {  // bf16 pools: the warp-split kernel
    switch (a.hq / a.hkv) {
      case 1: return launch_bf16_g<TO, D, 1>(a, st);
      case 2: return launch_bf16_g<TO, D, 2>(a, st);
      case 4: return launch_bf16_g<TO, D, 4>(a, st);
      case 8: return launch_bf16_g<TO, D, 8>(a, st);
      default: return cudaErrorInvalidValue;
    }
  }
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
