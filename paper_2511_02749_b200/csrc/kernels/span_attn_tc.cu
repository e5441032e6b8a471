// span_attn_tc.cu — K2/K3: span-masked flash attention over the paged KV pool on sm_100a
// tensor cores (SURVEY §8(a) a6 fragment/prefix prefill and a7 join).
//
// Semantics (work.h): for each (work item, q head) — up to 128 query rows — stream the item's
// KV tiles; q of row r is rotated to pos[r] - rot_delta of the tile's segment (fragment KV is
// cached at span-local positions and never touched: the join counter-rotates Q by Δ_f instead,
// "ReRoPE" P:610 done on the query side), keys are masked by n_valid and, in causal tiles,
// key_pos0 + t > pos[r] (block-diagonal fragment attention). O, LSE are written final
// (bf16, natural log) or as fp32 split-KV partials merged by combine.cu.
//
// B200 design (one persistent CTA per SM, 384 threads, ~193 KB smem, 512 TMEM columns):
//   warp 0      TMA producer: K and V tiles of 128 keys = 128/bs pool blocks, SWIZZLE_128B boxes
//               {64 cols, bs rows} from one 2D tensor map over the whole pool (block id -> row);
//               2-stage ring, separate K/V full/empty mbarriers.
//   warp 1      MMA issuer (one thread): S = Q K^T (kind::f16 SS, M=N=128, fp32 in TMEM,
//               double-buffered S at cols 0/128), then O += P V with P read from TMEM (TS form,
//               bf16 P aliased over its S columns) and V as an MN-major smem operand; order
//               S_j, PV_{j-1}, S_{j+1}, ... so softmax of tile j overlaps both MMAs.
//   warps 4-7   softmax/epilogue (thread = row, TMEM lane = row): two TMEM passes (max, then
//               exp2 + pack + tcgen05.st of P), conditional O rescale only when the running
//               max grows by > 8 (log2 units) — P stays <= 256, exact after normalisation —
//               then the epilogue (tcgen05.ld O, 1/l, store).
//   warps 8-11  Q prep: load pre-RoPE q rows, rotate (fp64-built cos/sin table), write the
//               SWIZZLE_128B K-major Q tile, double-buffered, re-done when rot_delta changes.
// Descriptor bit layouts and the TS / MN-major operand forms were validated on the B200 by
// tools/tc_probe.cu before use.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cmath>

#include "launch.h"
#include "sm100.cuh"

namespace spq {
namespace {

constexpr int kThreads = 384;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS0 = 0, kColO = 256;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

template <int D>
struct TcSmem {
  static constexpr int kChunks = D / 64;
  static constexpr int kChunkBytes = 128 * 128;  // 128 rows x 128 B
  alignas(1024) uint8_t q[2][kChunks][kChunkBytes];
  alignas(1024) uint8_t k[2][kChunks][kChunkBytes];
  alignas(1024) uint8_t v[2][kChunks][kChunkBytes];
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2], p_full[2], q_full[2], q_empty[2], o_done;
  uint32_t tmem_base;
};

struct TcParams {
  CUtensorMap tmk;
  CUtensorMap tmv;
  AttnArgs a;
  float scale_log2;
};

template <int D>
__device__ __forceinline__ TcSmem<D>& smem_ref(uint8_t* raw) {
  return *reinterpret_cast<TcSmem<D>*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
}

// ------------------------------------------------------------------ warp 0: TMA producer
template <int D>
__device__ void run_producer(const TcParams& P, TcSmem<D>& S, int it_begin, int it_end) {
  const AttnArgs& a = P.a;
  const int group = a.hq / a.hkv;
  const int bpt = kTileKeys / a.bs;
  constexpr uint32_t kStageBytes = 128 * D * 2;
  const int64_t layer_rows = static_cast<int64_t>(a.layer) * a.nblk * a.hkv * a.bs;
  uint32_t kt = 0;
  for (int ii = it_begin; ii < it_end; ++ii) {
    const int code = a.cta_items[ii];
    const WorkItem w = a.items[code / a.hq];
    const int kvh = (code % a.hq) / group;
    for (int t = w.tile_begin; t < w.tile_end; ++t, ++kt) {
      const int stage = kt & 1;
      const uint32_t ph = (kt >> 1) & 1;
      const int32_t boff = a.tiles[t].blk_off;
      mbar_wait(&S.k_empty[stage], ph ^ 1);
      mbar_arrive_expect_tx(&S.k_full[stage], kStageBytes);
      for (int j = 0; j < bpt; ++j) {
        const int32_t y = static_cast<int32_t>(
            layer_rows + (static_cast<int64_t>(a.tile_blocks[boff + j]) * a.hkv + kvh) * a.bs);
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          tma_load_2d(&S.k[stage][c][j * a.bs * 128], &P.tmk, &S.k_full[stage], c * 64, y);
      }
      mbar_wait(&S.v_empty[stage], ph ^ 1);
      mbar_arrive_expect_tx(&S.v_full[stage], kStageBytes);
      for (int j = 0; j < bpt; ++j) {
        const int32_t y = static_cast<int32_t>(
            layer_rows + (static_cast<int64_t>(a.tile_blocks[boff + j]) * a.hkv + kvh) * a.bs);
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          tma_load_2d(&S.v[stage][c][j * a.bs * 128], &P.tmv, &S.v_full[stage], c * 64, y);
      }
    }
  }
}

// ------------------------------------------------------------------ warp 1: MMA issuer
template <int D>
__device__ void run_mma(const TcParams& P, TcSmem<D>& S, uint32_t tmem, int it_begin, int it_end) {
  const AttnArgs& a = P.a;
  constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false);
  constexpr uint32_t idO = idesc_bf16_f32(128, D, false, true);
  uint32_t kt = 0, st = 0, qs = 0;
  struct Pend {
    int stage, sb;
    uint32_t kt, st;
    bool first;
  };
  auto issue_pv = [&](const Pend& p) {
    mbar_wait(&S.p_full[p.sb], (p.st >> 1) & 1);
    mbar_wait(&S.v_full[p.stage], (p.kt >> 1) & 1);
    tc_fence_after();
    const uint32_t vbase = smem_u32(&S.v[p.stage][0][0]);
#pragma unroll
    for (int kk = 0; kk < kTileKeys / 16; ++kk) {
      const uint64_t vd = desc_sw128(vbase + kk * 2048, 16384, 1024);
      mma_ts(tmem + kColO, tmem + kColS0 + p.sb * 128 + kk * 8, vd, idO, (!p.first || kk > 0) ? 1u : 0u);
    }
    mma_commit(&S.v_empty[p.stage]);
    mma_commit(&S.o_done);
  };
  for (int ii = it_begin; ii < it_end; ++ii) {
    const int code = a.cta_items[ii];
    const WorkItem w = a.items[code / a.hq];
    int qb = 0;
    Pend prev{0, 0, 0, 0, true};
    for (int t = w.tile_begin; t < w.tile_end; ++t) {
      const int k = t - w.tile_begin;
      if (k == 0 || a.tiles[t].rot_delta != a.tiles[t - 1].rot_delta) {
        if (k > 0) mma_commit(&S.q_empty[qb]);
        qb = qs & 1;
        mbar_wait(&S.q_full[qb], (qs >> 1) & 1);
        ++qs;
      }
      const int stage = kt & 1, sb = st & 1;
      mbar_wait(&S.k_full[stage], (kt >> 1) & 1);
      tc_fence_after();
      const uint32_t qbase = smem_u32(&S.q[qb][0][0]);
      const uint32_t kbase = smem_u32(&S.k[stage][0][0]);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off = (kk / 4) * TcSmem<D>::kChunkBytes + (kk % 4) * 32;
        mma_ss(tmem + kColS0 + sb * 128, desc_sw128(qbase + off, 16, 1024),
               desc_sw128(kbase + off, 16, 1024), idS, kk > 0 ? 1u : 0u);
      }
      mma_commit(&S.k_empty[stage]);
      mma_commit(&S.s_full[sb]);
      if (k > 0) issue_pv(prev);
      prev = Pend{stage, sb, kt, st, k == 0};
      ++kt;
      ++st;
    }
    issue_pv(prev);
    mma_commit(&S.q_empty[qb]);
  }
}

// ------------------------------------------------------------------ warps 4-7: softmax + epilogue
template <int D>
__device__ void run_softmax(const TcParams& P, TcSmem<D>& S, uint32_t tmem, int it_begin, int it_end) {
  const AttnArgs& a = P.a;
  const int r = threadIdx.x - 128;  // row within the tile == TMEM lane
  const uint32_t lane_base = static_cast<uint32_t>((r / 32) * 32) << 16;
  const float sl2 = P.scale_log2;
  uint32_t st = 0, pvw = 0;
  for (int ii = it_begin; ii < it_end; ++ii) {
    const int code = a.cta_items[ii];
    const int h = code % a.hq;
    const WorkItem w = a.items[code / a.hq];
    const bool valid = r < w.n_rows;
    const int64_t row = static_cast<int64_t>(w.row0) + r;
    const int p = valid ? a.pos[row] : 0;
    float m = -INFINITY, l = 0.f;
    for (int t = w.tile_begin; t < w.tile_end; ++t) {
      const int k = t - w.tile_begin;
      const KvTile tl = a.tiles[t];
      const int lim = min(tl.n_valid - 1, tl.causal ? p - tl.key_pos0 : kTileKeys - 1);
      const int sb = st & 1;
      const uint32_t scol = tmem + lane_base + kColS0 + sb * 128;
      mbar_wait(&S.s_full[sb], (st >> 1) & 1);
      tc_fence_after();
      // pass 1: row max — 8 independent accumulators (no 128-long dependency chain); the
      // per-key mask is only evaluated when some row of the warp sees a partial tile
      const bool full = __all_sync(0xffffffffu, lim >= kTileKeys - 1);
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(scol + c * 32, v);
        tmem_wait_ld();
        if (full) {
#pragma unroll
          for (int i = 0; i < 32; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], __uint_as_float(v[i]));
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i <= lim) mx8[i & 7] = fmaxf(mx8[i & 7], __uint_as_float(v[i]));
        }
      }
      float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      mx *= sl2;
      const float m_new = fmaxf(m, mx);
      const bool resc = m_new > m + kRescaleThreshold;
      const float m_use = resc ? m_new : m;
      const float alpha = resc ? ex2_approx(m - m_new) : 1.f;
      const float msub = (m_use == -INFINITY) ? 0.f : m_use;
      // pass 2: P = exp2(s*scale - m), packed bf16 over the first 64 columns of S
      float sum8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) sum8[i] = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(scol + c * 32, v);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j0 = c * 32 + 2 * i;
          float p0 = ex2_approx(fmaf(__uint_as_float(v[2 * i]), sl2, -msub));
          float p1 = ex2_approx(fmaf(__uint_as_float(v[2 * i + 1]), sl2, -msub));
          if (!full) {
            p0 = (j0 <= lim) ? p0 : 0.f;
            p1 = (j0 + 1 <= lim) ? p1 : 0.f;
          }
          sum8[(2 * i) & 7] += p0;
          sum8[(2 * i + 1) & 7] += p1;
          pk[i] = pack_bf16x2(p0, p1);
        }
        tmem_st16(scol + c * 16, pk);
      }
      const float sum = ((sum8[0] + sum8[1]) + (sum8[2] + sum8[3])) + ((sum8[4] + sum8[5]) + (sum8[6] + sum8[7]));
      tmem_wait_st();
      l = l * alpha + sum;
      if (k > 0) {
        mbar_wait(&S.o_done, pvw & 1);  // PV of the previous tile has landed in O
        ++pvw;
        tc_fence_after();
        if (__any_sync(0xffffffffu, resc)) {
          const uint32_t ocol = tmem + lane_base + kColO;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t v[32];
            tmem_ld32(ocol + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st32(ocol + c * 32, v);
          }
          tmem_wait_st();
        }
      }
      m = m_use;
      tc_fence_before();
      mbar_arrive(&S.p_full[sb]);
      ++st;
    }
    // epilogue: wait for the last PV, normalize, store
    mbar_wait(&S.o_done, pvw & 1);
    ++pvw;
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const float lse = l > 0.f ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
    const uint32_t ocol = tmem + lane_base + kColO;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(ocol + c * 32, v);
      tmem_wait_ld();
      if (valid) {
        if (w.part < 0 && a.out_fp32) {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.o) + (row * a.hq + h) * D + c * 32);
#pragma unroll
          for (int u = 0; u < 8; ++u)
            dst[u] = make_float4(__uint_as_float(v[4 * u]) * inv, __uint_as_float(v[4 * u + 1]) * inv,
                                 __uint_as_float(v[4 * u + 2]) * inv, __uint_as_float(v[4 * u + 3]) * inv);
        } else if (w.part < 0) {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.o) +
                                                (row * a.hq + h) * D + c * 32);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint4 pk;
            pk.x = pack_bf16x2(__uint_as_float(v[8 * u + 0]) * inv, __uint_as_float(v[8 * u + 1]) * inv);
            pk.y = pack_bf16x2(__uint_as_float(v[8 * u + 2]) * inv, __uint_as_float(v[8 * u + 3]) * inv);
            pk.z = pack_bf16x2(__uint_as_float(v[8 * u + 4]) * inv, __uint_as_float(v[8 * u + 5]) * inv);
            pk.w = pack_bf16x2(__uint_as_float(v[8 * u + 6]) * inv, __uint_as_float(v[8 * u + 7]) * inv);
            dst[u] = pk;
          }
        } else {
          float4* dst = reinterpret_cast<float4*>(
              a.opart + ((static_cast<int64_t>(w.part) * a.hq + h) * kTileRows + r) * D + c * 32);
#pragma unroll
          for (int u = 0; u < 8; ++u)
            dst[u] = make_float4(__uint_as_float(v[4 * u]) * inv, __uint_as_float(v[4 * u + 1]) * inv,
                                 __uint_as_float(v[4 * u + 2]) * inv, __uint_as_float(v[4 * u + 3]) * inv);
        }
      }
    }
    if (valid) {
      if (w.part < 0) {
        if (a.lse != nullptr) a.lse[row * a.hq + h] = lse;
      } else {
        a.lsepart[(static_cast<int64_t>(w.part) * a.hq + h) * kTileRows + r] = lse;
      }
    }
    tc_fence_before();
  }
}

// ------------------------------------------------------------------ warps 8-11: Q prep
template <int D>
__device__ void run_qprep(const TcParams& P, TcSmem<D>& S, int it_begin, int it_end) {
  const AttnArgs& a = P.a;
  const int r = threadIdx.x - 256;
  const __nv_bfloat16* qg = static_cast<const __nv_bfloat16*>(a.q);
  uint32_t qs = 0;
  for (int ii = it_begin; ii < it_end; ++ii) {
    const int code = a.cta_items[ii];
    const int h = code % a.hq;
    const WorkItem w = a.items[code / a.hq];
    const bool valid = r < w.n_rows;
    const int64_t row = static_cast<int64_t>(w.row0) + r;
    const int p = valid ? a.pos[row] : 0;
    const __nv_bfloat16* qrow = qg + (row * a.hq + h) * D;
    for (int t = w.tile_begin; t < w.tile_end; ++t) {
      const int k = t - w.tile_begin;
      const int rot = a.tiles[t].rot_delta;
      if (k > 0 && rot == a.tiles[t - 1].rot_delta) continue;
      const int qb = qs & 1;
      mbar_wait(&S.q_empty[qb], ((qs >> 1) & 1) ^ 1);
      uint8_t* qs_base = &S.q[qb][0][0];
      const int rp = min(max(p - rot, 0), a.max_pos - 1);
      const float4* cs = reinterpret_cast<const float4*>(a.rope + static_cast<int64_t>(rp) * (D / 2));
      // issue every q load of the row first (latency is paid once), then the cos/sin table in
      // batches of 8 pairs interleaved with the rotate + swizzled stores
      uint4 q1[D / 16], q2[D / 16];
#pragma unroll
      for (int g = 0; g < D / 16; ++g) {
        q1[g] = valid ? __ldg(reinterpret_cast<const uint4*>(qrow + g * 8)) : make_uint4(0, 0, 0, 0);
        q2[g] = valid ? __ldg(reinterpret_cast<const uint4*>(qrow + D / 2 + g * 8)) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int g0 = 0; g0 < D / 16; g0 += 2) {
        float4 cst[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) cst[e] = valid ? __ldg(cs + g0 * 4 + e) : make_float4(1.f, 0.f, 1.f, 0.f);
#pragma unroll
        for (int gg = 0; gg < 2; ++gg) {
          const int g = g0 + gg;
          const int i0 = g * 8;
          uint4 o1, o2;
          const __nv_bfloat162* b1 = reinterpret_cast<const __nv_bfloat162*>(&q1[g]);
          const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&q2[g]);
          uint32_t* w1 = reinterpret_cast<uint32_t*>(&o1);
          uint32_t* w2 = reinterpret_cast<uint32_t*>(&o2);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float4 c = cst[gg * 4 + e];  // (cos,sin) of pairs i0+2e, i0+2e+1
            const float2 x1 = __bfloat1622float2(b1[e]), x2 = __bfloat1622float2(b2[e]);
            w1[e] = pack_bf16x2(x1.x * c.x - x2.x * c.y, x1.y * c.z - x2.y * c.w);
            w2[e] = pack_bf16x2(x2.x * c.x + x1.x * c.y, x2.y * c.z + x1.y * c.w);
          }
          const int e1 = i0, e2 = D / 2 + i0;
          *reinterpret_cast<uint4*>(qs_base + (e1 / 64) * TcSmem<D>::kChunkBytes + r * 128 +
                                    ((((e1 % 64) / 8) ^ (r & 7)) * 16)) = o1;
          *reinterpret_cast<uint4*>(qs_base + (e2 / 64) * TcSmem<D>::kChunkBytes + r * 128 +
                                    ((((e2 % 64) / 8) ^ (r & 7)) * 16)) = o2;
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&S.q_full[qb]);
      ++qs;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) span_attn_tc_kernel(const __grid_constant__ TcParams P) {
  extern __shared__ uint8_t smem_raw[];
  TcSmem<D>& S = smem_ref<D>(smem_raw);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.k_full[i], 1);
      mbar_init(&S.k_empty[i], 1);
      mbar_init(&S.v_full[i], 1);
      mbar_init(&S.v_empty[i], 1);
      mbar_init(&S.s_full[i], 1);
      mbar_init(&S.p_full[i], 128);
      mbar_init(&S.q_full[i], 128);
      mbar_init(&S.q_empty[i], 1);
    }
    mbar_init(&S.o_done, 1);
    fence_barrier_init();
  }
  if (warp == 0 && (threadIdx.x & 31) == 0) {
    tma_prefetch_desc(&P.tmk);
    tma_prefetch_desc(&P.tmv);
  }
  if (warp == 2) tmem_alloc<kTmemCols>(&S.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  const int it_begin = P.a.cta_off[blockIdx.x], it_end = P.a.cta_off[blockIdx.x + 1];
  if (warp == 0) {
    if (elect_one()) run_producer<D>(P, S, it_begin, it_end);
  } else if (warp == 1) {
    if (elect_one()) run_mma<D>(P, S, tmem, it_begin, it_end);
  } else if (warp >= 4 && warp < 8) {
    run_softmax<D>(P, S, tmem, it_begin, it_end);
  } else if (warp >= 8) {
    run_qprep<D>(P, S, it_begin, it_end);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

template <int D>
cudaError_t launch_d(const AttnArgs& a, cudaStream_t st) {
  static bool attr_set = false;
  const int smem = static_cast<int>(sizeof(TcSmem<D>)) + 1024;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(span_attn_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  TcParams p;
  p.tmk = *a.tmap_k;
  p.tmv = *a.tmap_v;
  p.a = a;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  span_attn_tc_kernel<D><<<a.grid, kThreads, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_span_attn_tc(const AttnArgs& a, cudaStream_t st) {
  if (a.n_items == 0 || a.grid == 0) return cudaSuccess;
  if (a.bs < 16 || a.bs > 128 || (a.bs & (a.bs - 1)) != 0) return cudaErrorInvalidValue;
  switch (a.d) {
    case 64: return launch_d<64>(a, st);
    case 128: return launch_d<128>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace spq
