// span_attn_tc.cu — K2/K3: span-masked flash attention over the paged KV pool on sm_100a
// tensor cores (SURVEY §8(a) a6 fragment/prefix prefill and a7 join).
//
// Semantics (work.h): for each work unit — up to 128 query rows x one q head (or the two q
// heads of a GQA pair) — stream the item's KV tiles; q of row r is rotated to pos[r] - rot_delta
// of the tile's segment (fragment KV is cached at span-local positions and never touched: the
// join counter-rotates Q by Δ_f instead, "ReRoPE" P:610 done on the query side), keys are
// masked by n_valid and, in causal tiles, key_pos0 + t > pos[r] (block-diagonal fragment
// attention). O, LSE are written final or as fp32 split-KV partials (combine.cu).
//
// B200 design — one persistent CTA per SM, 512 threads, ~225 KB smem, 512 TMEM columns
// (DESIGN.md §6 has the measurements behind each choice):
//   * the two q heads h, h+1 of a GQA group share every K/V tile, so one CTA runs them as two
//     M=128 Q tiles (A, B) against the same TMA-loaded K/V (half the K/V traffic per FLOP), with
//     one MMA-issuing thread per head (warps 1 / 2) so each head's chain runs at its own pace.
//   * work is streamed in 64-key sub-tiles. TMEM: S_A [0,128) S_B [128,256) as two 64-column S
//     buffers per head, O_A [256,384) O_B [384,512) (fp32). P (bf16) is written over the first
//     32 columns of its S buffer and consumed by the TS-form MMA (A from TMEM). Per head the
//     issuer runs S(0), S(1), then PV(j), S(j+2), ...: softmax(j+1) never waits for PV(j).
//   * K/V: two TMA rings of 64-key sub-tiles (K 3 slots, V 3 at d=128; 8 / 4 at d=64), each with
//     its own producer warp (0 / 3), SWIZZLE_128B boxes {64 cols, min(bs, 64) rows} from one 2D
//     tensor map over the whole pool (block id -> row): the paged gather is done by TMA.
//   * work: prefill codes are claimed at run time (atomic counter, smem ring shared by all
//     roles, longest-first order); joins use a static stream-K cut with fp32 partials (combine.cu).
//   * Q: slot x = head x, prepared by warps 12-15 (TMA load of the pre-RoPE tile, in-place
//     rotate-half with the fp64-built fp32 table and an fp32 angle recurrence, packed fp32x2);
//     an epoch (an item or a change of rot_delta) reloads it once its last S MMA has completed.
//     Joins (an epoch per fragment segment) keep a 2-deep ring per head whose second slot is the
//     staging area, so the next fragment's Q is ready a whole epoch ahead.
//   * softmax (warps 4-7 head A, 8-11 head B; thread = row = TMEM lane): one pass per sub-tile
//     (LDTM.x64, FMNMX3 row max, exp2 on MUFU, packed FFMA2/FADD2, STTM.x32); O rescaled only
//     when the running max grows by > 8 (log2), so P <= 256; then the epilogue (TMEM -> swizzled
//     smem staging -> TMA bulk store, or fp32 split partials).
// Descriptor bit layouts and the TS / MN-major operand forms were validated on the B200 by
// tools/tc_probe.cu before use.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <climits>
#include <cmath>
#include <cstdlib>

#include "launch.h"
#include "sm100.cuh"

namespace spq {
namespace {

constexpr int kThreads = 512;
constexpr uint32_t kTmemCols = 512;
// TMEM columns of head x. Default: one S buffer per head [256x, +64), two P buffers (bf16, 32
// columns each) [256x + 64, +64), O [256x + 128, +128). The softmax releases S(j) as soon as its
// LDTM has landed, so S(j+1) is computed while softmax(j) runs and the chain per head is
// S(j) -> softmax load -> S(j+1), no longer S(j) -> softmax -> PV(j) -> S(j+2).
// SPANQ_S2 (A/B build): two S buffers per head with P written over its S buffer, O at 256 + 128x.
#ifdef SPANQ_S2
constexpr bool kSP = false;
#else
constexpr bool kSP = true;
#endif
#ifndef SPANQ_PP
#define SPANQ_PP 0
#endif
constexpr bool kPingPong = SPANQ_PP != 0;  // A/B build: -DSPANQ_PP=1 (measured slower: a WG alone
                                           // needs ~780 cycles per sub-tile, both together ~1150-1300)
__host__ __device__ constexpr uint32_t col_s(int x, int buf) {
  return kSP ? 256u * x : 128u * x + 64u * buf;
}
__host__ __device__ constexpr uint32_t col_p(int x, int buf) {
  return kSP ? 256u * x + 64u + 32u * buf : 128u * x + 64u * buf;
}
__host__ __device__ constexpr uint32_t col_o(int x) { return kSP ? 256u * x + 128u : 256u + 128u * x; }

template <int D, bool PR = false>
struct TcSmem {
  static constexpr int kChunks = D / 64;
  static constexpr int kChunkBytes = 128 * 128;  // Q: 128 rows x 128 B per 64-column chunk
  static constexpr int kSubBytes = 64 * 128;     // K/V: 64 keys x 128 B per 64-column chunk
  // CTA pair (PR): each CTA holds half of every K sub-tile (32 of its 64 keys, all d columns)
  // and half of every V sub-tile (all 64 keys, its 64 of the d columns), so the rings are twice
  // as deep in the same bytes
  static constexpr int kKChunkBytes = (PR ? 32 : 64) * 128;
  static constexpr int kVChunks = PR ? 1 : kChunks;
  // K(j+2) is needed one step after its slot frees (S(j+2) right after PV(j)), V(j) two steps
  // later. d=128: 3 + 3 slots measured faster than 4 + 2 (A/B on one GPU: prefill 0.248 ->
  // 0.245 ms, join 0.095 -> 0.093 ms) — the V producer no longer stalls the K stream's release
  static constexpr int kKSlots = PR ? 7 : (D == 64 ? 8 : 3);
  static constexpr int kVSlots = PR ? 5 : (D == 64 ? 4 : 3);
  static_assert(kVSlots <= kKSlots, "V uses the first kVSlots of the [K, V][kKSlots] barriers");
  static constexpr int kQSlots = 2;  // slot x = head x (the next epoch's tile is loaded after
                                     // this epoch's last S MMA: ~2 steps before the item ends)
  alignas(1024) uint8_t q[kQSlots][kChunks][kChunkBytes];
  alignas(1024) uint8_t k[kKSlots][kChunks][kKChunkBytes];  // ring of 64-key K sub-tiles
  alignas(1024) uint8_t v[kVSlots][kVChunks][kSubBytes];    // ring of 64-key V sub-tiles
  // prefill: epilogue transpose, 2 x 4 KB per softmax warp. join: the second Q slot of each
  // head (q2), so the next fragment's counter-rotated Q is prepared a whole epoch ahead; the
  // join epilogue stages in the Q slot of its item's last epoch instead
  alignas(1024) float stage[8][2][32 * 32];
  uint64_t kv_full[2][kKSlots], kv_empty[2][kKSlots];  // [K, V][slot] (V uses the first kVSlots)
  uint64_t q_full[2][2], q_empty[2][2], q_load[2][2];  // [head][Q ring slot]
  __device__ uint8_t* q2(int x) { return reinterpret_cast<uint8_t*>(&stage[0][0][0]) + x * kChunks * kChunkBytes; }
  uint64_t s_full[2][2], p_full[2][2], o_done[2][2];  // [head][S buffer / PV parity j & 1]
  uint64_t s_free[2][2];  // [head][j & 1]: softmax(j) has loaded S(j) (kSP: S(j+1) may overwrite it)
  // prefill: the epilogue runs on the Q-prep warps (12-15). The softmax WG of head x hands over
  // 1/l of every row through fin_inv[x][item & 1] (fin_full: 128 arrivals), the epilogue warps
  // drain O_x from TMEM into the staging area and arrive o_free[x] (128 threads), which the issuer
  // waits for before the next item's first PV overwrites O_x
  uint64_t o_free[2], fin_full[2][2];
  float fin_inv[2][2][128];
  static constexpr int kSched = 4;  // dynamic schedule: ring of claimed codes
  uint64_t sched_full[kSched], sched_empty[kSched];
  int32_t sched_code[kSched];
  uint32_t tmem_base;
  // ping-pong: a word that is always 0 (read after the barrier: the exponentials depend on it) and a
  // sink the row sums are stored to before the hand-over (the stores cannot sink below it)
  float pp_zero, pp_sink;
};

struct TcParams {
  CUtensorMap tmk;
  CUtensorMap tmk2;  // CTA pair: K boxes of min(bs, 32) rows (each CTA loads 32 keys per sub-tile)
  CUtensorMap tmv;
  CUtensorMap tmq;
  CUtensorMap tmo;   // fp32 O (valid when a.out_fp32)
  CUtensorMap tmop;  // fp32 partials (valid when the launch has split items)
  AttnArgs a;
  float scale_log2;
  int paired;     // 1: a unit is a GQA head pair (A = 2u, B = 2u+1); 0: one head (B idle)
  int poly_mask;  // pair i of a 32-key chunk uses the FMA-pipe exp2 when (i & 3) < poly_mask
  float rescale_threshold;  // log2 units; O is rescaled when the running max grows by more
  int qprep_mode;  // Q prep: bit 0 = issue head B's load early, bit 1 = L2-prefetch the next item's q
  int join;        // 1: 2-deep Q ring per head in the staging area, epilogue staged in Q slots
  int epi_q;       // 1 (prefill launches): the epilogue runs on the Q-prep warps (prefill_epilogue)
  int dbg_mode;  // profiling builds only: 1 = softmax does no math, 2 = max pass only,
                 // 3 = 1 + K/V always from the first block (L2-resident), 4 = 1 + MMA skips K/V waits,
                 // 5 = 1 + Q prep does no work
};

// The dynamic shared memory window starts 1024-byte aligned when a kernel has no static shared
// memory (SWIZZLE_128B operands need it); the launch requests exactly sizeof(TcSmem) (d=128 uses
// the whole 227 KB), so a misaligned base would be a fatal configuration error: trap loudly.
template <int D, bool PR>
__device__ __forceinline__ TcSmem<D, PR>& smem_ref(uint8_t* raw) {
  if (smem_u32(raw) & 1023u) __trap();
  return *reinterpret_cast<TcSmem<D, PR>*>(raw);
}

// Q ring of head x: epoch e uses slot e % depth (depth 1 for prefill, 2 for joins), its
// (e / depth)-th use
// (J = P.join: a runtime flag, so prefill and join launches run the same kernel binary — two
// binaries alternating per layer measured ~2% slower, their code evicting each other's)
__device__ __forceinline__ int q_slot(bool J, uint32_t e) {
  return J ? static_cast<int>(e & 1) : 0;
}
__device__ __forceinline__ uint32_t q_par(bool J, uint32_t e) {
  return (J ? e >> 1 : e) & 1;
}
template <int D, bool PR>
__device__ __forceinline__ uint8_t* q_tile(TcSmem<D, PR>& S, bool J, int x, uint32_t e) {
  return q_slot(J, e) ? S.q2(x) : &S.q[x][0][0];
}

// profiling only: CTA 0 records (event, clock) pairs per warp (lane 0 / the elected thread);
// 1024 events per warp
constexpr int kTraceWarps = 16;
// (profiling builds only: -DSPANQ_PROFILING, tools/; compiled out of the product library)
__device__ __forceinline__ void trace(const TcParams& P, int, uint32_t& cnt, int ev) {
#ifdef SPANQ_PROFILING
  // (mode bits 8+: the CTA to record, default 0)
  if (P.a.dbg_trace == nullptr || blockIdx.x != static_cast<unsigned>(P.dbg_mode >> 8) || cnt >= 1024) return;
  long long* t = P.a.dbg_trace + ((threadIdx.x / 32) * 1024 + cnt) * 2;
  t[0] = ev;
  t[1] = clock64();
  ++cnt;
#endif
}
// profiling builds: timing variants of the kernel (spq_set_trace); 0 in the product library
__device__ __forceinline__ int dbg_mode(const TcParams& P) {
#ifdef SPANQ_PROFILING
  return P.dbg_mode & 255;
#else
  return 0;
#endif
}

struct Unit {
  WorkItem w;
  int head_a, n_heads;
};

// CTA pair (PR): a unit is the 4 q heads 4x .. 4x+3 of a GQA group (one K/V stream); CTA rank r of
// the pair runs heads 4x + 2r and 4x + 2r + 1 as its A / B tiles
template <bool PR>
__device__ __forceinline__ Unit decode(const TcParams& P, int code) {
  Unit u;
  const int units = PR ? P.a.hq / 4 : (P.paired ? P.a.hq / 2 : P.a.hq);
  u.w = P.a.items[code / units];
  const int x = code % units;
  if constexpr (PR) {
    u.head_a = 4 * x + 2 * static_cast<int>(cluster_rank());
    u.n_heads = 2;
  } else {
    u.head_a = P.paired ? 2 * x : x;
    u.n_heads = P.paired ? 2 : 1;
  }
  return u;
}

// Barriers that only the leader CTA of a pair waits on (its MMA issuers / claimer) but that both
// CTAs arrive on: arrivals go to the leader's copy (cluster scope), waits acquire at cluster scope.
// Outside a pair these are the plain CTA-local forms.
template <bool PR>
__device__ __forceinline__ void arrive_lead(uint64_t* bar) {
  if constexpr (PR)
    mbar_arrive_cl(cluster_addr(bar, 0));
  else
    mbar_arrive(bar);
}
// Warp-wide form (all 32 lanes call it, converged): a pair sends ONE remote arrival per warp
// (after __syncwarp, which orders the lanes' earlier accesses before lane 0's release) — 32
// cluster-scope arrivals per warp cost DSMEM round trips on the step's critical path; the leader
// barrier then counts warps (kLeadUnit = 1 per warp), a single CTA keeps one arrival per thread
template <bool PR>
__device__ __forceinline__ void arrive_lead_warp(uint64_t* bar) {
  if constexpr (PR) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive_cl(cluster_addr(bar, 0));
  } else {
    mbar_arrive(bar);
  }
}
// Waits of the single-thread roles (TMA producers, MMA issuers). SPANQ_ISSWAIT (A/B builds): 0 =
// try_wait with the suspend-time hint, 1 = test_wait poll, 2 = try_wait without a hint
#ifndef SPANQ_ISSWAIT
#define SPANQ_ISSWAIT 0
#endif
__device__ __forceinline__ void mbar_wait_1t(uint64_t* bar, uint32_t parity) {
#if SPANQ_ISSWAIT == 1
  while (!mbar_test_wait(bar, parity)) {
  }
#elif SPANQ_ISSWAIT == 2
  while (!mbar_try_wait(bar, parity)) {
  }
#else
  mbar_wait(bar, parity);
#endif
}
// The softmax hand-overs on the MMA issuer's critical path (S loaded, P written): one arrival per
// warp (after __syncwarp) instead of 128 per-thread arrivals (SPANQ_WARPARRIVE=1, A/B build: no measurable gain, and
// compute-sanitizer racecheck does not credit the __syncwarp ordering)
#ifndef SPANQ_WARPARRIVE
#define SPANQ_WARPARRIVE 0
#endif
template <bool PR>
__device__ __forceinline__ void arrive_hand(uint64_t* bar) {
  if constexpr (PR || SPANQ_WARPARRIVE) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      if constexpr (PR)
        mbar_arrive_cl(cluster_addr(bar, 0));
      else
        mbar_arrive(bar);
    }
  } else {
    mbar_arrive(bar);
  }
}
__host__ __device__ constexpr uint32_t kHandCount(bool pr) { return (pr ? 8u : (SPANQ_WARPARRIVE ? 4u : 128u)); }
template <bool PR>
__device__ __forceinline__ void wait_lead(uint64_t* bar, uint32_t parity) {
  if constexpr (PR)
    mbar_wait_cl(bar, parity);
  else
    mbar_wait_1t(bar, parity);
}
// spin (no suspend-time hint) — A/B of the wake-up latency on the step's critical path
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// MMA completion: in a pair the commit arrives on the barrier of both CTAs
template <bool PR>
__device__ __forceinline__ void commit_x(uint64_t* bar) {
  if constexpr (PR)
    mma_commit2(bar);
  else
    mma_commit(bar);
}

// The CTA's sequence of work codes. Static: its slice of cta_items. Dynamic: the K producer
// claims codes from the launch's counter (atomicAdd) and hands them to the other roles through a
// smem ring; every role sees the same sequence, ending with -1.
constexpr int kSchedConsumers = 1 + 2 + 256 + 128;  // V producer, 2 MMA issuers, softmax, Q prep
// CTA pair: the leader's ring entry is free once the leader's consumers and the peer's (K and V
// producers, softmax, Q prep; its MMA warps idle) have read it
// (arrivals: one per producer / issuer thread, one per softmax / Q-prep warp)
constexpr int kSchedConsumersPair = (1 + 2 + 8 + 4) + (1 + 1 + 8 + 4);
template <int D, bool EPI, bool PR>
struct ItemSrc {
  const TcParams& P;
  TcSmem<D, PR>& S;
  int it, end;
  bool claimer;
  bool warp_wide;  // the caller is a whole converged warp (softmax, Q prep), not one elected thread
  uint32_t k = 0;
  __device__ ItemSrc(const TcParams& p, TcSmem<D, PR>& s, int b, int e, bool c, bool ww = false)
      : P(p), S(s), it(b), end(e), claimer(c), warp_wide(ww) {}
  int ahead = -1;  // claimer: the code published one entry ahead of the one it is working on
  // claim the next code of the launch and publish it as entry n of the ring (a pair: the leader
  // claims for both CTAs and publishes into the peer's ring too)
  __device__ int publish(uint32_t n) {
    constexpr int R = TcSmem<D, PR>::kSched;
    const int slot = n % R;
    wait_lead<PR>(&S.sched_empty[slot], ((n / R) & 1) ^ 1);
    const int idx = atomicAdd(P.a.sched, 1);
    const int code = idx < P.a.n_codes ? P.a.cta_items[idx] : -1;
    *reinterpret_cast<volatile int32_t*>(&S.sched_code[slot]) = code;
    if constexpr (PR) {
      st_cluster_u32(cluster_addr(&S.sched_code[slot], 1), static_cast<uint32_t>(code));
      mbar_arrive_cl(cluster_addr(&S.sched_full[slot], 1));
    }
    mbar_arrive(&S.sched_full[slot]);
    return code;
  }
  __device__ int next() {
    if (P.a.sched == nullptr) return it < end ? P.a.cta_items[it++] : -1;
    if (claimer) {
      // epi_q launches: one code of look-ahead, so the other roles learn item k+1 when the producer
      // starts item k (its Q is then prepared a whole item ahead)
      if (!EPI) return publish(k++);
      if (k == 0) ahead = publish(0);
      const int mine = ahead;
      if (mine >= 0) ahead = publish(k + 1);
      ++k;
      return mine;
    }
    constexpr int R = TcSmem<D, PR>::kSched;
    const int slot = k % R;
    const uint32_t par = (k / R) & 1;
    ++k;
    int code;
    {
      if constexpr (PR)
        mbar_wait_cl(&S.sched_full[slot], par);  // the peer's entries are written by the leader
      else
        mbar_wait(&S.sched_full[slot], par);
      code = *reinterpret_cast<volatile int32_t*>(&S.sched_code[slot]);
      if (warp_wide)
        arrive_lead_warp<PR>(&S.sched_empty[slot]);
      else
        arrive_lead<PR>(&S.sched_empty[slot]);
    }
    return code;
  }
};

// exp2 on the FMA pipe: x = n + f, n = rint(x) via the 1.5*2^23 trick, 2^f by a degree-3
// polynomial on [-0.5, 0.5] (max rel. error 1.0e-4), exponent added in the integer domain.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -120.f);
  const float t = x + 12582912.f;
  const float n = t - 12582912.f;
  const float f = x - n;
  const float p = fmaf(fmaf(fmaf(0.05500831f, f, 0.24220964f), f, 0.69328305f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}

// two exp2 on the FMA pipe in packed fp32x2 (FADD2 / FFMA2): the same rounding trick and
// polynomial as exp2_poly, ~5 instructions per value; the exponent is added with one IMAD per
// value — (t_bits - 0x4B400000) << 23 == t_bits << 23 mod 2^32, the magic's low 9 bits being 0
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -120.f);
  x.y = fmaxf(x.y, -120.f);
  const float2 t = fadd2(x, make_float2(12582912.f, 12582912.f));
  const float2 n = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = ffma2(n, make_float2(-1.f, -1.f), x);
  float2 p = ffma2(make_float2(0.05500831f, 0.05500831f), f, make_float2(0.24220964f, 0.24220964f));
  p = ffma2(p, f, make_float2(0.69328305f, 0.69328305f));
  p = ffma2(p, f, make_float2(1.0f, 1.0f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// two exp2 with one MUFU op: fp32 inputs rounded to f16 (the large-p keys have x near 0 where
// f16 is fine-grained: <= 0.07% error for p >= 1/16, below the bf16 rounding of P itself),
// packed ex2.approx.f16x2, widened back to fp32 for the row sum.
__device__ __forceinline__ void ex2_pair_f16(float x0, float x1, float& p0, float& p1) {
  uint32_t h, e;
  asm("cvt.rn.f16x2.f32 %0, %2, %1;" : "=r"(h) : "f"(x0), "f"(x1));
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(e) : "r"(h));
  asm("{\n\t.reg .f16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tcvt.f32.f16 %0, lo;\n\tcvt.f32.f16 %1, hi;\n\t}"
      : "=f"(p0), "=f"(p1)
      : "r"(e));
}

// ------------------------------------------------------------------ warps 0 / 3: TMA producers
// K (warp 0) and V (warp 3) are streamed per 64-key sub-tile (the MMA granularity) into two
// independent rings, so a K load never queues behind a V slot (S(j+2) needs K(j+2) one step
// after PV(j); V(j) is needed two steps later). Sub-tile s goes to slot s % (ring depth).
// Each sub-tile is 64/bs paged blocks (bs <= 64) or half of one 128-row block, gathered by TMA
// boxes {64 columns, min(bs, 64) rows}.
template <int D, bool EPI, bool PR>
__device__ void run_producer(const TcParams& P, TcSmem<D, PR>& S, int it_begin, int it_end, int kv) {
  const AttnArgs& a = P.a;
  // programmatic dependent launch: the pages this launch reads are written by the preceding
  // rope_kv_write — everything before this point (barriers, TMEM, work claims, Q loads and
  // rotation) may overlap that kernel's tail; the pool is read only after it has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int kSlots = kv == 0 ? TcSmem<D, PR>::kKSlots : TcSmem<D, PR>::kVSlots;
  const int group = a.hq / a.hkv;
  const int box = min(a.bs, 64);
  const int bps = 64 / box;  // boxes per sub-tile
  constexpr uint32_t kSubTileBytes = 64 * D * 2;  // (a pair: both CTAs' halves together)
  const int64_t layer_rows = static_cast<int64_t>(a.layer) * a.nblk * a.hkv * a.bs;
  const CUtensorMap* map = kv == 0 ? (PR ? &P.tmk2 : &P.tmk) : &P.tmv;
  const uint32_t rank = PR ? cluster_rank() : 0;
  uint32_t n = 0;
  uint32_t tc = 0;
#ifdef SPANQ_L2HINT
  const uint64_t pol = policy_evict_last();
#endif
  // a pair: the leader claims the work codes (K producer), the peer's K producer consumes them
  ItemSrc<D, EPI, PR> src(P, S, it_begin, it_end, kv == 0 && rank == 0);
  for (int code; (code = src.next()) >= 0;) {
    const Unit u = decode<PR>(P, code);
    const int kvh = u.head_a / group;
    for (int t = u.w.tile_begin; t < u.w.tile_end; ++t) {
      const KvTile tl = a.tiles[t];
      const int nsub = tl.n_valid > 64 ? 2 : 1;
#pragma unroll 1
      for (int h = 0; h < nsub; ++h, ++n) {
        const int slot = n % kSlots;
        trace(P, 0, tc, 12 + kv + (static_cast<int>(n) << 8));  // 12: K slot wanted, 13: V slot wanted
        mbar_wait_1t(&S.kv_empty[kv][slot], ((n / kSlots) & 1) ^ 1);
        trace(P, 0, tc, 10 + kv + (static_cast<int>(n) << 8));  // 10: K load issued, 11: V load issued
        if constexpr (PR) {
          // this CTA's half: K keys [64h + 32 rank, +32) (all d columns), V all 64 keys of its
          // d columns [64 rank, +64); completion counted on the leader's barrier, which expects
          // both halves
          if (rank == 0) mbar_arrive_expect_tx(&S.kv_full[kv][slot], kSubTileBytes);
          const uint32_t bar = cluster_addr(&S.kv_full[kv][slot], 0);
          if (kv == 0) {
            const int kbox = min(a.bs, 32);
            for (int j = 0; j < 32 / kbox; ++j) {
              const int key = 64 * h + 32 * static_cast<int>(rank) + j * kbox;
              const int32_t blk = a.tile_blocks[tl.blk_off + key / a.bs];
              const int32_t y =
                  static_cast<int32_t>(layer_rows + (static_cast<int64_t>(blk) * a.hkv + kvh) * a.bs + key % a.bs);
#pragma unroll
              for (int c = 0; c < D / 64; ++c) tma_load_2d_pair(&S.k[slot][c][0] + j * kbox * 128, map, bar, c * 64, y);
            }
          } else {
            for (int j = 0; j < bps; ++j) {
              const int key = 64 * h + j * box;
              const int32_t blk = a.tile_blocks[tl.blk_off + key / a.bs];
              const int32_t y =
                  static_cast<int32_t>(layer_rows + (static_cast<int64_t>(blk) * a.hkv + kvh) * a.bs + key % a.bs);
              tma_load_2d_pair(&S.v[slot][0][0] + j * box * 128, map, bar, 64 * static_cast<int>(rank), y);
            }
          }
          continue;
        }
        mbar_arrive_expect_tx(&S.kv_full[kv][slot], kSubTileBytes);
        for (int j = 0; j < bps; ++j) {
          // key 64h + j*box of the tile: block (64h + j*box) / bs, row offset (64h + j*box) % bs
          const int key = 64 * h + j * box;
          const int32_t blk = dbg_mode(P) == 3 ? a.tile_blocks[0] : a.tile_blocks[tl.blk_off + key / a.bs];
          const int32_t y = static_cast<int32_t>(layer_rows + (static_cast<int64_t>(blk) * a.hkv + kvh) * a.bs +
                                                 key % a.bs);
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
#ifdef SPANQ_L2HINT  // A/B: K/V pages kept in L2 (each is read by every q tile of its segment)
            tma_load_2d_hint((kv == 0 ? &S.k[slot][c][0] : &S.v[slot][c][0]) + j * box * 128, map,
                             &S.kv_full[kv][slot], c * 64, y, pol);
#else
            tma_load_2d((kv == 0 ? &S.k[slot][c][0] : &S.v[slot][c][0]) + j * box * 128, map, &S.kv_full[kv][slot],
                        c * 64, y);
#endif
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------------ warps 1 / 2: MMA issuers
// One issuing thread per head (warp 1: head A, warp 2: head B), so each head's chain
// softmax(j) -> PV(j) -> S(j+2) runs at its own pace and the tensor core interleaves the two.
// Work is issued per 64-key sub-tile j. Each head has two S buffers, so S(j+2) is issued as
// soon as PV(j) (which reads P(j) from S buffer j&1) is issued: softmax(j+1) never waits for the
// tensor core to finish PV(j). Per head: S(0), S(1), then PV(j), [release V_j], S(j+2), ...
// K_j / V_j slots are released when both heads' MMAs reading them are done (2 commits).
struct SubCursor {
  int t, h;  // KV tile, half (keys [64h, 64h+64))
};

// A pair (PR): only the leader runs this; its M = 256 MMAs take A rows 0-127 from its own smem /
// TMEM and rows 128-255 from the peer's at the same offsets, B halves from both, and write D into
// both CTAs' TMEM; commits arrive on both CTAs' barriers.
template <int D, bool EPI, bool PR>
__device__ void run_mma(const TcParams& P, TcSmem<D, PR>& S, uint32_t tmem, int it_begin, int it_end, int x) {
  const AttnArgs& a = P.a;
  const bool J = EPI || P.join != 0;  // 2-deep Q ring
  using Sm = TcSmem<D, PR>;
  constexpr int kKS = Sm::kKSlots, kVS = Sm::kVSlots;
  constexpr uint32_t idS = idesc_bf16_f32(PR ? 256 : 128, 64, false, false);
  constexpr uint32_t idO = idesc_bf16_f32(PR ? 256 : 128, D, false, true);
  uint32_t jg = 0;  // sub-tiles whose PV has been issued (global): S buffer j & 1, V slot j
  uint32_t ep = 0;    // Q epochs started
  uint32_t qcur = 0;  // the epoch whose Q tile the S MMAs read
  uint32_t n_items = 0;  // items of this head completed (prefill: o_free completions awaited)
  uint32_t tc = 0;
  auto wait_kv = [&](int kv, uint32_t n) {
    const uint32_t ns = kv == 0 ? kKS : kVS;
    wait_lead<PR>(&S.kv_full[kv][n % ns], (n / ns) & 1);
    tc_fence_after();
  };
  ItemSrc<D, EPI, PR> src(P, S, it_begin, it_end, false);
  for (int code; (code = src.next()) >= 0;) {
    const Unit u = decode<PR>(P, code);
    if (x >= u.n_heads) continue;  // unpaired launch: the B issuer idles
    const int tb = u.w.tile_begin, te = u.w.tile_end;
    auto nsub = [&](int t) { return a.tiles[t].n_valid > 64 ? 2 : 1; };
    auto advance = [&](SubCursor& c) {
      if (c.h == 0 && nsub(c.t) == 2)
        c.h = 1;
      else
        c = SubCursor{c.t + 1, 0};
    };
    SubCursor cs{tb, 0}, cp{tb, 0};
    uint32_t js = jg;  // global index of the next S sub-tile (K slot js)
    // Q: slot x holds head x's tile of the current epoch (an item or a change of rot_delta)
    auto release_q = [&]() {
      const int sl = q_slot(J, qcur);
      commit_x<PR>(&S.q_empty[x][sl]);
    };
    auto issue_s = [&]() {
      const int t = cs.t;
      if (kSP && js > 0) {  // the single S buffer: softmax(js - 1) has loaded it
        wait_lead<PR>(&S.s_free[x][(js - 1) & 1], ((js - 1) >> 1) & 1);
        tc_fence_after();
      }
      if (cs.h == 0 && (t == tb || a.tiles[t].rot_delta != a.tiles[t - 1].rot_delta)) {
        if (t != tb) release_q();  // the previous epoch's Q tile: free once its S MMAs are done
        wait_lead<PR>(&S.q_full[x][q_slot(J, ep)], q_par(J, ep));
        trace(P, 1, tc, 21);  // 21: Q ready for new epoch
        qcur = ep++;
      }
      wait_kv(0, js);
      trace(P, 1, tc, 22 + (static_cast<int>(js) << 8));  // 22: K ready
      const uint32_t qbase = smem_u32(q_tile<D, PR>(S, J, x, qcur));
      const uint32_t kb = smem_u32(&S.k[js % kKS][0][0]);
      const int buf = js & 1;
      const uint64_t ad0 = desc_sw128(qbase, 16, 1024), bd0 = desc_sw128(kb, 16, 1024);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint64_t ad = desc_add(ad0, (kk / 4) * Sm::kChunkBytes + (kk % 4) * 32);
        const uint64_t bd = desc_add(bd0, (kk / 4) * Sm::kKChunkBytes + (kk % 4) * 32);
        if constexpr (PR)
          mma2_ss(tmem + col_s(x, buf), ad, bd, idS, kk > 0 ? 1u : 0u);
        else
          mma_ss(tmem + col_s(x, buf), ad, bd, idS, kk > 0 ? 1u : 0u);
      }
      trace(P, 1, tc, 25 + (static_cast<int>(js) << 8));  // 25: S MMAs accepted
      commit_x<PR>(&S.s_full[x][buf]);
      commit_x<PR>(&S.kv_empty[0][js % kKS]);  // K_js (one of the heads' two arrivals)
      advance(cs);
      ++js;
      if (cs.t >= te) release_q();
    };
    auto issue_pv = [&](uint32_t j, bool first) {
      wait_kv(1, j);
      trace(P, 1, tc, 24 + (static_cast<int>(j) << 8));  // 24: V ready
      // V sub-tile, MN-major: 64-column d chunks kSubBytes apart (LBO), 16 keys = 2048 B per K step
      const uint32_t vb = smem_u32(&S.v[j % kVS][0][0]);
      const int buf = j & 1;
      const uint64_t vd0 = desc_sw128(vb, Sm::kSubBytes, 1024);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t vd = desc_add(vd0, kk * 2048);
        if constexpr (PR)
          mma2_ts(tmem + col_o(x), tmem + col_p(x, buf) + kk * 8, vd, idO, (!first || kk > 0) ? 1u : 0u);
        else
          mma_ts(tmem + col_o(x), tmem + col_p(x, buf) + kk * 8, vd, idO, (!first || kk > 0) ? 1u : 0u);
      }
      trace(P, 1, tc, 27 + (static_cast<int>(j) << 8));  // 27: PV MMAs accepted
      commit_x<PR>(&S.o_done[x][j & 1]);
      commit_x<PR>(&S.kv_empty[1][j % kVS]);  // V_j
    };
    if constexpr (EPI) {
      // prefill items are one epoch (rot_delta 0 on every tile) of w.n_sub sub-tiles: the issuer
      // walks them by count, with no work-list reads on its critical path (each tile read is an
      // L1-miss-prone global load: ~40-600 cycles per step otherwise)
      int ns = u.w.n_sub;  // sub-tiles of the item whose S MMAs are being issued
      int si = 0;          // S sub-tiles issued for that item
      auto issue_s_cnt = [&]() {
        if (kSP && js > 0) {  // the single S buffer: softmax(js - 1) has loaded it
          wait_lead<PR>(&S.s_free[x][(js - 1) & 1], ((js - 1) >> 1) & 1);
          tc_fence_after();
        }
        if (si == 0) {
          wait_lead<PR>(&S.q_full[x][q_slot(J, ep)], q_par(J, ep));
          trace(P, 1, tc, 21);  // 21: Q ready for new epoch
          qcur = ep++;
        }
        wait_kv(0, js);
        trace(P, 1, tc, 22 + (static_cast<int>(js) << 8));  // 22: K ready
        const uint32_t qbase = smem_u32(q_tile<D, PR>(S, J, x, qcur));
        const uint32_t kb = smem_u32(&S.k[js % kKS][0][0]);
        const int buf = js & 1;
        const uint64_t ad0 = desc_sw128(qbase, 16, 1024), bd0 = desc_sw128(kb, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = desc_add(ad0, (kk / 4) * Sm::kChunkBytes + (kk % 4) * 32);
          const uint64_t bd = desc_add(bd0, (kk / 4) * Sm::kKChunkBytes + (kk % 4) * 32);
          if constexpr (PR)
            mma2_ss(tmem + col_s(x, buf), ad, bd, idS, kk > 0 ? 1u : 0u);
          else
            mma_ss(tmem + col_s(x, buf), ad, bd, idS, kk > 0 ? 1u : 0u);
        }
        trace(P, 1, tc, 25 + (static_cast<int>(js) << 8));  // 25: S MMAs accepted
      commit_x<PR>(&S.s_full[x][buf]);
        commit_x<PR>(&S.kv_empty[0][js % kKS]);
        ++js;
        if (++si == ns) release_q();
      };
      if constexpr (kSP) {
        // one flat pipeline over the CTA's items: S(0) of the next item is issued as soon as the
        // softmax has loaded the current item's last S (its Q was prepared a whole item ahead), so
        // an item boundary costs no pipeline refill
        int pv_left = ns, pv_next = -1;
        bool pv_first = true, s_done = false;
        issue_s_cnt();
        for (;;) {
          const uint32_t j = jg;
          if (si == ns && pv_next < 0 && !s_done) {  // the S side moves on to the next item
            const int c = src.next();
            if (c < 0) {
              s_done = true;
            } else {
              ns = decode<PR>(P, c).w.n_sub;
              si = 0;
              pv_next = ns;
            }
          }
          if (si < ns) issue_s_cnt();  // S(j+1) as soon as softmax(j) has loaded S(j)
          wait_lead<PR>(&S.p_full[x][j & 1], (j >> 1) & 1);
          trace(P, 1, tc, 20);  // 20: P ready
          if (pv_first && n_items > 0) {
            // the previous item's O has been drained by the epilogue warps (the latest possible
            // completion: this thread waited for n_items - 2 before the previous item's first PV)
            wait_lead<PR>(&S.o_free[x], (n_items - 1) & 1);
            tc_fence_after();
            trace(P, 1, tc, 26);  // 26: O free for the next item
          }
          issue_pv(j, pv_first);
          ++jg;
          pv_first = false;
          if (--pv_left == 0) {
            ++n_items;
            if (pv_next < 0) break;
            pv_left = pv_next;
            pv_next = -1;
            pv_first = true;
          }
        }
        break;  // every code of the launch has been consumed
      }
      for (int i = 0; i < 2 && si < ns; ++i) issue_s_cnt();
      for (int pi = 0; pi < ns; ++pi) {
        const uint32_t j = jg;
#ifdef SPANQ_SPIN_ISSUER
        if constexpr (!PR) mbar_wait_spin(&S.p_full[x][j & 1], (j >> 1) & 1); else
#endif
        wait_lead<PR>(&S.p_full[x][j & 1], (j >> 1) & 1);
        trace(P, 1, tc, 20);  // 20: P ready
        if (pi == 0 && n_items > 0) {
          // the previous item's O has been drained by the epilogue warps. Completion n_items - 1
          // is the latest possible one (this thread waited for n_items - 2 before the previous
          // item's first PV), so the parity wait cannot be lapped
          wait_lead<PR>(&S.o_free[x], (n_items - 1) & 1);
          tc_fence_after();
          trace(P, 1, tc, 26);  // 26: O free for the next item
        }
        issue_pv(j, pi == 0);
        if (si < ns) issue_s_cnt();  // S(j+2) into the buffer PV(j) reads
        ++jg;
      }
      ++n_items;
      continue;
    }
    // prologue: S for the first two sub-tiles
    for (int i = 0; i < (kSP ? 1 : 2) && cs.t < te; ++i) issue_s();
    bool first = true;
    while (cp.t < te) {
      const uint32_t j = jg;
      if (kSP && cs.t < te) issue_s();  // S(j+1) as soon as softmax(j) has loaded S(j)
      wait_lead<PR>(&S.p_full[x][j & 1], (j >> 1) & 1);
      trace(P, 1, tc, 20);  // 20: P ready
      if (EPI && first && n_items > 0) {
        // prefill: the previous item's O has been drained by the epilogue warps. Completion
        // n_items - 1 is the latest possible one (this thread waited for n_items - 2 before the
        // previous item's first PV), so the parity wait cannot be lapped
        wait_lead<PR>(&S.o_free[x], (n_items - 1) & 1);
        tc_fence_after();
        trace(P, 1, tc, 26);  // 26: O free for the next item
      }
      issue_pv(j, first);
      if (!kSP && cs.t < te) issue_s();  // S(j+2) into the buffer PV(j) reads
      advance(cp);
      ++jg;
      first = false;
    }
    ++n_items;
  }
}

// Online softmax over one 64-key S sub-tile row in TMEM, single pass: one LDTM.x64 of the 64
// fp32 scores, row max with three-input FMNMX3, then P = exp2(s*scale - m) packed to bf16 and
// written back over the first 32 columns of the sub-tile with one STTM.x32. The running max m
// only moves when the new max exceeds it by more than `thr` (log2 units: P <= 2^thr), and then
// *alpha = 2^(m_old - m_new) is the factor for O and l. Returns the row sum of P (fp32, before
// bf16 rounding; 8 independent accumulators).
__device__ __forceinline__ float ld_shared_volatile(const float* p) {
  float v;
  asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_shared_volatile(float* p, float v) {
  asm volatile("st.volatile.shared.f32 [%0], %1;" ::"r"(smem_u32(p)), "f"(v) : "memory");
}

template <int PM, bool kMasked, bool PR>
__device__ __forceinline__ float softmax_sub(uint32_t scol, uint32_t pcol, uint64_t* sfree, int pp_wait, int pp_give,
                                             float* pp_words, float sl2, float thr, int lim, float& m, float& alpha,
                                             bool& resc) {
  uint32_t v[64];
  tmem_ld64(scol, v);
  tmem_wait_ld();
  if constexpr (kSP) {  // S(j) is in registers: the issuer may compute S(j+1) into the buffer
    tc_fence_before();
    arrive_hand<PR>(sfree);
  }
  // ping-pong: the two heads' softmax WGs take turns (named barriers 1 / 2), so each runs alone on
  // the SMSPs' MUFU / issue slots and the two heads' MMAs reach the tensor core staggered
  // (ptxas moves register-only math across a barrier freely: the exponentials are tied to it by
  // a dependency on a shared-memory word read after it, the hand-over by a store of the row sum)
  float pp_z = 0.f;
  if (pp_wait) {
    named_sync(pp_wait, 256);
    pp_z = ld_shared_volatile(pp_words);
  }
  if constexpr (kMasked) {
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = i <= lim ? v[i] : 0xff800000u;  // -inf
  }
  float mx4[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) mx4[k] = fmaxf(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
#pragma unroll
  for (int i = 4; i < 32; ++i)
    mx4[i & 3] = fmax3(mx4[i & 3], __uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
  const float mx = fmax3(fmaxf(mx4[0], mx4[1]), mx4[2], mx4[3]) * sl2;
  const float m_new = fmaxf(m, mx);
  resc = m_new > m + thr;
  const float m_use = resc ? m_new : m;
  alpha = resc ? ex2_approx(m - m_new) : 1.f;
  m = m_use;
  const float msub = ((m_use == -INFINITY) ? 0.f : m_use) + pp_z;
  // x = s * scale - m and the row sums in packed fp32x2 (FFMA2 / FADD2: half the instructions)
  float2 sum4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) sum4[i] = make_float2(0.f, 0.f);
  const float2 sl2v = make_float2(sl2, sl2), nmv = make_float2(-msub, -msub);
  uint32_t pk[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float2 xx = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), sl2v, nmv);
    float p0, p1;
    if constexpr (PM == 3) {
      ex2_pair_f16(xx.x, xx.y, p0, p1);
    } else {
      // PM 1 / 2: a quarter / half of the pairs on the FMA pipe (MUFU: 16 ex2 per SM per clock)
      constexpr bool kPoly[4] = {0 < PM, 2 < PM, 1 < PM, 3 < PM};
      if (kPoly[i & 3]) {
        const float2 pp = exp2_poly2(xx);
        p0 = pp.x;
        p1 = pp.y;
      } else {
        p0 = ex2_approx(xx.x);
        p1 = ex2_approx(xx.y);
      }
    }
    if constexpr (kMasked) {
      p0 = (2 * i <= lim) ? p0 : 0.f;
      p1 = (2 * i + 1 <= lim) ? p1 : 0.f;
    }
    sum4[i & 3] = fadd2(sum4[i & 3], make_float2(p0, p1));
    pk[i] = pack_bf16x2(p0, p1);
  }
  const float2 s01 = fadd2(sum4[0], sum4[1]), s23 = fadd2(sum4[2], sum4[3]);
  const float2 st = fadd2(s01, s23);
  const float rsum = st.x + st.y;
  if (pp_give) {
    st_shared_volatile(pp_words + 1, rsum);
    named_arrive(pp_give, 256);
  }
  tmem_st32(pcol, pk);
  tmem_wait_st();
  return rsum;
}

// ------------------------------------------------------------------ softmax + epilogue (one WG per head)
// A finished item whose O sits in TMEM.
struct Finished {
  WorkItem w;
  float m, l;
  int h, n_heads;
  uint32_t jlast;  // global index of the item's last sub-tile (its PV is the last write to O)
  uint32_t elast;  // Q epoch of the item's last sub-tile (join: its slot stages the epilogue)
};

// Epilogue of one finished item: wait for its last PV, read O from TMEM, normalise, store. Each warp stages 32 rows x 32 fp32 columns in its 4 KB SWIZZLE_128B buffer
// and one lane hands it to a TMA bulk store (the warp only waits until the TMA has READ the
// buffer before reusing it, never for the HBM write).
template <int D, bool PR>
__device__ __forceinline__ void epilogue(const TcParams& P, TcSmem<D, PR>& S, uint32_t ocol, int x, const Finished& f,
                                         uint32_t& tc, bool tr) {
  const AttnArgs& a = P.a;
  const bool J = P.join != 0;
  const WorkItem& w = f.w;
  const int r = threadIdx.x & 127;
  mbar_wait(&S.o_done[x][f.jlast & 1], (f.jlast >> 1) & 1);
  if (tr) trace(P, 2 + x, tc, 32);  // 32: O ready (epilogue start)
  tc_fence_after();
  // chunk c+1 is read from TMEM while chunk c is staged and stored
  uint32_t vv[2][32];
  tmem_ld32(ocol, vv[0]);
  tmem_wait_ld();
  const float inv = f.l > 0.f ? 1.f / f.l : 0.f;
  const float lse = f.l > 0.f ? (f.m + __log2f(f.l)) * 0.69314718055994531f : -INFINITY;
  const int wr = (threadIdx.x / 32) & 3;  // warp's 32-row slice of the tile
  const int lane = threadIdx.x & 31;
  // 4 KB staging buffers per warp, chunk c uses buffer c % kBufs. Prefill: the staging area. Join:
  // the Q slot of the item's last epoch (its S MMAs are done: they precede the last PV), handed
  // back to the Q prep only once the stores below have read it
  const int kBufs = (J && D == 64) ? 1 : 2;
  float* const stg2 = J ? reinterpret_cast<float*>(q_tile<D, PR>(S, J, x, f.elast)) + wr * kBufs * 1024
                        : &S.stage[x * 4 + wr][0][0];
  // TMA store for whole 32-row slices (and for split partials, whose padding rows are never
  // read); a slice that ends inside this item's rows is written directly (the next rows belong
  // to another item)
  const bool in_range = wr * 32 < w.n_rows;
  const bool use_tma = in_range && (w.part >= 0 || (a.out_fp32 && wr * 32 + 32 <= w.n_rows));
  const bool direct = in_range && !use_tma;
#pragma unroll
  for (int c = 0; c < D / 32; ++c) {
    if (c + 1 < D / 32) tmem_ld32(ocol + (c + 1) * 32, vv[(c + 1) & 1]);
    const uint32_t(&v)[32] = vv[c & 1];
    float* stg = stg2 + (c % kBufs) * 1024;
    if (lane == 0) {  // the store of chunk c-kBufs (same buffer) has read it
      if (kBufs == 1)
        bulk_wait_read<0>();
      else
        bulk_wait_read<1>();
    }
    __syncwarp();
    if (tr) trace(P, 2 + x, tc, 50 + c);  // 50+c: staging buffer of chunk c free
#pragma unroll
    for (int uu = 0; uu < 8; ++uu)
      *reinterpret_cast<float4*>(stg + lane * 32 + ((uu ^ (lane & 7)) * 4)) =
          make_float4(__uint_as_float(v[4 * uu]) * inv, __uint_as_float(v[4 * uu + 1]) * inv,
                      __uint_as_float(v[4 * uu + 2]) * inv, __uint_as_float(v[4 * uu + 3]) * inv);
    if (use_tma) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (w.part >= 0)
          tma_store_2d(&P.tmop, stg, c * 32, (w.part * f.n_heads + x) * kTileRows + wr * 32);
        else
          tma_store_3d(&P.tmo, stg, c * 32, f.h, w.row0 + wr * 32);
        bulk_commit();
      }
    } else {
      __syncwarp();
    }
    if (direct) {  // coalesced: each store instruction writes 4 rows x 128 B
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int rr = j * 4 + (lane >> 3);
        const int uu = lane & 7;
        const float4 val = *reinterpret_cast<const float4*>(stg + rr * 32 + ((uu ^ (rr & 7)) * 4));
        const int trow = wr * 32 + rr;
        const int col = c * 32 + uu * 4;
        if (trow < w.n_rows) {
          if (a.out_fp32) {
            *reinterpret_cast<float4*>(static_cast<float*>(a.o) +
                                       ((w.row0 + trow) * static_cast<int64_t>(a.hq) + f.h) * D + col) = val;
          } else {
            uint2 pk;
            pk.x = pack_bf16x2(val.x, val.y);
            pk.y = pack_bf16x2(val.z, val.w);
            *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.o) +
                                      ((w.row0 + trow) * static_cast<int64_t>(a.hq) + f.h) * D + col) = pk;
          }
        }
      }
      __syncwarp();
    }
    tmem_wait_ld();
  }
  if (r < w.n_rows) {
    if (w.part < 0) {
      if (a.lse != nullptr) a.lse[(static_cast<int64_t>(w.row0) + r) * a.hq + f.h] = lse;
    } else {
      a.lsepart[(static_cast<int64_t>(w.part) * f.n_heads + x) * kTileRows + r] = lse;
    }
  }
  if (J) {  // the Q slot is free again once this warp's stores have read it
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
    mbar_arrive(&S.q_empty[x][q_slot(J, f.elast)]);  // every lane (its staging writes are released)
  }
  if (tr) trace(P, 2 + x, tc, 33);  // 33: epilogue done
}

// Prefill epilogue, run by the Q-prep warps (warp wq = 12 + i reads TMEM lanes [32i, 32i+32)) so
// that it overlaps the softmax WGs' next item: per head x, wait for the row stats and the item's
// last PV, drain O_x (times 1/l) from TMEM into the item's own Q slot of head x (free since the
// item's last S MMA: the next item's Q is in the other slot of the 2-deep ring), release O_x
// (o_free) as soon as the last TMEM load has landed, and store: TMA bulk stores of whole 32-row
// slices, coalesced st.global for a ragged last slice (the rows after it belong to another item).
// The slot goes back to the Q prep (q_empty) once the stores have read it. Staging per warp: the
// warp's quarter of the slot (8 KB at d=128, 4 KB at d=64) as 4 KB chunks of 32 rows x 128 B,
// SWIZZLE_128B (fp32: 32 columns per chunk, bf16: 64); bf16 O always fits, fp32 O cycles through
// the chunk buffers (a chunk waits for the store of the chunk that used its buffer before).
template <int D, bool PR>
__device__ void prefill_epilogue(const TcParams& P, TcSmem<D, PR>& S, uint32_t tmem, const Unit& u, uint32_t jlast,
                                 uint32_t k, uint32_t& tc) {
  const AttnArgs& a = P.a;
  const WorkItem& w = u.w;
  const bool tr = (threadIdx.x & 31) == 0;
  const int lane = threadIdx.x & 31;
  const int wq = (threadIdx.x / 32) & 3;
  const int r = wq * 32 + lane;
  const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
  const bool in_range = wq * 32 < w.n_rows;
  const bool use_tma = in_range && wq * 32 + 32 <= w.n_rows;
  const bool direct = in_range && !use_tma;
  const bool f32 = a.out_fp32;
  constexpr int kBufs = D / 64;  // 4 KB chunk buffers per warp in its quarter of a Q slot
  const int n_chunks = f32 ? D / 32 : D / 64;
  for (int x = 0; x < u.n_heads; ++x) {
    uint8_t* const stg = q_tile<D, PR>(S, true, x, k) + wq * kBufs * 4096;
    mbar_wait(&S.fin_full[x][k & 1], (k >> 1) & 1);
    const float inv = S.fin_inv[x][k & 1][r];
    if (tr) trace(P, 4, tc, 60 + 4 * x);  // 60/64: row stats of head A/B ready
    mbar_wait(&S.o_done[x][jlast & 1], (jlast >> 1) & 1);
    tc_fence_after();
    if (tr) trace(P, 4, tc, 61 + 4 * x);  // 61/65: O ready
    const uint32_t ocol = tmem + lane_base + col_o(x);
    const int h = u.head_a + x;
    uint32_t vv[2][32];
    tmem_ld32(ocol, vv[0]);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      if (c + 1 < D / 32) tmem_ld32(ocol + (c + 1) * 32, vv[(c + 1) & 1]);
      const uint32_t(&v)[32] = vv[c & 1];
      if (c + 1 == D / 32) {
        // the last TMEM load has landed (waited at the end of the previous iteration): O_x is free
        tc_fence_before();
        arrive_lead_warp<PR>(&S.o_free[x]);  // every lane: its TMEM loads and fin_inv read are done
        if (tr) trace(P, 4, tc, 62 + 4 * x);  // 62/66: O drained (o_free)
      }
      const int chunk = f32 ? c : c / 2;
      uint8_t* ch = stg + (chunk % kBufs) * 4096;
      if (f32 && chunk >= kBufs) {  // this buffer's previous chunk must have been read
        if (lane == 0) {
          if constexpr (kBufs == 1)
            bulk_wait_read<0>();
          else
            bulk_wait_read<kBufs - 1>();
        }
        __syncwarp();
      }
      if (f32) {
#pragma unroll
        for (int uu = 0; uu < 8; ++uu)
          *reinterpret_cast<float4*>(ch + lane * 128 + ((uu ^ (lane & 7)) * 16)) =
              make_float4(__uint_as_float(v[4 * uu]) * inv, __uint_as_float(v[4 * uu + 1]) * inv,
                          __uint_as_float(v[4 * uu + 2]) * inv, __uint_as_float(v[4 * uu + 3]) * inv);
      } else {  // 64 columns (two fp32 chunks) per 128-byte row, 16-byte unit = 8 columns
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int uu = (c & 1) * 4 + q;
          uint4 pk;
          pk.x = pack_bf16x2(__uint_as_float(v[8 * q]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
          pk.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
          pk.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
          pk.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
          *reinterpret_cast<uint4*>(ch + lane * 128 + ((uu ^ (lane & 7)) * 16)) = pk;
        }
      }
      const bool chunk_done = f32 || (c & 1);
      if (chunk_done && use_tma) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
#ifdef SPANQ_L2HINT  // O is written once
          tma_store_3d_hint(&P.tmo, ch, f32 ? c * 32 : (c / 2) * 64, h, w.row0 + wq * 32, policy_evict_first());
#else
          tma_store_3d(&P.tmo, ch, f32 ? c * 32 : (c / 2) * 64, h, w.row0 + wq * 32);
#endif
          bulk_commit();
        }
      } else if (chunk_done && direct) {
        __syncwarp();
        // coalesced: 8 lanes cover one 128-byte staging row, 4 rows per instruction
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int rr = j * 4 + (lane >> 3);
          const int uu = lane & 7;
          const int trow = wq * 32 + rr;
          if (trow < w.n_rows) {
            const uint4 val = *reinterpret_cast<const uint4*>(ch + rr * 128 + ((uu ^ (rr & 7)) * 16));
            const int64_t base = (static_cast<int64_t>(w.row0) + trow) * a.hq + h;
            if (f32)
              *reinterpret_cast<uint4*>(static_cast<float*>(a.o) + base * D + c * 32 + uu * 4) = val;
            else
              *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.o) + base * D + (c / 2) * 64 + uu * 8) = val;
          }
        }
        __syncwarp();
      }
      tmem_wait_ld();
    }
    // the slot returns to the Q prep once this warp's stores have read it (every lane arrives, so
    // each lane's own staging writes are released by its own arrive)
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
    mbar_arrive(&S.q_empty[x][k & 1]);
  }
}

template <int D, int PM, bool EPI, bool PR>
__device__ void run_softmax(const TcParams& P, TcSmem<D, PR>& S, uint32_t tmem, int it_begin, int it_end, int x) {
  const AttnArgs& a = P.a;
  const bool J = P.join != 0;
  const int r = threadIdx.x & 127;  // row within the tile == TMEM lane
  const uint32_t lane_base = static_cast<uint32_t>((r / 32) * 32) << 16;
  const float sl2 = P.scale_log2;
  const uint32_t ocol = tmem + lane_base + col_o(x);
  uint32_t js = 0;  // sub-tiles processed (global; == the MMA warps' PV index)
  uint32_t eps = 0, ecur = 0;  // Q epochs seen / current (join: Q slots are also epilogue staging)
  uint32_t ni = 0;             // prefill: items finished by this WG (fin_inv buffer ni & 1)
  uint32_t tc = 0;
  const bool tr = (threadIdx.x & 31) == 0;
  // ping-pong of the two WGs (paired launches: both see the same sub-tile sequence). Barrier 1:
  // A -> B ("A has finished its exponentials of sub-tile j"), barrier 2: B -> A (j -> j + 1)
  const bool pp = kPingPong && P.paired && dbg_mode(P) == 0;
  const int pp_give = pp ? 1 + x : 0;
  ItemSrc<D, EPI, PR> src(P, S, it_begin, it_end, false, true);
  for (int code; (code = src.next()) >= 0;) {
    const Unit u = decode<PR>(P, code);
    if (x >= u.n_heads) continue;  // single-head unit: WG B idles
    const WorkItem& w = u.w;
    const bool valid = r < w.n_rows;
    const int64_t row = static_cast<int64_t>(w.row0) + r;
    const int p = valid ? a.pos[row] : 0;
    float m = -INFINITY, l = 0.f;
    bool first = true;
    // tile descriptors one tile ahead: the next tile's (global) load overlaps this tile's
    // sub-tiles instead of sitting between two of them (~150 cycles per tile in CTA-0 traces)
    KvTile tl_next = a.tiles[w.tile_begin];
    int prev_rot = 0;
    for (int t = w.tile_begin; t < w.tile_end; ++t) {
      const KvTile tl = tl_next;
      if (t + 1 < w.tile_end) tl_next = a.tiles[t + 1];
      const int nsub = tl.n_valid > 64 ? 2 : 1;
      const bool new_epoch = t == w.tile_begin || tl.rot_delta != prev_rot;
      prev_rot = tl.rot_delta;
      if (J && new_epoch) {
        // a new epoch: this warp has no use for the previous epoch's Q slot (mid-item)
        if (t != w.tile_begin) mbar_arrive(&S.q_empty[x][q_slot(J, ecur)]);
        ecur = eps++;
      }
      for (int hh = 0; hh < nsub; ++hh, ++js) {
        const int buf = js & 1;
        const uint32_t scol = tmem + lane_base + col_s(x, buf);
        const uint32_t pcol = tmem + lane_base + col_p(x, buf);
        // key index i of this sub-tile is visible iff i <= lim
        const int lim = min(tl.n_valid - 1, tl.causal ? p - tl.key_pos0 : kTileKeys - 1) - 64 * hh;
#ifdef SPANQ_SPIN_SOFTMAX
        mbar_wait_spin(&S.s_full[x][buf], (js >> 1) & 1);
#else
        mbar_wait(&S.s_full[x][buf], (js >> 1) & 1);
#endif
        if (tr) trace(P, 2 + x, tc, 30 + (static_cast<int>(js) << 8));  // 30: S ready
        tc_fence_after();
        // masks only on partial sub-tiles
        const bool full = __all_sync(0xffffffffu, lim >= 63);
        float alpha;
        bool resc;
        float sum;
        if (dbg_mode(P) == 1) {  // profiling only: no softmax work (timing of the other roles)
          alpha = 1.f;
          resc = false;
          sum = 1.f;
          m = 0.f;
          if (kSP) {
            tc_fence_before();
            arrive_hand<PR>(&S.s_free[x][buf]);
          }
        } else {
          const int pp_wait = !pp ? 0 : (x == 1 ? 1 : (js > 0 ? 2 : 0));
          sum = full ? softmax_sub<PM, false, PR>(scol, pcol, &S.s_free[x][buf], pp_wait, pp_give, &S.pp_zero, sl2,
                                                  P.rescale_threshold, lim, m, alpha, resc)
                     : softmax_sub<PM, true, PR>(scol, pcol, &S.s_free[x][buf], pp_wait, pp_give, &S.pp_zero, sl2,
                                                 P.rescale_threshold, lim, m, alpha, resc);
        }
        l = l * alpha + sum;
        // O is only touched when a row's running max moved (rare with the threshold): then PV of
        // the previous sub-tile must have landed first. PV(j) commits to o_done[x][j & 1], phase
        // j >> 1; PV(j + 2) cannot complete before this warp releases P(j + 2), so a parity wait
        // is exact even though most phases are never observed.
        if (!first && __any_sync(0xffffffffu, resc)) {
          const uint32_t jp = js - 1;
          mbar_wait(&S.o_done[x][jp & 1], (jp >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
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
        if (tr) trace(P, 2 + x, tc, 31 + (static_cast<int>(js) << 8));  // 31: P written
        tc_fence_before();
        arrive_hand<PR>(&S.p_full[x][buf]);
        first = false;
      }
    }
    if constexpr (EPI) {
      // prefill: LSE straight from the row's thread; 1/l to the epilogue warps (Q prep), which
      // drain O_x while this WG starts the next item. Buffer ni & 1 is rewritten two items
      // later, which needs S of that item, issued only after the next item's first PV — after
      // the epilogue warps arrived o_free, i.e. after they read this buffer
      const float inv = l > 0.f ? 1.f / l : 0.f;
      if (valid && a.lse != nullptr)
        a.lse[row * a.hq + u.head_a + x] = l > 0.f ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
      S.fin_inv[x][ni & 1][r] = inv;
      mbar_arrive(&S.fin_full[x][ni & 1]);
      ++ni;
      continue;
    }
    Finished f;
    f.w = w;
    f.m = m;
    f.l = l;
    f.h = u.head_a + x;
    f.n_heads = u.n_heads;
    f.jlast = js - 1;
    f.elast = ecur;
    epilogue<D, PR>(P, S, ocol, x, f, tc, tr);
  }
  if (pp && x == 0 && js > 0) named_sync(2, 256);  // B's last hand-over
  tc_fence_before();
}

// ------------------------------------------------------------------ warps 12-15: Q prep
// The pre-RoPE q tile of one head (128 rows x d, bf16) is TMA-loaded straight into its Q slot in
// the SWIZZLE_128B K-major layout the MMA reads, then rotated in place: warp wq owns rows
// [32wq, 32wq+32), one row per step, lane l holding elements [l*E, l*E+E) (E = d/32) — its
// rotate-half partner sits in lane l^16 (one shuffle) — with the fp32 (cos, sin) of its pairs
// loaded coalesced from the table, 8 rows per batch. Rows past n_rows are rotated too but never
// stored by the epilogue; rows past the tensor are zero (TMA out-of-bounds fill).
// One step rotates R rows (R = 4 at d=128, 8 at d=64): lane l owns 8 rotate-half pairs
// (i, i + d/2) of row g = l / (32/R): the 16-byte unit u of the first half and the same unit of
// the second half (d=128: the same offset in the second 64-column chunk; d=64: unit u + 4), so
// no shuffles are needed. (cos, sin) of the 8 pairs live in registers.
// (cos, sin) of a lane's 8 pairs are kept as float2 pairs of adjacent pairs — cc[k] = (cos of
// pair 2k, cos of pair 2k+1), ss[k] likewise — the operand layout of the packed fp32x2
// instructions, so the rotation and the angle recurrence need no register shuffles.
template <int D>
__device__ __forceinline__ void rotate_step(uint8_t* qs_base, int r, int u, const float2 (&cc)[4], const float2 (&ss)[4]) {
  uint8_t* p0;
  uint8_t* p1;
  if constexpr (D == 128) {
    p0 = qs_base + r * 128 + ((u ^ (r & 7)) * 16);
    p1 = p0 + TcSmem<D>::kChunkBytes;
  } else {
    p0 = qs_base + r * 128 + ((u ^ (r & 7)) * 16);
    p1 = qs_base + r * 128 + (((u + 4) ^ (r & 7)) * 16);
  }
  const uint4 a = *reinterpret_cast<const uint4*>(p0);
  const uint4 b = *reinterpret_cast<const uint4*>(p1);
  const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
  uint32_t oa[4], ob[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 xx = make_float2(__uint_as_float(av[k] << 16), __uint_as_float(av[k] & 0xFFFF0000u));
    const float2 yy = make_float2(__uint_as_float(bv[k] << 16), __uint_as_float(bv[k] & 0xFFFF0000u));
    // first half: x cos - y sin ; second half: y cos + x sin (packed fp32x2, same roundings)
    const float2 o1 = ffma2(yy, fmul2(ss[k], make_float2(-1.f, -1.f)), fmul2(xx, cc[k]));
    const float2 o2 = ffma2(xx, ss[k], fmul2(yy, cc[k]));
    oa[k] = pack_bf16x2(o1.x, o1.y);
    ob[k] = pack_bf16x2(o2.x, o2.y);
  }
  *reinterpret_cast<uint4*>(p0) = make_uint4(oa[0], oa[1], oa[2], oa[3]);
  *reinterpret_cast<uint4*>(p1) = make_uint4(ob[0], ob[1], ob[2], ob[3]);
}

// the (cos, sin) table entries of 8 consecutive pairs, regrouped into cos / sin pairs
__device__ __forceinline__ void load_cs8(const float2* rope, int64_t idx, float2 (&cc)[4], float2 (&ss)[4]) {
  const float4* t = reinterpret_cast<const float4*>(rope + idx);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float4 v = __ldg(t + e);  // (cos i, sin i, cos i+1, sin i+1)
    cc[e] = make_float2(v.x, v.z);
    ss[e] = make_float2(v.y, v.w);
  }
}

template <int D>
__device__ __forceinline__ void rotate_q_tile(uint8_t* qs_base, const float2* rope, int my_pos, int my_valid, int rot,
                                              int max_pos, const TcParams* tp = nullptr, uint32_t* tc = nullptr) {
  constexpr int kLanesPerRow = D / 16;       // 8 pairs per lane
  constexpr int R = 32 / kLanesPerRow;       // rows per step
  const int lane = threadIdx.x & 31;
  const int wq = (threadIdx.x / 32) & 3;
  const int g = lane / kLanesPerRow, u = lane % kLanesPerRow;
  const int pair0 = u * 8;
  const int p_first = __shfl_sync(0xffffffffu, my_pos, 0);
  // rows of a tile normally have consecutive positions (a job's rows, a query's cross rows):
  // then (cos, sin) advance by R*theta per step — 4 FMAs per pair (fp32, <= 7 steps from a
  // table value: ~1e-6 drift vs bf16's 4e-3) instead of a table row per row.
  const bool consecutive = __all_sync(0xffffffffu, !my_valid || my_pos == p_first + lane) && p_first - rot >= 0 &&
                           p_first - rot + 31 < max_pos;
  float2 cc[4], ss[4];
  if (tp != nullptr && lane == 0) trace(*tp, 4, *tc, consecutive ? 46 : 47);  // 46/47: rotation (fast/slow path)
  if (consecutive) {
    float2 cd[4], sd[4];
    load_cs8(rope, static_cast<int64_t>(p_first - rot + g) * (D / 2) + pair0, cc, ss);
    load_cs8(rope, static_cast<int64_t>(R) * (D / 2) + pair0, cd, sd);  // position R: (cos R th, sin R th)
    float2 sdn[4];
    if (tp != nullptr && lane == 0) trace(*tp, 4, *tc, 48 + (__float_as_int(cc[0].x) == 0x7fffffff));  // 48: table read
#pragma unroll
    for (int e = 0; e < 4; ++e) sdn[e] = fmul2(sd[e], make_float2(-1.f, -1.f));
    // rolled: the unrolled 8-step body is ~8 KB of SASS, and a cold instruction cache made the
    // first rotation of a launch ~10K cycles (CTA-0 trace of a C2 join)
#pragma unroll 1
    for (int st = 0; st < 32 / R; ++st) {
      rotate_step<D>(qs_base, wq * 32 + st * R + g, u, cc, ss);
#pragma unroll
      for (int e = 0; e < 4; ++e) {  // advance the angles by R*theta (packed, same roundings)
        const float2 cn = ffma2(cc[e], cd[e], fmul2(ss[e], sdn[e]));  // c cosR - s sinR
        ss[e] = ffma2(ss[e], cd[e], fmul2(cc[e], sd[e]));            // s cosR + c sinR
        cc[e] = cn;
      }
    }
  } else {
#pragma unroll 1
    for (int st = 0; st < 32 / R; ++st) {
      const int p = __shfl_sync(0xffffffffu, my_pos, st * R + g);
      const int rp = min(max(p - rot, 0), max_pos - 1);
      load_cs8(rope, static_cast<int64_t>(rp) * (D / 2) + pair0, cc, ss);
      rotate_step<D>(qs_base, wq * 32 + st * R + g, u, cc, ss);
    }
  }
}

template <int D, bool EPI, bool PR>
__device__ void run_qprep(const TcParams& P, TcSmem<D, PR>& S, int it_begin, int it_end) {
  const AttnArgs& a = P.a;
  const bool J = P.join != 0;
  const int r = threadIdx.x & 127;
  const int lane = threadIdx.x & 31;
  const int wq = (threadIdx.x / 32) & 3;
  constexpr uint32_t kQBytes = 128 * D * 2;
  uint32_t ep = 0;
  uint32_t tc = 0;
  uint32_t load_phase = 0;  // bit 2x + s: parity of the next q_load[x][s] completion
  const bool tr = lane == 0;
  ItemSrc<D, EPI, PR> src(P, S, it_begin, it_end, false, true);
  const bool early_b = (P.qprep_mode & 1) != 0, prefetch = (P.qprep_mode & 2) != 0;
  // thread 0: TMA of head x's pre-RoPE tile into its slot of epoch ep
  auto load = [&](int x, const Unit& u) {
    uint64_t* bar = &S.q_load[x][q_slot(J, ep)];
    uint8_t* dst = q_tile<D, PR>(S, J, x, ep);
    mbar_arrive_expect_tx(bar, kQBytes);
#pragma unroll
    for (int c = 0; c < D / 64; ++c)
      tma_load_3d(dst + c * TcSmem<D>::kChunkBytes, &P.tmq, bar, c * 64, u.head_a + x, u.w.row0);
  };
  int code = src.next();
  while (code >= 0) {
    const Unit u = decode<PR>(P, code);
    const WorkItem& w = u.w;
    const int my_row = wq * 32 + lane;  // this lane's row position, shuffled to the warp per row
    const int my_pos = my_row < w.n_rows ? a.pos[static_cast<int64_t>(w.row0) + my_row] : 0;
    const bool work = dbg_mode(P) != 5;
    for (int t = w.tile_begin; t < w.tile_end; ++t) {
      const int rot = a.tiles[t].rot_delta;
      if (t > w.tile_begin && rot == a.tiles[t - 1].rot_delta) continue;
      // warp 12 (converged: a warp never splits across two long waits) waits for slot A and its
      // lane 0 issues head A's load, and head B's right away if slot B is already free too (both
      // loads then overlap A's rotation); the other warps only wait for the data
      const int sl = q_slot(J, ep);
      const uint32_t epar = q_par(J, ep) ^ 1;
      bool b_issued = false;  // (warp 12 only, warp-uniform)
      if (wq == 0) {
        mbar_wait(&S.q_empty[0][sl], epar);
        if (tr) trace(P, 4, tc, 40);  // 40: slot free for head A
        if (work && lane == 0) load(0, u);
        if (work && early_b && u.n_heads == 2) {
          const bool free_b = lane == 0 && mbar_try_wait(&S.q_empty[1][sl], epar);
          b_issued = __shfl_sync(0xffffffffu, free_b, 0);
          if (b_issued && lane == 0) load(1, u);
        }
        __syncwarp();
      }
      // an unpaired launch never touches slot B: no issuer waits on it, and waiting on its empty
      // barrier (committed once per epoch by the A issuer) could be lapped — the A issuer can
      // finish a one-sub-tile epoch and complete the next phase before a late warp arrives, and
      // a parity wait then blocks on a phase that needs this warp's next Q (a deadlock)
      for (int x = 0; x < u.n_heads; ++x) {
        if (work) {
          if (x == 1 && wq == 0 && !b_issued) {
            mbar_wait(&S.q_empty[1][sl], epar);
            if (tr) trace(P, 4, tc, 41);  // 41: slot free for head B
            if (lane == 0) load(1, u);
            __syncwarp();
          }
          // the load is issued only once the slot is free, so its completion implies that
          const int bit = 2 * x + sl;
          mbar_wait(&S.q_load[x][sl], (load_phase >> bit) & 1);
          load_phase ^= 1u << bit;
          if (tr) trace(P, 4, tc, 44 + x);  // 44/45: Q tile A/B loaded
          rotate_q_tile<D>(q_tile<D, PR>(S, J, x, ep), a.rope, my_pos, my_row < w.n_rows, rot, a.max_pos, &P, &tc);
          fence_proxy_async_smem();
        } else {
          mbar_wait(&S.q_empty[x][sl], epar);
        }
        if (tr) trace(P, 4, tc, 42 + x);  // 42/43: Q tile A/B written
        arrive_lead_warp<PR>(&S.q_full[x][sl]);
      }
      ++ep;
    }
    // the next item's code is known long before its Q slots free: warm L2 with its q tiles
    code = src.next();
    if (prefetch && code >= 0 && r == 0 && work) {
      const Unit n = decode<PR>(P, code);
      for (int x = 0; x < n.n_heads; ++x)
#pragma unroll
        for (int c = 0; c < D / 64; ++c) tma_prefetch_3d(&P.tmq, c * 64, n.head_a + x, n.w.row0);
    }
    __syncwarp();
  }
}

// Prefill launches (paired heads): Q prep through a 2-deep ring (item k in slot k & 1, prepared
// while item k - 1 runs: the rotation is off the item boundary) and the epilogue of every item
// (prefill_epilogue, staged in that item's own slot). Order: Q(0); then per item k: Q(k+1), the
// epilogue of k. Q(k+1) waits for slot (k+1) & 1, released by the epilogue of k - 1 (done in the
// previous iteration) and item k - 1's last S MMA; the epilogue of k waits for item k's last PV.
template <int D, bool EPI, bool PR>
__device__ void run_qprep_epi(const TcParams& P, TcSmem<D, PR>& S, uint32_t tmem, int it_begin, int it_end) {
  const AttnArgs& a = P.a;
  const int lane = threadIdx.x & 31;
  const int wq = (threadIdx.x / 32) & 3;
  constexpr uint32_t kQBytes = 128 * D * 2;
  uint32_t tc = 0;
  uint32_t load_phase = 0;  // bit 2x + s: parity of the next q_load[x][s] completion
  const bool tr = lane == 0;
  ItemSrc<D, EPI, PR> src(P, S, it_begin, it_end, false, true);
  const int my_row = wq * 32 + lane;
  // prepare the (single-epoch) Q tiles of item e in slot e & 1
  auto prep = [&](const Unit& u, uint32_t e) {
    const WorkItem& w = u.w;
    const int sl = static_cast<int>(e & 1);
    const uint32_t epar = ((e >> 1) & 1) ^ 1;
    const int my_pos = my_row < w.n_rows ? a.pos[static_cast<int64_t>(w.row0) + my_row] : 0;
    if (wq == 0) {
      // warp 12 waits for both slots (converged), lane 0 issues both loads (they overlap A's rotation)
      for (int x = 0; x < u.n_heads; ++x) {
        mbar_wait(&S.q_empty[x][sl], epar);
        if (tr) trace(P, 4, tc, 40 + x);  // 40/41: slot free for head A/B
        if (lane == 0) {
          uint64_t* bar = &S.q_load[x][sl];
          uint8_t* dst = q_tile<D, PR>(S, true, x, e);
          mbar_arrive_expect_tx(bar, kQBytes);
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
#ifdef SPANQ_L2HINT  // q rows are read once
            tma_load_3d_hint(dst + c * TcSmem<D>::kChunkBytes, &P.tmq, bar, c * 64, u.head_a + x, w.row0,
                             policy_evict_first());
#else
            tma_load_3d(dst + c * TcSmem<D>::kChunkBytes, &P.tmq, bar, c * 64, u.head_a + x, w.row0);
#endif
          }
        }
        __syncwarp();
      }
    }
    for (int x = 0; x < u.n_heads; ++x) {
      const int bit = 2 * x + sl;
      mbar_wait(&S.q_load[x][sl], (load_phase >> bit) & 1);
      load_phase ^= 1u << bit;
      if (tr) trace(P, 4, tc, 44 + x);  // 44/45: Q tile A/B loaded
      rotate_q_tile<D>(q_tile<D, PR>(S, true, x, e), a.rope, my_pos, my_row < w.n_rows, 0, a.max_pos);
      fence_proxy_async_smem();
      if (tr) trace(P, 4, tc, 42 + x);  // 42/43: Q tile A/B written
      arrive_lead_warp<PR>(&S.q_full[x][sl]);
    }
  };
  int code = src.next();
  if (code < 0) return;
  Unit cur = decode<PR>(P, code);
  uint32_t jtot = static_cast<uint32_t>(cur.w.n_sub);
  uint32_t cur_jlast = jtot - 1;
  prep(cur, 0);
  for (uint32_t k = 0;; ++k) {
    code = src.next();
    const bool more = code >= 0;
    Unit nxt{};
    uint32_t nxt_jlast = 0;
    if (more) {
      nxt = decode<PR>(P, code);
      jtot += static_cast<uint32_t>(nxt.w.n_sub);
      nxt_jlast = jtot - 1;
      prep(nxt, k + 1);
    }
    prefill_epilogue<D, PR>(P, S, tmem, cur, cur_jlast, k, tc);
    if (!more) break;
    cur = nxt;
    cur_jlast = nxt_jlast;
  }
}

// PR: a CTA pair (cluster of 2 on one TPC, cta_group::2 MMAs issued by the leader); each CTA
// initialises every barrier, the leader's copies of q_full / p_full / o_free / sched_empty count
// both CTAs' arrivals
template <int D, int PM, bool EPI, bool PR>
__global__ void __launch_bounds__(kThreads, 1) span_attn_tc_kernel(const __grid_constant__ TcParams P) {
  extern __shared__ uint8_t smem_raw[];
  TcSmem<D, PR>& S = smem_ref<D, PR>(smem_raw);
  const int warp = threadIdx.x / 32;
  const uint32_t rank = PR ? cluster_rank() : 0;
  constexpr uint32_t kBoth = PR ? 2 : 1;  // CTAs arriving on a leader barrier
  // arrivals of a 128-thread role on a leader barrier: one per thread, or in a pair one per warp
  // of each CTA (arrive_lead_warp)
  constexpr uint32_t kRole = PR ? 4 * 2 : 128;
  if (threadIdx.x == 0) {
    for (int kv = 0; kv < 2; ++kv)
      for (int i = 0; i < TcSmem<D, PR>::kKSlots; ++i) {
        mbar_init(&S.kv_full[kv][i], 1);
        mbar_init(&S.kv_empty[kv][i], P.paired ? 2 : 1);  // released by each head's issuer
      }
    for (int i = 0; i < TcSmem<D, PR>::kQSlots; ++i)
      for (int sl = 0; sl < 2; ++sl) {
        mbar_init(&S.q_full[i][sl], kRole);
        // 2-deep ring: + the 128 threads whose epilogue stages in the slot (join: softmax WG of
        // head i, prefill: the Q-prep warps)
        mbar_init(&S.q_empty[i][sl], (EPI || P.join) ? 1 + 128 : 1);
        mbar_init(&S.q_load[i][sl], 1);
      }
    for (int i = 0; i < 2; ++i) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(&S.s_full[i][b], 1);
        mbar_init(&S.p_full[i][b], kHandCount(PR));
        mbar_init(&S.s_free[i][b], kHandCount(PR));
      }
      mbar_init(&S.o_done[i][0], 1);
      mbar_init(&S.sched_full[2 * i], 1);
      mbar_init(&S.sched_full[2 * i + 1], 1);
      mbar_init(&S.sched_empty[2 * i], PR ? kSchedConsumersPair : kSchedConsumers);
      mbar_init(&S.sched_empty[2 * i + 1], PR ? kSchedConsumersPair : kSchedConsumers);
      mbar_init(&S.o_done[i][1], 1);
      mbar_init(&S.o_free[i], kRole);  // every epilogue (Q-prep) thread (a pair: warp)
      mbar_init(&S.fin_full[i][0], 128);
      mbar_init(&S.fin_full[i][1], 128);
    }
    S.pp_zero = 0.f;
    fence_barrier_init();
  }
  if (warp == 0 && (threadIdx.x & 31) == 0) {
    tma_prefetch_desc(PR ? &P.tmk2 : &P.tmk);
    tma_prefetch_desc(&P.tmv);
    tma_prefetch_desc(&P.tmq);
  }
  if (warp == 2) {
    if constexpr (PR)
      tmem_alloc2<kTmemCols>(&S.tmem_base);
    else
      tmem_alloc<kTmemCols>(&S.tmem_base);
  }
  tc_fence_before();
  if constexpr (PR)
    cluster_sync_all();  // both CTAs' barriers are initialised before any remote arrive
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  const bool dyn = P.a.sched != nullptr;
  const int it_begin = dyn ? 0 : P.a.cta_off[blockIdx.x], it_end = dyn ? 0 : P.a.cta_off[blockIdx.x + 1];
#ifdef SPANQ_PROFILING
  if (P.a.dbg_trace != nullptr && threadIdx.x == 0) {  // profiling only: per-CTA start (ns)
    uint64_t g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    P.a.dbg_trace[kTraceWarps * 2048 + 2 * blockIdx.x] = static_cast<long long>(g);
  }
#endif
  // register budget 65536 >= 128 x (56 + 160 + 160 + 120): TMA/MMA warps need few
  if (warp < 4) {
    reg_dealloc<56>();
    if (warp == 0 || warp == 3) {
      if (elect_one()) run_producer<D, EPI, PR>(P, S, it_begin, it_end, warp == 0 ? 0 : 1);
    } else if (rank == 0) {  // a pair: the leader issues the MMAs of both CTAs
      if (elect_one()) run_mma<D, EPI, PR>(P, S, tmem, it_begin, it_end, warp - 1);
    }
  } else if (warp < 12) {
    reg_alloc<160>();
    run_softmax<D, PM, EPI, PR>(P, S, tmem, it_begin, it_end, warp < 8 ? 0 : 1);
  } else {
    reg_dealloc<120>();
    if constexpr (EPI)
      run_qprep_epi<D, EPI, PR>(P, S, tmem, it_begin, it_end);
    else
      run_qprep<D, EPI, PR>(P, S, it_begin, it_end);
  }
  if (warp >= 4 && (threadIdx.x & 31) == 0) bulk_wait<0>();  // epilogue stores done
  tc_fence_before();
  if constexpr (PR)
    cluster_sync_all();  // neither CTA leaves while the other may still touch its smem / TMEM
  else
    __syncthreads();
  if (P.a.sched != nullptr && threadIdx.x == 0 && rank == 0) {
    // the last CTA (pair) to finish (all claims of all CTAs are done) resets the counters for the
    // next launch of this work list
    __threadfence();
    if (atomicAdd(P.a.sched + 1, 1) == static_cast<int>(gridDim.x / kBoth) - 1) {
      P.a.sched[0] = 0;
      P.a.sched[1] = 0;
      __threadfence();
    }
  }
#ifdef SPANQ_PROFILING
  if (P.a.dbg_trace != nullptr && threadIdx.x == 0) {  // profiling only: per-CTA end (ns)
    uint64_t g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    P.a.dbg_trace[kTraceWarps * 2048 + 2 * blockIdx.x + 1] = static_cast<long long>(g);
  }
#endif
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PR)
      tmem_dealloc2<kTmemCols>(tmem);
    else
      tmem_dealloc<kTmemCols>(tmem);
  }
}

template <int D, int PM, bool EPI, bool PR = false>
cudaError_t launch_dp(const AttnArgs& a, cudaStream_t st) {
  // the large-smem attribute is per device: one bit per device ordinal that has it set
  static std::atomic<uint64_t> attr_set{0};
  const int smem = static_cast<int>(sizeof(TcSmem<D, PR>));
  static_assert(sizeof(TcSmem<D, PR>) <= 232448, "shared memory budget (227 KB per CTA)");
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load() & bit)) {
    e = cudaFuncSetAttribute(span_attn_tc_kernel<D, PM, EPI, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit);
  }
  TcParams p;
  p.tmk = *a.tmap_k;
  if (PR) p.tmk2 = *a.tmap_k2;
  p.tmv = *a.tmap_v;
  p.tmq = *a.tmap_q;
  if (a.tmap_o) p.tmo = *a.tmap_o;
  if (a.tmap_op) p.tmop = *a.tmap_op;
  p.a = a;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  p.paired = a.paired ? 1 : 0;
  p.poly_mask = PM;
  p.rescale_threshold = a.rescale_threshold;
  p.dbg_mode = a.dbg_mode;
  p.qprep_mode = 3;
  // joins of paired launches: 2-deep Q ring per head in the staging area
  p.join = a.paired && a.join ? 1 : 0;
  p.epi_q = EPI ? 1 : 0;
  // launched as a programmatic dependent of the preceding K1 when the caller says it directly
  // precedes (a.pdl; the ctx option SPQ_OPT_PDL = 0 turns it off): the prologue and Q
  // preparation overlap K1's tail (see run_producer)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(a.grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (a.pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (PR) {  // CTA pairs: clusters of 2 (one TPC each)
    if (a.grid % 2 != 0) return cudaErrorInvalidValue;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, span_attn_tc_kernel<D, PM, EPI, PR>, p);
}

template <int D>
cudaError_t launch_d(const AttnArgs& a, cudaStream_t st) {
  // Q-prep-warp epilogue + 2-deep Q ring (a separate kernel instance, EPI) for the prefill
  // launches where it measured faster: bf16 O (C2 prefill 0.270 -> 0.256 ms) and d = 64 (C4
  // 0.311 -> 0.296 ms); fp32 O at d = 128 keeps the softmax-WG epilogue (its fp32 drain cycles
  // through 2 x 4 KB per warp of the Q slot, and measured 0.255 vs 0.247 ms)
  const bool epi = a.paired && !a.join && (!a.out_fp32 || D == 64);
  if (a.cluster == 2) {
    // CTA-pair kernel (d = 128 prefill with bf16 O, GQA groups of 4k): work codes are 4-head units
    // (exp2: MUFU fp32 or f16x2 only)
    if constexpr (D == 128) {
      if (!epi || a.tmap_k2 == nullptr || (a.hq / a.hkv) % 4 != 0) return cudaErrorInvalidValue;
      return a.poly_mask != 3 ? launch_dp<D, 0, true, true>(a, st) : launch_dp<D, 3, true, true>(a, st);
    }
    return cudaErrorInvalidValue;
  }
  // a quarter / half of the exponentials on the FMA pipe
  if (a.poly_mask == 1) return epi ? launch_dp<D, 1, true>(a, st) : launch_dp<D, 1, false>(a, st);
  if (a.poly_mask == 2) return epi ? launch_dp<D, 2, true>(a, st) : launch_dp<D, 2, false>(a, st);
  // exp2: 0 = MUFU ex2 (fp32), else MUFU ex2.f16x2 (two exponentials per op)
  if (a.poly_mask == 0) return epi ? launch_dp<D, 0, true>(a, st) : launch_dp<D, 0, false>(a, st);
  return epi ? launch_dp<D, 3, true>(a, st) : launch_dp<D, 3, false>(a, st);
}

}  // namespace

cudaError_t launch_span_attn_tc(const AttnArgs& a, cudaStream_t st) {
  if (a.n_items == 0 || a.grid == 0) return cudaSuccess;
  if (a.bs < 16 || a.bs > 128 || (a.bs & (a.bs - 1)) != 0) return cudaErrorInvalidValue;
  if (a.paired && (a.hq / a.hkv) % 2 != 0) return cudaErrorInvalidValue;
  switch (a.d) {
    case 64: return launch_d<64>(a, st);
    case 128: return launch_d<128>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace spq
