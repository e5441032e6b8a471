// launch.h — host-side launchers of the device kernels (called by the C-ABI layer only).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "work.h"

// K9 bf16 decode: per-warp ring depth (16-key K / V groups in flight + 1 being consumed); the host
// sizes decode chunks for one wave of resident CTAs from the same constant
#ifndef SPQ_DEC_STAGES
#define SPQ_DEC_STAGES 2
#endif
constexpr int kDecStages = SPQ_DEC_STAGES;

namespace spq {

struct KvWriteArgs {
  const void* k;  // [rows][hkv][d] pre-RoPE
  const void* v;
  const int32_t* pos;
  const int64_t* slot;
  int64_t rows;
  const int64_t* pad_slots;
  int64_t n_pad;
  void* k_pool;
  void* v_pool;
  int hkv, d, bs;
  int64_t nblk;
  int layer;
  const float2* rope;
  bool fp32;
};
cudaError_t launch_rope_kv_write(const KvWriteArgs& a, cudaStream_t st);

struct AttnArgs {
  // work list (device)
  const KvTile* tiles;
  const int32_t* tile_blocks;
  const WorkItem* items;
  int32_t n_items;
  const int32_t* cta_off;  // persistent schedule (tcgen05 kernel): static per-CTA lists, or
  const int32_t* cta_items;
  int32_t grid;
  int32_t* sched;          // dynamic: {next, done} claim counters (zero between launches), or null
  int32_t n_codes;         // dynamic: codes in cta_items
  // rows
  const int32_t* pos;  // [rows] position of each query row
  const void* q;       // [rows][hq][d]
  void* o;             // [rows][hq][d]
  float* lse;          // [rows][hq] or null
  float* opart;        // [parts][hq][128][d] fp32
  float* lsepart;      // [parts][hq][128]
  // pools
  const void* k_pool;
  const void* v_pool;
  const CUtensorMap* tmap_k;  // host copies (bf16 path)
  const CUtensorMap* tmap_k2; // K with boxes of min(bs, 32) rows (CTA-pair kernel), or null
  const CUtensorMap* tmap_v;
  const CUtensorMap* tmap_q;  // per call: q [rows][hq][d] as 3D {d, hq, rows}, box {64, 1, 128}
  const CUtensorMap* tmap_o;  // per call (fp32 o): 3D {d, hq, rows}, box {32, 1, 32}, SWIZZLE_128B
  const CUtensorMap* tmap_op; // per plan (fp32 partials): 2D {d, parts*hq*128}, box {32, 32}
  int hq, hkv, d, bs;
  int64_t nblk;
  int layer;
  const float2* rope;
  int max_pos;
  bool out_fp32;  // o is fp32 (else ctx dtype)
  bool paired;    // tcgen05 path: work codes are (item, GQA head pair) — see span_attn_tc.cu
  int cluster;    // tcgen05 path: 2 = CTA-pair kernel, codes are (item, 4-head unit), grid even
  bool join;      // tcgen05 path: a join launch (2-deep Q ring, epilogue staged in Q slots)
  bool pdl;       // tcgen05 path: launch as a programmatic dependent of the preceding K1
  int poly_mask;  // tcgen05 path: exp2 on MUFU: 0 = ex2 fp32, else ex2.f16x2 (SPQ_OPT_EXP2)
  float rescale_threshold;  // tcgen05 path: conditional O rescale threshold (log2 units, 8)
  long long* dbg_trace;     // profiling builds only: CTA-0 event timeline (null = off)
  int dbg_mode;             // profiling builds only: timing variants (0 = off)
};
cudaError_t launch_span_attn_tc(const AttnArgs& a, cudaStream_t st);   // bf16 tcgen05
cudaError_t launch_span_attn_f32(const AttnArgs& a, cudaStream_t st);  // fp32 SIMT

struct CombineArgs {
  const CombineDesc* desc;
  int32_t n_desc;
  const float* opart;
  const float* lsepart;
  void* o;
  float* lse;
  int hq, d;
  int heads_per_desc;  // max CombineDesc::n_heads
  int rows_per_part;   // rows of one (partial slot, head): kTileRows (joins) or 1 (decode)
  bool out_fp32;
  bool pdl;  // launch as a programmatic dependent of the join kernel right before it
};

// K9 decode (decode.cu): one work item = (home query row, kv head, chunk of KV tiles)
struct DecodeItem {
  int32_t row, kvh, tile_begin, tile_end, part;  // part -1: write o / lse directly
  int32_t n_chunks, part0, pair;                 // (row, kv head): chunks, first partial, index
};
struct DecodeArgs {
  const DecodeItem* items;
  int32_t n_items;
  const KvTile* tiles;
  const int32_t* tile_blocks;
  const int32_t* pos_base;  // [rows] N_q: position of generated token 0
  int32_t step;             // generated token t: the row sits at pos_base + t
  const void* q;            // [rows][hq][d] pre-RoPE, pool dtype
  void* o;                  // [rows][hq][d] out dtype
  float* lse;               // [rows][hq] or null
  float* opart;             // [parts][g][d]
  float* lsepart;           // [parts][g]
  int32_t* done;            // bf16 path: [rows * hkv] chunks finished per (row, kv head), zero
                            // between launches (the last chunk merges the partials and resets it)
  const void* k_pool;
  const void* v_pool;
  const float2* rope;
  int max_pos;
  int hq, hkv, d, bs;
  int64_t nblk;
  int layer;
  bool fp32, out_fp32;
};
cudaError_t launch_decode(const DecodeArgs& a, cudaStream_t st);

// owner-side split join (split_join.cu): K10 row gather (Q send buffer) and K11 merge
cudaError_t launch_gather_rows(const int32_t* rows, int64_t n, const void* src, void* dst, int64_t row_bytes,
                               int num_sms, cudaStream_t st);
struct SplitMergeDesc {  // one home query: join rows [row0, row0 + n_rows), partial sources
  int64_t row0;
  int32_t n_rows, src_begin, src_end, pad;  // merge_src[src_begin, src_end): first partial row per owner
};
struct SplitMergeArgs {
  const SplitMergeDesc* desc;
  int32_t n_desc;
  const int64_t* src;   // [..] row offsets into o_rem / lse_rem
  const float* o_loc;   // [rows][hq][d] local join (normalized), fp32
  const float* lse_loc; // [rows][hq]
  const float* o_rem;   // [recv rows][hq][d] owners' partials (normalized), fp32
  const float* lse_rem; // [recv rows][hq]
  void* o;              // [rows][hq][d] out dtype
  float* lse;           // [rows][hq] or null
  int hq, d, num_sms;
  int64_t total_rows;
  bool out_fp32;
};
cudaError_t launch_merge_split(const SplitMergeArgs& a, cudaStream_t st);
cudaError_t launch_combine(const CombineArgs& a, cudaStream_t st);

struct KvExchangeArgs {
  const int32_t* blocks;  // device [n] block ids
  int64_t n;
  void* k_pool;
  void* v_pool;
  void* buf;  // device [n][2][Hkv*bs*d] elements
  int hkv, bs, d, elt, layer, num_sms;
  int64_t nblk;
  int scatter;  // 0: pool -> buf (pack), 1: buf -> pool (unpack)
};
cudaError_t launch_kv_exchange(const KvExchangeArgs& a, cudaStream_t st);

struct CidraArgs {
  const int4* ops;         // device [n_ops] {dst, src, delta, mode} (host/cidra.h)
  const int32_t* comp_off; // device [n_comp + 1]
  int32_t n_comp;
  void* k_pool;
  void* v_pool;
  const float2* rope;      // [max_pos][d/2] (cos, sin)
  int hkv, d, bs;
  int64_t nblk;
  int layer_begin, layer_end;
  bool fp32;
  int num_sms;
};
cudaError_t launch_cidra(const CidraArgs& a, cudaStream_t st);  // in-place repositioning (K8)

}  // namespace spq
