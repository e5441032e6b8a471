// work_builder.h — turn a plan's segments into attention work lists.
#pragma once
#include <cstdint>
#include <map>
#include <utility>
#include <vector>

#include "../kernels/work.h"
#include "planner.h"

namespace spq {

struct DecodeItemHost {
  int32_t row, kvh, tile_begin, tile_end, part;  // mirrors kernels/launch.h DecodeItem
  int32_t n_chunks, part0, pair;                 // (row, kv head): chunks, first partial, index
};

struct AttnWorkHost {
  std::vector<KvTile> tiles;
  std::vector<int32_t> tile_blocks;
  std::vector<WorkItem> items;
  std::vector<int32_t> cta_off;    // [grid+1] static schedule (unused when dynamic)
  std::vector<int32_t> cta_items;  // item * units + unit: per CTA in execution order (static), or
                                   // one global list in claim order (dynamic)
  bool dynamic = false;            // CTAs claim codes from cta_items with an atomic counter
  std::vector<CombineDesc> combine;
  int32_t n_parts = 0;
  int32_t grid = 0;
  int32_t cluster = 1;  // 2: CTA-pair launch (codes are 4-head units, grid even)
  double flops = 0;  // algorithmic 4·d·Hq·visible pairs
};

struct WorkOpts {
  int hq, d, bs;
  int num_sms;       // persistent grid upper bound
  bool allow_split;  // split-KV (join only)
  bool persistent;   // build per-CTA LPT lists
  int units;         // work units per item: hq (one head each), hq/2 (GQA head pairs) or hq/4
                     // (CTA pairs: 4 heads of a GQA group, cluster = 2)
  int cluster = 1;   // CTAs per cluster of the launch (grid a multiple of it)
};

// Prefill jobs [job_begin, job_end): rows relative to job_row_off[job_begin].
void build_prefill_work(const PlanHost& p, const WorkOpts& o, int job_begin, int job_end,
                        AttnWorkHost* w);
// W > 1 joins in two launches around the fragment-KV exchange: sel 1 = the
// segments this rank holds (prefix, local fragments, cross), sel 2 = the received fragments.
// remote[s] marks plan segment s as received. A query with received fragments writes partials
// in both phases (ranges[(row0, unit)] = its phase-1 (first slot, count)), merged by phase 2's
// combine list; partial slots of phase 2 start at part_base (= phase 1's n_parts).
struct JoinPhase {
  int sel;
  const std::vector<uint8_t>& remote;
  int32_t part_base;
  std::map<std::pair<int32_t, int32_t>, std::pair<int32_t, int32_t>>* ranges;
};

// Joins of queries [q_begin, q_end): rows relative to query_join_row_off[q_begin]. ph == null: one
// launch over every segment.
void build_join_work(const PlanHost& p, const WorkOpts& o, int q_begin, int q_end, AttnWorkHost* w,
                     const JoinPhase* ph = nullptr);
// Algorithmic FLOPs of the join of queries [q_begin, q_end) (the `flops` build_join_work reports,
// without building the work list): 4·d·Hq per visible (cross row, key) pair
double join_flops(const PlanHost& p, const WorkOpts& o, int q_begin, int q_end);

// Owner-side split join: the plan's tasks — each a home query's cross rows
// (rows in task order, packed) over the fragments of it owned here at Δ_f — as one join work list.
void build_task_join_work(const PlanHost& p, const WorkOpts& o, AttnWorkHost* w);

// Decode after the join: the KV tiles of one home query for its generated
// rows — prefix (non-causal), fragments at Δ_f (non-causal, Q counter-rotated), then the cross +
// generated tokens as one causal segment of gen_ctx tokens over `cross_gen_blocks` — split per kv
// head into chunks of <= chunk_tiles tiles (K9 items; a (row, kv head) with several chunks writes
// partials merged by combine, rows_per_part = 1).
struct DecodeWorkHost {
  std::vector<KvTile> tiles;
  std::vector<int32_t> tile_blocks;
  std::vector<DecodeItemHost> items;
  std::vector<CombineDesc> combine;
  int32_t n_parts = 0;
};
// Tiles of one decode row, appended to w; returns [first, end) tile range.
std::pair<int32_t, int32_t> decode_row_tiles(const PlanHost& p, int32_t query, const std::vector<int32_t>& cross_gen_blocks,
                                             int32_t gen_ctx, int bs, DecodeWorkHost* w);
// Items for rows whose tile ranges are given: chunks of <= chunk_tiles per (row, kv head).
void decode_items(const std::vector<std::pair<int32_t, int32_t>>& row_tiles, int hkv, int group, int chunk_tiles,
                  DecodeWorkHost* w);

}  // namespace spq
