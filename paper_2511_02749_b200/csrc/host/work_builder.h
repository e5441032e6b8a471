// work_builder.h — turn a plan's segments into attention work lists.
#pragma once
#include <cstdint>
#include <vector>

#include "../kernels/work.h"
#include "planner.h"

namespace spq {

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
  double flops = 0;  // algorithmic 4·d·Hq·visible pairs
};

struct WorkOpts {
  int hq, d, bs;
  int num_sms;       // persistent grid upper bound
  bool allow_split;  // split-KV (join only)
  bool persistent;   // build per-CTA LPT lists
  int units;         // work units per item: hq (one head each) or hq/2 (GQA head pairs)
};

// Prefill jobs [job_begin, job_end): rows relative to job_row_off[job_begin].
void build_prefill_work(const PlanHost& p, const WorkOpts& o, int job_begin, int job_end,
                        AttnWorkHost* w);
// Joins of queries [q_begin, q_end): rows relative to query_join_row_off[q_begin].
void build_join_work(const PlanHost& p, const WorkOpts& o, int q_begin, int q_end, AttnWorkHost* w);

}  // namespace spq
