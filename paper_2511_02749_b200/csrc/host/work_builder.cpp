// work_builder.cpp — see work_builder.h.
#include "work_builder.h"

#include <algorithm>
#include <cmath>

namespace spq {
namespace {

// Append the KV tiles of one segment; returns the index of its first tile.
int32_t add_tiles(const PlanHost& p, const Segment& s, int bs, int32_t key_base, int32_t rot,
                  int32_t causal, AttnWorkHost* w) {
  const int32_t first = static_cast<int32_t>(w->tiles.size());
  const int bpt = kTileKeys / bs;
  for (int32_t t0 = 0; t0 < s.tok_len; t0 += kTileKeys) {
    KvTile k{};
    k.blk_off = static_cast<int32_t>(w->tile_blocks.size());
    k.n_valid = std::min(kTileKeys, s.tok_len - t0);
    k.key_pos0 = key_base + t0;
    k.rot_delta = rot;
    k.causal = causal;
    const int32_t b0 = t0 / bs;
    const int32_t nb = (k.n_valid + bs - 1) / bs;
    for (int j = 0; j < bpt; ++j) w->tile_blocks.push_back(p.blocks[s.block_off + b0 + std::min(j, nb - 1)]);
    w->tiles.push_back(k);
  }
  return first;
}

// Static schedule of (item, head) pairs over `grid` persistent CTAs: pairs sorted by cost
// (longest first, heads of one item adjacent so a KV head's tiles are reused from L2), dealt in
// boustrophedon waves (0..grid-1, grid-1..0, ...) — O(pairs), close to LPT for sorted costs.
void schedule(const std::vector<double>& item_cost, int hq, int num_sms, AttnWorkHost* w) {
  std::vector<int32_t> order(item_cost.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int32_t>(i);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return item_cost[a] > item_cost[b]; });
  const size_t pairs = item_cost.size() * static_cast<size_t>(hq);
  const int grid = static_cast<int>(std::min<size_t>(num_sms, std::max<size_t>(1, pairs)));
  std::vector<int32_t> count(grid, 0);
  std::vector<int32_t> bin_of(pairs);
  for (size_t i = 0; i < pairs; ++i) {
    const size_t wave = i / grid, pos = i % grid;
    const int b = static_cast<int>((wave & 1) ? grid - 1 - pos : pos);
    bin_of[i] = b;
    count[b]++;
  }
  w->grid = grid;
  w->cta_off.assign(grid + 1, 0);
  for (int c = 0; c < grid; ++c) w->cta_off[c + 1] = w->cta_off[c] + count[c];
  w->cta_items.assign(pairs, 0);
  std::vector<int32_t> fill(w->cta_off.begin(), w->cta_off.end() - 1);
  size_t i = 0;
  for (int32_t it : order)
    for (int h = 0; h < hq; ++h, ++i) w->cta_items[fill[bin_of[i]]++] = it * hq + h;
}

constexpr double kItemOverhead = 1.0;   // q-prep + epilogue, in KV-tile units
constexpr double kSplitOverhead = 0.5;  // partial write + combine read, per split

}  // namespace

void build_prefill_work(const PlanHost& p, const WorkOpts& o, int job_begin, int job_end,
                        AttnWorkHost* w) {
  *w = AttnWorkHost();
  const int64_t base = p.job_row_off[job_begin];
  std::vector<double> cost;
  for (int j = job_begin; j < job_end; ++j) {
    const Segment& s = p.segs[p.jobs[j]];
    const int32_t t0 = add_tiles(p, s, o.bs, 0, 0, 1, w);
    const int64_t row_off = p.job_row_off[j] - base;
    const int32_t nrows = s.tok_len - s.compute_begin;
    for (int32_t r = 0; r < nrows; r += kTileRows) {
      WorkItem it{};
      it.row0 = static_cast<int32_t>(row_off + r);
      it.n_rows = std::min(kTileRows, nrows - r);
      const int32_t max_pos = s.compute_begin + r + it.n_rows - 1;
      it.tile_begin = t0;
      it.tile_end = t0 + max_pos / kTileKeys + 1;
      it.part = -1;
      w->items.push_back(it);
      cost.push_back(it.tile_end - it.tile_begin + kItemOverhead);
    }
    for (int64_t i = s.compute_begin; i < s.tok_len; ++i) w->flops += static_cast<double>(i + 1);
  }
  w->flops *= 4.0 * o.d * o.hq;
  if (o.persistent) schedule(cost, o.units, o.num_sms, w);
}

void build_join_work(const PlanHost& p, const WorkOpts& o, int q_begin, int q_end, AttnWorkHost* w) {
  *w = AttnWorkHost();
  const int64_t base = p.query_join_row_off[q_begin];
  struct QTile {
    int32_t row0, n_rows, tb, te;
  };
  std::vector<QTile> qt;
  for (size_t si = 0; si < p.segs.size(); ++si) {
    const Segment& c = p.segs[si];
    if (c.kind != kCross || c.query < q_begin || c.query >= q_end) continue;
    int32_t first = -1;
    // the query's segments precede its cross segment contiguously
    size_t s0 = si;
    while (s0 > 0 && p.segs[s0 - 1].query == c.query) --s0;
    for (size_t k = s0; k < si; ++k) {
      const Segment& s = p.segs[k];
      const int32_t t = s.kind == kPrefix ? add_tiles(p, s, o.bs, 0, 0, 0, w)
                                          : add_tiles(p, s, o.bs, s.pos0, s.pos0, 0, w);
      if (first < 0) first = t;
    }
    const int32_t tc = add_tiles(p, c, o.bs, c.pos0, 0, 1, w);
    if (first < 0) first = tc;
    const int64_t row_off = p.query_join_row_off[c.query] - base;
    for (int32_t r = 0; r < c.tok_len; r += kTileRows) {
      QTile q{static_cast<int32_t>(row_off + r), std::min(kTileRows, c.tok_len - r), first,
              tc + r / kTileKeys + 1};
      qt.push_back(q);
    }
    const double before = static_cast<double>(c.pos0);
    for (int32_t j = 0; j < c.tok_len; ++j) w->flops += before + j + 1;
  }
  w->flops *= 4.0 * o.d * o.hq;
  // choose the split count K (same for all q tiles, capped by each tile count): minimise the
  // wave-quantised makespan ceil(pairs / SMs) * (largest chunk cost) — closed form, O(K·tiles)
  int best_k = 1;
  if (o.allow_split && !qt.empty()) {
    const size_t pairs1 = qt.size() * static_cast<size_t>(o.units);
    if (pairs1 < static_cast<size_t>(4 * o.num_sms)) {
      double best = 1e300;
      int max_n = 0;
      for (const QTile& q : qt) max_n = std::max(max_n, q.te - q.tb);
      for (int k = 1; k <= std::min(64, max_n); ++k) {
        size_t items = 0;
        double cmax = 0;
        for (const QTile& q : qt) {
          const int n = q.te - q.tb, kk = std::min(k, n);
          items += kk;
          cmax = std::max(cmax, (n + kk - 1) / kk + kItemOverhead + (kk > 1 ? kSplitOverhead : 0.0));
        }
        const double waves = std::ceil(static_cast<double>(items * o.units) / o.num_sms);
        const double mk = waves * cmax;
        if (mk < best * 0.98) {
          best = mk;
          best_k = k;
        }
      }
    }
  }
  std::vector<double> cost;
  for (const QTile& q : qt) {
    const int n = q.te - q.tb, kk = std::min(best_k, n);
    if (kk > 1) w->combine.push_back({q.row0, q.n_rows, w->n_parts, kk});
    for (int s = 0; s < kk; ++s) {
      WorkItem it{};
      it.row0 = q.row0;
      it.n_rows = q.n_rows;
      it.tile_begin = q.tb + (n * s) / kk;
      it.tile_end = q.tb + (n * (s + 1)) / kk;
      it.part = kk > 1 ? w->n_parts + s : -1;
      w->items.push_back(it);
      cost.push_back(it.tile_end - it.tile_begin + kItemOverhead + (kk > 1 ? kSplitOverhead : 0.0));
    }
    if (kk > 1) w->n_parts += kk;
  }
  if (o.persistent) schedule(cost, o.units, o.num_sms, w);
}

}  // namespace spq
