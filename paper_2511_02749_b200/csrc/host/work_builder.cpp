// work_builder.cpp — see work_builder.h.
#include "work_builder.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

namespace spq {
namespace {

// Append the KV tiles of n_tok tokens held densely in blocks[0..]; returns the first tile index.
int32_t append_tiles(const int32_t* blocks, int32_t n_tok, int bs, int32_t key_base, int32_t rot, int32_t causal,
                     std::vector<KvTile>* tiles, std::vector<int32_t>* tile_blocks) {
  const int32_t first = static_cast<int32_t>(tiles->size());
  const int bpt = kTileKeys / bs;
  for (int32_t t0 = 0; t0 < n_tok; t0 += kTileKeys) {
    KvTile k{};
    k.blk_off = static_cast<int32_t>(tile_blocks->size());
    k.n_valid = std::min(kTileKeys, n_tok - t0);
    k.key_pos0 = key_base + t0;
    k.rot_delta = rot;
    k.causal = causal;
    const int32_t b0 = t0 / bs;
    const int32_t nb = (k.n_valid + bs - 1) / bs;
    for (int j = 0; j < bpt; ++j) tile_blocks->push_back(blocks[b0 + std::min(j, nb - 1)]);
    tiles->push_back(k);
  }
  return first;
}

// Append the KV tiles of one segment; returns the index of its first tile.
int32_t add_tiles(const PlanHost& p, const Segment& s, int bs, int32_t key_base, int32_t rot,
                  int32_t causal, AttnWorkHost* w) {
  return append_tiles(p.blocks.data() + s.block_off, s.tok_len, bs, key_base, rot, causal, &w->tiles,
                      &w->tile_blocks);
}

// Schedule of (item, unit) codes over `grid` persistent CTAs: codes sorted by cost, longest
// first (units of one item adjacent, so a KV head's tiles are reused from L2), claimed at run time
// by the CTAs with an atomic counter — a CTA takes the next code when it needs one, so the
// makespan adapts to the real per-item cost (LPT list scheduling, no cost model in the loop).
void schedule(const std::vector<double>& item_cost, int units, int num_sms, AttnWorkHost* w,
              const std::vector<int32_t>* group = nullptr, int cluster = 1) {
  std::vector<int32_t> order(item_cost.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int32_t>(i);
#ifdef SPANQ_SCHED_GROUP
  // A/B: the items of one job (segment) claimed together, longest first inside the job, so the
  // CTAs reading one segment's K/V run at the same time (L2 reuse)
  if (group != nullptr) {
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      if ((*group)[a] != (*group)[b]) return (*group)[a] < (*group)[b];
      return item_cost[a] > item_cost[b];
    });
  } else
#else
  (void)group;
#endif
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return item_cost[a] > item_cost[b]; });
  const size_t codes = item_cost.size() * static_cast<size_t>(units);
  // a cluster (CTA pair) takes one code at a time: at most num_sms / cluster clusters
  w->cluster = cluster;
  w->grid = cluster * static_cast<int>(std::min<size_t>(num_sms / cluster, std::max<size_t>(1, codes)));
  // host-built static lists (boustrophedon waves) measured slower than run-time claims
  // (0.296 vs 0.276 ms); kept for hosts that build lists without a counter
  constexpr bool kStaticSched = false;
  if (kStaticSched) {
    // boustrophedon waves (0..grid-1, grid-1..0, ...) over the sorted codes
    const int grid = w->grid;
    std::vector<int32_t> count(grid, 0), bin_of(codes);
    for (size_t i = 0; i < codes; ++i) {
      const size_t wave = i / grid, pos = i % grid;
      bin_of[i] = static_cast<int32_t>((wave & 1) ? grid - 1 - pos : pos);
      count[bin_of[i]]++;
    }
    w->dynamic = false;
    w->cta_off.assign(grid + 1, 0);
    for (int c = 0; c < grid; ++c) w->cta_off[c + 1] = w->cta_off[c] + count[c];
    w->cta_items.assign(codes, 0);
    std::vector<int32_t> fill(w->cta_off.begin(), w->cta_off.end() - 1);
    size_t i = 0;
    for (int32_t it : order)
      for (int u = 0; u < units; ++u, ++i) w->cta_items[fill[bin_of[i]]++] = it * units + u;
    return;
  }
  w->dynamic = true;
  w->cta_off.assign({0, static_cast<int32_t>(codes)});
  w->cta_items.clear();
  w->cta_items.reserve(codes);
  for (int32_t it : order)
    for (int u = 0; u < units; ++u) w->cta_items.push_back(it * units + u);
}

constexpr double kItemOverhead = 1.0;   // q-prep + epilogue, in KV-tile units
constexpr double kSplitOverhead = 0.5;  // partial write + combine read, per split
// per work item, in 64-key sub-tiles (epilogue + Q + pipeline fill; measured)
constexpr double kSubOverhead = 3.0;
// per Q-rotation change inside a join piece, in sub-tiles
constexpr double kEpochCost = 1.5;

// Per-item sub-tile counts (the kernel's roles need them without walking the tiles).
void count_subtiles(AttnWorkHost* w) {
  for (WorkItem& it : w->items) {
    it.n_sub = 0;
    for (int32_t t = it.tile_begin; t < it.tile_end; ++t) it.n_sub += w->tiles[t].n_valid > 64 ? 2 : 1;
  }
}

}  // namespace

void build_prefill_work(const PlanHost& p, const WorkOpts& o, int job_begin, int job_end,
                        AttnWorkHost* w) {
  *w = AttnWorkHost();
  const int64_t base = p.job_row_off[job_begin];
  std::vector<double> cost;
  std::vector<int32_t> group;  // the item's job
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
      group.push_back(j);
    }
    for (int64_t i = s.compute_begin; i < s.tok_len; ++i) w->flops += static_cast<double>(i + 1);
  }
  w->flops *= 4.0 * o.d * o.hq;
  count_subtiles(w);
  if (o.persistent) schedule(cost, o.units, o.num_sms, w, &group, o.cluster);
}

namespace {
struct QTile {
  int32_t row0, n_rows, tb, te;
  bool force;  // write partials even when one piece covers it (its other phase adds more)
};
void finish_join(const std::vector<QTile>& qt, const WorkOpts& o, const JoinPhase* ph, AttnWorkHost* w);
}  // namespace

void build_task_join_work(const PlanHost& p, const WorkOpts& o, AttnWorkHost* w) {
  *w = AttnWorkHost();
  std::vector<QTile> qt;
  int64_t row = 0;
  for (const PlanHost::Task& t : p.tasks) {
    const int32_t first = static_cast<int32_t>(w->tiles.size());
    int64_t keys = 0;
    for (int32_t si = t.seg_begin; si < t.seg_end; ++si) {
      const Segment& s = p.segs[si];
      add_tiles(p, s, o.bs, s.pos0, s.pos0, 0, w);
      keys += s.tok_len;
    }
    const int32_t last = static_cast<int32_t>(w->tiles.size());
    for (int32_t r = 0; r < t.n_rows; r += kTileRows)
      qt.push_back({static_cast<int32_t>(row + r), std::min(kTileRows, t.n_rows - r), first, last, false});
    w->flops += static_cast<double>(keys) * t.n_rows;
    row += t.n_rows;
  }
  w->flops *= 4.0 * o.d * o.hq;
  finish_join(qt, o, nullptr, w);
}

void build_join_work(const PlanHost& p, const WorkOpts& o, int q_begin, int q_end, AttnWorkHost* w,
                     const JoinPhase* ph) {
  *w = AttnWorkHost();
  const int64_t base = p.query_join_row_off[q_begin];
  std::vector<QTile> qt;
  const int sel = ph ? ph->sel : 0;
  for (size_t si = 0; si < p.segs.size(); ++si) {
    const Segment& c = p.segs[si];
    if (c.kind != kCross || c.query < q_begin || c.query >= q_end) continue;
    int32_t first = -1, last = -1;
    // the query's segments precede its cross segment contiguously
    size_t s0 = si;
    while (s0 > 0 && p.segs[s0 - 1].query == c.query) --s0;
    bool has_remote = false;
    for (size_t k = s0; k < si; ++k) has_remote |= ph && ph->remote[k] != 0;
    if (sel == 2 && !has_remote) continue;  // nothing of this query arrives by the exchange
    for (size_t k = s0; k < si; ++k) {
      const Segment& s = p.segs[k];
      if (sel == 1 && ph->remote[k]) continue;  // phase 1: the segments this rank holds
      if (sel == 2 && !ph->remote[k]) continue;  // phase 2: the received fragments
      const int32_t t = s.kind == kPrefix ? add_tiles(p, s, o.bs, 0, 0, 0, w)
                                          : add_tiles(p, s, o.bs, s.pos0, s.pos0, 0, w);
      if (first < 0) first = t;
      last = static_cast<int32_t>(w->tiles.size());
    }
    const int32_t tc = sel == 2 ? -1 : add_tiles(p, c, o.bs, c.pos0, 0, 1, w);
    if (first < 0) first = tc;
    const int64_t row_off = p.query_join_row_off[c.query] - base;
    for (int32_t r = 0; r < c.tok_len; r += kTileRows) {
      QTile q{static_cast<int32_t>(row_off + r), std::min(kTileRows, c.tok_len - r), first,
              sel == 2 ? last : tc + r / kTileKeys + 1, has_remote};
      qt.push_back(q);
    }
    const double before = static_cast<double>(c.pos0);
    for (int32_t j = 0; j < c.tok_len; ++j) w->flops += before + j + 1;
  }
  w->flops *= 4.0 * o.d * o.hq;
  finish_join(qt, o, ph, w);
}

double join_flops(const PlanHost& p, const WorkOpts& o, int q_begin, int q_end) {
  double f = 0;
  for (const Segment& c : p.segs) {
    if (c.kind != kCross || c.query < q_begin || c.query >= q_end) continue;
    const double before = static_cast<double>(c.pos0);
    for (int32_t j = 0; j < c.tok_len; ++j) f += before + j + 1;
  }
  return f * 4.0 * o.d * o.hq;
}

namespace {
// Items of a join work list from its q tiles: one item per (q tile, unit), or (allow_split +
// persistent) the stream-K cut into <= num_sms equal-cost contiguous ranges.
void finish_join(const std::vector<QTile>& qt, const WorkOpts& o, const JoinPhase* ph, AttnWorkHost* w) {
  const int sel = ph ? ph->sel : 0;
  if (!(o.allow_split && o.persistent) || qt.empty()) {
    std::vector<double> cost;
    for (const QTile& q : qt) {
      WorkItem it{};
      it.row0 = q.row0;
      it.n_rows = q.n_rows;
      it.tile_begin = q.tb;
      it.tile_end = q.te;
      it.part = -1;
      w->items.push_back(it);
      cost.push_back(q.te - q.tb + kItemOverhead);
    }
    count_subtiles(w);
    if (o.persistent) schedule(cost, o.units, o.num_sms, w);
    return;
  }
  // Stream-K split: the (q tile, unit) pairs' KV sub-tiles, flattened pair-major (units of one q
  // tile adjacent: the two units of a KV head read the same tiles close in time), are cut into
  // num_sms contiguous ranges of equal cost (sub-tiles + a per-item overhead). A pair covered by
  // one CTA writes its final O; a pair cut across CTAs writes partials (per unit: hpu heads)
  // merged by combine. Every CTA gets <= ceil(range) work and at most a few items.
  const int hpu = o.hq / o.units;
  std::vector<int32_t> sub(w->tiles.size());
  double total = 0;
  for (size_t t = 0; t < w->tiles.size(); ++t) sub[t] = w->tiles[t].n_valid > 64 ? 2 : 1;
  const int grid = o.num_sms;
  struct Piece {
    int cta, t0, t1;
  };
  // prefix sums of the cost per tile (tiles of one q tile are contiguous): its sub-tiles, plus
  // kEpochCost where the Q rotation changes (a new fragment segment: the Q tiles are reloaded and
  // re-rotated inside the piece)
  std::vector<double> pre(w->tiles.size() + 1, 0.0);
  for (size_t t = 0; t < w->tiles.size(); ++t)
    pre[t + 1] = pre[t] + sub[t] +
                 (t > 0 && w->tiles[t].rot_delta != w->tiles[t - 1].rot_delta ? kEpochCost : 0.0);
  for (const QTile& q : qt) total += (pre[q.te] - pre[q.tb]) * o.units;
  // greedy cut at cost budget `target` per CTA; returns the CTAs used (unbounded), pieces per pair
  auto cut = [&](double target, std::vector<std::vector<Piece>>* out) {
    int cta = 0;
    double load = 0;
    if (out) out->clear();
    for (const QTile& q : qt) {
      for (int u = 0; u < o.units; ++u) {
        if (out) out->emplace_back();
        int t = q.tb;
        while (t < q.te) {
          const double cap = target - load - kSubOverhead;
          if (cap < 2 && load > 0) {
            ++cta;
            load = 0;
            continue;
          }
          // largest t1 > t with pre[t1] - pre[t] <= cap (at least one tile)
          const double lim = pre[t] + cap;
          int t1 = static_cast<int>(std::upper_bound(pre.begin() + t + 1, pre.begin() + q.te + 1, lim) - pre.begin()) - 1;
          t1 = std::max(t1, t + 1);
          if (out) out->back().push_back({cta, t, t1});
          load += pre[t1] - pre[t] + kSubOverhead;
          t = t1;
        }
      }
    }
    return cta + (load > 0 ? 1 : 0);
  };
  // smallest budget whose greedy cut fits in `grid` CTAs (bisection; the cost is monotone enough)
  double lo = total / grid, hi = total / grid + 4 * kSubOverhead + 64;
  while (cut(hi, nullptr) > grid) hi *= 1.5;
  for (int it = 0; it < 16 && hi - lo > 0.5; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (cut(mid, nullptr) <= grid)
      hi = mid;
    else
      lo = mid;
  }
  std::vector<std::vector<Piece>> all;
  cut(hi, &all);
  std::vector<std::vector<int32_t>> per_cta(grid);
  size_t pi = 0;
  for (const QTile& q : qt) {
    for (int u = 0; u < o.units; ++u, ++pi) {
      const std::vector<Piece>& pieces = all[pi];
      const int np = static_cast<int>(pieces.size());
      const bool part = np > 1 || q.force;
      const int32_t pb = (ph ? ph->part_base : 0) + w->n_parts;  // global partial slot of piece 0
      if (part) {
        if (sel == 1 && q.force) {
          (*ph->ranges)[{q.row0, u}] = {pb, np};  // merged after phase 2
        } else if (sel == 2) {
          const std::pair<int32_t, int32_t> r1 = ph->ranges->at({q.row0, u});
          w->combine.push_back({q.row0, q.n_rows, r1.first, r1.second, u * hpu, hpu, pb, np});
        } else {
          w->combine.push_back({q.row0, q.n_rows, pb, np, u * hpu, hpu, 0, 0});
        }
      }
      for (int k = 0; k < np; ++k) {
        WorkItem it{};
        it.row0 = q.row0;
        it.n_rows = q.n_rows;
        it.tile_begin = pieces[k].t0;
        it.tile_end = pieces[k].t1;
        it.part = part ? pb + k : -1;
        per_cta[pieces[k].cta].push_back(static_cast<int32_t>(w->items.size()) * o.units + u);
        w->items.push_back(it);
      }
      if (part) w->n_parts += np;
    }
  }
  count_subtiles(w);
  int used = grid;
  while (used > 1 && per_cta[used - 1].empty()) --used;
  (void)sel;
  w->grid = used;
  w->cta_off.assign(used + 1, 0);
  for (int c = 0; c < used; ++c) {
    w->cta_off[c + 1] = w->cta_off[c] + static_cast<int32_t>(per_cta[c].size());
    w->cta_items.insert(w->cta_items.end(), per_cta[c].begin(), per_cta[c].end());
  }
}

}  // namespace

std::pair<int32_t, int32_t> decode_row_tiles(const PlanHost& p, int32_t query, const std::vector<int32_t>& cross_gen_blocks,
                                             int32_t gen_ctx, int bs, DecodeWorkHost* w) {
  const int32_t first = static_cast<int32_t>(w->tiles.size());
  for (const Segment& s : p.segs) {
    if (s.query != query) continue;
    const int32_t* blk = p.blocks.data() + s.block_off;
    if (s.kind == kPrefix)
      append_tiles(blk, s.tok_len, bs, 0, 0, 0, &w->tiles, &w->tile_blocks);
    else if (s.kind == kFrag)
      append_tiles(blk, s.tok_len, bs, s.pos0, s.pos0, 0, &w->tiles, &w->tile_blocks);
    else
      append_tiles(cross_gen_blocks.data(), gen_ctx, bs, s.pos0, 0, 1, &w->tiles, &w->tile_blocks);
  }
  return {first, static_cast<int32_t>(w->tiles.size())};
}

void decode_items(const std::vector<std::pair<int32_t, int32_t>>& row_tiles, int hkv, int group, int chunk_tiles,
                  DecodeWorkHost* w) {
  for (size_t r = 0; r < row_tiles.size(); ++r) {
    const int32_t tb = row_tiles[r].first, te = row_tiles[r].second;
    const int32_t n = std::max<int32_t>(1, (te - tb + chunk_tiles - 1) / chunk_tiles);
    for (int32_t h = 0; h < hkv; ++h) {
      const int32_t pb = n > 1 ? w->n_parts : -1;
      for (int32_t c = 0; c < n; ++c) {
        DecodeItemHost it{};
        it.row = static_cast<int32_t>(r);
        it.kvh = h;
        it.tile_begin = tb + c * chunk_tiles;
        it.tile_end = std::min(te, tb + (c + 1) * chunk_tiles);
        it.part = n > 1 ? pb + c : -1;
        it.n_chunks = n;                                                   // chunks of this (row, kv head)
        it.part0 = n > 1 ? pb : -1;                                     // its first partial slot
        it.pair = static_cast<int32_t>(r) * hkv + h;                   // (row, kv head) index
        w->items.push_back(it);
      }
      if (n > 1) {
        w->combine.push_back({static_cast<int32_t>(r), 1, pb, n, h * group, group, 0, 0});
        w->n_parts += n;
      }
    }
  }
}

}  // namespace spq
