// cidra.cpp — see cidra.h.
#include "cidra.h"

#include <algorithm>
#include <unordered_map>

namespace spq {

bool cidra_schedule(const int32_t* src, const int32_t* dst, const int32_t* delta, int64_t n, int64_t num_blocks,
                    CidraSchedule* out, std::string* err) {
  *out = CidraSchedule();
  out->comp_off.push_back(0);
  // node ids: every block a move touches
  std::unordered_map<int32_t, int32_t> id;
  std::vector<int32_t> block;
  auto node = [&](int32_t b) {
    auto it = id.find(b);
    if (it != id.end()) return it->second;
    const int32_t k = static_cast<int32_t>(block.size());
    id.emplace(b, k);
    block.push_back(b);
    return k;
  };
  std::vector<int32_t> in_move;              // node -> the move writing it, or -1
  std::vector<std::vector<int32_t>> out_mv;  // node -> moves reading it
  for (int64_t i = 0; i < n; ++i) {
    if (src[i] < 0 || src[i] >= num_blocks || dst[i] < 0 || dst[i] >= num_blocks) {
      *err = "block id out of range";
      return false;
    }
    const int32_t s = node(src[i]), d = node(dst[i]);
    if (static_cast<size_t>(std::max(s, d)) >= in_move.size()) {
      in_move.resize(block.size(), -1);
      out_mv.resize(block.size());
    }
    if (in_move[d] >= 0) {
      *err = "block " + std::to_string(dst[i]) + " is the destination of two moves";
      return false;
    }
    in_move[d] = static_cast<int32_t>(i);
    out_mv[s].push_back(static_cast<int32_t>(i));
  }
  for (const auto& m : out_mv) out->duplicates += std::max<int64_t>(0, static_cast<int64_t>(m.size()) - 1);
  const int32_t nn = static_cast<int32_t>(block.size());
  std::vector<int32_t> done(nn, 0), stamp(nn, -1);
  std::vector<int32_t> level;  // BFS frontier of nodes
  std::vector<int32_t> tree;   // BFS-ordered moves of the current component
  for (int32_t start = 0; start < nn; ++start) {
    if (done[start]) continue;
    // walk up (to each node's source) until a root (nobody writes it) or a node seen twice (a cycle)
    int32_t v = start;
    while (in_move[v] >= 0 && stamp[v] != start) {
      stamp[v] = start;
      v = id[src[in_move[v]]];
    }
    std::vector<int32_t> cyc;  // W[0..k): W[j+1] = source of W[j]
    if (in_move[v] >= 0) {
      int32_t u = v;
      do {
        cyc.push_back(u);
        u = id[src[in_move[u]]];
      } while (u != v);
    }
    // BFS over the moves leaving the core (root, or the cycle nodes), skipping cycle edges
    level.clear();
    tree.clear();
    if (cyc.empty()) {
      level.push_back(v);
    } else {
      level = cyc;
    }
    for (int32_t c : level) done[c] = 1;
    while (!level.empty()) {
      std::vector<int32_t> next;
      for (int32_t u : level)
        for (int32_t m : out_mv[u]) {
          const int32_t w = id[dst[m]];
          if (done[w]) continue;  // a cycle edge (its destination is a core node)
          done[w] = 1;
          tree.push_back(m);
          next.push_back(w);
        }
      level.swap(next);
    }
    // reverse BFS: every move reading a block runs before the move overwriting it
    for (auto it = tree.rbegin(); it != tree.rend(); ++it) out->ops.push_back({dst[*it], src[*it], delta[*it], 0});
    if (!cyc.empty()) {
      const int k = static_cast<int>(cyc.size());
      out->ops.push_back({-1, block[cyc[0]], 0, 1});  // tmp <- W[0]
      for (int j = 0; j + 1 < k; ++j) {
        const int32_t m = in_move[cyc[j]];  // W[j] <- R(W[j+1])
        out->ops.push_back({block[cyc[j]], block[cyc[j + 1]], delta[m], 0});
      }
      out->ops.push_back({block[cyc[k - 1]], -1, delta[in_move[cyc[k - 1]]], 2});  // W[k-1] <- R(tmp)
      out->cycles++;
    }
    const int32_t c0 = out->comp_off.back();
    out->comp_off.push_back(static_cast<int32_t>(out->ops.size()));
    out->max_component_ops = std::max<int64_t>(out->max_component_ops, out->comp_off.back() - c0);
  }
  return true;
}

}  // namespace spq
