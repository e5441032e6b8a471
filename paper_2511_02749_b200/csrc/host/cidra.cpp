// cidra.cpp — see cidra.h.
#include "cidra.h"

#include <algorithm>

namespace spq {

bool cidra_schedule(const int32_t* src, const int32_t* dst, const int32_t* delta, int64_t n, int64_t num_blocks,
                    CidraSchedule* out, std::string* err) {
  *out = CidraSchedule();
  out->comp_off.push_back(0);
  for (int64_t i = 0; i < n; ++i)
    if (src[i] < 0 || src[i] >= num_blocks || dst[i] < 0 || dst[i] >= num_blocks) {
      *err = "block id out of range";
      return false;
    }
  // node ids: every block a move touches, compacted by sorting (no per-node allocation)
  std::vector<int32_t> block(src, src + n);
  block.insert(block.end(), dst, dst + n);
  std::sort(block.begin(), block.end());
  block.erase(std::unique(block.begin(), block.end()), block.end());
  auto node = [&](int32_t b) {
    return static_cast<int32_t>(std::lower_bound(block.begin(), block.end(), b) - block.begin());
  };
  const int32_t nn = static_cast<int32_t>(block.size());
  std::vector<int32_t> s_id(n), d_id(n);
  std::vector<int32_t> in_move(nn, -1);  // node -> the move writing it, or -1
  std::vector<int32_t> out_off(nn + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    s_id[i] = node(src[i]);
    d_id[i] = node(dst[i]);
    if (in_move[d_id[i]] >= 0) {
      *err = "block " + std::to_string(dst[i]) + " is the destination of two moves";
      return false;
    }
    in_move[d_id[i]] = static_cast<int32_t>(i);
    out_off[s_id[i] + 1]++;
  }
  // node -> moves reading it (CSR, in move order)
  for (int32_t v = 0; v < nn; ++v) out_off[v + 1] += out_off[v];
  std::vector<int32_t> out_mv(n), fill(out_off.begin(), out_off.end() - 1);
  for (int64_t i = 0; i < n; ++i) out_mv[fill[s_id[i]]++] = static_cast<int32_t>(i);
  for (int32_t v = 0; v < nn; ++v) out->duplicates += std::max<int32_t>(0, out_off[v + 1] - out_off[v] - 1);
  std::vector<int32_t> done(nn, 0), stamp(nn, -1);
  std::vector<int32_t> level;  // BFS frontier of nodes
  std::vector<int32_t> tree;   // BFS-ordered moves of the current component
  for (int32_t start = 0; start < nn; ++start) {
    if (done[start]) continue;
    // walk up (to each node's source) until a root (nobody writes it) or a node seen twice (a cycle)
    int32_t v = start;
    while (in_move[v] >= 0 && stamp[v] != start) {
      stamp[v] = start;
      v = s_id[in_move[v]];
    }
    std::vector<int32_t> cyc;  // W[0..k): W[j+1] = source of W[j]
    if (in_move[v] >= 0) {
      int32_t u = v;
      do {
        cyc.push_back(u);
        u = s_id[in_move[u]];
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
        for (int32_t e = out_off[u]; e < out_off[u + 1]; ++e) {
          const int32_t m = out_mv[e];
          const int32_t w = d_id[m];
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
