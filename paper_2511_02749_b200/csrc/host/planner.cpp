// planner.cpp — see planner.h. Semantics are the contract of DESIGN.md (readings R1-R13,
// hash contract); the CPU oracle (oracle/store.py) implements the same contract separately
// and tests/test_planner_parity.py checks the two bit-for-bit.
#include "planner.h"

#include <unordered_set>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../../include/spanq.h"

namespace spq {

// ------------------------------------------------------------------ tree normalization
namespace {

struct TreeParser {
  const spq_query& q;
  std::string* err;
  bool fail(const char* m) {
    *err = m;
    return false;
  }
  // index after the subtree rooted at i, or -1
  int64_t subtree_end(int64_t i) {
    if (i >= q.num_nodes) return -1;
    const spq_node& n = q.nodes[i];
    if (n.op < 0 || n.op > 2 || n.num_children < 0) return -1;
    int64_t j = i + 1;
    for (int c = 0; c < n.num_children; ++c) {
      j = subtree_end(j);
      if (j < 0) return -1;
    }
    return j;
  }
  bool leaf(int64_t i, std::vector<int32_t>* out) {
    const spq_node& n = q.nodes[i];
    if (n.op != SPQ_TOKENS || n.num_children != 0) return fail("expected TOKENS leaf");
    if (n.tok_len <= 0) return fail("empty token leaf");
    if (n.tok_begin < 0 || n.tok_begin + n.tok_len > q.num_tokens) return fail("token range out of bounds");
    const int32_t* t0 = q.tokens + n.tok_begin;
    int32_t mn = 0;
    for (int64_t t = 0; t < n.tok_len; ++t) mn = std::min(mn, t0[t]);
    if (mn < 0) return fail("negative token id");
    out->insert(out->end(), t0, t0 + n.tok_len);
    return true;
  }
  // fragments under a PLUS node (nested PLUS flattened); *next = index after it
  bool plus(int64_t i, std::vector<std::vector<int32_t>>* frags, int64_t* next) {
    const spq_node& n = q.nodes[i];
    if (n.op != SPQ_PLUS) return fail("expected PLUS");
    if (n.num_children < 1) return fail("PLUS needs >= 1 child");
    int64_t j = i + 1;
    for (int c = 0; c < n.num_children; ++c) {
      const spq_node& k = q.nodes[j];
      if (k.op == SPQ_TOKENS) {
        frags->emplace_back();
        if (!leaf(j, &frags->back())) return false;
        j += 1;
      } else if (k.op == SPQ_PLUS) {
        if (!plus(j, frags, &j)) return false;
      } else {  // CROSS of TOKENS leaves = one fragment
        if (k.num_children < 1) return fail("CROSS needs >= 1 child");
        frags->emplace_back();
        int64_t m = j + 1;
        for (int cc = 0; cc < k.num_children; ++cc, ++m)
          if (!leaf(m, &frags->back())) return false;
        j = m;
      }
    }
    *next = j;
    return true;
  }
};

}  // namespace

bool normalize_tree(const spq_query& q, FlatQuery* out, std::string* err) {
  TreeParser p{q, err};
  if (q.num_nodes <= 0 || q.nodes == nullptr) return p.fail("empty tree");
  if (q.num_tokens > 0 && q.tokens == nullptr) return p.fail("null tokens");
  if (p.subtree_end(0) != q.num_nodes) return p.fail("malformed tree (op, arity or node count)");
  const spq_node& root = q.nodes[0];
  if (root.op != SPQ_CROSS || root.num_children < 1) return p.fail("root must be CROSS with >= 1 child");
  std::vector<int64_t> kids;
  int64_t j = 1;
  for (int c = 0; c < root.num_children; ++c) {
    kids.push_back(j);
    j = p.subtree_end(j);
  }
  if (q.nodes[kids.back()].op != SPQ_TOKENS) return p.fail("last child must be the cross TOKENS leaf");
  *out = FlatQuery();
  if (!p.leaf(kids.back(), &out->cross)) return false;
  kids.pop_back();
  std::vector<int32_t> ops;
  for (int64_t k : kids) ops.push_back(q.nodes[k].op);
  int64_t dummy;
  if (ops == std::vector<int32_t>{SPQ_TOKENS, SPQ_PLUS}) {
    if (!p.leaf(kids[0], &out->prefix)) return false;
    if (!p.plus(kids[1], &out->frags, &dummy)) return false;
  } else if (ops == std::vector<int32_t>{SPQ_TOKENS}) {
    if (!p.leaf(kids[0], &out->prefix)) return false;
  } else if (ops == std::vector<int32_t>{SPQ_PLUS}) {
    if (!p.plus(kids[0], &out->frags, &dummy)) return false;
  } else if (!ops.empty()) {
    return p.fail("unsupported tree shape");
  }
  return true;
}

// ------------------------------------------------------------------ digests
namespace {
inline void put_u32(std::vector<uint8_t>* b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b->push_back(static_cast<uint8_t>(v >> (8 * i)));
}
inline Digest b2(const std::vector<uint8_t>& buf) {
  Digest d;
  blake2b(d.b, 16, buf.data(), buf.size());
  return d;
}
}  // namespace

Digest root_digest(int hq, int hkv, int d, int bs, double rope_base, uint64_t salt) {
  std::vector<uint8_t> buf = {'S', 'P', 'Q', 'v', '1'};
  put_u32(&buf, hq);
  put_u32(&buf, hkv);
  put_u32(&buf, d);
  put_u32(&buf, bs);
  uint8_t f[8];
  std::memcpy(f, &rope_base, 8);
  buf.insert(buf.end(), f, f + 8);
  for (int i = 0; i < 8; ++i) buf.push_back(static_cast<uint8_t>(salt >> (8 * i)));
  return b2(buf);
}

void chain(char tag, const Digest& seed, const int32_t* tok, int64_t n, int bs,
           std::vector<Digest>* out) {
  // message = tag ‖ prev digest ‖ u32 n ‖ n × u32 token (little-endian host)
  std::vector<uint8_t> buf(1 + 16 + 4 + 4 * static_cast<size_t>(bs));
  buf[0] = static_cast<uint8_t>(tag);
  Digest prev = seed;
  for (int64_t s = 0; s < n; s += bs) {
    const uint32_t m = static_cast<uint32_t>(std::min<int64_t>(bs, n - s));
    std::memcpy(buf.data() + 1, prev.b, 16);
    std::memcpy(buf.data() + 17, &m, 4);
    std::memcpy(buf.data() + 21, tok + s, 4 * static_cast<size_t>(m));
    blake2b(prev.b, 16, buf.data(), 21 + 4 * static_cast<size_t>(m));
    out->push_back(prev);
  }
}

Digest join_fold(const Digest& h_last, const std::vector<Digest>& frag_lasts) {
  std::vector<uint8_t> buf = {'J'};
  buf.insert(buf.end(), h_last.b, h_last.b + 16);
  put_u32(&buf, static_cast<uint32_t>(frag_lasts.size()));
  for (const Digest& d : frag_lasts) buf.insert(buf.end(), d.b, d.b + 16);
  return b2(buf);
}

// ------------------------------------------------------------------ store
Store::Store(int64_t num_blocks, int block_size, const Digest& root)
    : nblocks_(num_blocks), bs_(block_size), root_(root) {
  meta_.resize(num_blocks);
  for (auto& m : meta_) m = Meta{Digest{}, 0, 0, false};
  pins_.assign(num_blocks, 0);
  pinned_mark_.assign(num_blocks, 0);
  free_.init(num_blocks);
  index_.init(num_blocks);
}

int64_t Store::pinned_count() const {
  int64_t n = 0;
  for (int32_t p : pins_) n += p > 0;
  return n;
}

int32_t Store::lookup(const Digest& d) const {
  return index_.find(d);
}

void Store::set_evictable(int32_t b, bool on) {
  if (on)
    evictable_.insert({meta_[b].last_use, b});
  else
    evictable_.erase({meta_[b].last_use, b});
}

int32_t Store::alloc(bool* ok) {
  if (!free_.empty()) {
    const int32_t b = free_.pop_lowest();
    if (journaling_) journal_.push_back({kUndoFreePop, b, Meta{}});
    return b;
  }
  if (evictable_.empty()) {
    *ok = false;
    return -1;
  }
  const int32_t b = evictable_.begin()->second;
  evictable_.erase(evictable_.begin());
  if (journaling_) journal_.push_back({kUndoEvict, b, meta_[b]});
  index_.erase(meta_[b].dig);
  meta_[b].resident = false;
  stats_.evictions++;
  return b;
}

void Store::pin(int32_t b) {
  if (pinned_mark_[b]) return;
  pinned_mark_[b] = 1;
  cur_pinned_->push_back(b);
  if (pins_[b] == 0 && meta_[b].resident) set_evictable(b, false);
  pins_[b]++;
  journal_.push_back({kUndoPin, b, Meta{}});
}

void Store::touch(int32_t b) {
  journal_.push_back({kUndoTouch, b, meta_[b]});
  meta_[b].last_use = plan_no_;
}

void Store::rollback() {
  for (auto it = journal_.rbegin(); it != journal_.rend(); ++it) {
    const int32_t b = it->block;
    switch (it->kind) {
      case kUndoFreePop:
        free_.insert(b);
        break;
      case kUndoEvict:
        meta_[b] = it->meta;
        index_.set(meta_[b].dig, b);
        if (pins_[b] == 0) set_evictable(b, true);
        break;
      case kUndoInsert:
        if (pins_[b] == 0) set_evictable(b, false);  // no-op unless the insert was unpinned
        index_.erase(meta_[b].dig);
        meta_[b].resident = false;
        break;
      case kUndoPin:
        pins_[b]--;
        pinned_mark_[b] = 0;
        if (pins_[b] == 0 && meta_[b].resident) set_evictable(b, true);
        break;
      case kUndoTouch:
        meta_[b].last_use = it->meta.last_use;
        break;
    }
  }
  journal_.clear();
}

namespace {
struct QueryDigests {
  std::vector<Digest> prefix, cross;
  std::vector<std::vector<Digest>> frags;
  Digest join;
};

void hash_all(const std::vector<FlatQuery>& qs, int bs, const Digest& root, ThreadPool* pool,
              std::vector<QueryDigests>* out) {
  out->assign(qs.size(), QueryDigests());
  std::vector<std::pair<int32_t, int32_t>> tasks;  // (query, -1 prefix | fragment index)
  int64_t ntok = 0;
  for (size_t q = 0; q < qs.size(); ++q) {
    (*out)[q].frags.resize(qs[q].frags.size());
    tasks.push_back({static_cast<int32_t>(q), -1});
    ntok += static_cast<int64_t>(qs[q].prefix.size() + qs[q].cross.size());
    for (size_t f = 0; f < qs[q].frags.size(); ++f) {
      tasks.push_back({static_cast<int32_t>(q), static_cast<int32_t>(f)});
      ntok += static_cast<int64_t>(qs[q].frags[f].size());
    }
  }
  const bool par = pool != nullptr && ntok >= 4096;
  std::function<void(int64_t)> chains = [&](int64_t i) {
    const auto [q, f] = tasks[i];
    if (f < 0)
      chain('P', root, qs[q].prefix.data(), static_cast<int64_t>(qs[q].prefix.size()), bs, &(*out)[q].prefix);
    else
      chain('F', root, qs[q].frags[f].data(), static_cast<int64_t>(qs[q].frags[f].size()), bs,
            &(*out)[q].frags[f]);
  };
  std::function<void(int64_t)> crosses = [&](int64_t q) {
    QueryDigests& d = (*out)[q];
    std::vector<Digest> lasts;
    for (const auto& f : d.frags) lasts.push_back(f.back());
    d.join = join_fold(d.prefix.empty() ? root : d.prefix.back(), lasts);
    chain('X', d.join, qs[q].cross.data(), static_cast<int64_t>(qs[q].cross.size()), bs, &d.cross);
  };
  if (par) {
    pool->parallel_for(static_cast<int64_t>(tasks.size()), chains);
    pool->parallel_for(static_cast<int64_t>(qs.size()), crosses);
  } else {
    for (size_t i = 0; i < tasks.size(); ++i) chains(static_cast<int64_t>(i));
    for (size_t q = 0; q < qs.size(); ++q) crosses(static_cast<int64_t>(q));
  }
}
}  // namespace

int owner_rank(const Digest& d, int world) {
  uint64_t v;
  std::memcpy(&v, d.b, 8);  // u64 little-endian of s_last[0:8]
  return static_cast<int>(v % static_cast<uint64_t>(world));
}

int Store::plan(const std::vector<FlatQuery>& qs, PlanHost* out, ThreadPool* pool, int rank, int world, bool split) {
  std::vector<QueryDigests> qd;
#ifdef SPANQ_PROFILING
  static const bool prof = std::getenv("SPANQ_PROFILE") != nullptr;  // profiling builds only
#else
  constexpr bool prof = false;
#endif
  auto t0 = std::chrono::steady_clock::now();
  hash_all(qs, bs_, root_, pool, &qd);
  if (prof)
    std::fprintf(stderr, "[spanq]   store.hash_all %8.1f us\n",
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  const StoreStats saved_stats = stats_;
  const int64_t saved_plan = plan_no_;
  journal_.clear();
  journaling_ = true;
  *out = PlanHost();
  PlanHost& P = *out;
  P.n_queries = static_cast<int32_t>(qs.size());
  P.join_digests.assign(qs.size(), Digest{});  // zero for queries homed on another rank
  cur_pinned_ = &P.pinned;
  plan_no_++;
  const int bs = bs_;
  bool ok = true;

  auto insert_new = [&](const Digest& d, int32_t ntok) -> int32_t {
    const int32_t b = alloc(&ok);
    if (!ok) return -1;
    index_.set(d, b);
    meta_[b] = Meta{d, ntok, plan_no_, true};
    journal_.push_back({kUndoInsert, b, Meta{}});
    stats_.inserted_blocks++;
    pin(b);
    for (int64_t s = static_cast<int64_t>(b) * bs + ntok; s < static_cast<int64_t>(b) * bs + bs; ++s)
      P.pad_slots.push_back(s);
    return b;
  };
  auto new_private = [&](int32_t ntok) -> int32_t {
    const int32_t b = alloc(&ok);
    if (!ok) return -1;
    P.priv.push_back(b);
    pin(b);
    for (int64_t s = static_cast<int64_t>(b) * bs + ntok; s < static_cast<int64_t>(b) * bs + bs; ++s)
      P.pad_slots.push_back(s);
    return b;
  };
  // a received block, indexed under its digest (R38 replica): no pad slots — the owner's pages
  // carry their zeroed pads and blocks move whole
  // blocks whose KV this plan receives: an owned fragment of the same plan that shares one (a common
  // token prefix) must not count it as resident — it is filled only by the exchange, after the
  // prefill and after the pack of the owner's own sends — so it recomputes and writes it
  std::unordered_set<int32_t> pending;
  auto insert_replica = [&](const Digest& d, int32_t ntok) -> int32_t {
    const int32_t b = alloc(&ok);
    if (!ok) return -1;
    pending.insert(b);
    P.replicas.push_back(b);
    index_.set(d, b);
    meta_[b] = Meta{d, ntok, plan_no_, true};
    journal_.push_back({kUndoInsert, b, Meta{}});
    stats_.inserted_blocks++;
    pin(b);
    return b;
  };
  auto add_seg = [&](int32_t qi, int32_t kind, int32_t fi, int32_t len, int32_t pos0, int32_t hit,
                     int32_t cb, const std::vector<int32_t>& blocks, const std::vector<uint8_t>& wr,
                     const std::vector<Digest>& dig) {
    P.segs.push_back(Segment{qi, kind, fi, len, pos0, hit, cb, static_cast<int32_t>(P.blocks.size()),
                             static_cast<int32_t>(blocks.size())});
    P.blocks.insert(P.blocks.end(), blocks.begin(), blocks.end());
    P.block_write.insert(P.block_write.end(), wr.begin(), wr.end());
    P.digests.insert(P.digests.end(), dig.begin(), dig.end());
  };

  std::vector<Digest> dig;
  std::vector<int32_t> blocks;
  std::vector<uint8_t> wr;
  std::unordered_map<Digest, std::vector<int32_t>, DigestHash> owned_blocks, recv_blocks;
  std::unordered_map<Digest, uint8_t, DigestHash> recv_hit;  // remote fragment: replica resident
  std::vector<std::vector<Digest>> send_list(world), recv_list(world), cand_recv(world);
  std::vector<std::vector<int32_t>> xq(world);  // split mode: home queries per owner peer
  // all-or-nothing lookup of one locally owned fragment; pins resident blocks before allocating
  auto owned_fragment = [&](int32_t qi, int32_t fi, int32_t flen, int32_t off, const std::vector<Digest>& fd) {
    stats_.lookups++;
    std::vector<int32_t> res(fd.size());
    bool all = true;
    for (size_t i = 0; i < fd.size(); ++i) {
      res[i] = lookup(fd[i]);
      all = all && res[i] >= 0 && !pending.count(res[i]);
    }
    for (int32_t b : res)
      if (b >= 0) {
        pin(b);
        touch(b);
      }
    std::vector<int32_t> fb;
    std::vector<uint8_t> fw;
    if (all) {
      stats_.hit_blocks += static_cast<int64_t>(fd.size());
      stats_.hit_tokens += flen;
      fw.assign(fd.size(), 0);
      add_seg(qi, kFrag, fi, flen, off, 1, flen, res, fw, fd);
      fb = res;
    } else {
      stats_.miss_blocks += static_cast<int64_t>(fd.size());
      for (size_t i = 0; i < fd.size() && ok; ++i) {
        if (res[i] >= 0) {
          fb.push_back(res[i]);
          fw.push_back(pending.count(res[i]) ? 1 : 0);
        } else {
          fb.push_back(insert_new(fd[i], std::min<int32_t>(bs, flen - static_cast<int32_t>(i) * bs)));
          fw.push_back(1);
        }
      }
      if (!ok) return;
      add_seg(qi, kFrag, fi, flen, off, 0, 0, fb, fw, fd);
    }
    owned_blocks.emplace(fd.back(), fb);
  };
  for (int32_t qi = 0; qi < P.n_queries && ok; ++qi) {
    const FlatQuery& q = qs[qi];
    const int home = qi % world;
    if (home != rank) {
      // only the fragments this rank owns: prefill/cache them, send them to the home rank (split
      // mode: keep them at their offset Δ_f in the query, for this rank's task)
      const int32_t first = static_cast<int32_t>(P.segs.size());
      int32_t off = static_cast<int32_t>(q.prefix.size());
      for (size_t fi = 0; fi < q.frags.size() && ok; ++fi) {
        const std::vector<Digest>& fd = qd[qi].frags[fi];
        const int32_t delta = off;
        off += static_cast<int32_t>(q.frags[fi].size());
        if (owner_rank(fd.back(), world) != rank) continue;
        owned_fragment(qi, static_cast<int32_t>(fi), static_cast<int32_t>(q.frags[fi].size()), split ? delta : 0, fd);
        if (split) continue;
        auto& lst = send_list[home];
        if (std::find(lst.begin(), lst.end(), fd.back()) == lst.end()) lst.push_back(fd.back());
      }
      if (split && ok && static_cast<int32_t>(P.segs.size()) > first)
        P.tasks.push_back({qi, static_cast<int32_t>(home), static_cast<int32_t>(q.cross.size()), off, first,
                           static_cast<int32_t>(P.segs.size())});
      continue;
    }
    P.n_join_queries++;
    int64_t ntot = static_cast<int64_t>(q.prefix.size()) + static_cast<int64_t>(q.cross.size());
    for (const auto& f : q.frags) ntot += static_cast<int64_t>(f.size());
    stats_.input_tokens += ntot;
    // ---- prefix: chained digests + prefix scan; partial tail plan-private (R9)
    const int32_t plen = static_cast<int32_t>(q.prefix.size());
    dig = qd[qi].prefix;
    blocks.clear();
    wr.clear();
    bool hit_run = true;
    int32_t n_hit = 0;
    for (size_t i = 0; i < dig.size() && ok; ++i) {
      const int32_t ntok = std::min<int32_t>(bs, plen - static_cast<int32_t>(i) * bs);
      const bool full = ntok == bs;
      if (full) stats_.lookups++;
      const int32_t r = full ? lookup(dig[i]) : -1;
      if (r >= 0) {
        pin(r);
        touch(r);
        blocks.push_back(r);
        wr.push_back(0);
        if (hit_run) {
          n_hit++;
          stats_.hit_blocks++;
          stats_.hit_tokens += bs;
        } else {
          stats_.miss_blocks++;
        }
        continue;
      }
      hit_run = false;
      if (full) {
        stats_.miss_blocks++;
        blocks.push_back(insert_new(dig[i], bs));
      } else {
        blocks.push_back(new_private(ntok));
      }
      wr.push_back(1);
    }
    if (!ok) break;
    if (plen > 0)
      add_seg(qi, kPrefix, -1, plen, 0, n_hit, std::min(n_hit * bs, plen), blocks, wr, dig);
    const Digest h_last = dig.empty() ? root_ : dig.back();
    // ---- fragments: suspended chains, all-or-nothing lookup (R10, R11); with W > 1
    // a fragment owned by another rank is received into plan-private blocks (no prefill)
    int32_t off = plen;
    for (size_t fi = 0; fi < q.frags.size() && ok; ++fi) {
      const int32_t flen = static_cast<int32_t>(q.frags[fi].size());
      const std::vector<Digest>& fd = qd[qi].frags[fi];
      const int owner = owner_rank(fd.back(), world);
      if (owner == rank) {
        owned_fragment(qi, static_cast<int32_t>(fi), flen, off, fd);
      } else if (split) {  // computed by its owner (a task there); this rank merges the partial
        if (xq[owner].empty() || xq[owner].back() != qi) xq[owner].push_back(qi);
      } else {
        // remote-owned (R38): an all-or-nothing lookup of its replica; a miss is received whole
        // into its resident blocks and newly indexed ones (pinned before any allocation, R24)
        auto it = recv_blocks.find(fd.back());
        if (it == recv_blocks.end()) {
          stats_.lookups++;
          std::vector<int32_t> res(fd.size());
          bool all = true;
          for (size_t i = 0; i < fd.size(); ++i) {
            res[i] = lookup(fd[i]);
            all = all && res[i] >= 0;
          }
          for (int32_t b : res)
            if (b >= 0) {
              pin(b);
              touch(b);
            }
          if (all) {
            stats_.hit_blocks += static_cast<int64_t>(fd.size());
            stats_.hit_tokens += flen;
          } else {
            stats_.miss_blocks += static_cast<int64_t>(fd.size());
            for (size_t i = 0; i < fd.size() && ok; ++i)
              if (res[i] < 0) res[i] = insert_replica(fd[i], std::min<int32_t>(bs, flen - static_cast<int32_t>(i) * bs));
            if (!ok) break;
            recv_list[owner].push_back(fd.back());
          }
          it = recv_blocks.emplace(fd.back(), res).first;
          recv_hit[fd.back()] = all ? 1 : 0;
          cand_recv[owner].push_back(fd.back());
        }
        wr.assign(fd.size(), 0);
        add_seg(qi, kFrag, static_cast<int32_t>(fi), flen, off, recv_hit[fd.back()], flen, it->second, wr, fd);
      }
      off += flen;
    }
    if (!ok) break;
    (void)h_last;
    const Digest J = qd[qi].join;
    P.join_digests[qi] = J;
    // ---- cross: always computed; full blocks under the X chain (R9)
    const int32_t clen = static_cast<int32_t>(q.cross.size());
    dig = qd[qi].cross;
    blocks.clear();
    wr.clear();
    for (size_t i = 0; i < dig.size() && ok; ++i) {
      const int32_t ntok = std::min<int32_t>(bs, clen - static_cast<int32_t>(i) * bs);
      const int32_t r = ntok == bs ? lookup(dig[i]) : -1;
      if (r >= 0) {
        pin(r);
        touch(r);
        blocks.push_back(r);
        wr.push_back(0);
      } else if (ntok == bs) {
        blocks.push_back(insert_new(dig[i], bs));
        wr.push_back(1);
      } else {
        blocks.push_back(new_private(ntok));
        wr.push_back(1);
      }
    }
    if (!ok) break;
    add_seg(qi, kCross, -1, clen, off, 0, 0, blocks, wr, dig);
  }
  if (prof)
    std::fprintf(stderr, "[spanq]   store.segments %8.1f us\n",
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  if (!ok) {
    rollback();
    for (int32_t b : P.pinned) pinned_mark_[b] = 0;
    stats_ = saved_stats;
    plan_no_ = saved_plan;
    journaling_ = false;
    cur_pinned_ = nullptr;
    *out = PlanHost();
    return 2;
  }
  journal_.clear();
  journaling_ = false;
  for (int32_t b : P.pinned) pinned_mark_[b] = 0;
  cur_pinned_ = nullptr;

  // ---- packed rows (job order for prefill, query order for joins)
  auto rows = [&](const Segment& s, int32_t begin, std::vector<int32_t>* pos,
                  std::vector<int64_t>* slot, std::vector<int32_t>* segi, int32_t si) {
    const int32_t p0 = s.kind == kCross ? s.pos0 : 0;
    const size_t n0 = pos->size();
    const size_t n = static_cast<size_t>(std::max(0, s.tok_len - begin));
    pos->resize(n0 + n);
    slot->resize(n0 + n);
    segi->resize(n0 + n, si);
    int32_t* pp = pos->data() + n0;
    int64_t* sp = slot->data() + n0;
    for (int32_t b = begin / bs; b * bs < s.tok_len; ++b) {
      const int32_t t0 = std::max(begin, b * bs), t1 = std::min(s.tok_len, (b + 1) * bs);
      const bool w = P.block_write[s.block_off + b] != 0;
      const int64_t base = static_cast<int64_t>(P.blocks[s.block_off + b]) * bs - static_cast<int64_t>(b) * bs;
      for (int32_t t = t0; t < t1; ++t) {
        *pp++ = p0 + t;
        *sp++ = w ? base + t : -1;
      }
    }
  };
  {
    int64_t np = 0, nj = 0;
    for (const Segment& s : P.segs) {
      if (s.kind == kCross) nj += s.tok_len;
      else if (s.compute_begin < s.tok_len) np += s.tok_len - s.compute_begin;
    }
    P.prefill_pos.reserve(np);
    P.prefill_slot.reserve(np);
    P.prefill_seg.reserve(np);
    P.join_pos.reserve(nj);
    P.join_slot.reserve(nj);
    P.join_seg.reserve(nj);
  }
  P.job_row_off.push_back(0);
  for (size_t i = 0; i < P.segs.size(); ++i) {
    const Segment& s = P.segs[i];
    if (s.kind != kCross && s.compute_begin < s.tok_len) {
      P.jobs.push_back(static_cast<int32_t>(i));
      rows(s, s.compute_begin, &P.prefill_pos, &P.prefill_slot, &P.prefill_seg, static_cast<int32_t>(i));
      P.job_row_off.push_back(static_cast<int64_t>(P.prefill_pos.size()));
    }
  }
  if (prof)
    std::fprintf(stderr, "[spanq]   store.rows %8.1f us\n",
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  // exchange lists: per peer, fragments in first-occurrence order, each fragment's blocks. The
  // owner's send list starts as every candidate (select_send prunes it by the home's need flags)
  P.send_off.assign(1, 0);
  P.recv_off.assign(1, 0);
  P.cand_send_off.assign(1, 0);
  P.cand_send_blk.assign(1, 0);
  P.cand_recv_off.assign(1, 0);
  for (int w = 0; w < world; ++w) {
    for (const Digest& d : send_list[w]) {
      const auto& b = owned_blocks.at(d);
      P.send_blocks.insert(P.send_blocks.end(), b.begin(), b.end());
      P.cand_send_blocks.insert(P.cand_send_blocks.end(), b.begin(), b.end());
      P.cand_send_blk.push_back(static_cast<int64_t>(P.cand_send_blocks.size()));
      P.cand_send_need.push_back(1);
    }
    P.send_off.push_back(static_cast<int64_t>(P.send_blocks.size()));
    P.cand_send_off.push_back(static_cast<int64_t>(P.cand_send_need.size()));
    for (const Digest& d : cand_recv[w]) P.cand_recv_need.push_back(recv_hit.at(d) ? 0 : 1);
    P.cand_recv_off.push_back(static_cast<int64_t>(P.cand_recv_need.size()));
    for (const Digest& d : recv_list[w]) {
      const auto& b = recv_blocks.at(d);
      P.recv_blocks.insert(P.recv_blocks.end(), b.begin(), b.end());
    }
    P.recv_off.push_back(static_cast<int64_t>(P.recv_blocks.size()));
  }
  std::stable_sort(P.tasks.begin(), P.tasks.end(), [](const PlanHost::Task& a, const PlanHost::Task& b) {
    return a.home != b.home ? a.home < b.home : a.query < b.query;
  });
  P.xq_off.assign(1, 0);
  for (int w = 0; w < world; ++w) {
    P.xq_queries.insert(P.xq_queries.end(), xq[w].begin(), xq[w].end());
    P.xq_off.push_back(static_cast<int32_t>(P.xq_queries.size()));
  }
  // join rows in query order; query_join_row_off is indexed by the global query id (queries
  // homed elsewhere have an empty range)
  std::vector<int32_t> cross_of(P.n_queries, -1);
  for (size_t i = 0; i < P.segs.size(); ++i)
    if (P.segs[i].kind == kCross) cross_of[P.segs[i].query] = static_cast<int32_t>(i);
  P.query_join_row_off.reserve(P.n_queries + 1);
  P.query_join_row_off.push_back(0);
  for (int32_t qi = 0; qi < P.n_queries; ++qi) {
    if (cross_of[qi] >= 0) rows(P.segs[cross_of[qi]], 0, &P.join_pos, &P.join_slot, &P.join_seg, cross_of[qi]);
    P.query_join_row_off.push_back(static_cast<int64_t>(P.join_pos.size()));
  }
  return 0;
}

bool select_send(PlanHost* p, int peer, const uint8_t* need, int64_t n) {
  if (peer < 0 || peer + 1 >= static_cast<int>(p->cand_send_off.size())) return false;
  const int64_t c0 = p->cand_send_off[peer], c1 = p->cand_send_off[peer + 1];
  if (n != c1 - c0) return false;
  for (int64_t i = 0; i < n; ++i) p->cand_send_need[c0 + i] = need[i] ? 1 : 0;
  p->send_blocks.clear();
  p->send_off.assign(1, 0);
  const int world = static_cast<int>(p->cand_send_off.size()) - 1;
  for (int w = 0; w < world; ++w) {
    for (int64_t c = p->cand_send_off[w]; c < p->cand_send_off[w + 1]; ++c)
      if (p->cand_send_need[c])
        p->send_blocks.insert(p->send_blocks.end(), p->cand_send_blocks.begin() + p->cand_send_blk[c],
                              p->cand_send_blocks.begin() + p->cand_send_blk[c + 1]);
    p->send_off.push_back(static_cast<int64_t>(p->send_blocks.size()));
  }
  return true;
}

void Store::release(const PlanHost& p) {
  for (int32_t b : p.pinned) {
    pins_[b]--;
    if (pins_[b] == 0 && meta_[b].resident) set_evictable(b, true);
  }
  for (int32_t b : p.priv) free_.insert(b);
}

void Store::abort(const PlanHost& p) {
  release(p);
  std::vector<uint8_t> priv(static_cast<size_t>(nblocks_), 0);
  for (int32_t b : p.priv) priv[b] = 1;
  for (size_t i = 0; i < p.blocks.size(); ++i) {
    const int32_t b = p.blocks[i];
    if (!p.block_write[i] || priv[b] || !meta_[b].resident) continue;
    if (index_.find(p.digests[i]) == b && pins_[b] == 0) drop(b);
  }
  for (int32_t b : p.replicas)  // indexed, but the exchange never delivered their KV
    if (meta_[b].resident && pins_[b] == 0) drop(b);
}

int Store::extend_private(PlanHost* p, int64_t n, std::vector<int32_t>* out) {
  std::vector<int32_t> got;
  journal_.clear();
  journaling_ = true;
  bool ok = true;
  for (int64_t i = 0; i < n && ok; ++i) {
    const int32_t b = alloc(&ok);
    if (ok) got.push_back(b);
  }
  if (!ok) {
    rollback();
    journaling_ = false;
    return 2;
  }
  journal_.clear();
  journaling_ = false;
  for (int32_t b : got) {
    p->priv.push_back(b);
    p->pinned.push_back(b);
    pins_[b]++;
  }
  out->insert(out->end(), got.begin(), got.end());
  return 0;
}

int64_t Store::commit(PlanHost* p, const int32_t* blocks, const Digest* dig, const int32_t* ntok, int64_t n) {
  int64_t done = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t b = blocks[i];
    if (index_.find(dig[i]) >= 0) continue;  // resident already (here or in an equal-content block)
    if (meta_[b].resident) {           // re-key (e.g. a full cross block under its X digest)
      if (pins_[b] == 0) set_evictable(b, false);
      index_.erase(meta_[b].dig);
    }
    index_.set(dig[i], b);
    meta_[b] = Meta{dig[i], ntok[i], plan_no_, true};
    auto pv = std::find(p->priv.begin(), p->priv.end(), b);
    if (pv != p->priv.end()) p->priv.erase(pv);
    if (std::find(p->pinned.begin(), p->pinned.end(), b) == p->pinned.end()) {
      p->pinned.push_back(b);
      pins_[b]++;
    }
    stats_.inserted_blocks++;
    ++done;
  }
  return done;
}

void Store::drop(int32_t b) {
  if (!meta_[b].resident) return;
  set_evictable(b, false);
  index_.erase(meta_[b].dig);
  meta_[b].resident = false;
  free_.insert(b);
}

void Store::evict_all() {
  std::vector<int32_t> victims;
  for (int32_t b = 0; b < static_cast<int32_t>(nblocks_); ++b)
    if (meta_[b].resident && pins_[b] == 0) victims.push_back(b);
  for (int32_t b : victims) {
    set_evictable(b, false);
    index_.erase(meta_[b].dig);
    meta_[b].resident = false;
    free_.insert(b);
  }
}

int Store::insert(const Digest* d, const int32_t* ntok, int64_t n, int32_t* ids) {
  const StoreStats saved = stats_;
  journal_.clear();
  journaling_ = true;
  bool ok = true;
  for (int64_t i = 0; i < n && ok; ++i) {
    const int32_t r = lookup(d[i]);
    if (r >= 0) {
      ids[i] = r;
      continue;
    }
    const int32_t b = alloc(&ok);
    if (!ok) break;
    index_.set(d[i], b);
    meta_[b] = Meta{d[i], ntok[i], plan_no_, true};
    journal_.push_back({kUndoInsert, b, Meta{}});
    set_evictable(b, true);
    stats_.inserted_blocks++;
    ids[i] = b;
  }
  if (!ok) {
    rollback();
    stats_ = saved;
    journaling_ = false;
    return 2;
  }
  journal_.clear();
  journaling_ = false;
  return 0;
}

}  // namespace spq
