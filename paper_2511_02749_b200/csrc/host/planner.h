// planner.h — span-query planner and content-hash block store (host, C++17).
//
// Step a1-a3 of SURVEY §8(a): normalize the tree (plus simplification
// P:439), hash blocks (prefix chain P:97-98, suspended fragment chain P:603, ordered join fold,
// cross chain), prefix-scan / all-or-nothing lookup, in-plan dedupe, lowest-id allocation, LRU
// eviction of unpinned blocks, pinning, rollback on ENOMEM. Readings R8-R13.
#pragma once
#include <algorithm>
#include <cstdint>
#include <set>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "blake2b.h"
#include "thread_pool.h"

#include "../../../include/spanq.h"

namespace spq {

enum SegKind : int32_t { kPrefix = 0, kFrag = 1, kCross = 2 };

struct FlatQuery {
  std::vector<int32_t> prefix;
  std::vector<std::vector<int32_t>> frags;
  std::vector<int32_t> cross;
};

// Validate + flatten an ABI tree. Returns false and sets *err on an invalid tree.
bool normalize_tree(const spq_query& q, FlatQuery* out, std::string* err);

struct Segment {
  int32_t query, kind, frag_idx, tok_len, pos0, hit, compute_begin, block_off, n_blocks;
};

struct StoreStats {
  int64_t lookups = 0, hit_blocks = 0, miss_blocks = 0, hit_tokens = 0, input_tokens = 0,
          evictions = 0, inserted_blocks = 0;
};

struct PlanHost {
  std::vector<Segment> segs;
  std::vector<int32_t> blocks;
  std::vector<uint8_t> block_write;
  std::vector<Digest> digests;
  std::vector<Digest> join_digests;
  std::vector<int32_t> jobs;
  std::vector<int64_t> job_row_off;
  std::vector<int32_t> prefill_pos;
  std::vector<int64_t> prefill_slot;
  std::vector<int32_t> prefill_seg;
  std::vector<int32_t> join_pos;
  std::vector<int64_t> join_slot;
  std::vector<int32_t> join_seg;
  std::vector<int64_t> query_join_row_off;
  std::vector<int64_t> pad_slots;
  std::vector<int32_t> pinned;
  std::vector<int32_t> priv;
  int32_t n_queries = 0;
  int32_t n_join_queries = 0;  // queries homed on this rank (all when world == 1)
  // W > 1 fragment exchange: blocks sent to / received from each peer
  std::vector<int64_t> send_off, recv_off;  // [world+1]
  std::vector<int32_t> send_blocks, recv_blocks;
  // owner-side split join (split mode): tasks this rank computes for other homes
  // in (home, query) order — the home query's cross rows over the fragments of it owned here
  // (segments [seg_begin, seg_end), pos0 = Δ_f) — and, per peer owner, the home queries whose
  // cross Q this rank sends there and whose partials come back (query order)
  struct Task {
    int32_t query, home, n_rows, pos0, seg_begin, seg_end;
  };
  std::vector<Task> tasks;
  std::vector<int32_t> xq_off;  // [world+1]
  std::vector<int32_t> xq_queries;
  // digest-keyed replicas (reading R38). Home side: per owner peer, the remote fragments its joins
  // read (first-occurrence order) and whether their KV must be sent — 0 when a replica kept from an
  // earlier exchange is resident here (received fragments are indexed under their digests). Owner
  // side: per home peer, the same candidate sequence with each fragment's block range; the home's
  // need flags select which of them the send list carries (select_send; all until then).
  std::vector<int64_t> cand_recv_off;  // [world+1]
  std::vector<uint8_t> cand_recv_need;
  std::vector<int64_t> cand_send_off;  // [world+1]
  std::vector<int64_t> cand_send_blk;  // [n_cand+1] ranges into cand_send_blocks
  std::vector<int32_t> cand_send_blocks;
  std::vector<uint8_t> cand_send_need;
  std::vector<int32_t> replicas;  // blocks indexed by this plan whose KV only the exchange delivers
};

// Owner side: keep in the send list to `peer` only the candidates the home flagged (need[i] != 0,
// n = the peer's candidate count); rebuilds send_blocks / send_off. Returns false on a count mismatch.
bool select_send(PlanHost* p, int peer, const uint8_t* need, int64_t n);

// Fragment owner rank: u64le(s_last[0:8]) mod W.
int owner_rank(const Digest& d, int world);

// Digest chains (hash contract): ROOT, 'P' prefix, 'F' fragment, 'J' fold, 'X' cross.
Digest root_digest(int hq, int hkv, int d, int bs, double rope_base, uint64_t salt);
void chain(char tag, const Digest& seed, const int32_t* tok, int64_t n, int bs,
           std::vector<Digest>* out);
Digest join_fold(const Digest& h_last, const std::vector<Digest>& frag_lasts);

// Free block ids with O(1) amortized "pop the lowest" (a bitmap plus a hint: every word before
// `hint_` is empty) — the lowest-id allocation policy (R12) without a tree node per block.
class FreeSet {
 public:
  void init(int64_t n) {
    bits_.assign(static_cast<size_t>((n + 63) / 64), ~0ULL);
    if (n % 64) bits_.back() = (1ULL << (n % 64)) - 1;
    count_ = n;
    hint_ = 0;
  }
  bool empty() const { return count_ == 0; }
  int64_t size() const { return count_; }
  void insert(int32_t b) {
    uint64_t& w = bits_[static_cast<size_t>(b) >> 6];
    const uint64_t m = 1ULL << (b & 63);
    if (w & m) return;
    w |= m;
    ++count_;
    hint_ = std::min<int64_t>(hint_, b >> 6);
  }
  int32_t pop_lowest() {  // requires !empty()
    while (bits_[static_cast<size_t>(hint_)] == 0) ++hint_;
    uint64_t& w = bits_[static_cast<size_t>(hint_)];
    const int bit = __builtin_ctzll(w);
    w &= w - 1;
    --count_;
    return static_cast<int32_t>(hint_ * 64 + bit);
  }

 private:
  std::vector<uint64_t> bits_;
  int64_t count_ = 0, hint_ = 0;
};

// Digest -> block id, open addressing with linear probing and backward-shift deletion (no
// tombstones) over a power-of-two table of >= 2x the pool's blocks: no allocation per insert
// (std::unordered_map allocated a node for every block a plan inserted)
class DigestIndex {
 public:
  void init(int64_t max_entries) {
    size_t cap = 16;
    while (cap < static_cast<size_t>(2 * max_entries)) cap <<= 1;
    keys_.assign(cap, Digest{});
    vals_.assign(cap, -1);
    mask_ = cap - 1;
    n_ = 0;
  }
  int32_t find(const Digest& d) const {
    for (size_t i = slot(d);; i = (i + 1) & mask_) {
      if (vals_[i] < 0) return -1;
      if (keys_[i] == d) return vals_[i];
    }
  }
  void set(const Digest& d, int32_t v) {  // insert or overwrite
    size_t i = slot(d);
    for (; vals_[i] >= 0; i = (i + 1) & mask_)
      if (keys_[i] == d) {
        vals_[i] = v;
        return;
      }
    keys_[i] = d;
    vals_[i] = v;
    ++n_;
  }
  void erase(const Digest& d) {
    size_t i = slot(d);
    for (;; i = (i + 1) & mask_) {
      if (vals_[i] < 0) return;
      if (keys_[i] == d) break;
    }
    // backward shift: pull later entries of the probe run into the hole when their home slot
    // does not lie (cyclically) after the hole
    for (size_t j = (i + 1) & mask_; vals_[j] >= 0; j = (j + 1) & mask_) {
      const size_t k = slot(keys_[j]);
      if (((j - k) & mask_) >= ((j - i) & mask_)) {
        keys_[i] = keys_[j];
        vals_[i] = vals_[j];
        i = j;
      }
    }
    vals_[i] = -1;
    --n_;
  }
  size_t size() const { return n_; }

 private:
  size_t slot(const Digest& d) const { return DigestHash()(d) & mask_; }
  std::vector<Digest> keys_;
  std::vector<int32_t> vals_;
  size_t mask_ = 0, n_ = 0;
};

class Store {
 public:
  Store(int64_t num_blocks, int block_size, const Digest& root);

  // Plan a batch. Returns 0 on success, 2 on ENOMEM (state rolled back). Block digests do
  // not depend on store state, so they are computed first, in parallel on `pool` if given.
  int plan(const std::vector<FlatQuery>& qs, PlanHost* out, ThreadPool* pool = nullptr, int rank = 0,
           int world = 1, bool split = false);
  void release(const PlanHost& p);
  // Undo a committed plan whose device side failed: release it and forget the blocks it inserted
  // (their KV was never written, so their digests must not produce cache hits).
  void abort(const PlanHost& p);
  // Forget the digest held by block b (its content was rewritten in place): resident -> free.
  // Pinned blocks are the caller's to exclude.
  void drop(int32_t b);
  bool is_pinned(int32_t b) const { return pins_[b] > 0; }
  // Allocate n more plan-private blocks for a live plan (lowest free id, LRU eviction; pinned,
  // freed at release). All-or-nothing: returns 2 (ENOMEM, nothing allocated) or 0.
  int extend_private(PlanHost* p, int64_t n, std::vector<int32_t>* out);
  // Plus distribution: index blocks[i] under dig[i] (ntok[i] tokens) as cached KV of a
  // live plan. A block already indexed under another digest is re-keyed; a digest already
  // resident elsewhere is left alone (the two blocks hold the same content); plan-private blocks
  // leave the plan's private list (they are no longer freed at release, only unpinned).
  // Returns the number of blocks indexed.
  int64_t commit(PlanHost* p, const int32_t* blocks, const Digest* dig, const int32_t* ntok, int64_t n);
  void evict_all();
  int32_t lookup(const Digest& d) const;
  // Low-level insert: returns 0 or 2 (ENOMEM, rolled back).
  int insert(const Digest* d, const int32_t* ntok, int64_t n, int32_t* ids);

  const StoreStats& stats() const { return stats_; }
  int64_t resident() const { return static_cast<int64_t>(index_.size()); }
  int64_t free_count() const { return static_cast<int64_t>(free_.size()); }
  int64_t pinned_count() const;
  int64_t plans() const { return plan_no_; }
  const Digest& root() const { return root_; }
  int block_size() const { return bs_; }

 private:
  struct Meta {
    Digest dig;
    int32_t ntok;
    int64_t last_use;
    bool resident;
  };
  enum UndoKind { kUndoFreePop, kUndoEvict, kUndoInsert, kUndoPin, kUndoTouch };
  struct Undo {
    UndoKind kind;
    int32_t block;
    Meta meta;  // previous meta (evict / touch)
  };

  int32_t alloc(bool* ok);
  void pin(int32_t b);
  void touch(int32_t b);
  int32_t insert_new(const Digest& d, int32_t ntok);
  void rollback();
  void set_evictable(int32_t b, bool on);

  int64_t nblocks_;
  int bs_;
  Digest root_;
  DigestIndex index_;
  std::vector<Meta> meta_;
  std::vector<int32_t> pins_;
  FreeSet free_;
  std::set<std::pair<int64_t, int32_t>> evictable_;  // (last_use, id), resident & unpinned
  int64_t plan_no_ = 0;
  StoreStats stats_;
  std::vector<Undo> journal_;
  bool journaling_ = false;
  // per-plan pin bookkeeping
  std::vector<uint8_t> pinned_mark_;
  std::vector<int32_t>* cur_pinned_ = nullptr;
};

}  // namespace spq
