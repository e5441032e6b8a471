// work.h — device work lists of the span-attention kernels (host builds, device reads).
//
// One attention launch = a list of WorkItems; item i covers up to 128 query rows (one "q tile")
// of one job (fragment/prefix prefill) or one query's cross rows (join), and a contiguous range
// of KvTiles. A KvTile is <=128 keys of one KV segment, made of 128/bs pool blocks:
//   key t of the tile is visible to row r  iff  t < n_valid  and  (!causal or key_pos0+t <= pos[r])
//   before scoring against the tile, q of row r is rotated to position pos[r] - rot_delta.
// rot_delta is 0 for KV stored in the row's frame (prefix, cross, a fragment's own job) and
// Δ_f (the fragment's global start) for fragment KV read by the join: the cached KV stays at
// span-local positions and the query is counter-rotated instead ("ReRoPE", P:610 — relative
// RoPE makes q(p)·k(Δ+t) = q(p-Δ)·k(t)).
#pragma once
#include <cstdint>

namespace spq {

constexpr int kTileKeys = 128;  // keys per KV tile
constexpr int kTileRows = 128;  // query rows per work item (tcgen05 M = 128)

struct KvTile {
  int32_t blk_off;   // first of (kTileKeys / bs) entries in tile_blocks (padded by repetition)
  int32_t n_valid;   // valid keys in the tile, 1..128
  int32_t key_pos0;  // position of key 0 in the query rows' frame (causal test)
  int32_t rot_delta; // q rotated to pos[r] - rot_delta for this tile
  int32_t causal;    // 1 = causal segment
  int32_t pad0, pad1, pad2;
};

struct WorkItem {
  int32_t row0;        // first query row, in the launch's packed row space
  int32_t n_rows;      // 1..128
  int32_t tile_begin;  // KV tile range [tile_begin, tile_end)
  int32_t tile_end;
  int32_t part;        // -1: write final O/LSE; >= 0: split-KV partial slot
  int32_t n_sub;       // 64-key sub-tiles of the item (tiles with n_valid > 64 count twice)
  int32_t pad1, pad2;
};

// Split-KV partials are per work unit: partial slot p holds the unit's heads, rows
// ((p * n_heads + x) * kTileRows + r) of opart / lsepart (x = head - head0). A (q tile, unit)'s
// partials are the slots [part_base, part_base + n_split) followed by [part_base2, part_base2 +
// n_split2) (the second range: the remote-segment phase of a W > 1 join), merged in that order.
struct CombineDesc {
  int32_t row0, n_rows, part_base, n_split, head0, n_heads, part_base2, n_split2;
};

}  // namespace spq
