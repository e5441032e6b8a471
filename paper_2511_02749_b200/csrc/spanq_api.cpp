// spanq_api.cpp — implementation of include/spanq.h (the C ABI).
//
// Host side of the path: ctx (config, content-hash store, RoPE table, TMA descriptors, staging),
// plans (planner output + device work lists uploaded with one H2D copy), and the per-call
// kernel sequence:
//   spq_prefill_jobs: rope_kv_write (K1) -> span_attn (K2; tcgen05 bf16 or SIMT fp32)
//   spq_join:         rope_kv_write (K1) -> span_attn (K3, split-KV) -> combine (K4)
// No CPU fallback: a ctx with device >= 0 requires an sm_100 GPU and fails loudly otherwise.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <deque>
#include <map>
#include <unordered_set>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/spanq.h"
#include "host/cidra.h"
#include "host/planner.h"
#include "host/work_builder.h"
#include "kernels/launch.h"

namespace {

thread_local std::string g_err;

spq_status fail(spq_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(SPQ_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));             \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// One device buffer holding several arrays (one H2D copy): offsets are assigned first, the bytes
// are copied once, straight into the destination (pinned staging). Sources must outlive write().
struct Packer {
  size_t size = 0;
  std::vector<std::pair<size_t, std::pair<const void*, size_t>>> parts;
  template <typename T>
  size_t add(const std::vector<T>& v) {
    const size_t off = align_up(size, 256);
    parts.push_back({off, {v.data(), v.size() * sizeof(T)}});
    size = off + v.size() * sizeof(T);
    return off;
  }
  void write(uint8_t* dst) const {
    for (const auto& p : parts)
      if (p.second.second) std::memcpy(dst + p.first, p.second.first, p.second.second);
  }
};

const std::vector<int32_t> kZeros2 = {0, 0};  // claim counters of a dynamic work list

struct DevWork {  // offsets of one attention work list inside a plan buffer
  size_t tiles, tile_blocks, items, cta_off, cta_items, combine, sched;
  int32_t n_items = 0, grid = 0, n_combine = 0, n_parts = 0, n_codes = 0, cluster = 1;
  bool dynamic = false;
  double flops = 0;
};

}  // namespace

struct spq_ctx {
  spq_config cfg;
  std::unique_ptr<spq::Store> store;
  std::unique_ptr<spq::ThreadPool> pool;  // host planning (block hashing)
  int num_sms = 0;
  float2* rope = nullptr;  // device [max_position][d/2] (cos, sin) fp32: K1 (K pages) + fp32 path
  CUtensorMap tmk, tmv;
  CUtensorMap tmk2;  // K pool with boxes of min(bs, 32) rows (CTA-pair kernel, d = 128)
  bool have_tmk2 = false;
  bool have_tmap = false;
  std::vector<cudaEvent_t> pending;  // stream-ordered releases
  int64_t launches = 0;
  bool timing = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  float last_prefill_ms = 0.f, last_join_ms = 0.f;
  bool prefill_timed = false, join_timed = false;
  // pinned upload staging
  uint8_t* staging = nullptr;
  size_t staging_size = 0;
  cudaEvent_t staging_ev = nullptr;
  // a second one for the lazily built join work lists (W = 1 plans, ensure_join_work): with one
  // buffer a join's upload would wait for its own plan's upload and the next plan for that join's,
  // so the host could no longer run a whole query ahead of the GPU
  uint8_t* jstaging = nullptr;
  size_t jstaging_size = 0;
  cudaEvent_t jstaging_ev = nullptr;
  // options (spq_set_option)
  int exp2_mode = -1;              // SPQ_OPT_EXP2 (kernel poly_mask; -1 = auto: prefill 0, joins 1)
  float rescale_threshold = 8.0f;  // SPQ_OPT_RESCALE_THRESHOLD (log2 units)
  bool pdl = true;                 // SPQ_OPT_PDL
  bool pair = false;               // SPQ_OPT_PAIR (measured slower: DESIGN.md §6)
  // profiling builds only (spq_set_trace)
  long long* trace = nullptr;
  int dbg_mode = 0;
  // plan handles: live plans, and released ones kept (emptied) for kQuarantine more releases so
  // that a call on a released handle reports SPQ_ESTATE instead of touching freed memory
  std::unordered_set<spq_plan*> live;
  std::deque<spq_plan*> quarantine;
};
constexpr size_t kQuarantine = 1024;

struct spq_plan {
  spq::PlanHost host;
  bool released = false;
  // flat view arrays
  std::vector<int32_t> seg_query, seg_kind, seg_frag_idx, seg_tok_len, seg_pos0, seg_hit, seg_cb,
      seg_block_off, seg_n_blocks;
  std::vector<uint8_t> digests, join_digests;
  double prefill_flops = 0, join_flops = 0;
  int64_t prefill_kv_bytes = 0, join_kv_bytes = 0;
  // device
  uint8_t* dbuf = nullptr;
  size_t off_ppos = 0, off_pslot = 0, off_pad = 0, off_jpos = 0, off_jslot = 0, off_send = 0, off_recv = 0;
  DevWork pw, jw;
  bool phased = false;  // W > 1 with received fragments: the join also as two phases (jw1, jw2)
  DevWork jw1, jw2;
  spq::AttnWorkHost jw1_host, jw2_host;
  float* opart = nullptr;
  float* lsepart = nullptr;
  std::vector<uint8_t> padded_layers;
  spq::AttnWorkHost pw_host, jw_host;  // kept for sub-range rebuilds / inspection
  // W = 1 GPU plans build and upload the join's work list at the first full join call (its own
  // device buffer, partials included): that host work then overlaps the prefill on the GPU
  bool jw_lazy = false;
  uint8_t* jbuf = nullptr;
  std::vector<std::vector<int32_t>> cross_tokens;  // per query (plus distribution: commit)
  // owner-side split join (world > 1, cfg.split_join)
  bool split = false;
  spq::AttnWorkHost tw_host;  // the tasks' join (owner side)
  struct Split {
    DevWork tw;
    int64_t task_rows = 0, xq_rows = 0, home_rows = 0;
    size_t off_tpos = 0, off_xrows = 0, off_mdesc = 0, off_msrc = 0;
    int32_t n_mdesc = 0;
    float *o_loc = nullptr, *lse_loc = nullptr;    // home: the local join, fp32
    float *topart = nullptr, *tlsepart = nullptr;  // owner: split pieces of the task join
  } sp;
  // decode after the join (spq_decode_reserve / spq_decode_step / spq_commit_span)
  struct Decode {
    int32_t max_new = 0;
    std::vector<int32_t> rows;                      // home query of each decode row
    std::vector<std::vector<int32_t>> blocks;       // per row: cross blocks + generation blocks
    uint8_t* dbuf = nullptr;
    size_t off_tiles = 0, off_tb = 0, off_items = 0, off_comb = 0, off_posb = 0, off_kpos = 0, off_kslot = 0,
           off_done = 0;
    float* opart = nullptr;
    float* lsepart = nullptr;
    int32_t n_items = 0, n_comb = 0;
  } dec;
};

using Decode = spq_plan::Decode;

namespace {

bool is_gpu(const spq_ctx* c) { return c->cfg.device >= 0; }

// tcgen05 path pairs the two q heads of a GQA group (shared K/V) when the group size is even
bool paired(const spq_ctx* c) {
  return c->cfg.dtype == SPQ_BF16 && (c->cfg.num_q_heads / c->cfg.num_kv_heads) % 2 == 0;
}

// heads per attention work unit (a split-KV partial slot holds one unit's heads)
int heads_per_unit(const spq_ctx* c) { return paired(c) ? 2 : 1; }

// host-only contexts plan for a B200 (148 SMs) so their work lists match a GPU ctx's
spq::WorkOpts work_opts(const spq_ctx* c, bool allow_split) {
  spq::WorkOpts o{};
  o.hq = c->cfg.num_q_heads;
  o.d = c->cfg.head_dim;
  o.bs = c->cfg.block_size;
  o.num_sms = c->num_sms > 0 ? c->num_sms : 148;
  o.allow_split = allow_split;
  o.persistent = c->cfg.dtype == SPQ_BF16;
  o.units = paired(c) ? o.hq / 2 : o.hq;
  return o;
}
// The prefill launches run on CTA pairs (cta_group::2, span_attn_tc.cu PR) when the shape allows
// it: bf16, d = 128, GQA groups of 4k heads, bf16 O (the Q-prep-warp epilogue), an even SM count.
// Decided when a plan's work list is built (the launch follows the list's cluster size).
bool pair_prefill(const spq_ctx* c) {
  const spq_config& g = c->cfg;
  const int sms = c->num_sms > 0 ? c->num_sms : 148;
  return c->pair && g.dtype == SPQ_BF16 && g.head_dim == 128 && (g.num_q_heads / g.num_kv_heads) % 4 == 0 &&
         g.out_dtype != SPQ_FP32 && sms % 2 == 0 && (!is_gpu(c) || c->have_tmk2);
}
spq::WorkOpts prefill_opts(const spq_ctx* c) {
  spq::WorkOpts o = work_opts(c, false);
  if (pair_prefill(c)) {
    o.units = o.hq / 4;
    o.cluster = 2;
  }
  return o;
}

int elt_size(const spq_ctx* c) { return c->cfg.dtype == SPQ_FP32 ? 4 : 2; }

spq_status make_tmap(spq_ctx* c, void* pool, CUtensorMap* out, int max_box_rows = 64) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (fn == nullptr || q != cudaDriverEntryPointSuccess)
    return fail(SPQ_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const spq_config& g = c->cfg;
  const uint64_t rows = static_cast<uint64_t>(g.num_layers) * g.num_blocks * g.num_kv_heads * g.block_size;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.head_dim), rows};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.head_dim) * 2};
  // one box = 64 columns x min(bs, 64) rows: the attention kernel streams 64-key sub-tiles
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(std::min(g.block_size, max_box_rows))};
  cuuint32_t es[2] = {1, 1};
  CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(
      out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SPQ_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return SPQ_OK;
}

// per-call TMA map of the packed q rows: 3D {d, hq, rows}, box {64, 1, 128}, SWIZZLE_128B
spq_status make_qmap(const spq_ctx* c, const void* q, int64_t rows, CUtensorMap* out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
  if (fn == nullptr || qr != cudaDriverEntryPointSuccess) return fail(SPQ_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(q) & 15) return fail(SPQ_EINVAL, "q must be 16-byte aligned");
  const spq_config& g = c->cfg;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.head_dim), static_cast<cuuint64_t>(g.num_q_heads),
                        static_cast<cuuint64_t>(std::max<int64_t>(rows, 1))};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(g.head_dim) * 2,
                           static_cast<cuuint64_t>(g.head_dim) * 2 * g.num_q_heads};
  cuuint32_t box[3] = {64, 1, 128};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(q), dims,
                                                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SPQ_ECUDA, "cuTensorMapEncodeTiled(q) failed: " + std::to_string(r));
  return SPQ_OK;
}

// output maps for the epilogue's TMA stores: o as 3D {d, hq, rows}, box {32, 1, 32} (fp32) or
// {64, 1, 32} (bf16): 128-byte rows; partials as 2D {d, parts*hq*128} box {32, 32}; all
// SWIZZLE_128B (the staging layout)
spq_status make_omap(const spq_ctx* c, const void* o, int64_t rows, CUtensorMap* out, int f32_override = -1) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
  if (reinterpret_cast<uintptr_t>(o) & 15) return fail(SPQ_EINVAL, "o must be 16-byte aligned");
  const spq_config& g = c->cfg;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.head_dim), static_cast<cuuint64_t>(g.num_q_heads),
                        static_cast<cuuint64_t>(std::max<int64_t>(rows, 1))};
  const bool f32 = f32_override >= 0 ? f32_override != 0 : g.out_dtype == SPQ_FP32;
  const cuuint64_t elt = f32 ? 4 : 2;
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(g.head_dim) * elt,
                           static_cast<cuuint64_t>(g.head_dim) * elt * g.num_q_heads};
  cuuint32_t box[3] = {f32 ? 32u : 64u, 1, 32};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(out, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(o), dims,
                                                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SPQ_ECUDA, "cuTensorMapEncodeTiled(o) failed: " + std::to_string(r));
  return SPQ_OK;
}

spq_status make_partmap(const spq_ctx* c, const float* opart, int64_t parts, CUtensorMap* out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
  const spq_config& g = c->cfg;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.head_dim),
                        static_cast<cuuint64_t>(parts) * heads_per_unit(c) * spq::kTileRows};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.head_dim) * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(opart),
                                                   dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SPQ_ECUDA, "cuTensorMapEncodeTiled(opart) failed: " + std::to_string(r));
  return SPQ_OK;
}

spq_status wait_pending(spq_ctx* c, cudaStream_t st) {
  std::vector<cudaEvent_t> keep;
  for (cudaEvent_t e : c->pending) {
    if (cudaEventQuery(e) == cudaSuccess) {
      cudaEventDestroy(e);
      continue;
    }
    CUDA_TRY(cudaStreamWaitEvent(st, e, 0));
    keep.push_back(e);
  }
  c->pending.swap(keep);
  return SPQ_OK;
}

template <typename T>
T* at(const spq_plan* p, size_t off) {
  return reinterpret_cast<T*>(p->dbuf + off);
}

void fill_attn(spq_ctx* c, const spq_plan* p, const DevWork& w, spq::AttnArgs* a) {
  a->tiles = at<spq::KvTile>(p, w.tiles);
  a->tile_blocks = at<int32_t>(p, w.tile_blocks);
  a->items = at<spq::WorkItem>(p, w.items);
  a->n_items = w.n_items;
  a->cta_off = at<int32_t>(p, w.cta_off);
  a->cta_items = at<int32_t>(p, w.cta_items);
  a->sched = w.dynamic ? at<int32_t>(p, w.sched) : nullptr;
  a->cluster = w.cluster;
  a->tmap_k2 = c->have_tmk2 ? &c->tmk2 : nullptr;
  a->n_codes = w.n_codes;
  a->grid = w.grid;
  a->k_pool = c->cfg.k_pool;
  a->v_pool = c->cfg.v_pool;
  a->tmap_k = &c->tmk;
  a->tmap_v = &c->tmv;
  a->hq = c->cfg.num_q_heads;
  a->hkv = c->cfg.num_kv_heads;
  a->d = c->cfg.head_dim;
  a->bs = c->cfg.block_size;
  a->nblk = c->cfg.num_blocks;
  a->rope = c->rope;
  a->max_pos = c->cfg.max_position;
  a->opart = p->opart;
  a->lsepart = p->lsepart;
  a->out_fp32 = c->cfg.out_dtype == SPQ_FP32;
  a->paired = paired(c);
  a->poly_mask = c->exp2_mode < 0 ? 0 : c->exp2_mode;
  a->rescale_threshold = c->rescale_threshold;
  a->dbg_trace = c->trace;  // null unless a profiling build set it (spq_set_trace)
  a->dbg_mode = c->dbg_mode;
}

spq_status run_attn(spq_ctx* c, const spq::AttnArgs& a, cudaStream_t st) {
  cudaError_t e = c->cfg.dtype == SPQ_FP32 ? spq::launch_span_attn_f32(a, st) : spq::launch_span_attn_tc(a, st);
  if (e != cudaSuccess) return fail(SPQ_ECUDA, std::string("span_attn launch: ") + cudaGetErrorString(e));
  if (a.n_items > 0) c->launches++;
  return SPQ_OK;
}

spq_status kv_write(spq_ctx* c, spq_plan* p, int32_t layer, const void* k, const void* v,
                    const int32_t* pos, const int64_t* slot, int64_t rows, cudaStream_t st,
                    bool* launched = nullptr) {
  if (launched) *launched = false;
  spq::KvWriteArgs w{};
  w.k = k;
  w.v = v;
  w.pos = pos;
  w.slot = slot;
  w.rows = rows;
  const bool pad = !p->padded_layers[layer];
  w.pad_slots = at<int64_t>(p, p->off_pad);
  w.n_pad = pad ? static_cast<int64_t>(p->host.pad_slots.size()) : 0;
  w.k_pool = c->cfg.k_pool;
  w.v_pool = c->cfg.v_pool;
  w.hkv = c->cfg.num_kv_heads;
  w.d = c->cfg.head_dim;
  w.bs = c->cfg.block_size;
  w.nblk = c->cfg.num_blocks;
  w.layer = layer;
  w.rope = c->rope;
  w.fp32 = c->cfg.dtype == SPQ_FP32;
  if (rows + w.n_pad == 0) return SPQ_OK;
  cudaError_t e = spq::launch_rope_kv_write(w, st);
  if (e != cudaSuccess) return fail(SPQ_ECUDA, std::string("rope_kv_write launch: ") + cudaGetErrorString(e));
  p->padded_layers[layer] = 1;
  c->launches++;
  if (launched) *launched = true;
  return SPQ_OK;
}

spq_status check_call(spq_ctx* c, spq_plan* p, int32_t layer) {
  if (c == nullptr || p == nullptr) return fail(SPQ_EINVAL, "null ctx/plan");
  if (!c->live.count(p)) return fail(SPQ_ESTATE, "plan used after release (or not a plan of this ctx)");
  if (!is_gpu(c)) return fail(SPQ_ESTATE, "host-only ctx (device < 0) cannot run kernels");
  if (layer < 0 || layer >= c->cfg.num_layers) return fail(SPQ_ESTATE, "layer out of range");
  return SPQ_OK;
}

// Upload a sub-range work list (not the precomputed full range) into a temporary buffer.
struct TempWork {
  uint8_t* buf = nullptr;
  DevWork w;
};

spq_status upload_work(spq_ctx* c, const spq::AttnWorkHost& h, cudaStream_t st, TempWork* tw) {
  Packer pk;
  tw->w.tiles = pk.add(h.tiles);
  tw->w.tile_blocks = pk.add(h.tile_blocks);
  tw->w.items = pk.add(h.items);
  tw->w.cta_off = pk.add(h.cta_off);
  tw->w.cta_items = pk.add(h.cta_items);
  tw->w.sched = pk.add(kZeros2);  // claim counters (self-resetting)
  tw->w.dynamic = h.dynamic;
  tw->w.n_codes = static_cast<int32_t>(h.cta_items.size());
  tw->w.combine = pk.add(h.combine);
  tw->w.n_items = static_cast<int32_t>(h.items.size());
  tw->w.grid = h.grid;
  tw->w.cluster = h.cluster;
  tw->w.n_combine = static_cast<int32_t>(h.combine.size());
  tw->w.n_parts = h.n_parts;
  std::vector<uint8_t> host(pk.size);
  pk.write(host.data());
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tw->buf), std::max<size_t>(pk.size, 256), st));
  CUDA_TRY(cudaMemcpyAsync(tw->buf, host.data(), pk.size, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));  // pageable source: keep it alive until the copy is done
  return SPQ_OK;
}

}  // namespace

extern "C" {

const char* spq_last_error(void) { return g_err.c_str(); }
const char* spq_version(void) { return "spanq-b200 0.1 (sm_100a tcgen05)"; }

spq_status spq_create(const spq_config* cfg, spq_ctx** out) {
  if (cfg == nullptr || out == nullptr) return fail(SPQ_EINVAL, "null argument");
  const spq_config& g = *cfg;
  if (g.num_q_heads <= 0 || g.num_kv_heads <= 0 || g.num_q_heads % g.num_kv_heads != 0)
    return fail(SPQ_EINVAL, "Hq must be a positive multiple of Hkv");
  if (g.num_layers <= 0 || g.block_size <= 0 || g.num_blocks <= 0 || g.num_blocks > INT32_MAX)
    return fail(SPQ_EINVAL, "bad layers/block_size/num_blocks");
  if (g.dtype != SPQ_BF16 && g.dtype != SPQ_FP32) return fail(SPQ_EINVAL, "bad dtype");
  if (g.out_dtype != SPQ_BF16 && g.out_dtype != SPQ_FP32) return fail(SPQ_EINVAL, "bad out_dtype");
  if (g.dtype == SPQ_FP32 && g.out_dtype != SPQ_FP32) return fail(SPQ_EINVAL, "fp32 ctx needs fp32 outputs");
  if (g.world_size < 1 || g.rank < 0 || g.rank >= g.world_size) return fail(SPQ_EINVAL, "bad rank/world_size");
  if (g.max_position <= 0 || !(g.rope_base > 0)) return fail(SPQ_EINVAL, "bad rope parameters");
  std::unique_ptr<spq_ctx> c(new spq_ctx());
  c->cfg = g;
  {
    const unsigned hw = std::thread::hardware_concurrency();
    c->pool.reset(new spq::ThreadPool(static_cast<int>(std::min(15u, hw > 1 ? hw - 1 : 0u))));
  }
  c->store.reset(new spq::Store(g.num_blocks, g.block_size,
                                spq::root_digest(g.num_q_heads, g.num_kv_heads, g.head_dim, g.block_size,
                                                 g.rope_base, g.model_salt)));
  if (g.device >= 0) {
    if (g.head_dim != 64 && g.head_dim != 128) return fail(SPQ_EINVAL, "head_dim must be 64 or 128 on the GPU");
    if (g.block_size > 128 || (g.block_size & (g.block_size - 1)) != 0)
      return fail(SPQ_EINVAL, "block_size must be a power of two <= 128 on the GPU");
    if (g.dtype == SPQ_BF16 && g.block_size < 16) return fail(SPQ_EINVAL, "bf16 path needs block_size >= 16");
    if (g.k_pool == nullptr || g.v_pool == nullptr) return fail(SPQ_EINVAL, "null KV pool");
    if ((reinterpret_cast<uintptr_t>(g.k_pool) | reinterpret_cast<uintptr_t>(g.v_pool)) & 127)
      return fail(SPQ_EINVAL, "KV pools must be 128-byte aligned");
    CUDA_TRY(cudaSetDevice(g.device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, g.device));
    if (prop.major != 10 || prop.minor != 0)
      return fail(SPQ_ECUDA, "device is sm_" + std::to_string(prop.major) + std::to_string(prop.minor) +
                                 "; this library is built for sm_100a only");
    c->num_sms = prop.multiProcessorCount;
    // plans allocate their device arrays with cudaMallocAsync: keep freed memory in the pool
    // (the default threshold 0 returns it at every sync and re-maps it on the next plan)
    cudaMemPool_t mp;
    CUDA_TRY(cudaDeviceGetDefaultMemPool(&mp, g.device));
    uint64_t thr = UINT64_MAX;
    CUDA_TRY(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr));
    // RoPE table from fp64: cos/sin(p * base^(-2i/d)) rounded once to fp32
    const int half = g.head_dim / 2;
    std::vector<float2> tab(static_cast<size_t>(g.max_position) * half);
    for (int i = 0; i < half; ++i) {
      const double th = std::pow(g.rope_base, -2.0 * i / g.head_dim);
      for (int64_t p = 0; p < g.max_position; ++p) {
        const double a = static_cast<double>(p) * th;
        tab[p * half + i] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
      }
    }
    CUDA_TRY(cudaMalloc(&c->rope, tab.size() * sizeof(float2)));
    CUDA_TRY(cudaMemcpy(c->rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
    if (g.dtype == SPQ_BF16) {
      spq_status s = make_tmap(c.get(), g.k_pool, &c->tmk);
      if (s != SPQ_OK) return s;
      s = make_tmap(c.get(), g.v_pool, &c->tmv);
      if (s != SPQ_OK) return s;
      c->have_tmap = true;
      if (g.head_dim == 128) {  // CTA-pair prefill: each CTA loads 32 keys of a K sub-tile
        s = make_tmap(c.get(), g.k_pool, &c->tmk2, 32);
        if (s != SPQ_OK) return s;
        c->have_tmk2 = true;
      }
    }
    for (auto& e : c->ev) CUDA_TRY(cudaEventCreate(&e));
    CUDA_TRY(cudaEventCreateWithFlags(&c->staging_ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->jstaging_ev, cudaEventDisableTiming));
  }
  *out = c.release();
  return SPQ_OK;
}

void spq_destroy(spq_ctx* c) {
  if (c == nullptr) return;
  if (is_gpu(c)) {
    cudaSetDevice(c->cfg.device);
    cudaDeviceSynchronize();
    for (cudaEvent_t e : c->pending) cudaEventDestroy(e);
    for (auto& e : c->ev)
      if (e) cudaEventDestroy(e);
    if (c->staging_ev) cudaEventDestroy(c->staging_ev);
    if (c->staging) cudaFreeHost(c->staging);
    if (c->jstaging_ev) cudaEventDestroy(c->jstaging_ev);
    if (c->jstaging) cudaFreeHost(c->jstaging);
    if (c->rope) cudaFree(c->rope);
  }
  for (spq_plan* p : c->live) {  // plans never released: their device arrays go with the ctx
    if (p->dbuf) cudaFree(p->dbuf);
    if (p->dec.dbuf) cudaFree(p->dec.dbuf);
    delete p;
  }
  for (spq_plan* p : c->quarantine) delete p;
  delete c;
}

spq_status spq_block_hashes(const spq_ctx* c, const spq_query* q, uint8_t* digests, int64_t cap, int64_t* n) {
  if (c == nullptr || q == nullptr || n == nullptr) return fail(SPQ_EINVAL, "null argument");
  spq::FlatQuery fq;
  std::string err;
  if (!spq::normalize_tree(*q, &fq, &err)) return fail(SPQ_EINVAL, err);
  const int bs = c->cfg.block_size;
  const spq::Digest& root = c->store->root();
  std::vector<spq::Digest> all, tmp;
  spq::chain('P', root, fq.prefix.data(), static_cast<int64_t>(fq.prefix.size()), bs, &tmp);
  all = tmp;
  const spq::Digest h_last = tmp.empty() ? root : tmp.back();
  std::vector<spq::Digest> lasts;
  for (const auto& f : fq.frags) {
    tmp.clear();
    spq::chain('F', root, f.data(), static_cast<int64_t>(f.size()), bs, &tmp);
    lasts.push_back(tmp.back());
    all.insert(all.end(), tmp.begin(), tmp.end());
  }
  const spq::Digest J = spq::join_fold(h_last, lasts);
  all.push_back(J);
  tmp.clear();
  spq::chain('X', J, fq.cross.data(), static_cast<int64_t>(fq.cross.size()), bs, &tmp);
  all.insert(all.end(), tmp.begin(), tmp.end());
  *n = static_cast<int64_t>(all.size());
  if (cap < *n || digests == nullptr) return fail(SPQ_EINVAL, "digest buffer too small");
  for (size_t i = 0; i < all.size(); ++i) std::memcpy(digests + 16 * i, all[i].b, 16);
  return SPQ_OK;
}

spq_status spq_lookup(const spq_ctx* c, const uint8_t* digests, int64_t n, int32_t* ids) {
  if (c == nullptr || (n > 0 && (digests == nullptr || ids == nullptr))) return fail(SPQ_EINVAL, "null argument");
  for (int64_t i = 0; i < n; ++i) {
    spq::Digest d;
    std::memcpy(d.b, digests + 16 * i, 16);
    ids[i] = c->store->lookup(d);
  }
  return SPQ_OK;
}

spq_status spq_insert(spq_ctx* c, const uint8_t* digests, const int32_t* ntok, int64_t n, int32_t* ids) {
  if (c == nullptr || (n > 0 && (digests == nullptr || ntok == nullptr || ids == nullptr)))
    return fail(SPQ_EINVAL, "null argument");
  std::vector<spq::Digest> d(n);
  for (int64_t i = 0; i < n; ++i) {
    if (ntok[i] < 1 || ntok[i] > c->cfg.block_size) return fail(SPQ_EINVAL, "ntok out of range");
    std::memcpy(d[i].b, digests + 16 * i, 16);
  }
  if (c->store->insert(d.data(), ntok, n, ids) != 0) return fail(SPQ_ENOMEM, "block pool exhausted (insert rolled back)");
  return SPQ_OK;
}

spq_status spq_plan_create(spq_ctx* c, const spq_query* queries, int32_t n_queries, void* stream, spq_plan** out) {
  if (c == nullptr || out == nullptr || (n_queries > 0 && queries == nullptr)) return fail(SPQ_EINVAL, "null argument");
  if (n_queries <= 0) return fail(SPQ_EINVAL, "n_queries must be >= 1");
  using clk = std::chrono::steady_clock;
#ifdef SPANQ_PROFILING
  static const bool prof = std::getenv("SPANQ_PROFILE") != nullptr;  // profiling builds only
#else
  constexpr bool prof = false;
#endif
  auto t0 = clk::now();
  auto lap = [&](const char* what) {
    if (!prof) return;
    auto t = clk::now();
    std::fprintf(stderr, "[spanq] plan_create %-12s %8.1f us\n", what,
                 std::chrono::duration<double, std::micro>(t - t0).count());
    t0 = t;
  };
  std::vector<spq::FlatQuery> fq(n_queries);
  for (int32_t i = 0; i < n_queries; ++i) {
    std::string err;
    if (!spq::normalize_tree(queries[i], &fq[i], &err))
      return fail(SPQ_EINVAL, "query " + std::to_string(i) + ": " + err);
    int64_t n = static_cast<int64_t>(fq[i].prefix.size() + fq[i].cross.size());
    for (const auto& f : fq[i].frags) n += static_cast<int64_t>(f.size());
    if (n > c->cfg.max_position)
      return fail(SPQ_EINVAL, "query " + std::to_string(i) + " exceeds max_position");
  }
  lap("normalize");
  std::unique_ptr<spq_plan> p(new spq_plan());
  if (c->store->plan(fq, &p->host, c->pool.get(), c->cfg.rank, c->cfg.world_size,
                     c->cfg.world_size > 1 && c->cfg.split_join != 0) != 0)
    return fail(SPQ_ENOMEM, "block pool cannot hold the plan (rolled back)");
  // from here on the store holds the plan's pins and inserted digests: any failure undoes them
  struct Guard {
    spq_ctx* c;
    spq_plan* p;
    bool armed = true;
    ~Guard() {
      if (!armed) return;
      c->store->abort(p->host);
      if (p->dbuf) cudaFree(p->dbuf);
    }
  } guard{c, p.get()};
  lap("store.plan");
  const spq::PlanHost& H = p->host;
  for (const spq::Segment& s : H.segs) {
    p->seg_query.push_back(s.query);
    p->seg_kind.push_back(s.kind);
    p->seg_frag_idx.push_back(s.frag_idx);
    p->seg_tok_len.push_back(s.tok_len);
    p->seg_pos0.push_back(s.pos0);
    p->seg_hit.push_back(s.hit);
    p->seg_cb.push_back(s.compute_begin);
    p->seg_block_off.push_back(s.block_off);
    p->seg_n_blocks.push_back(s.n_blocks);
  }
  for (const auto& q : fq) p->cross_tokens.push_back(q.cross);
  for (const auto& d : H.digests) p->digests.insert(p->digests.end(), d.b, d.b + 16);
  for (const auto& d : H.join_digests) p->join_digests.insert(p->join_digests.end(), d.b, d.b + 16);
  p->padded_layers.assign(c->cfg.num_layers, 0);
  // host-only contexts plan for a B200 (148 SMs) so their work lists match a GPU ctx's
  spq::WorkOpts o = work_opts(c, c->cfg.dtype == SPQ_BF16);
  lap("view arrays");
  spq::build_prefill_work(H, prefill_opts(c), 0, static_cast<int>(H.jobs.size()), &p->pw_host);
  lap("prefill work");
  p->jw_lazy = is_gpu(c) && c->cfg.world_size == 1;
  if (!p->jw_lazy) spq::build_join_work(H, o, 0, H.n_queries, &p->jw_host);
  // W > 1: the join again as two phases around the exchange (held segments, then the received
  // fragments), for spq_join_phase; needs split partials (the persistent bf16 path)
  if (is_gpu(c) && o.allow_split && o.persistent && !H.recv_blocks.empty()) {
    std::vector<uint8_t> remote(H.segs.size(), 0);
    std::unordered_set<int32_t> rs(H.recv_blocks.begin(), H.recv_blocks.end());
    for (size_t i = 0; i < H.segs.size(); ++i) {
      const spq::Segment& sg = H.segs[i];
      remote[i] = sg.kind == spq::kFrag && sg.n_blocks > 0 && rs.count(H.blocks[sg.block_off]) ? 1 : 0;
    }
    std::map<std::pair<int32_t, int32_t>, std::pair<int32_t, int32_t>> ranges;
    const spq::JoinPhase ph1{1, remote, 0, &ranges};
    spq::build_join_work(H, o, 0, H.n_queries, &p->jw1_host, &ph1);
    const spq::JoinPhase ph2{2, remote, p->jw1_host.n_parts, &ranges};
    spq::build_join_work(H, o, 0, H.n_queries, &p->jw2_host, &ph2);
    p->phased = true;
  }
  // split join: the tasks' join work (owner side) and the exchange / merge tables (home side)
  std::vector<int32_t> task_pos, xq_rows;
  std::vector<spq::SplitMergeDesc> mdesc;
  std::vector<int64_t> msrc;
  if (c->cfg.world_size > 1 && c->cfg.split_join) {
    p->split = true;
    spq::build_task_join_work(H, o, &p->tw_host);
    for (const spq::PlanHost::Task& t : H.tasks)
      for (int32_t i = 0; i < t.n_rows; ++i) task_pos.push_back(t.pos0 + i);
    std::vector<std::vector<int64_t>> first_row(H.n_queries);  // per home query: source rows (peer order)
    int64_t off = 0;
    for (int w = 0; w < c->cfg.world_size; ++w)
      for (int32_t k = H.xq_off[w]; k < H.xq_off[w + 1]; ++k) {
        const int32_t qi = H.xq_queries[k];
        first_row[qi].push_back(off);
        for (int64_t r = H.query_join_row_off[qi]; r < H.query_join_row_off[qi + 1]; ++r)
          xq_rows.push_back(static_cast<int32_t>(r));
        off += H.query_join_row_off[qi + 1] - H.query_join_row_off[qi];
      }
    for (int32_t qi = 0; qi < H.n_queries; ++qi) {
      const int64_t r0 = H.query_join_row_off[qi], r1 = H.query_join_row_off[qi + 1];
      if (r0 == r1) continue;
      spq::SplitMergeDesc d{};
      d.row0 = r0;
      d.n_rows = static_cast<int32_t>(r1 - r0);
      d.src_begin = static_cast<int32_t>(msrc.size());
      msrc.insert(msrc.end(), first_row[qi].begin(), first_row[qi].end());
      d.src_end = static_cast<int32_t>(msrc.size());
      mdesc.push_back(d);
    }
    p->sp.task_rows = static_cast<int64_t>(task_pos.size());
    p->sp.xq_rows = static_cast<int64_t>(xq_rows.size());
    p->sp.home_rows = H.query_join_row_off.empty() ? 0 : H.query_join_row_off.back();
    p->sp.n_mdesc = static_cast<int32_t>(mdesc.size());
  }
  lap("join work");
  if (prof) {
    for (const spq::AttnWorkHost* wh : {&p->pw_host, &p->jw_host}) {
      if (wh->dynamic) {
        std::fprintf(stderr, "[spanq]   work: items %zu codes %zu grid %d (dynamic claims)\n", wh->items.size(),
                     wh->cta_items.size(), wh->grid);
        continue;
      }
      int64_t mn = INT64_MAX, mx = 0, imn = INT64_MAX, imx = 0;
      double cmx = 0, cmn = 1e30;
      for (int32_t cta = 0; cta < wh->grid; ++cta) {
        const int64_t ni = wh->cta_off[cta + 1] - wh->cta_off[cta];
        imn = std::min(imn, ni);
        imx = std::max(imx, ni);
        int64_t subs = 0;
        for (int32_t i = wh->cta_off[cta]; i < wh->cta_off[cta + 1]; ++i) {
          const spq::WorkItem& it = wh->items[wh->cta_items[i] / o.units];
          for (int32_t t = it.tile_begin; t < it.tile_end; ++t) subs += wh->tiles[t].n_valid > 64 ? 2 : 1;
        }
        mn = std::min(mn, subs);
        mx = std::max(mx, subs);
        const double cost = static_cast<double>(subs) + 3.5 * static_cast<double>(ni);
        cmx = std::max(cmx, cost);
        cmn = std::min(cmn, cost);
      }
      std::fprintf(stderr, "[spanq]   work: items/CTA min %ld max %ld; cost (sub-tiles + 3.5/item) min %.1f max %.1f\n",
                   static_cast<long>(imn), static_cast<long>(imx), cmn, cmx);
      std::fprintf(stderr, "[spanq]   work: items %zu codes %zu grid %d parts %d combine %zu sub-tiles/CTA min %ld max %ld\n",
                   wh->items.size(), wh->cta_items.size(), wh->grid, wh->n_parts, wh->combine.size(),
                   static_cast<long>(mn), static_cast<long>(mx));
    }
  }
  p->prefill_flops = p->pw_host.flops;
  p->join_flops = p->jw_lazy ? spq::join_flops(H, o, 0, H.n_queries) : p->jw_host.flops;
  // algorithmic bytes of rope_kv_write: per written row, read k,v and write both pages
  // (4*Hkv*d*elt), plus 12 B of pos/slot metadata per row
  const int64_t row_bytes = 4LL * c->cfg.num_kv_heads * c->cfg.head_dim * elt_size(c);
  {
    int64_t written = 0;
    for (int64_t s : H.prefill_slot) written += s >= 0;
    p->prefill_kv_bytes = 12 * static_cast<int64_t>(H.prefill_slot.size()) + written * row_bytes;
    written = 0;
    for (int64_t s : H.join_slot) written += s >= 0;
    p->join_kv_bytes = 12 * static_cast<int64_t>(H.join_slot.size()) + written * row_bytes;
  }
  lap("flops/bytes");
  if (is_gpu(c)) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaSetDevice(c->cfg.device));
    Packer pk;
    p->off_ppos = pk.add(H.prefill_pos);
    p->off_pslot = pk.add(H.prefill_slot);
    p->off_pad = pk.add(H.pad_slots);
    p->off_jpos = pk.add(H.join_pos);
    p->off_jslot = pk.add(H.join_slot);
    p->off_send = pk.add(H.send_blocks);
    p->off_recv = pk.add(H.recv_blocks);
    auto add_work = [&](const spq::AttnWorkHost& h, DevWork* w) {
      w->tiles = pk.add(h.tiles);
      w->tile_blocks = pk.add(h.tile_blocks);
      w->items = pk.add(h.items);
      w->cta_off = pk.add(h.cta_off);
      w->cta_items = pk.add(h.cta_items);
      w->sched = pk.add(kZeros2);  // claim counters (self-resetting)
      w->dynamic = h.dynamic;
      w->n_codes = static_cast<int32_t>(h.cta_items.size());
      w->combine = pk.add(h.combine);
      w->n_items = static_cast<int32_t>(h.items.size());
      w->grid = h.grid;
      w->cluster = h.cluster;
      w->n_combine = static_cast<int32_t>(h.combine.size());
      w->n_parts = h.n_parts;
      w->flops = h.flops;
    };
    add_work(p->pw_host, &p->pw);
    if (!p->jw_lazy) add_work(p->jw_host, &p->jw);
    if (p->phased) {
      add_work(p->jw1_host, &p->jw1);
      add_work(p->jw2_host, &p->jw2);
    }
    if (p->split) {
      add_work(p->tw_host, &p->sp.tw);
      p->sp.off_tpos = pk.add(task_pos);
      p->sp.off_xrows = pk.add(xq_rows);
      p->sp.off_mdesc = pk.add(mdesc);
      p->sp.off_msrc = pk.add(msrc);
    }
    // one device allocation: packed arrays, then the split-KV partials (O, LSE)
    size_t bytes = std::max<size_t>(pk.size, 256);
    size_t off_opart = 0, off_lsepart = 0;
    const int32_t n_parts = std::max(p->jw.n_parts, p->jw1.n_parts + p->jw2.n_parts);
    if (n_parts > 0) {
      const size_t rows = static_cast<size_t>(n_parts) * heads_per_unit(c) * spq::kTileRows;
      off_opart = align_up(bytes, 1024);
      off_lsepart = align_up(off_opart + rows * c->cfg.head_dim * sizeof(float), 1024);
      bytes = off_lsepart + rows * sizeof(float);
    }
    size_t off_oloc = 0, off_lloc = 0, off_top = 0, off_tlp = 0;
    if (p->split) {  // fp32 local join result (home) and the task join's split pieces (owner)
      const size_t hr = static_cast<size_t>(p->sp.home_rows) * c->cfg.num_q_heads;
      off_oloc = align_up(bytes, 1024);
      off_lloc = align_up(off_oloc + hr * c->cfg.head_dim * sizeof(float), 1024);
      bytes = off_lloc + hr * sizeof(float);
      const size_t tr = static_cast<size_t>(p->sp.tw.n_parts) * heads_per_unit(c) * spq::kTileRows;
      off_top = align_up(bytes, 1024);
      off_tlp = align_up(off_top + tr * c->cfg.head_dim * sizeof(float), 1024);
      bytes = off_tlp + tr * sizeof(float) + 256;
    }
    // pinned staging, reused once its previous upload has completed
    if (c->staging_size < pk.size) {
      CUDA_TRY(cudaEventSynchronize(c->staging_ev));
      if (c->staging) CUDA_TRY(cudaFreeHost(c->staging));
      c->staging_size = std::max(pk.size, static_cast<size_t>(1) << 20);
      CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&c->staging), c->staging_size));
    } else {
      CUDA_TRY(cudaEventSynchronize(c->staging_ev));
    }
    pk.write(c->staging);
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&p->dbuf), bytes, st));
    CUDA_TRY(cudaMemcpyAsync(p->dbuf, c->staging, pk.size, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaEventRecord(c->staging_ev, st));
    if (n_parts > 0) {
      p->opart = reinterpret_cast<float*>(p->dbuf + off_opart);
      p->lsepart = reinterpret_cast<float*>(p->dbuf + off_lsepart);
    }
    if (p->split) {
      p->sp.o_loc = reinterpret_cast<float*>(p->dbuf + off_oloc);
      p->sp.lse_loc = reinterpret_cast<float*>(p->dbuf + off_lloc);
      p->sp.topart = reinterpret_cast<float*>(p->dbuf + off_top);
      p->sp.tlsepart = reinterpret_cast<float*>(p->dbuf + off_tlp);
    }
    lap("upload");
  }
  guard.armed = false;
  c->live.insert(p.get());
  *out = p.release();
  return SPQ_OK;
}

spq_status spq_plan_view_get(const spq_plan* p, spq_plan_view* v) {
  if (p == nullptr || v == nullptr) return fail(SPQ_EINVAL, "null argument");
  if (p->released) return fail(SPQ_ESTATE, "plan used after release");
  const spq::PlanHost& H = p->host;
  std::memset(v, 0, sizeof(*v));
  v->n_queries = H.n_queries;
  v->n_segments = static_cast<int32_t>(H.segs.size());
  v->n_jobs = static_cast<int32_t>(H.jobs.size());
  v->n_blocks_total = static_cast<int64_t>(H.blocks.size());
  v->seg_query = p->seg_query.data();
  v->seg_kind = p->seg_kind.data();
  v->seg_frag_idx = p->seg_frag_idx.data();
  v->seg_tok_len = p->seg_tok_len.data();
  v->seg_pos0 = p->seg_pos0.data();
  v->seg_hit = p->seg_hit.data();
  v->seg_compute_begin = p->seg_cb.data();
  v->seg_block_off = p->seg_block_off.data();
  v->seg_n_blocks = p->seg_n_blocks.data();
  v->blocks = H.blocks.data();
  v->block_write = H.block_write.data();
  v->digests = p->digests.data();
  v->join_digests = p->join_digests.data();
  v->jobs = H.jobs.data();
  v->job_row_off = H.job_row_off.data();
  v->n_prefill_rows = static_cast<int64_t>(H.prefill_pos.size());
  v->prefill_pos = H.prefill_pos.data();
  v->prefill_slot = H.prefill_slot.data();
  v->n_join_rows = static_cast<int64_t>(H.join_pos.size());
  v->query_join_row_off = H.query_join_row_off.data();
  v->join_pos = H.join_pos.data();
  v->join_slot = H.join_slot.data();
  v->n_pad_slots = static_cast<int64_t>(H.pad_slots.size());
  v->pad_slots = H.pad_slots.data();
  v->prefill_flops = p->prefill_flops;
  v->join_flops = p->join_flops;
  v->prefill_kv_bytes = p->prefill_kv_bytes;
  v->join_kv_bytes = p->join_kv_bytes;
  v->n_join_queries = H.n_join_queries;
  v->world_size = static_cast<int32_t>(H.send_off.size()) - 1;
  v->send_off = H.send_off.data();
  v->send_blocks = H.send_blocks.data();
  v->recv_off = H.recv_off.data();
  v->cand_recv_off = H.cand_recv_off.data();
  v->cand_recv_need = H.cand_recv_need.data();
  v->cand_send_off = H.cand_send_off.data();
  v->recv_blocks = H.recv_blocks.data();
  v->n_tasks = static_cast<int32_t>(H.tasks.size());
  v->tasks = H.tasks.empty() ? nullptr : &H.tasks[0].query;
  v->xq_off = H.xq_off.data();
  v->xq_queries = H.xq_queries.data();
  return SPQ_OK;
}

spq_status spq_prefill_jobs(spq_ctx* c, spq_plan* p, int32_t layer, int32_t a, int32_t b, const void* q,
                            const void* k, const void* v, void* o, float* lse, void* stream) {
  spq_status s = check_call(c, p, layer);
  if (s != SPQ_OK) return s;
  const int32_t nj = static_cast<int32_t>(p->host.jobs.size());
  if (a < 0 || b > nj || a > b) return fail(SPQ_ESTATE, "job range out of bounds");
  if (a == b) return SPQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  s = wait_pending(c, st);
  if (s != SPQ_OK) return s;
  const int64_t r0 = p->host.job_row_off[a], r1 = p->host.job_row_off[b];
  bool k1 = false;
  s = kv_write(c, p, layer, k, v, at<int32_t>(p, p->off_ppos) + r0, at<int64_t>(p, p->off_pslot) + r0, r1 - r0, st,
               &k1);
  if (s != SPQ_OK) return s;
  spq::AttnArgs args{};
  TempWork tw;
  const bool full = (a == 0 && b == nj);
  if (full) {
    fill_attn(c, p, p->pw, &args);
  } else {
    spq::AttnWorkHost h;
    spq::build_prefill_work(p->host, prefill_opts(c), a, b, &h);
    s = upload_work(c, h, st, &tw);
    if (s != SPQ_OK) return s;
    spq_plan tmp_view;  // only dbuf is read by fill_attn through `at`
    tmp_view.dbuf = tw.buf;
    tmp_view.opart = nullptr;
    tmp_view.lsepart = nullptr;
    fill_attn(c, &tmp_view, tw.w, &args);
  }
  args.pos = at<int32_t>(p, p->off_ppos) + r0;
  args.q = q;
  args.o = o;
  args.lse = lse;
  args.layer = layer;
  // programmatic dependent launch only right behind our own K1 (nothing else in between on the
  // stream: no work-list upload, no timing event) — then every input but the pool is complete
  args.pdl = k1 && full && !c->timing && c->pdl;
  CUtensorMap qmap, omap;
  if (c->cfg.dtype == SPQ_BF16) {
    s = make_qmap(c, q, r1 - r0, &qmap);
    if (s != SPQ_OK) return s;
    args.tmap_q = &qmap;
    s = make_omap(c, o, r1 - r0, &omap);  // prefill epilogue: TMA stores in either out dtype
    if (s != SPQ_OK) return s;
    args.tmap_o = &omap;
  }
  if (c->timing) CUDA_TRY(cudaEventRecord(c->ev[0], st));
  s = run_attn(c, args, st);
  if (s != SPQ_OK) return s;
  if (c->timing) {
    CUDA_TRY(cudaEventRecord(c->ev[1], st));
    c->prefill_timed = true;
  }
  if (tw.buf) CUDA_TRY(cudaFreeAsync(tw.buf, st));
  return SPQ_OK;
}

namespace {
// mode -1: the whole join of queries [a, b) (spq_join); 0 / 1: phase 0 / 1 of a phased plan's
// join (spq_join_phase: K1 + the held segments, then the received fragments + the combine)
// One join-shaped launch (K3 + K4) of work list w (device arrays in `buf`): rows of q at pos,
// output o / lse in fp32 (f32) or the ctx out dtype; split pieces in opart / lsepart.
spq_status launch_join_list(spq_ctx* c, const DevWork& w, uint8_t* buf, spq::AttnArgs& args, float* opart,
                            float* lsepart, int32_t part_extent, const void* q, const int32_t* pos, int64_t rows,
                            int32_t layer, void* o, float* lse, bool f32, bool pdl, cudaStream_t st) {
  spq_status s = SPQ_OK;
  args.opart = opart;
  args.lsepart = lsepart;
  args.pos = pos;
  args.join = true;
  // auto exp2: joins run MUFU-bound steady-state steps; a quarter of their exponentials on the FMA
  // pipe measured faster (C2 join 0.0860 -> 0.0830 ms), the prefill (item boundaries) did not
  if (c->exp2_mode < 0) args.poly_mask = 1;
  args.pdl = pdl;  // see spq_prefill_jobs
  args.q = q;
  args.o = o;
  args.lse = lse;
  args.layer = layer;
  args.out_fp32 = f32;
  CUtensorMap qmap, omap, pmap;
  if (c->cfg.dtype == SPQ_BF16) {
    s = make_qmap(c, q, rows, &qmap);
    if (s != SPQ_OK) return s;
    args.tmap_q = &qmap;
    if (f32) {
      s = make_omap(c, o, rows, &omap, 1);
      if (s != SPQ_OK) return s;
      args.tmap_o = &omap;
    }
    if (w.n_parts > 0 && opart != nullptr) {
      s = make_partmap(c, opart, part_extent, &pmap);
      if (s != SPQ_OK) return s;
      args.tmap_op = &pmap;
    }
  }
  if (c->timing) CUDA_TRY(cudaEventRecord(c->ev[2], st));
  s = run_attn(c, args, st);
  if (s != SPQ_OK) return s;
  if (c->timing) {
    CUDA_TRY(cudaEventRecord(c->ev[3], st));
    c->join_timed = true;
  }
  if (w.n_combine > 0) {
    spq::CombineArgs ca{};
    ca.desc = reinterpret_cast<const spq::CombineDesc*>(buf + w.combine);
    ca.n_desc = w.n_combine;
    ca.opart = opart;
    ca.lsepart = lsepart;
    ca.o = o;
    ca.lse = lse;
    ca.hq = c->cfg.num_q_heads;
    ca.heads_per_desc = heads_per_unit(c);
    ca.d = c->cfg.head_dim;
    ca.out_fp32 = f32;
    // the join kernel is the preceding stream operation unless a timing event sits between
    ca.pdl = !c->timing && c->cfg.dtype == SPQ_BF16 && c->pdl;
    cudaError_t e = spq::launch_combine(ca, st);
    if (e != cudaSuccess) return fail(SPQ_ECUDA, std::string("combine launch: ") + cudaGetErrorString(e));
    c->launches++;
  }
  return SPQ_OK;
}

// The join's work list of a lazy (W = 1) plan, built and uploaded at its first full join: the
// packed arrays then the split-KV partials in one device buffer, copied from the ctx's second
// pinned staging buffer (reused once the previous join-work upload has completed)
spq_status ensure_join_work(spq_ctx* c, spq_plan* p, cudaStream_t st) {
  if (p->jbuf != nullptr) return SPQ_OK;
  spq::build_join_work(p->host, work_opts(c, c->cfg.dtype == SPQ_BF16), 0, p->host.n_queries, &p->jw_host);
  const spq::AttnWorkHost& h = p->jw_host;
  Packer pk;
  DevWork& w = p->jw;
  w.tiles = pk.add(h.tiles);
  w.tile_blocks = pk.add(h.tile_blocks);
  w.items = pk.add(h.items);
  w.cta_off = pk.add(h.cta_off);
  w.cta_items = pk.add(h.cta_items);
  w.sched = pk.add(kZeros2);  // claim counters (self-resetting)
  w.dynamic = h.dynamic;
  w.n_codes = static_cast<int32_t>(h.cta_items.size());
  w.combine = pk.add(h.combine);
  w.n_items = static_cast<int32_t>(h.items.size());
  w.grid = h.grid;
  w.cluster = h.cluster;
  w.n_combine = static_cast<int32_t>(h.combine.size());
  w.n_parts = h.n_parts;
  w.flops = h.flops;
  size_t bytes = std::max<size_t>(pk.size, 256);
  size_t off_opart = 0, off_lsepart = 0;
  if (w.n_parts > 0) {
    const size_t rows = static_cast<size_t>(w.n_parts) * heads_per_unit(c) * spq::kTileRows;
    off_opart = align_up(bytes, 1024);
    off_lsepart = align_up(off_opart + rows * c->cfg.head_dim * sizeof(float), 1024);
    bytes = off_lsepart + rows * sizeof(float);
  }
  CUDA_TRY(cudaEventSynchronize(c->jstaging_ev));  // the previous join-work upload has read it
  if (c->jstaging_size < pk.size) {
    if (c->jstaging) CUDA_TRY(cudaFreeHost(c->jstaging));
    c->jstaging_size = std::max(pk.size, static_cast<size_t>(1) << 20);
    CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&c->jstaging), c->jstaging_size));
  }
  pk.write(c->jstaging);
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&p->jbuf), bytes, st));
  CUDA_TRY(cudaMemcpyAsync(p->jbuf, c->jstaging, pk.size, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaEventRecord(c->jstaging_ev, st));
  if (w.n_parts > 0) {
    p->opart = reinterpret_cast<float*>(p->jbuf + off_opart);
    p->lsepart = reinterpret_cast<float*>(p->jbuf + off_lsepart);
  }
  return SPQ_OK;
}

spq_status join_impl(spq_ctx* c, spq_plan* p, int32_t layer, int32_t a, int32_t b, const void* q, const void* k,
                     const void* v, void* o, float* lse, void* stream, int mode, float* split_out = nullptr,
                     float* split_lse = nullptr) {
  spq_status s = check_call(c, p, layer);
  if (s != SPQ_OK) return s;
  const int32_t nq = p->host.n_queries;
  if (a < 0 || b > nq || a > b) return fail(SPQ_ESTATE, "query range out of bounds");
  if (a == b) return SPQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  s = wait_pending(c, st);
  if (s != SPQ_OK) return s;
  const int64_t r0 = p->host.query_join_row_off[a], r1 = p->host.query_join_row_off[b];
  if (r0 == r1) return SPQ_OK;  // only queries homed on other ranks
  const bool full = (a == 0 && b == nq);
  if (full && p->jw_lazy && mode < 0) {
    // before K1, so that K1 stays the attention kernel's immediate predecessor (PDL)
    s = ensure_join_work(c, p, st);
    if (s != SPQ_OK) return s;
  }
  bool k1 = false;
  if (mode != 1) {
    s = kv_write(c, p, layer, k, v, at<int32_t>(p, p->off_jpos) + r0, at<int64_t>(p, p->off_jslot) + r0, r1 - r0, st,
                 &k1);
    if (s != SPQ_OK) return s;
  }
  spq::AttnArgs args{};
  TempWork tw;
  float* opart = p->opart;
  float* lsepart = p->lsepart;
  DevWork w;
  int32_t part_extent = 0;  // partial slots the launch may address
  if (mode >= 0) {
    w = mode == 0 ? p->jw1 : p->jw2;
    fill_attn(c, p, w, &args);
    part_extent = p->jw1.n_parts + p->jw2.n_parts;
  } else if (full && p->jw_lazy) {
    w = p->jw;
    spq_plan view;  // the work list lives in jbuf (fill_attn reads through dbuf)
    view.dbuf = p->jbuf;
    fill_attn(c, &view, p->jw, &args);
    part_extent = w.n_parts;
  } else if (full) {
    w = p->jw;
    fill_attn(c, p, p->jw, &args);
    part_extent = w.n_parts;
  } else {
    spq::AttnWorkHost h;
    spq::WorkOpts o = work_opts(c, false);
    spq::build_join_work(p->host, o, a, b, &h);
    s = upload_work(c, h, st, &tw);
    if (s != SPQ_OK) return s;
    spq_plan tmp_view;
    tmp_view.dbuf = tw.buf;
    tmp_view.opart = nullptr;
    tmp_view.lsepart = nullptr;
    fill_attn(c, &tmp_view, tw.w, &args);
    w = tw.w;
    part_extent = w.n_parts;
  }
  const bool f32 = split_out != nullptr || c->cfg.out_dtype == SPQ_FP32;
  s = launch_join_list(c, w, full && p->jw_lazy ? p->jbuf : (full || mode >= 0 ? p->dbuf : tw.buf), args, opart,
                       lsepart, part_extent, q,
                       at<int32_t>(p, p->off_jpos) + r0, r1 - r0, layer, split_out ? split_out : o,
                       split_out ? split_lse : lse, f32, k1 && (full || mode >= 0) && !c->timing && c->pdl, st);
  if (s != SPQ_OK) return s;
  if (tw.buf) CUDA_TRY(cudaFreeAsync(tw.buf, st));
  return SPQ_OK;
}
}  // namespace

spq_status spq_join(spq_ctx* c, spq_plan* p, int32_t layer, int32_t a, int32_t b, const void* q, const void* k,
                    const void* v, void* o, float* lse, void* stream) {
  if (p != nullptr && c != nullptr && c->live.count(p) && p->split)
    return fail(SPQ_ESTATE, "split-join plan: use spq_split_join_local / spq_split_merge");
  return join_impl(c, p, layer, a, b, q, k, v, o, lse, stream, -1);
}

// ------------------------------------------------------------------ owner-side split join (f1)
spq_status spq_split_pack_q(spq_ctx* c, spq_plan* p, const void* q, void* sendbuf, void* stream) {
  spq_status s = check_call(c, p, 0);
  if (s != SPQ_OK) return s;
  if (!p->split) return fail(SPQ_ESTATE, "not a split-join plan");
  if (p->sp.xq_rows == 0) return SPQ_OK;
  if (q == nullptr || sendbuf == nullptr) return fail(SPQ_EINVAL, "null buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  const int64_t row_bytes = static_cast<int64_t>(c->cfg.num_q_heads) * c->cfg.head_dim * elt_size(c);
  cudaError_t e = spq::launch_gather_rows(at<int32_t>(p, p->sp.off_xrows), p->sp.xq_rows, q, sendbuf, row_bytes,
                                          c->num_sms, st);
  if (e != cudaSuccess) return fail(SPQ_ECUDA, std::string("gather_rows launch: ") + cudaGetErrorString(e));
  c->launches++;
  return SPQ_OK;
}

spq_status spq_split_task_join(spq_ctx* c, spq_plan* p, int32_t layer, const void* q_recv, float* part_o,
                               float* part_lse, void* stream) {
  spq_status s = check_call(c, p, layer);
  if (s != SPQ_OK) return s;
  if (!p->split) return fail(SPQ_ESTATE, "not a split-join plan");
  if (p->sp.task_rows == 0) return SPQ_OK;
  if (q_recv == nullptr || part_o == nullptr || part_lse == nullptr) return fail(SPQ_EINVAL, "null buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  s = wait_pending(c, st);
  if (s != SPQ_OK) return s;
  spq::AttnArgs args{};
  fill_attn(c, p, p->sp.tw, &args);
  return launch_join_list(c, p->sp.tw, p->dbuf, args, p->sp.topart, p->sp.tlsepart, p->sp.tw.n_parts, q_recv,
                          at<int32_t>(p, p->sp.off_tpos), p->sp.task_rows, layer, part_o, part_lse, true, false, st);
}

spq_status spq_split_join_local(spq_ctx* c, spq_plan* p, int32_t layer, const void* q, const void* k, const void* v,
                                void* stream) {
  spq_status s = check_call(c, p, layer);
  if (s != SPQ_OK) return s;
  if (!p->split) return fail(SPQ_ESTATE, "not a split-join plan");
  return join_impl(c, p, layer, 0, p->host.n_queries, q, k, v, nullptr, nullptr, stream, -1, p->sp.o_loc,
                   p->sp.lse_loc);
}

spq_status spq_split_merge(spq_ctx* c, spq_plan* p, const float* part_o_recv, const float* part_lse_recv, void* o,
                           float* lse, void* stream) {
  spq_status s = check_call(c, p, 0);
  if (s != SPQ_OK) return s;
  if (!p->split) return fail(SPQ_ESTATE, "not a split-join plan");
  if (p->sp.home_rows == 0) return SPQ_OK;
  if (o == nullptr || (p->sp.xq_rows > 0 && (part_o_recv == nullptr || part_lse_recv == nullptr)))
    return fail(SPQ_EINVAL, "null buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  spq::SplitMergeArgs m{};
  m.desc = at<spq::SplitMergeDesc>(p, p->sp.off_mdesc);
  m.n_desc = p->sp.n_mdesc;
  m.src = at<int64_t>(p, p->sp.off_msrc);
  m.o_loc = p->sp.o_loc;
  m.lse_loc = p->sp.lse_loc;
  m.o_rem = part_o_recv;
  m.lse_rem = part_lse_recv;
  m.o = o;
  m.lse = lse;
  m.hq = c->cfg.num_q_heads;
  m.d = c->cfg.head_dim;
  m.num_sms = c->num_sms;
  m.total_rows = p->sp.home_rows;
  m.out_fp32 = c->cfg.out_dtype == SPQ_FP32;
  cudaError_t e = spq::launch_merge_split(m, st);
  if (e != cudaSuccess) return fail(SPQ_ECUDA, std::string("merge_split launch: ") + cudaGetErrorString(e));
  c->launches++;
  return SPQ_OK;
}

spq_status spq_join_phase(spq_ctx* c, spq_plan* p, int32_t layer, int32_t phase, const void* q, const void* k,
                          const void* v, void* o, float* lse, void* stream) {
  if (phase != 0 && phase != 1) return fail(SPQ_EINVAL, "phase must be 0 or 1");
  spq_status s = check_call(c, p, layer);
  if (s != SPQ_OK) return s;
  const int32_t nq = p->host.n_queries;
  if (p->phased) return join_impl(c, p, layer, 0, nq, q, k, v, o, lse, stream, phase);
  // not split (no received fragments, or a path without partials): the whole join in phase 1
  return phase == 0 ? SPQ_OK : join_impl(c, p, layer, 0, nq, q, k, v, o, lse, stream, -1);
}

static spq_status exchange(spq_ctx* c, spq_plan* p, int32_t layer, int32_t peer, void* buf, void* stream,
                           int scatter) {
  spq_status s = check_call(c, p, layer);
  if (s != SPQ_OK) return s;
  const spq::PlanHost& H = p->host;
  if (peer < 0 || peer >= static_cast<int32_t>(H.send_off.size()) - 1) return fail(SPQ_ESTATE, "peer out of range");
  const std::vector<int64_t>& off = scatter ? H.recv_off : H.send_off;
  const int64_t a = off[peer], n = off[peer + 1] - a;
  if (n == 0) return SPQ_OK;
  if (buf == nullptr || (reinterpret_cast<uintptr_t>(buf) & 15)) return fail(SPQ_EINVAL, "buf must be 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  s = wait_pending(c, st);
  if (s != SPQ_OK) return s;
  spq::KvExchangeArgs x{};
  x.blocks = at<int32_t>(p, scatter ? p->off_recv : p->off_send) + a;
  x.n = n;
  x.k_pool = c->cfg.k_pool;
  x.v_pool = c->cfg.v_pool;
  x.buf = buf;
  x.hkv = c->cfg.num_kv_heads;
  x.bs = c->cfg.block_size;
  x.d = c->cfg.head_dim;
  x.elt = elt_size(c);
  x.layer = layer;
  x.num_sms = c->num_sms;
  x.nblk = c->cfg.num_blocks;
  x.scatter = scatter;
  cudaError_t e = spq::launch_kv_exchange(x, st);
  if (e != cudaSuccess) return fail(SPQ_ECUDA, std::string("kv_exchange launch: ") + cudaGetErrorString(e));
  c->launches++;
  return SPQ_OK;
}

spq_status spq_exchange_set_need(spq_ctx* c, spq_plan* p, int32_t peer, const uint8_t* need, int64_t n,
                                 void* stream) {
  if (c == nullptr || p == nullptr) return fail(SPQ_EINVAL, "null ctx/plan");
  if (!c->live.count(p)) return fail(SPQ_ESTATE, "plan used after release (or not a plan of this ctx)");
  spq::PlanHost& H = p->host;
  if (peer < 0 || peer >= static_cast<int32_t>(H.cand_send_off.size()) - 1) return fail(SPQ_ESTATE, "peer out of range");
  if (n > 0 && need == nullptr) return fail(SPQ_EINVAL, "null need flags");
  if (!spq::select_send(&H, peer, need, n)) return fail(SPQ_EINVAL, "need flags: count differs from the candidates");
  if (is_gpu(c) && !H.send_blocks.empty()) {
    // the pruned list is a prefix-sized rewrite of the region the full candidate list was uploaded to
    CUDA_TRY(cudaSetDevice(c->cfg.device));
    CUDA_TRY(cudaMemcpyAsync(p->dbuf + p->off_send, H.send_blocks.data(), H.send_blocks.size() * sizeof(int32_t),
                             cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)));
  }
  return SPQ_OK;
}

spq_status spq_exchange_pack(spq_ctx* c, spq_plan* p, int32_t layer, int32_t peer, void* buf, void* stream) {
  return exchange(c, p, layer, peer, buf, stream, 0);
}

spq_status spq_exchange_unpack(spq_ctx* c, spq_plan* p, int32_t layer, int32_t peer, const void* buf,
                               void* stream) {
  return exchange(c, p, layer, peer, const_cast<void*>(buf), stream, 1);
}

spq_status spq_plan_release(spq_ctx* c, spq_plan* p, void* stream) {
  if (c == nullptr || p == nullptr) return fail(SPQ_EINVAL, "null argument");
  if (!c->live.count(p)) return fail(SPQ_ESTATE, "plan released twice (or not a plan of this ctx)");
  if (is_gpu(c)) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaSetDevice(c->cfg.device));
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(e, st));
    c->pending.push_back(e);
    if (p->dbuf) CUDA_TRY(cudaFreeAsync(p->dbuf, st));
    if (p->jbuf) CUDA_TRY(cudaFreeAsync(p->jbuf, st));
    if (p->dec.dbuf) CUDA_TRY(cudaFreeAsync(p->dec.dbuf, st));
    // opart / lsepart live inside dbuf (or jbuf)
    p->dbuf = nullptr;
    p->jbuf = nullptr;
    p->dec.dbuf = nullptr;
  }
  c->store->release(p->host);
  c->live.erase(p);
  // keep the (emptied) object for a while: a later call on this handle reports SPQ_ESTATE
  *p = spq_plan();
  p->released = true;
  c->quarantine.push_back(p);
  if (c->quarantine.size() > kQuarantine) {
    delete c->quarantine.front();
    c->quarantine.pop_front();
  }
  return SPQ_OK;
}

// ------------------------------------------------------------------ decode after the join (f3)
spq_status spq_decode_reserve(spq_ctx* c, spq_plan* p, int32_t max_new) {
  if (c == nullptr || p == nullptr) return fail(SPQ_EINVAL, "null argument");
  if (!c->live.count(p)) return fail(SPQ_ESTATE, "plan used after release (or not a plan of this ctx)");
  if (max_new < 1) return fail(SPQ_EINVAL, "max_new must be >= 1");
  if (p->dec.max_new > 0) return fail(SPQ_ESTATE, "decode already reserved for this plan");
  const spq::PlanHost& H = p->host;
  const int bs = c->cfg.block_size;
  // decode rows: home queries in query order; generation blocks continue each cross segment
  std::vector<int32_t> rows, cross_seg;
  int64_t extra = 0;
  for (size_t i = 0; i < H.segs.size(); ++i) {
    const spq::Segment& sg = H.segs[i];
    if (sg.kind != spq::kCross) continue;
    if (static_cast<int64_t>(sg.pos0) + sg.tok_len + max_new > c->cfg.max_position)
      return fail(SPQ_EINVAL, "query " + std::to_string(sg.query) + ": generation exceeds max_position");
    rows.push_back(sg.query);
    cross_seg.push_back(static_cast<int32_t>(i));
    extra += (static_cast<int64_t>(sg.tok_len) + max_new + bs - 1) / bs - sg.n_blocks;
  }
  if (rows.empty()) return fail(SPQ_ESTATE, "no query of the plan is homed on this rank");
  std::vector<int32_t> fresh;
  if (c->store->extend_private(&p->host, extra, &fresh) != 0)
    return fail(SPQ_ENOMEM, "block pool cannot hold the generation blocks (nothing reserved)");
  Decode& D = p->dec;
  D.rows = rows;
  D.blocks.assign(rows.size(), {});
  const int64_t B = static_cast<int64_t>(rows.size());
  std::vector<int32_t> pos_base(B), kpos(static_cast<size_t>(max_new) * B);
  std::vector<int64_t> kslot(static_cast<size_t>(max_new) * B);
  spq::DecodeWorkHost w;
  std::vector<std::pair<int32_t, int32_t>> row_tiles;
  size_t fi = 0;
  for (int64_t b = 0; b < B; ++b) {
    const spq::Segment& sg = H.segs[cross_seg[b]];
    std::vector<int32_t>& bl = D.blocks[b];
    bl.assign(H.blocks.begin() + sg.block_off, H.blocks.begin() + sg.block_off + sg.n_blocks);
    const int64_t need = (static_cast<int64_t>(sg.tok_len) + max_new + bs - 1) / bs - sg.n_blocks;
    for (int64_t i = 0; i < need; ++i) bl.push_back(fresh[fi++]);
    pos_base[b] = sg.pos0 + sg.tok_len;
    for (int32_t t = 0; t < max_new; ++t) {
      const int64_t idx = static_cast<int64_t>(sg.tok_len) + t;
      kpos[t * B + b] = pos_base[b] + t;
      kslot[t * B + b] = static_cast<int64_t>(bl[idx / bs]) * bs + idx % bs;
    }
    row_tiles.push_back(spq::decode_row_tiles(H, sg.query, bl, sg.tok_len + max_new, bs, &w));
  }
  // chunks of <= T tiles per (row, kv head), sized so that the whole batch is ONE wave of
  // resident CTAs (a second, partial wave of a memory-bound kernel costs a whole CTA time): the
  // bf16 kernel holds 4 warps x kDecStages stages x 16 keys of K and V plus per-warp P^T and merge state
  int64_t max_tiles = 1;
  for (const auto& rt : row_tiles) max_tiles = std::max<int64_t>(max_tiles, rt.second - rt.first);
  const int64_t gq = c->cfg.num_q_heads / c->cfg.num_kv_heads, dd = c->cfg.head_dim;
  const int64_t smem = c->cfg.dtype == SPQ_BF16
                           ? 4 * kDecStages * 2 * 16 * dd * 2 + 4 * 8 * 16 * 2 + 4 * 2 * gq * 4
                           : 2 * (64 * (dd + 4) + 64 * dd) * 4 + 4 * (gq * dd + gq * 64 + gq * 3);
  const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(232448 / smem, 16));
  const int64_t slots = per_sm * (c->num_sms > 0 ? c->num_sms : 148);
  const int64_t pairs = B * c->cfg.num_kv_heads;  // (row, kv head) pairs
#ifndef SPQ_DEC_CHUNK_DIV
#define SPQ_DEC_CHUNK_DIV 1
#endif
  const int64_t per_pair = std::max<int64_t>(1, slots / pairs / SPQ_DEC_CHUNK_DIV);
  const int chunk = static_cast<int>(std::max<int64_t>(1, (max_tiles + per_pair - 1) / per_pair));
  spq::decode_items(row_tiles, c->cfg.num_kv_heads, c->cfg.num_q_heads / c->cfg.num_kv_heads, chunk, &w);
  D.max_new = max_new;
  D.n_items = static_cast<int32_t>(w.items.size());
  D.n_comb = static_cast<int32_t>(w.combine.size());
  if (!is_gpu(c)) return SPQ_OK;
  Packer pk;
  D.off_tiles = pk.add(w.tiles);
  D.off_tb = pk.add(w.tile_blocks);
  D.off_items = pk.add(w.items);
  D.off_comb = pk.add(w.combine);
  D.off_posb = pk.add(pos_base);
  D.off_kpos = pk.add(kpos);
  D.off_kslot = pk.add(kslot);
  const std::vector<int32_t> done0(static_cast<size_t>(B) * c->cfg.num_kv_heads, 0);  // (alive until pk.write)
  D.off_done = pk.add(done0);
  const int g = c->cfg.num_q_heads / c->cfg.num_kv_heads;
  const size_t off_op = align_up(pk.size, 256);
  const size_t off_lp = align_up(off_op + static_cast<size_t>(w.n_parts) * g * c->cfg.head_dim * sizeof(float), 256);
  const size_t bytes = off_lp + static_cast<size_t>(w.n_parts) * g * sizeof(float) + 256;
  std::vector<uint8_t> host(pk.size);
  pk.write(host.data());
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  CUDA_TRY(cudaMalloc(&D.dbuf, bytes));
  CUDA_TRY(cudaMemcpy(D.dbuf, host.data(), pk.size, cudaMemcpyHostToDevice));
  D.opart = reinterpret_cast<float*>(D.dbuf + off_op);
  D.lsepart = reinterpret_cast<float*>(D.dbuf + off_lp);
  return SPQ_OK;
}

spq_status spq_decode_step(spq_ctx* c, spq_plan* p, int32_t layer, int32_t t, const void* q, const void* k,
                           const void* v, void* o, float* lse, void* stream) {
  spq_status s = check_call(c, p, layer);
  if (s != SPQ_OK) return s;
  Decode& D = p->dec;
  if (D.max_new == 0) return fail(SPQ_ESTATE, "spq_decode_reserve was not called for this plan");
  if (t < 0 || t >= D.max_new) return fail(SPQ_ESTATE, "step outside the reserved generation range");
  if (q == nullptr || k == nullptr || v == nullptr || o == nullptr) return fail(SPQ_EINVAL, "null buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  s = wait_pending(c, st);
  if (s != SPQ_OK) return s;
  const int64_t B = static_cast<int64_t>(D.rows.size());
  // K1: the new tokens' K (RoPE at N_q + t) and V into their reserved slots
  spq::KvWriteArgs kw{};
  kw.k = k;
  kw.v = v;
  kw.pos = reinterpret_cast<const int32_t*>(D.dbuf + D.off_kpos) + t * B;
  kw.slot = reinterpret_cast<const int64_t*>(D.dbuf + D.off_kslot) + t * B;
  kw.rows = B;
  kw.n_pad = 0;
  kw.k_pool = c->cfg.k_pool;
  kw.v_pool = c->cfg.v_pool;
  kw.hkv = c->cfg.num_kv_heads;
  kw.d = c->cfg.head_dim;
  kw.bs = c->cfg.block_size;
  kw.nblk = c->cfg.num_blocks;
  kw.layer = layer;
  kw.rope = c->rope;
  kw.fp32 = c->cfg.dtype == SPQ_FP32;
  cudaError_t e = spq::launch_rope_kv_write(kw, st);
  if (e != cudaSuccess) return fail(SPQ_ECUDA, std::string("rope_kv_write launch: ") + cudaGetErrorString(e));
  c->launches++;
  // K9: the new rows over every segment, split-KV
  spq::DecodeArgs a{};
  a.items = reinterpret_cast<const spq::DecodeItem*>(D.dbuf + D.off_items);
  a.n_items = D.n_items;
  a.tiles = reinterpret_cast<const spq::KvTile*>(D.dbuf + D.off_tiles);
  a.tile_blocks = reinterpret_cast<const int32_t*>(D.dbuf + D.off_tb);
  a.pos_base = reinterpret_cast<const int32_t*>(D.dbuf + D.off_posb);
  a.step = t;
  a.q = q;
  a.o = o;
  a.lse = lse;
  a.opart = D.opart;
  a.lsepart = D.lsepart;
  a.done = c->cfg.dtype == SPQ_BF16 ? reinterpret_cast<int32_t*>(D.dbuf + D.off_done) : nullptr;
  a.k_pool = c->cfg.k_pool;
  a.v_pool = c->cfg.v_pool;
  a.rope = c->rope;
  a.max_pos = c->cfg.max_position;
  a.hq = c->cfg.num_q_heads;
  a.hkv = c->cfg.num_kv_heads;
  a.d = c->cfg.head_dim;
  a.bs = c->cfg.block_size;
  a.nblk = c->cfg.num_blocks;
  a.layer = layer;
  a.fp32 = c->cfg.dtype == SPQ_FP32;
  a.out_fp32 = c->cfg.out_dtype == SPQ_FP32;
  e = spq::launch_decode(a, st);
  if (e != cudaSuccess) return fail(SPQ_ECUDA, std::string("decode launch: ") + cudaGetErrorString(e));
  c->launches++;
  // the bf16 kernel merges a (row, kv head)'s chunks itself (its last chunk to finish); the fp32
  // path runs K4
  if (D.n_comb > 0 && a.done == nullptr) {
    spq::CombineArgs ca{};
    ca.desc = reinterpret_cast<const spq::CombineDesc*>(D.dbuf + D.off_comb);
    ca.n_desc = D.n_comb;
    ca.opart = D.opart;
    ca.lsepart = D.lsepart;
    ca.o = o;
    ca.lse = lse;
    ca.hq = c->cfg.num_q_heads;
    ca.heads_per_desc = c->cfg.num_q_heads / c->cfg.num_kv_heads;
    ca.rows_per_part = 1;
    ca.d = c->cfg.head_dim;
    ca.out_fp32 = c->cfg.out_dtype == SPQ_FP32;
    ca.pdl = false;
    e = spq::launch_combine(ca, st);
    if (e != cudaSuccess) return fail(SPQ_ECUDA, std::string("combine launch: ") + cudaGetErrorString(e));
    c->launches++;
  }
  return SPQ_OK;
}

spq_status spq_commit_span(spq_ctx* c, spq_plan* p, int32_t query, const int32_t* gen_tokens, int32_t n_gen,
                           int32_t crop, int32_t* n_committed) {
  if (c == nullptr || p == nullptr || (n_gen > 0 && gen_tokens == nullptr)) return fail(SPQ_EINVAL, "null argument");
  if (!c->live.count(p)) return fail(SPQ_ESTATE, "plan used after release (or not a plan of this ctx)");
  const spq::PlanHost& H = p->host;
  if (query < 0 || query >= H.n_queries) return fail(SPQ_EINVAL, "query out of range");
  const Decode& D = p->dec;
  int64_t row = -1;
  for (size_t b = 0; b < D.rows.size(); ++b)
    if (D.rows[b] == query) row = static_cast<int64_t>(b);
  if (n_gen < 0 || (n_gen > 0 && row < 0) || n_gen > D.max_new)
    return fail(SPQ_ESTATE, "n_gen outside the reserved generation range of this query");
  for (const spq::Segment& sg : H.segs)
    if (sg.query == query && sg.kind != spq::kCross)
      return fail(SPQ_EINVAL, "only a query without prefix and fragments (an inner generate ⋈[input]) "
                              "is a span at positions 0..: plus distribution needs its KV span-local");
  const int bs = c->cfg.block_size;
  std::vector<int32_t> toks = p->cross_tokens[query];
  for (int32_t i = 0; i < n_gen; ++i) {
    if (gen_tokens[i] < 0) return fail(SPQ_EINVAL, "negative token");
    toks.push_back(gen_tokens[i]);
  }
  int64_t keep = static_cast<int64_t>(toks.size());
  if (crop) keep = keep / bs * bs;  // trailing partial block cropped
  if (n_committed) *n_committed = static_cast<int32_t>(keep);
  if (keep == 0) return SPQ_OK;
  std::vector<int32_t> blocks;
  if (row >= 0) {
    blocks = D.blocks[row];
  } else {  // no generation reserved: the cross blocks themselves
    for (const spq::Segment& sg : H.segs)
      if (sg.query == query && sg.kind == spq::kCross)
        blocks.assign(H.blocks.begin() + sg.block_off, H.blocks.begin() + sg.block_off + sg.n_blocks);
  }
  std::vector<spq::Digest> dig;
  spq::chain('F', c->store->root(), toks.data(), keep, bs, &dig);
  std::vector<int32_t> ntok(dig.size());
  for (size_t i = 0; i < dig.size(); ++i) ntok[i] = static_cast<int32_t>(std::min<int64_t>(bs, keep - static_cast<int64_t>(i) * bs));
  c->store->commit(&p->host, blocks.data(), dig.data(), ntok.data(), static_cast<int64_t>(dig.size()));
  return SPQ_OK;
}

spq_status spq_get_stats(const spq_ctx* c, spq_stats* out) {
  if (c == nullptr || out == nullptr) return fail(SPQ_EINVAL, "null argument");
  const spq::StoreStats& s = c->store->stats();
  out->lookups = s.lookups;
  out->hit_blocks = s.hit_blocks;
  out->miss_blocks = s.miss_blocks;
  out->hit_tokens = s.hit_tokens;
  out->input_tokens = s.input_tokens;
  out->evictions = s.evictions;
  out->inserted_blocks = s.inserted_blocks;
  out->resident_blocks = c->store->resident();
  out->free_blocks = c->store->free_count();
  out->pinned_blocks = c->store->pinned_count();
  out->plans = c->store->plans();
  return SPQ_OK;
}

spq_status spq_evict_all(spq_ctx* c) {
  if (c == nullptr) return fail(SPQ_EINVAL, "null argument");
  c->store->evict_all();
  return SPQ_OK;
}

spq_status spq_read_blocks(spq_ctx* c, int32_t layer, const int32_t* ids, int64_t n, void* k, void* v,
                           void* stream) {
  if (c == nullptr || (n > 0 && (ids == nullptr || k == nullptr || v == nullptr)))
    return fail(SPQ_EINVAL, "null argument");
  if (!is_gpu(c)) return fail(SPQ_ESTATE, "host-only ctx (device < 0) has no pool");
  if (layer < 0 || layer >= c->cfg.num_layers) return fail(SPQ_ESTATE, "layer out of range");
  for (int64_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= c->cfg.num_blocks) return fail(SPQ_EINVAL, "block id out of range");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  const size_t blk = static_cast<size_t>(c->cfg.num_kv_heads) * c->cfg.block_size * c->cfg.head_dim * elt_size(c);
  const size_t layer_off = static_cast<size_t>(layer) * c->cfg.num_blocks * blk;
  for (int64_t i = 0; i < n; ++i) {
    const size_t src = layer_off + static_cast<size_t>(ids[i]) * blk;
    CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(k) + i * blk, static_cast<const uint8_t*>(c->cfg.k_pool) + src, blk,
                             cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(v) + i * blk, static_cast<const uint8_t*>(c->cfg.v_pool) + src, blk,
                             cudaMemcpyDeviceToDevice, st));
  }
  return SPQ_OK;
}

// ------------------------------------------------------------------ CIDRA
namespace {
spq_status cidra_plan(const spq_ctx* c, const int32_t* src, const int32_t* dst, const int32_t* delta, int64_t n,
                      spq::CidraSchedule* sch, spq_cidra_stats* stats) {
  if (c == nullptr || (n > 0 && (src == nullptr || dst == nullptr || delta == nullptr)))
    return fail(SPQ_EINVAL, "null argument");
  if (n < 0) return fail(SPQ_EINVAL, "negative move count");
  for (int64_t i = 0; i < n; ++i)
    if (delta[i] <= -c->cfg.max_position || delta[i] >= c->cfg.max_position)
      return fail(SPQ_EINVAL, "|delta| >= max_position (no RoPE table row)");
  std::string err;
  if (!spq::cidra_schedule(src, dst, delta, n, c->cfg.num_blocks, sch, &err)) return fail(SPQ_EINVAL, err);
  if (stats != nullptr) {
    stats->moves = n;
    stats->components = static_cast<int64_t>(sch->comp_off.size()) - 1;
    stats->cycles = sch->cycles;
    stats->duplicates = sch->duplicates;
    stats->ops = static_cast<int64_t>(sch->ops.size());
    stats->max_component_ops = sch->max_component_ops;
  }
  return SPQ_OK;
}
}  // namespace

spq_status spq_cidra_schedule(const spq_ctx* c, const int32_t* src, const int32_t* dst, const int32_t* delta,
                              int64_t n, int32_t* ops, int64_t cap, int64_t* n_ops, int32_t* comp_off,
                              int64_t comp_cap, int64_t* n_comp, spq_cidra_stats* stats) {
  if (n_ops == nullptr || n_comp == nullptr) return fail(SPQ_EINVAL, "null argument");
  spq::CidraSchedule sch;
  spq_status s = cidra_plan(c, src, dst, delta, n, &sch, stats);
  if (s != SPQ_OK) return s;
  *n_ops = static_cast<int64_t>(sch.ops.size());
  *n_comp = static_cast<int64_t>(sch.comp_off.size()) - 1;
  if (*n_ops > cap || *n_comp + 1 > comp_cap || (*n_ops > 0 && ops == nullptr) || comp_off == nullptr)
    return fail(SPQ_EINVAL, "schedule capacity too small");
  std::memcpy(ops, sch.ops.data(), sch.ops.size() * sizeof(spq::CidraOp));
  std::memcpy(comp_off, sch.comp_off.data(), sch.comp_off.size() * sizeof(int32_t));
  return SPQ_OK;
}

namespace {
// Run a CIDRA schedule on the ctx's pools for layers [lb, le) (K8), stream-ordered.
spq_status cidra_run(spq_ctx* c, const spq::CidraSchedule& sch, int32_t layer_begin, int32_t layer_end, void* stream) {
  const int64_t n_comp = static_cast<int64_t>(sch.comp_off.size()) - 1;
  if (n_comp == 0 || layer_begin == layer_end) return SPQ_OK;
  if (n_comp > INT32_MAX || static_cast<int64_t>(layer_end - layer_begin) * c->cfg.num_kv_heads > 65535)
    return fail(SPQ_EINVAL, "too many components or layers x kv heads for one launch");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  spq_status s = wait_pending(c, st);
  if (s != SPQ_OK) return s;
  // one stream-ordered device buffer: ops then component offsets (pageable H2D: staged before return)
  const size_t ob = sch.ops.size() * sizeof(spq::CidraOp), cb = sch.comp_off.size() * sizeof(int32_t);
  std::vector<uint8_t> host(ob + cb);  // one copy instead of two
  std::memcpy(host.data(), sch.ops.data(), ob);
  std::memcpy(host.data() + ob, sch.comp_off.data(), cb);
  void* buf = nullptr;
  CUDA_TRY(cudaMallocAsync(&buf, ob + cb, st));
  CUDA_TRY(cudaMemcpyAsync(buf, host.data(), ob + cb, cudaMemcpyHostToDevice, st));
  spq::CidraArgs a{};
  a.ops = static_cast<const int4*>(buf);
  a.comp_off = reinterpret_cast<const int32_t*>(static_cast<uint8_t*>(buf) + ob);
  a.n_comp = static_cast<int32_t>(n_comp);
  a.k_pool = c->cfg.k_pool;
  a.v_pool = c->cfg.v_pool;
  a.rope = c->rope;
  a.hkv = c->cfg.num_kv_heads;
  a.d = c->cfg.head_dim;
  a.bs = c->cfg.block_size;
  a.nblk = c->cfg.num_blocks;
  a.layer_begin = layer_begin;
  a.layer_end = layer_end;
  a.fp32 = c->cfg.dtype == SPQ_FP32;
  a.num_sms = c->num_sms;
  cudaError_t e = spq::launch_cidra(a, st);
  if (e != cudaSuccess) return fail(SPQ_ECUDA, std::string("cidra launch: ") + cudaGetErrorString(e));
  c->launches++;
  CUDA_TRY(cudaFreeAsync(buf, st));
  return SPQ_OK;
}
}  // namespace

spq_status spq_reposition(spq_ctx* c, const int32_t* src, const int32_t* dst, const int32_t* delta, int64_t n,
                          int32_t layer_begin, int32_t layer_end, void* stream, spq_cidra_stats* stats) {
  spq::CidraSchedule sch;
  spq_status s = cidra_plan(c, src, dst, delta, n, &sch, stats);
  if (s != SPQ_OK) return s;
  if (!is_gpu(c)) return fail(SPQ_ESTATE, "host-only ctx (device < 0) has no pool");
  if (layer_begin < 0 || layer_end > c->cfg.num_layers || layer_begin > layer_end)
    return fail(SPQ_ESTATE, "layer range out of bounds");
  if (c->cfg.head_dim != 64 && c->cfg.head_dim != 128) return fail(SPQ_EINVAL, "head_dim must be 64 or 128");
  // blocks a live plan reads or writes must not move under it
  for (int64_t i = 0; i < n; ++i)
    if (c->store->is_pinned(src[i]) || c->store->is_pinned(dst[i]))
      return fail(SPQ_ESTATE, "block " + std::to_string(c->store->is_pinned(src[i]) ? src[i] : dst[i]) +
                                  " is pinned by a live plan");
  s = cidra_run(c, sch, layer_begin, layer_end, stream);
  if (s != SPQ_OK) return s;
  // a destination now holds other KV than its digest names: the store forgets it (no later plan
  // may hit it); the caller owns the moved content from here on
  for (int64_t i = 0; i < n; ++i) c->store->drop(dst[i]);
  return SPQ_OK;
}

spq_status spq_commit_output(spq_ctx* c, spq_plan* p, int32_t query, const int32_t* gen_tokens, int32_t n_gen,
                             void* stream, int32_t* n_committed) {
  if (c == nullptr || p == nullptr || (n_gen > 0 && gen_tokens == nullptr)) return fail(SPQ_EINVAL, "null argument");
  if (!c->live.count(p)) return fail(SPQ_ESTATE, "plan used after release (or not a plan of this ctx)");
  if (!is_gpu(c)) return fail(SPQ_ESTATE, "host-only ctx (device < 0) has no pool");
  const spq::PlanHost& H = p->host;
  const Decode& D = p->dec;
  int64_t row = -1;
  for (size_t b = 0; b < D.rows.size(); ++b)
    if (D.rows[b] == query) row = static_cast<int64_t>(b);
  if (row < 0 || n_gen < 1 || n_gen > D.max_new)
    return fail(SPQ_ESTATE, "query has no reserved generation range holding n_gen tokens");
  const int bs = c->cfg.block_size;
  int32_t C = 0, pos0 = 0;
  for (const spq::Segment& sg : H.segs)
    if (sg.query == query && sg.kind == spq::kCross) {
      C = sg.tok_len;
      pos0 = sg.pos0;
    }
  if (C % bs != 0)
    return fail(SPQ_EINVAL, "the generated tokens must start a block: cross length a multiple of block_size "
                            "(block alignment, P:565-568)");
  for (int32_t i = 0; i < n_gen; ++i)
    if (gen_tokens[i] < 0) return fail(SPQ_EINVAL, "negative token");
  // the output's blocks: generated token t sits at N_q + t; re-encode its K to position t (ReRoPE
  // by -N_q, in place: CIDRA self-moves) on every layer, then index it under its fragment chain
  const std::vector<int32_t>& bl = D.blocks[row];
  const int32_t b0 = C / bs, b1 = (C + n_gen + bs - 1) / bs;
  std::vector<int32_t> ids(bl.begin() + b0, bl.begin() + b1), dl(ids.size(), -(pos0 + C));
  spq::CidraSchedule sch;
  spq_status s = cidra_plan(c, ids.data(), ids.data(), dl.data(), static_cast<int64_t>(ids.size()), &sch, nullptr);
  if (s != SPQ_OK) return s;
  CUDA_TRY(cudaSetDevice(c->cfg.device));
  s = wait_pending(c, static_cast<cudaStream_t>(stream));
  if (s != SPQ_OK) return s;
  s = cidra_run(c, sch, 0, c->cfg.num_layers, stream);
  if (s != SPQ_OK) return s;
  std::vector<spq::Digest> dig;
  spq::chain('F', c->store->root(), gen_tokens, n_gen, bs, &dig);
  std::vector<int32_t> ntok(dig.size());
  for (size_t i = 0; i < dig.size(); ++i) ntok[i] = std::min<int32_t>(bs, n_gen - static_cast<int32_t>(i) * bs);
  c->store->commit(&p->host, ids.data(), dig.data(), ntok.data(), static_cast<int64_t>(dig.size()));
  if (n_committed) *n_committed = n_gen;
  return SPQ_OK;
}

spq_status spq_bulk_order(const spq_ctx* c, const spq_query* queries, int32_t n, int64_t window_blocks,
                          int32_t* order) {
  if (c == nullptr || order == nullptr || (n > 0 && queries == nullptr)) return fail(SPQ_EINVAL, "null argument");
  if (n < 0) return fail(SPQ_EINVAL, "negative query count");
  const int bs = c->cfg.block_size;
  const spq::Digest& root = c->store->root();
  // per query: its set of cached units — each fragment's identity (s_last) and its whole prefix
  // (h_last) — and its block count
  std::vector<std::vector<spq::Digest>> units(n);
  int64_t blocks_total = 0;
  for (int32_t i = 0; i < n; ++i) {
    spq::FlatQuery fq;
    std::string err;
    if (!spq::normalize_tree(queries[i], &fq, &err)) return fail(SPQ_EINVAL, "query " + std::to_string(i) + ": " + err);
    std::vector<spq::Digest> tmp;
    if (!fq.prefix.empty()) {
      spq::chain('P', root, fq.prefix.data(), static_cast<int64_t>(fq.prefix.size()), bs, &tmp);
      units[i].push_back(tmp.back());
      blocks_total += static_cast<int64_t>(tmp.size());
    }
    for (const auto& f : fq.frags) {
      tmp.clear();
      spq::chain('F', root, f.data(), static_cast<int64_t>(f.size()), bs, &tmp);
      units[i].push_back(tmp.back());
      blocks_total += static_cast<int64_t>(tmp.size());
    }
    std::sort(units[i].begin(), units[i].end(), [](const spq::Digest& a, const spq::Digest& b) {
      return std::memcmp(a.b, b.b, 16) < 0;
    });
    units[i].erase(std::unique(units[i].begin(), units[i].end()), units[i].end());
  }
  // window: how many recent queries' blocks the pool holds (reading R34)
  const int64_t cap = window_blocks > 0 ? window_blocks : c->cfg.num_blocks;
  const int64_t per_q = n > 0 ? std::max<int64_t>(1, blocks_total / n) : 1;
  const int64_t win = std::max<int64_t>(1, cap / per_q);
  std::vector<uint8_t> done(n, 0);
  std::unordered_map<spq::Digest, int32_t, spq::DigestHash> recent;  // unit -> count in window
  std::vector<int32_t> out;
  for (int32_t step = 0; step < n; ++step) {
    int32_t best = -1;
    int64_t best_ov = -1;
    for (int32_t i = 0; i < n; ++i) {
      if (done[i]) continue;
      int64_t ov = 0;
      for (const spq::Digest& d : units[i]) ov += recent.count(d) ? 1 : 0;
      if (ov > best_ov) {  // ties: lowest index (arrival order)
        best_ov = ov;
        best = i;
      }
    }
    done[best] = 1;
    out.push_back(best);
    for (const spq::Digest& d : units[best]) recent[d]++;
    if (static_cast<int64_t>(out.size()) > win) {  // slide: forget the query leaving the window
      for (const spq::Digest& d : units[out[out.size() - 1 - win]]) {
        auto it = recent.find(d);
        if (--it->second == 0) recent.erase(it);
      }
    }
  }
  std::memcpy(order, out.data(), out.size() * sizeof(int32_t));
  return SPQ_OK;
}

spq_status spq_reduce_tree(int32_t n, int32_t k, int32_t* ply_off, int64_t ply_cap, int32_t* child_off,
                           int32_t* children, int64_t judge_cap, int32_t* n_plies, int32_t* n_judges) {
  if (n_plies == nullptr || n_judges == nullptr) return fail(SPQ_EINVAL, "null argument");
  if (n < 1 || k < 2) return fail(SPQ_EINVAL, "need n >= 1 candidates and branching factor k >= 2");
  std::vector<int32_t> po{0}, co{0}, ch;
  std::vector<int32_t> level(n);
  for (int32_t i = 0; i < n; ++i) level[i] = i;  // items of the current ply: candidates 0..n-1
  int32_t next_id = n;
  do {  // n <= k: one judge over every candidate (the query unchanged)
    std::vector<int32_t> up;
    for (size_t g = 0; g < level.size(); g += static_cast<size_t>(k)) {
      const size_t e = std::min(level.size(), g + static_cast<size_t>(k));
      if (e - g == 1 && level.size() > 1) {  // a lone item passes up unjudged (reading R33)
        up.push_back(level[g]);
        continue;
      }
      ch.insert(ch.end(), level.begin() + static_cast<std::ptrdiff_t>(g), level.begin() + static_cast<std::ptrdiff_t>(e));
      co.push_back(static_cast<int32_t>(ch.size()));
      up.push_back(next_id++);
    }
    po.push_back(static_cast<int32_t>(co.size()) - 1);
    level.swap(up);
  } while (level.size() > 1);
  *n_plies = static_cast<int32_t>(po.size()) - 1;
  *n_judges = static_cast<int32_t>(co.size()) - 1;
  if (ply_cap < static_cast<int64_t>(po.size()) || judge_cap < static_cast<int64_t>(co.size()) ||
      ply_off == nullptr || child_off == nullptr || children == nullptr)
    return fail(SPQ_EINVAL, "capacity too small (n_plies / n_judges report the sizes)");
  std::memcpy(ply_off, po.data(), po.size() * sizeof(int32_t));
  std::memcpy(child_off, co.data(), co.size() * sizeof(int32_t));
  std::memcpy(children, ch.data(), ch.size() * sizeof(int32_t));
  return SPQ_OK;
}

spq_status spq_set_option(spq_ctx* c, int32_t key, double value) {
  if (c == nullptr) return fail(SPQ_EINVAL, "null argument");
  switch (key) {
    case SPQ_OPT_EXP2:
      if (value != 0 && value != 1 && value != 2 && value != 3 && value != 4)
        return fail(SPQ_EINVAL, "SPQ_OPT_EXP2 must be 0, 1, 2, 3 or 4");
      // kernel poly_mask: 0 MUFU ex2, 3 MUFU ex2.f16x2, 1 / 2 a quarter / half on the FMA pipe,
      // -1 auto (prefill 0, joins 1)
      c->exp2_mode = value == 1 ? 3 : value == 2 ? 1 : value == 3 ? 2 : value == 4 ? -1 : 0;
      return SPQ_OK;
    case SPQ_OPT_RESCALE_THRESHOLD:
      if (!(value >= 0 && value <= 64)) return fail(SPQ_EINVAL, "SPQ_OPT_RESCALE_THRESHOLD must be in [0, 64]");
      c->rescale_threshold = static_cast<float>(value);
      return SPQ_OK;
    case SPQ_OPT_PDL:
      c->pdl = value != 0;
      return SPQ_OK;
    case SPQ_OPT_HASH_SCALAR:
      spq::blake2b_force_scalar(value != 0);
      return SPQ_OK;
    case SPQ_OPT_PAIR:
      c->pair = value != 0;
      return SPQ_OK;
    default:
      return fail(SPQ_EINVAL, "unknown option " + std::to_string(key));
  }
}

spq_status spq_set_trace(spq_ctx* c, void* buf, int32_t mode) {
  if (c == nullptr) return fail(SPQ_EINVAL, "null argument");
#ifdef SPANQ_PROFILING
  c->trace = static_cast<long long*>(buf);
  c->dbg_mode = mode;
  return SPQ_OK;
#else
  (void)buf;
  (void)mode;
  return fail(SPQ_EINVAL, "tracing needs a profiling build (build.py --profiling)");
#endif
}

spq_status spq_launch_count(const spq_ctx* c, int64_t* n) {
  if (c == nullptr || n == nullptr) return fail(SPQ_EINVAL, "null argument");
  *n = c->launches;
  return SPQ_OK;
}

spq_status spq_set_timing(spq_ctx* c, int32_t enable) {
  if (c == nullptr) return fail(SPQ_EINVAL, "null argument");
  if (!is_gpu(c)) return fail(SPQ_ESTATE, "host-only ctx");
  c->timing = enable != 0;
  return SPQ_OK;
}

spq_status spq_last_attn_ms(spq_ctx* c, float* prefill_ms, float* join_ms) {
  if (c == nullptr) return fail(SPQ_EINVAL, "null argument");
  if (!is_gpu(c)) return fail(SPQ_ESTATE, "host-only ctx");
  if (prefill_ms) {
    *prefill_ms = 0.f;
    if (c->prefill_timed) CUDA_TRY(cudaEventElapsedTime(prefill_ms, c->ev[0], c->ev[1]));
  }
  if (join_ms) {
    *join_ms = 0.f;
    if (c->join_timed) CUDA_TRY(cudaEventElapsedTime(join_ms, c->ev[2], c->ev[3]));
  }
  return SPQ_OK;
}

}  // extern "C"
