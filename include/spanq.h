/* spanq.h — C ABI of the B200-native span-query prefill path (arXiv 2511.02749).
 *
 * The calls follow the paper's statement of the problem:
 *   plan a span-query expression tree      — Def. "Span Query" PAPER.md §4.1,
 *                                            joins ⊕ / ⋈ Def. P:333-335;
 *   look up and insert fragment KV         — block hashing with suspended accumulation
 *                                            §5.4, prefix scan §2;
 *   run fragment prefill                   — fragments "prepared" independently of context,
 *                                            §5.1 footnote; span-sparse attention;
 *   run join prefill                       — the final ⋈ over cached, repositioned blocks
 *                                            ("ReRoPE", §5.5) + the cross tokens.
 *
 * Conventions
 *  - extern "C", plain pointers and sizes. "device" pointers live on ctx's CUDA device;
 *    "host" pointers in host memory. Streams are `cudaStream_t` passed as `void*` (NULL = the
 *    legacy default stream).
 *  - Every call returns spq_status; no exception crosses the ABI. On failure the message is
 *    available from spq_last_error() (thread-local, valid until the next failing call on
 *    the same thread).
 *  - Layouts are row-major. Activations: q [rows, Hq, d], k/v [rows, Hkv, d] in the ctx dtype,
 *    o [rows, Hq, d] in cfg.out_dtype (bf16 = IEEE bfloat16 bit patterns, or fp32), lse [rows, Hq] fp32 natural
 *    log. KV pools: [num_layers][num_blocks][Hkv][block_size][d] in the ctx dtype; slot
 *    s = block_id * block_size + offset addresses one token row of one block.
 *  - A ctx is single-writer (not thread-safe); plans execute in stream order.
 */
#ifndef SPANQ_H_
#define SPANQ_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPQ_OK = 0,
  SPQ_EINVAL = 1, /* bad argument, tree shape, op code, arity, empty leaf, negative token   */
  SPQ_ENOMEM = 2, /* the block pool cannot hold the plan's blocks; the plan is rolled back  */
  SPQ_ECUDA = 3,  /* CUDA launch/runtime failure, or no usable sm_100 device               */
  SPQ_ENCCL = 4,  /* reserved: the library issues no collective (reading R35)     */
  SPQ_ESTATE = 5  /* plan used after release, job/query range out of bounds, wrong mode     */
} spq_status;

typedef enum { SPQ_BF16 = 0, SPQ_FP32 = 1 } spq_dtype;

typedef struct {
  int32_t num_q_heads;  /* Hq  (multiple of Hkv; GQA q-head h uses kv-head h / (Hq/Hkv))    */
  int32_t num_kv_heads; /* Hkv                                                               */
  int32_t head_dim;     /* d: 64 or 128 on the GPU (either dtype); any >= 2 for host-only ctx */
  int32_t num_layers;   /* L                                                                 */
  int32_t block_size;   /* bs tokens per KV block: 16/32/64/128 on the GPU; any >=1
                           for host-only contexts                                            */
  int64_t num_blocks;   /* pool capacity in blocks on this device                            */
  int32_t dtype;        /* spq_dtype                                                         */
  double rope_base;     /* θ_i = rope_base^(-2i/d); rotate-half pairs (R15)     */
  int32_t max_position; /* RoPE table length (positions 0..max_position-1)                   */
  uint64_t model_salt;  /* folded into the root digest                                       */
  void *k_pool;         /* device, CALLER-owned, [L][num_blocks][Hkv][bs][d]; must outlive ctx */
  void *v_pool;         /* device, CALLER-owned, same layout                                 */
  int32_t device;       /* CUDA device ordinal; -1 = host-only ctx (planner/store, no kernels) */
  int32_t rank;         /* this rank, 0..world_size-1 (SURVEY §8(e) partitioning)             */
  int32_t world_size;   /* ranks sharing a batch: query q is homed on q mod W, fragment f owned
                           by u64le(s_last(f)[0:8]) mod W; each rank plans only its share       */
  int32_t out_dtype;    /* spq_dtype of o (attention outputs); SPQ_FP32 is allowed with a bf16
                           ctx (bf16 MMAs, fp32 outputs: removes the final bf16 rounding of O)  */
  int32_t split_join;   /* world_size > 1: 0 = remote fragments' KV moves to the home rank
                           (spq_exchange_*), 1 = owner-side split join: the home query's cross Q
                           moves to the fragment owners and their partial (O, LSE) come back
                           (spq_split_*)                                       */
} spq_config;

typedef struct spq_ctx spq_ctx;
typedef struct spq_plan spq_plan;

/* Create a context: validates cfg, builds the fp64->fp32 RoPE cos/sin table on the device
 * and the TMA descriptors of both pools. Fails with SPQ_ECUDA if device >= 0 and the device
 * is not sm_100. */
spq_status spq_create(const spq_config *cfg, spq_ctx **out);
void spq_destroy(spq_ctx *ctx); /* synchronizes ctx's device work; NULL is a no-op */
const char *spq_last_error(void);
const char *spq_version(void);

/* ------------------------------------------------------------------ span-query trees */
typedef enum { SPQ_TOKENS = 0, SPQ_PLUS = 1, SPQ_CROSS = 2 } spq_op; /* leaf, ⊕, ⋈ */
typedef struct {
  int32_t op;           /* spq_op                                                       */
  int32_t num_children; /* children follow in pre-order                                 */
  int64_t tok_begin;    /* TOKENS: first token index into spq_query.tokens              */
  int64_t tok_len;      /* TOKENS: token count (>= 1)                                   */
} spq_node;
/* Accepted tree (v1): root ⋈ with children [TOKENS prefix]? [⊕ ...]? TOKENS cross, where a ⊕
 * child is a TOKENS fragment, a nested ⊕ (flattened — "plus simplification") or a ⋈ of
 * TOKENS leaves (concatenated into one fragment). This is the optimized RAG form
 * G[⋈[S, ⊕[F…], U]] and the judge form ⋈[prefix, ⊕[c…], suffix]. */
typedef struct {
  const spq_node *nodes; /* host */
  int32_t num_nodes;
  const int32_t *tokens; /* host, token ids >= 0 */
  int64_t num_tokens;
} spq_query;

/* ------------------------------------------------------------------ low level */
/* Digests of one query, 16 bytes each, in the order: prefix blocks, each fragment's blocks (⊕
 * order), the join fold J, cross blocks. BLAKE2b-128 chains. *n is
 * set to the count; if cap is smaller, SPQ_EINVAL and nothing is written. */
spq_status spq_block_hashes(const spq_ctx *ctx, const spq_query *q, uint8_t *digests /*host [cap][16]*/,
                            int64_t cap, int64_t *n);
/* Pure lookup: block id of each resident digest, -1 on miss. No stats/LRU side effects. */
spq_status spq_lookup(const spq_ctx *ctx, const uint8_t *digests, int64_t n, int32_t *block_ids);
/* Insert digests (ntok tokens each, 1..bs): resident digests return their id, others get the
 * lowest free block id (evicting LRU unpinned blocks). Blocks are not pinned and their
 * contents are not written. All-or-nothing: SPQ_ENOMEM rolls back. */
spq_status spq_insert(spq_ctx *ctx, const uint8_t *digests, const int32_t *ntok, int64_t n,
                      int32_t *block_ids);

/* ------------------------------------------------------------------ plans */
/* Plan a batch of queries: validate + flatten trees, assign positions (prefix 0..P-1,
 * fragment f local 0..L_f-1 stored / global Δ_f = P + Σ_{g<f} L_g, cross P+S+j), hash,
 * prefix-scan the prefix, all-or-nothing lookup per fragment, dedupe within the plan,
 * allocate (lowest free id) + insert, evict LRU unpinned, pin everything referenced, build the
 * kernels' work lists and upload them with one H2D copy on `stream`. Readings R8-R13 in
 * DESIGN.md. On SPQ_ENOMEM/SPQ_EINVAL the store is unchanged. */
spq_status spq_plan_create(spq_ctx *ctx, const spq_query *queries, int32_t n_queries, void *stream,
                           spq_plan **out);

typedef struct {
  int32_t n_queries, n_segments, n_jobs;
  int64_t n_blocks_total;
  /* per segment (query order; within a query: prefix?, fragments in ⊕ order, cross) */
  const int32_t *seg_query, *seg_kind /*0 prefix 1 fragment 2 cross*/, *seg_frag_idx, *seg_tok_len,
      *seg_pos0 /*global position of first token*/, *seg_hit /*prefix: #hit blocks; fragment: 0/1*/,
      *seg_compute_begin /*first recomputed row (tok_len = none)*/, *seg_block_off, *seg_n_blocks;
  const int32_t *blocks;      /* [n_blocks_total] block ids, segment-major                   */
  const uint8_t *block_write; /* [n_blocks_total] 1 = written by this plan                   */
  const uint8_t *digests;     /* [n_blocks_total][16]                                        */
  const uint8_t *join_digests;/* [n_queries][16]                                             */
  const int32_t *jobs;        /* [n_jobs] segment index of each prefill job, plan order      */
  const int64_t *job_row_off; /* [n_jobs+1] packed prefill row offsets                       */
  int64_t n_prefill_rows;
  const int32_t *prefill_pos; /* stored position of each packed prefill row                  */
  const int64_t *prefill_slot;/* pool slot or -1 (resident block: read, not rewritten)       */
  int64_t n_join_rows;
  const int64_t *query_join_row_off; /* [n_queries+1]                                        */
  const int32_t *join_pos;
  const int64_t *join_slot;
  int64_t n_pad_slots;
  const int64_t *pad_slots;   /* slots zero-filled by the first prefill/join call of a plan  */
  double prefill_flops;       /* algorithmic 4·d·Hq·(visible pairs) of all prefill jobs      */
  double join_flops;          /* same for all joins                                          */
  int64_t prefill_kv_bytes;   /* K/V bytes written by rope_kv_write for prefill rows         */
  int64_t join_kv_bytes;
  /* world_size > 1: queries homed here (q mod W == rank) and the fragment-KV
   * exchange lists. Peer w: send_blocks[send_off[w] .. send_off[w+1]) are this rank's blocks of
   * the fragments it owns that w's joins read (all of them until spq_exchange_set_need narrows the
   * list to the ones w flagged); recv_blocks[recv_off[w] .. recv_off[w+1]) are the blocks that
   * receive the fragments owned by w which have no resident replica here. Received fragments are
   * indexed under their digests (reading R38: digest-keyed replicas, later plans on this rank hit
   * them). Fragments in first-occurrence (query, ⊕) order, each fragment's blocks in order — both
   * sides derive the same candidate sequence. With world_size 1 all lists are empty. */
  int32_t n_join_queries;
  int32_t world_size;
  const int64_t *send_off;    /* [world_size+1] */
  const int32_t *send_blocks;
  const int64_t *recv_off;    /* [world_size+1] */
  const int32_t *recv_blocks;
  /* split_join: the tasks this rank computes for other homes, [n_tasks][6] = {query, home,
   * n_rows (the query's cross rows), pos0 (global position of cross row 0), seg_begin, seg_end
   * (its fragment segments owned here, pos0 = Δ_f)}, in (home, query) order; and per peer w the
   * home queries whose cross Q this rank sends to w and whose partials w returns:
   * xq_queries[xq_off[w] .. xq_off[w+1]), query order. Empty unless split_join. */
  int32_t n_tasks;
  const int32_t *tasks;
  const int32_t *xq_off;      /* [world_size+1] */
  const int32_t *xq_queries;
  /* Replica need flags (R38). Home side, per owner peer w: cand_recv_need[cand_recv_off[w] ..
   * cand_recv_off[w+1]), one byte per remote fragment its joins read (first-occurrence order):
   * 1 = its KV must be sent, 0 = a replica is resident here. Owner side: cand_send_off[w+1] -
   * cand_send_off[w] = how many such fragments home peer w will flag. The home sends its flags to
   * each owner (a byte all-to-all), which passes them to spq_exchange_set_need. */
  const int64_t *cand_recv_off;  /* [world_size+1] */
  const uint8_t *cand_recv_need;
  const int64_t *cand_send_off;  /* [world_size+1] */
} spq_plan_view;
/* Read-only host arrays, valid until spq_plan_release. */
spq_status spq_plan_view_get(const spq_plan *plan, spq_plan_view *out);

/* Fragment / prefix prefill for jobs [job_begin, job_end): rope_kv_write of the jobs' rows
 * with slot >= 0 (RoPE at the stored position, fused with the paged write), then block-diagonal
 * causal attention (each job attends only within itself).
 *  q, k, v: device, packed pre-RoPE rows of those jobs, rows [job_row_off[a], job_row_off[b]).
 *  o: device [rows, Hq, d]; lse: device [rows, Hq] (may be NULL).  ctx must have device >= 0. */
spq_status spq_prefill_jobs(spq_ctx *ctx, spq_plan *plan, int32_t layer, int32_t job_begin,
                            int32_t job_end, const void *q, const void *k, const void *v, void *o,
                            float *lse, void *stream);

/* Join prefill for queries [q_begin, q_end): rope_kv_write of the cross rows, then the cross
 * rows attend over [prefix | every fragment at its Δ_f | cross causal] from the pool (Q is
 * counter-rotated by p - Δ_f per fragment: repositioning without touching cached KV), split
 * over the KV range and merged by `combine`.
 *  q/k/v: device, cross rows of those queries packed in query order
 *  (rows [query_join_row_off[a], query_join_row_off[b])). o/lse as above.
 * All prefill jobs of the plan that precede these queries must have been issued first on the
 * same stream (their KV is read here). */
spq_status spq_join(spq_ctx *ctx, spq_plan *plan, int32_t layer, int32_t q_begin, int32_t q_end,
                    const void *q, const void *k, const void *v, void *o, float *lse, void *stream);

/* Fragment-KV exchange, HBM side. One layer's blocks of the plan's exchange list
 * for `peer` (see spq_plan_view) are copied between the pool and a packed device buffer laid out
 * [n][2 (K then V)][Hkv][bs][d] in the pool dtype, n = send (pack) or recv (unpack) block count.
 * The transfer between ranks is the caller's (one NCCL all-to-all per layer). Pack must follow
 * the prefill jobs that write those blocks on `stream`; unpack must precede spq_join. Blocks are
 * copied whole (pads included: the owner zero-filled them). SPQ_ESTATE on a bad peer/layer. */
spq_status spq_exchange_pack(spq_ctx *ctx, spq_plan *plan, int32_t layer, int32_t peer, void *buf,
                             void *stream);
spq_status spq_exchange_unpack(spq_ctx *ctx, spq_plan *plan, int32_t layer, int32_t peer,
                               const void *buf, void *stream);
/* Owner side of the replica protocol (R38): keep in the send list to home peer `peer` only the
 * candidate fragments that peer flagged (need[i] != 0, host array of n = its candidate count,
 * cand_send_off in the view). Call once per peer before the plan's first spq_exchange_pack; the
 * view's send lists change (re-read the view). The device copy of the list is rewritten on
 * `stream`. SPQ_EINVAL: n differs from the candidate count or need is NULL with n > 0;
 * SPQ_ESTATE: released plan or bad peer. */
spq_status spq_exchange_set_need(spq_ctx *ctx, spq_plan *plan, int32_t peer, const uint8_t *need,
                                 int64_t n, void *stream);

/* The same join of all of the plan's home queries in two launches, so that on W > 1 the
 * fragment-KV exchange overlaps the first: phase 0 = rope_kv_write of the cross
 * rows and the attention over the segments this rank holds (prefix, locally owned fragments,
 * cross causal); phase 1 — after spq_exchange_unpack of this layer — the attention over the
 * received fragments and the combine of both phases' fp32 split partials into o / lse (in a
 * fixed order: phase-0 pieces, then phase-1 pieces). A plan without received fragments, or on
 * the fp32 path (no split partials), runs the whole join in phase 1 and phase 0 is a no-op.
 * Arguments as spq_join over [0, n_queries); phase must be 0 or 1 (SPQ_EINVAL). Both phases
 * must be issued, in order, for the layer. */
spq_status spq_join_phase(spq_ctx *ctx, spq_plan *plan, int32_t layer, int32_t phase, const void *q,
                          const void *k, const void *v, void *o, float *lse, void *stream);

/* ------------------------------------------------------------------ decode after the join
 * Token generation G over a span query (§4.1, Def. "Span Query" P:205-207; nested
 * generation P:170). Generated token t of home query q
 * sits at position N_q + t (N_q = P + S + C, reading R3) and its KV continues the cross
 * segment's blocks (the partial cross tail block, then plan-private generation blocks).
 *
 * Reserve generation blocks for max_new tokens of every home query of the plan (rows in query
 * order) and build the decode work lists (one H2D). Call once per plan, after spq_plan_create.
 * SPQ_ENOMEM: the pool cannot hold them (nothing reserved); SPQ_EINVAL: max_new < 1 or a query
 * would exceed max_position; SPQ_ESTATE: released plan, reserved twice, or no home query. */
spq_status spq_decode_reserve(spq_ctx *ctx, spq_plan *plan, int32_t max_new);
/* Decode step t (0 <= t < max_new) of layer `layer` for every home query: rope_kv_write of the
 * new token's k/v at position N_q + t into its reserved slot, then its row attends over
 * [prefix | every fragment at Δ_f (Q counter-rotated) | cross + generated 0..t] (K9,
 * split-KV + combine). q: device [rows, Hq, d], k/v: device [rows, Hkv, d] (pre-RoPE, ctx
 * dtype), o: device [rows, Hq, d] (out dtype), lse: device [rows, Hq] fp32 or NULL; rows = the
 * plan's home queries in query order. Steps of a layer must be issued in order t = 0, 1, ...
 * after that layer's spq_join (same stream). SPQ_ESTATE: not reserved, t out of range, bad layer,
 * released plan, host-only ctx. */
spq_status spq_decode_step(spq_ctx *ctx, spq_plan *plan, int32_t layer, int32_t t, const void *q,
                           const void *k, const void *v, void *o, float *lse, void *stream);
/* Plus distribution: commit query `query`'s sequence — its cross tokens followed by
 * its first n_gen generated tokens (host array, the caller's sampled ids) — as a cached
 * fragment: its blocks are indexed under the fragment chain ('F', DESIGN.md hash contract) of
 * those tokens, so a later query with the sequence as a ⊕ fragment hits without prefill (the KV
 * is already at span-local positions 0..len-1). crop = 1 drops the trailing partial block
 * (the paper's cropping); crop = 0 keeps it with its true token count (reading R8).
 * *n_committed = tokens committed (the fragment the caller must use). The query must have no
 * prefix and no fragments (an inner generate ⋈[input], positions from 0): SPQ_EINVAL otherwise.
 * The decode steps 0..n_gen-1 of every layer must have been issued. The blocks stay pinned until
 * the plan's release, then are ordinary cached blocks (LRU). SPQ_ESTATE: released plan or n_gen
 * beyond the reservation. */
spq_status spq_commit_span(spq_ctx *ctx, spq_plan *plan, int32_t query, const int32_t *gen_tokens /*host*/,
                           int32_t n_gen, int32_t crop, int32_t *n_committed /*or NULL*/);

/* Plus distribution for an inner generate whose output feeds a later span (the k-ary judge
 * reduction, §6): commit only the n_gen generated tokens of `query` as a
 * cached fragment. They sit at positions N_q + t; their K is re-encoded to the span-local
 * positions t (CIDRA / ReRoPE by -N_q, in place on every layer, on `stream`)
 * and their blocks are indexed under the fragment chain of gen_tokens (host). Needs block
 * alignment: the cross length must be a multiple of block_size (SPQ_EINVAL
 * otherwise). Ends the query's generation (its KV has moved). The decode steps 0..n_gen-1 of
 * every layer must precede on `stream`. SPQ_ESTATE: no reservation covering n_gen, released plan,
 * host-only ctx. */
spq_status spq_commit_output(spq_ctx *ctx, spq_plan *plan, int32_t query, const int32_t *gen_tokens /*host*/,
                             int32_t n_gen, void *stream, int32_t *n_committed /*or NULL*/);

/* The k-ary judge reduction (§6, Fig. 13 "3 2-way judge steps"; SPEC
 * reduce_for_attention) as a schedule: items 0..n-1 are the candidates, judge j is item n + j.
 * Each ply groups its items k at a time, in order, under one judge; a lone last item passes up
 * unjudged (reading R33); plies repeat until one item remains (n <= k: one judge over all n).
 * Judges are numbered ply by ply: ply p = judges [ply_off[p], ply_off[p+1]), judge j reads items
 * children[child_off[j] .. child_off[j+1]). Host only. SPQ_EINVAL: n < 1, k < 2, or a capacity
 * too small (*n_plies / *n_judges still report the sizes: ply_off needs n_plies + 1 entries,
 * child_off n_judges + 1, children <= n + n_judges). */
spq_status spq_reduce_tree(int32_t n, int32_t k, int32_t *ply_off, int64_t ply_cap, int32_t *child_off,
                           int32_t *children, int64_t judge_cap, int32_t *n_plies, int32_t *n_judges);

/* Bulk execution order (§5.8: "a greedy heuristic that clusters the requests in a
 * given bulk to increase temporal locality"), reading R34: a query's cached units are its
 * fragments (s_last digests) and its whole prefix (h_last); the pool is taken to hold the last
 * W queries' units, W = window_blocks (0: the ctx's capacity) / the bulk's mean blocks per
 * query; starting from query 0, repeatedly schedule the unscheduled query sharing the most units
 * with those W (ties: lowest index). order: host [n], a permutation of 0..n-1. Host only; the
 * store is not touched. SPQ_EINVAL: invalid tree, null argument. */
spq_status spq_bulk_order(const spq_ctx *ctx, const spq_query *queries, int32_t n, int64_t window_blocks,
                          int32_t *order);

/* ------------------------------------------------------------------ owner-side split join
 * (cfg.split_join = 1, world_size > 1; §4.3: independent
 * sub-trees run in parallel). Per layer, with the transfers done by the caller's collective (one
 * all-to-all each way, NCCL):
 *   home:  spq_split_pack_q(q_join -> qsend)         [Q all-to-all]    spq_split_join_local(...)
 *   owner: spq_split_task_join(qrecv -> partials)    [partial all-to-all]
 *   home:  spq_split_merge(partials_recv -> o, lse)
 * Buffer layouts (row = one query row, all Hq heads): qsend = for each owner peer w (rank order),
 * the rows of the home queries xq_queries[xq_off[w]..) (query order) — [rows][Hq][d], ctx dtype,
 * pre-RoPE; qrecv = for each home peer h (rank order) the rows of this rank's tasks with home h
 * (task order = the view's tasks) — the same layout as the tasks' row space; partials:
 * O [rows][Hq][d] fp32 (normalized) and LSE [rows][Hq] fp32 (natural log), sent back in the same
 * row order (partials_recv laid out like qsend). All calls: SPQ_ESTATE on a plan that is not a
 * split-join plan, a released plan or a host-only ctx; SPQ_EINVAL on a null buffer. */
spq_status spq_split_pack_q(spq_ctx *ctx, spq_plan *plan, const void *q_join /*[join rows][Hq][d]*/,
                            void *qsend, void *stream);
/* The tasks' join: each task's query rows attend over its fragments owned here (Q counter-rotated
 * by Δ_f, the join kernel + combine) -> fp32 partials. */
spq_status spq_split_task_join(spq_ctx *ctx, spq_plan *plan, int32_t layer, const void *qrecv, float *part_o,
                               float *part_lse, void *stream);
/* Home side: rope_kv_write of the cross rows + the join over the segments held here (prefix,
 * locally owned fragments, cross causal) into a plan-owned fp32 result (overlaps the exchange). */
spq_status spq_split_join_local(spq_ctx *ctx, spq_plan *plan, int32_t layer, const void *q, const void *k,
                                const void *v, void *stream);
/* Home side: o / lse = LSE merge of the local result and the owners' partials, in a fixed order
 * (local, then owners by rank): every home query row, out dtype. */
spq_status spq_split_merge(spq_ctx *ctx, spq_plan *plan, const float *part_o_recv, const float *part_lse_recv,
                           void *o, float *lse, void *stream);

/* Stream-ordered release: unpins the plan's blocks and frees its plan-private blocks; later
 * kernel calls on any stream wait for `stream` to pass this point before touching them. The
 * handle stays reserved (emptied) for the next 1024 releases of the ctx: any call on it in that
 * window returns SPQ_ESTATE ("plan used after release"); after it the handle must not be used.
 * Plans never released are freed by spq_destroy. */
spq_status spq_plan_release(spq_ctx *ctx, spq_plan *plan, void *stream);

/* ------------------------------------------------------------------ store admin / stats */
typedef struct {
  int64_t lookups, hit_blocks, miss_blocks, hit_tokens, input_tokens, evictions, inserted_blocks;
  int64_t resident_blocks, free_blocks, pinned_blocks, plans;
} spq_stats;
spq_status spq_get_stats(const spq_ctx *ctx, spq_stats *out); /* hit rate = hit/input tokens */
/* Drop every unpinned resident block (cold-cache reset). */
spq_status spq_evict_all(spq_ctx *ctx);
/* Copy the K and V pages of blocks ids[0..n) of one layer out of the pool (inspection / parity,
 * SURVEY §8(b)): k and v are caller-owned device buffers [n][Hkv][bs][d] in the pool dtype,
 * stream-ordered on `stream`. SPQ_EINVAL on a null buffer or an id outside [0, num_blocks),
 * SPQ_ESTATE on a host-only ctx or a bad layer. */
spq_status spq_read_blocks(spq_ctx *ctx, int32_t layer, const int32_t *block_ids /*host*/, int64_t n,
                           void *k, void *v, void *stream);

/* ------------------------------------------------------------------ CIDRA repositioning
 * PAPER.md §5.5.1 "Concurrent In-place Duplicating ReRoPE": for consumers that need
 * cached KV at absolute positions (the span path itself never does — the join counter-rotates Q,
 * SURVEY §8(f) f2). Move i: block dst[i] of every layer in [layer_begin, layer_end) ends
 * up holding the ORIGINAL content of block src[i], K re-encoded delta[i] positions later (ReRoPE
 * P:610, rotate-half pairs; all tokens of a block share delta) and V copied — the result of the
 * out-of-place definition (SPEC), reached in place: the move graph is split into
 * independent components (trees, and cycles with trees attached); inside one a block is
 * overwritten only after every move reading it, and a cycle rotates through one scratch slot.
 * A source may feed several destinations ("duplication"); a destination appears once.
 * src/dst/delta are HOST arrays of n entries; the pools are the ctx's; stream-ordered on
 * `stream`. Store effect: every destination block is dropped from the content-hash index (it no
 * longer holds what its digest names; it becomes a free block whose moved content the caller
 * owns until a later plan allocates it), so no later plan can hit stale KV. SPQ_EINVAL: null
 * array, id outside [0, num_blocks), a destination written twice, |delta| >= max_position,
 * head_dim not 64/128; SPQ_ESTATE: host-only ctx, bad layer range, or a source/destination block
 * pinned by a live plan (nothing is moved); SPQ_ECUDA: launch failure. */
typedef struct {
  int64_t moves, components, cycles, duplicates, ops, max_component_ops;
} spq_cidra_stats;
spq_status spq_reposition(spq_ctx *ctx, const int32_t *src, const int32_t *dst, const int32_t *delta, int64_t n,
                          int32_t layer_begin, int32_t layer_end, void *stream, spq_cidra_stats *stats /*or null*/);
/* The in-place schedule spq_reposition runs (host only; inspection / tests): ops[cap][4] =
 * {dst, src, delta, mode} with mode 0: dst <- R(src), 1: scratch <- src, 2: dst <- R(scratch);
 * comp_off[comp_cap] = component boundaries (n_comp + 1 entries). SPQ_EINVAL as above, or when
 * a capacity is too small (*n_ops / *n_comp still report the sizes needed). */
spq_status spq_cidra_schedule(const spq_ctx *ctx, const int32_t *src, const int32_t *dst, const int32_t *delta,
                              int64_t n, int32_t *ops, int64_t cap, int64_t *n_ops, int32_t *comp_off,
                              int64_t comp_cap, int64_t *n_comp, spq_cidra_stats *stats /*or null*/);

/* ------------------------------------------------------------------ options */
typedef enum {
  SPQ_OPT_EXP2 = 1,              /* softmax exp2: 0 = MUFU ex2 fp32, 1 = MUFU ex2.f16x2 (two
                                    exponentials per op; inputs rounded to f16), 2 / 3 = a
                                    quarter / half of them by an FMA-pipe polynomial (rel. error
                                    1e-4, below the bf16 rounding of P), 4 = auto (default:
                                    prefill 0, joins 2 — measured fastest for each)            */
  SPQ_OPT_RESCALE_THRESHOLD = 2, /* O is rescaled when a row max grows by more than this (log2
                                    units, default 8; 0 = on every growth). Exact either way  */
  SPQ_OPT_PDL = 3,               /* 1 (default): attention/combine launched as programmatic
                                    dependents of the kernel before them; 0: plain launches  */
  SPQ_OPT_HASH_SCALAR = 4,       /* process-wide: 1 = scalar BLAKE2b compression even with AVX2
                                    (same digests; lets tests cover both), 0 = default        */
  SPQ_OPT_PAIR = 5               /* 1: prefill of d = 128, GQA 4k, bf16 O on CTA pairs
                                    (cta_group::2, M = 256); 0 (default, measured faster): one
                                    CTA per head pair. Read when a plan is created (its prefill
                                    work list fixes the launch shape)                         */
} spq_option;
/* Set a ctx option (applies to later calls). SPQ_EINVAL on an unknown key or a bad value. */
spq_status spq_set_option(spq_ctx *ctx, int32_t key, double value);
/* Profiling builds only (build.py --profiling defines SPANQ_PROFILING): a device buffer of
 * int64 [16 warps][1024][2] (event, clock64) + [2 * grid] (%globaltimer per CTA) that the
 * attention kernel's CTA 0 fills, and a timing-variant mode (0 = off). The product library
 * returns SPQ_EINVAL. */
spq_status spq_set_trace(spq_ctx *ctx, void *device_buf, int32_t mode);

/* Instrumentation: kernel launches issued by this ctx so far, and the CUDA events bracketing
 * the most recent attention launch (for roofline timing on the launching stream). */
spq_status spq_launch_count(const spq_ctx *ctx, int64_t *n);
spq_status spq_last_attn_ms(spq_ctx *ctx, float *prefill_ms, float *join_ms);
/* Enable/disable recording of those events (off by default; recording adds 4 event records
 * per call). */
spq_status spq_set_timing(spq_ctx *ctx, int32_t enable);

#ifdef __cplusplus
}
#endif
#endif /* SPANQ_H_ */
