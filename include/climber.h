/*
 * climber.h — C ABI of libclimber.so: B200-native "single user, multiple items"
 * (SUMI) ranking inference for Climber (arXiv 2502.09888).
 *
 * The calls follow the paper's statement of the serving problem (PAPER.md
 * L257, §3.2 Deployment): "the system first generates multi-layered key-value
 * (KV) cache vectors from user features, then fetches candidate item features
 * from the feature server, and finally computes attention-based interactions
 * between the item features and cached KV representations."
 *
 *   climber_encode_user(events, r)        -> kv handle   (multi-layer K/V cache)
 *   climber_score_items(kv, items[M])     -> scores[M]   (SUMI attention + BGF)
 *
 * What is computed (PAPER.md, readings G1-G28 of SURVEY.md §8(c)):
 *   - MSE extraction (Eq. 1-2): per strategy a_k, the most recent n_k
 *     events whose action/scenario pass the strategy's filters, chronological.
 *   - N_b blocks of L adaptive Transformer layers (Eq. 3): pre-RMSNorm,
 *     QKV, softmax(QK^T / (sqrt(d_h) * tau[l][k][r][head])) V, W_O + residual,
 *     RMSNorm, FFN (d -> 4d SiLU -> d) + residual.  History attention is causal
 *     (hist_causal = 1) or bidirectional (0); every candidate attends to the
 *     whole history of its block plus itself only (L255: full-visible +
 *     diagonal masks).  Relative bias f_b is 0 (G6) unless the config sets
 *     rel_bias = 1 (Eq. 3's f_b^{p,t}(a_k, r), see climber_config).
 *   - Bit-wise gating fusion (Eq. 4): one fusion ATL over the N_b block
 *     outputs (temperature tau_f[r][head], no mask), squeeze-and-excitation gate
 *     FC(N_b d -> N_b d / se_reduction) + b, ReLU, FC + b, sigmoid, product.
 *   - Head: score = w_head . vec(Y) + b_head, an fp32 logit (G18).
 *
 * Conventions for every call:
 *   - Return value: climber_status.  No C++ exception or abort crosses the ABI.
 *     On failure climber_last_error() (thread-local) describes the cause.
 *   - Host-checkable errors (NULL, sizes, config) return synchronously and
 *     enqueue nothing.  Data-dependent errors (ids out of range, decreasing
 *     timestamps) are detected on the device: they set the ctx's device error
 *     word, the affected scores become NaN, and climber_stream_status() reports
 *     them.
 *   - "dev" pointers are CUDA device pointers, "host" pointers are CPU memory.
 *     Device inputs are borrowed until the stream reaches the call.  Outputs
 *     written to device memory are valid after the stream is synchronised.
 *   - One ctx owns one scratch workspace: calls that compute (encode / score)
 *     must be issued on one stream at a time per ctx (or externally ordered).
 *   - Determinism: same inputs give bit-identical scores; no float atomics, no
 *     split-K.  Permuting candidates permutes scores bit-exactly.
 */
#ifndef CLIMBER_H_
#define CLIMBER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CLIMBER_ABI_VERSION 2  /* 2: climber_config.rel_bias, climber_weights.b_pos / b_time */

typedef enum {
  CLIMBER_OK = 0,
  CLIMBER_E_INVALID_ARG = 1,   /* NULL pointer, M < 1, M > max_candidates, B < 1, ... */
  CLIMBER_E_CONFIG = 2,        /* d % h, unequal budgets, tau <= 0 or non-finite, empty masks */
  CLIMBER_E_OUT_OF_RANGE = 3,  /* item/action/scenario id outside the vocabulary (device-detected) */
  CLIMBER_E_UNSORTED = 4,      /* decreasing timestamps in a lifecycle sequence (device-detected) */
  CLIMBER_E_CAPACITY = 5,      /* K/V page pool, handle table or arena exhausted */
  CLIMBER_E_STALE = 6,         /* handle released, from another ctx, or double release */
  CLIMBER_E_CUDA = 7,          /* a CUDA runtime call failed */
  CLIMBER_E_NCCL = 8,          /* a collective failed */
  CLIMBER_E_NUMERIC = 9,       /* non-finite score (checked when CLIMBER_SYNC_CHECK=1) */
  CLIMBER_E_UNSUPPORTED = 10   /* valid request this build does not implement */
} climber_status;

typedef enum { CLIMBER_BF16 = 0, CLIMBER_FP32 = 1 } climber_dtype;

/* Model + capacity configuration.  Budgets are equal by construction
 * (n_k = n / N_b), so a single n_k describes all blocks. */
typedef struct {
  int32_t abi_version;      /* must be CLIMBER_ABI_VERSION */
  int32_t d;                /* model width; d % n_heads == 0; d % 32 == 0 */
  int32_t n_heads;          /* h; d_h = d / h in {16, 32, 64} */
  int32_t n_layers;         /* L >= 1, ATLs per block */
  int32_t n_blocks;         /* N_b in [1, 8], one per extraction strategy */
  int32_t n_k;              /* per-block budget, multiple of 32, <= 1024 */
  int32_t ffn_mult;         /* F = ffn_mult * d (4, G8) */
  int32_t se_reduction;     /* squeeze-and-excitation reduction (4, G17) */
  int32_t vocab;            /* item vocabulary size V */
  int32_t n_actions;        /* action vocabulary (<= 64) */
  int32_t n_scenarios;      /* R (<= 64) */
  int32_t max_candidates;   /* max M per request */
  int32_t hist_causal;      /* 1: causal history attention (G1), 0: bidirectional */
  int32_t dtype;            /* climber_dtype: BF16 (tcgen05 path) or FP32 (verification build) */
  int32_t page_tokens;      /* K/V page size in tokens; must be 64 */
  float rms_eps;            /* RMSNorm epsilon (1e-6, G7) */
  int32_t max_batch_users;  /* max users per batched call */
  int32_t max_wave_users;   /* users encoded per internal wave (scratch sizing) */
  int32_t max_wave_pairs;   /* candidate pairs scored per internal wave (scratch sizing) */
  int64_t kv_pages;         /* K/V page-pool capacity in pages */
  int32_t rel_bias;         /* 0: f_b = 0 (the north-star formula, G6); 1: Eq. 3's relative
                             * attention bias f_b^{p,t}(a_k, r):
                             * R = QK^T + b_pos[bucket_p(i - j)] + b_time[bucket_t(t_i - t_j)],
                             * divided by sqrt(d_h) tau with the scores (G6b).  Position =
                             * index within S_k, a candidate sits at v_k; time = event
                             * timestamp, a candidate at the request time = the last
                             * event's timestamp (G6d, G6e).  BF16 needs d_h in {32, 64} and
                             * n_k % 128 == 0 (tcgen05 attention), else CLIMBER_E_CONFIG. */
} climber_config;

/* One extraction strategy a_k (Eq. 2): keep event e iff
 * (action_mask >> action[e]) & 1 and (scenario_mask >> scenario[e]) & 1. */
typedef struct {
  uint64_t action_mask;
  uint64_t scenario_mask;
} climber_strategy;

/* A lifecycle sequence S (Eq. 1), structure of arrays, chronological
 * (non-decreasing ts; ties keep input order).  DEVICE pointers. */
typedef struct {
  const int32_t* item;      /* [n_s] item ids in [0, vocab) */
  const uint8_t* action;    /* [n_s] action ids in [0, n_actions) */
  const uint8_t* scenario;  /* [n_s] scenario ids in [0, n_scenarios) */
  const int64_t* ts;        /* [n_s] timestamps, non-decreasing */
} climber_events;

/* Parameters: HOST fp32 arrays, row-major, matrices in [in][out] layout.
 * They are copied (and, for BF16, rounded RNE to bf16 and transposed to the
 * K-major layout the tensor cores read) into the arena at climber_create; the
 * caller may free them afterwards.  Shapes (F = ffn_mult d, D = N_b d,
 * Hs = D / se_reduction, QKV columns are [Q | K | V], heads contiguous d_h): */
typedef struct {
  const float* emb_item;  /* [vocab][d]        */
  const float* emb_act;   /* [n_actions][d]    */
  const float* emb_scn;   /* [n_scenarios][d]  */
  const float* g1;        /* [N_b][L][d]       pre-attention RMSNorm gain */
  const float* w_qkv;     /* [N_b][L][d][3d]   f_QKV */
  const float* w_o;       /* [N_b][L][d][d]    */
  const float* g2;        /* [N_b][L][d]       pre-FFN RMSNorm gain */
  const float* w1;        /* [N_b][L][d][F]    */
  const float* w2;        /* [N_b][L][F][d]    */
  const float* tau;       /* [L][N_b][R][h]    f_tc(a_k, r) per head, > 0 */
  const float* f_g1;      /* fusion ATL: [d]   */
  const float* f_w_qkv;   /* [d][3d] */
  const float* f_w_o;     /* [d][d]  */
  const float* f_g2;      /* [d]     */
  const float* f_w1;      /* [d][F]  */
  const float* f_w2;      /* [F][d]  */
  const float* tau_f;     /* [R][h]  */
  const float* w_se1;     /* [D][Hs] */
  const float* b_se1;     /* [Hs]    */
  const float* w_se2;     /* [Hs][D] */
  const float* b_se2;     /* [D]     */
  const float* w_head;    /* [D]     */
  float b_head;
  const float* b_pos;     /* [L][N_b][R][h][128] position-offset buckets (rel_bias = 1, else NULL):
                           * |i-j| < 16 -> |i-j|; else 16 + 4 (e - 4) + the 2 bits after the
                           * leading one of |i-j| (e = floor log2), capped at 63; +64 if i < j */
  const float* b_time;    /* [L][N_b][R][h][14] time-delta buckets in seconds {0, <1m, <1h, <1d,
                           * <1w, <30d, >=30d}; +7 if t_i < t_j (rel_bias = 1, else NULL) */
} climber_weights;

typedef struct climber_ctx_s* climber_ctx_t;
typedef struct climber_kv_s* climber_kv_t;   /* one user's multi-layer K/V cache */
typedef void* climber_stream_t;               /* a cudaStream_t (NULL = legacy default) */

/* Device bytes climber_create needs for this config (weights + K/V page pool +
 * handle tables + scratch).  Returns 0 for an invalid config. */
size_t climber_arena_bytes(const climber_config* cfg);

/* Create a context.  `arena` is a DEVICE buffer of >= climber_arena_bytes(cfg)
 * bytes, 256-byte aligned, borrowed for the ctx's lifetime (e.g. a torch
 * tensor).  `strategies` is a host array of n_blocks entries.  Multi-GPU:
 * world > 1 needs `nccl_uid` (128 bytes from climber_nccl_unique_id on one
 * rank); every rank then calls climber_create concurrently (collective) and
 * the ctx holds an NCCL communicator for climber_kv_broadcast.  With world ==
 * 1, nccl_uid may be NULL (no communicator).  Synchronous. */
climber_status climber_create(const climber_config* cfg, const climber_strategy* strategies,
                              const climber_weights* weights, void* arena, size_t arena_bytes,
                              int32_t rank, int32_t world, const void* nccl_uid,
                              climber_ctx_t* out);

/* Destroy: synchronises the device, releases host state; the arena is the
 * caller's to free afterwards.  Outstanding handles become invalid. */
climber_status climber_destroy(climber_ctx_t ctx);

/* Encode one user (PAPER.md L257 step 1): validate and extract (Eq. 2), embed,
 * run the N_b block stacks over the history and write every layer's K and V
 * (bf16 or fp32 per dtype) into pages of the ctx pool.  `events` holds DEVICE
 * pointers to n_s >= 0 events; `scenario_r` is the request scenario r (G4).
 * The handle is returned synchronously; its contents are valid in stream order. */
climber_status climber_encode_user(climber_ctx_t ctx, const climber_events* events, int64_t n_s,
                                   int32_t scenario_r, climber_stream_t stream, climber_kv_t* out);

/* Batched encode of B users.  ev_offsets: HOST int64[B+1], user b's events are
 * [ev_offsets[b], ev_offsets[b+1]) of the DEVICE arrays in `events`.
 * scenario_r: HOST int32[B].  out: HOST array of B handles. */
climber_status climber_encode_users(climber_ctx_t ctx, int32_t B, const int64_t* ev_offsets,
                                    const climber_events* events, const int32_t* scenario_r,
                                    climber_stream_t stream, climber_kv_t* out);

/* Score M candidates of one user against its cache (PAPER.md L255, L257 step
 * 3).  items: DEVICE int32[M], 1 <= M <= max_candidates; scores: DEVICE
 * float[M], logits in candidate order. */
climber_status climber_score_items(climber_ctx_t ctx, climber_kv_t kv, const int32_t* items,
                                   int32_t M, float* scores, climber_stream_t stream);

/* Batched scoring: user b's candidates are items[cand_offsets[b] ..
 * cand_offsets[b+1]) (cand_offsets: HOST int64[B+1], each count in
 * [1, max_candidates]); scores are written at the same positions. */
climber_status climber_score_items_batched(climber_ctx_t ctx, int32_t B, const climber_kv_t* kvs,
                                           const int64_t* cand_offsets, const int32_t* items,
                                           float* scores, climber_stream_t stream);

/* SUMI forward of compressed training records (SURVEY
 * §8(f) NEXT-3): each user's "single user, multiple items" record — the
 * history plus its items, causal history, items full-visible to the history
 * and isolated from each other (diagonal) — is scored in one call without
 * keeping a cache (encode + score with transient handles, released when the
 * call returns).  Layouts as climber_encode_users + climber_score_items_batched
 * (DEVICE events / items / scores, HOST offsets and scenarios).  The pages
 * return to the pool on return: a later call on the SAME stream is ordered
 * after this one; on another stream, synchronise first.  Backward is out of
 * scope. */
climber_status climber_forward(climber_ctx_t ctx, int32_t B, const int64_t* ev_offsets,
                               const climber_events* events, const int32_t* scenario_r,
                               const int64_t* cand_offsets, const int32_t* items, float* scores,
                               climber_stream_t stream);

/* End-to-end convenience call with HOST buffers: copies the events and the
 * candidates to the device, encodes, scores, copies the scores back to
 * `scores` (HOST float[cand_offsets[B]]), releases the handles and
 * synchronises `stream`.  Same layouts as the batched calls, host memory. */
climber_status climber_rank_host(climber_ctx_t ctx, int32_t B, const int64_t* ev_offsets,
                                 const int32_t* item, const uint8_t* action, const uint8_t* scenario,
                                 const int64_t* ts, const int32_t* scenario_r,
                                 const int64_t* cand_offsets, const int32_t* items, float* scores,
                                 climber_stream_t stream);

/* ---- Block-parallel serving (PAPER.md L155
 * "block-parallel KV cache", L203: the N_b blocks are independent until the
 * fusion step).  G processes each own a block range [k0, k1) (G divides N_b):
 * each encodes and scores only its blocks, the block outputs E(S_k) (the
 * candidate rows after the last layer, G13) are exchanged with one
 * all-gather, and one process fuses (BGF + head).  Every block runs the same
 * kernels as the single-GPU path, and the fusion input is rebuilt in the
 * same summation order, so the scores are bit-identical to climber_score_items.
 * These calls need the bf16 grouped tcgen05 path (d_h in {32, 64}, n_k %
 * 128 == 0), else CLIMBER_E_UNSUPPORTED. */

/* climber_encode_users restricted to blocks [k0, k1): extraction, embedding
 * and the layer stacks of those blocks only; the handle holds their K/V and
 * can only be scored on a sub-range (else CLIMBER_E_INVALID_ARG). */
climber_status climber_encode_users_blocks(climber_ctx_t ctx, int32_t B, const int64_t* ev_offsets,
                                           const climber_events* events, const int32_t* scenario_r,
                                           int32_t k0, int32_t k1, climber_stream_t stream,
                                           climber_kv_t* out);

/* The candidate stacks of blocks [k0, k1) (layouts as climber_score_items_batched):
 * E is a DEVICE float [P][k1 - k0][d] (P = cand_offsets[B] - cand_offsets[0]),
 * E[p][k - k0] = block k's output row of pair p. */
climber_status climber_score_blocks(climber_ctx_t ctx, int32_t B, const climber_kv_t* kvs,
                                    const int64_t* cand_offsets, const int32_t* items, int32_t k0, int32_t k1,
                                    float* E, climber_stream_t stream);

/* BGF (Eq. 4) + squeeze-and-excitation gate + head from gathered block outputs.
 * E: DEVICE float [n_slices][P][N_b / n_slices][d] (slice g = blocks
 * [g N_b / n_slices, (g + 1) N_b / n_slices), i.e. the rank-major result of an
 * all-gather of climber_score_blocks outputs); scenario_r: HOST int32[B] (the
 * request scenarios, G4); cand_offsets: HOST int64[B + 1]; scores: DEVICE
 * float[P].  No handle is needed. */
climber_status climber_fuse_scores(climber_ctx_t ctx, int32_t B, const int64_t* cand_offsets,
                                   const int32_t* scenario_r, int32_t n_slices, const float* E, float* scores,
                                   climber_stream_t stream);

/* Return a handle's pages to the pool.  The caller must ensure no enqueued
 * work still reads it.  Double release -> CLIMBER_E_STALE. */
climber_status climber_kv_release(climber_ctx_t ctx, climber_kv_t kv);

/* ---- serving cache store ("concurrent
 * readers, atomic cache build"; PAPER.md L161 on static caches) ----
 * Handles keyed by (user_key, scenario r) with the caller's digest of the
 * event log (e.g. a hash of ids + timestamps; "digest mismatch ->
 * staleness").  An entry is pinned while any caller holds it; unpinned
 * entries are evicted least-recently-used when an encode needs pages.  The
 * store owns its handles: never climber_kv_release one; call
 * climber_cache_release to unpin.  Thread-safe (one mutex; a miss encodes
 * under it, so concurrent acquires of one key build the cache once). */
typedef enum {
  CLIMBER_CACHE_HIT = 0,        /* same key, same digest: the cached K/V is returned */
  CLIMBER_CACHE_ENCODED = 1,    /* miss or stale digest: encoded now and cached */
  CLIMBER_CACHE_UNCACHED = 2,   /* stale, but the old entry is pinned by another caller:
                                 * encoded now, returned pinned, dropped on release */
  CLIMBER_CACHE_APPENDED = 3    /* incremental update in place (climber_cache_append) */
} climber_cache_result;

/* Pin (and build if needed) the cache of one user.  events: DEVICE arrays of
 * n_s events (as climber_encode_user); result: HOST out, climber_cache_result.
 * CLIMBER_E_CAPACITY when every page is held by pinned entries. */
climber_status climber_cache_acquire(climber_ctx_t ctx, uint64_t user_key, int32_t scenario_r, uint64_t digest,
                                     const climber_events* events, int64_t n_s, climber_stream_t stream,
                                     climber_kv_t* out, int32_t* result);

/* Incremental update after the user's event log grew by appending
 * (static caches go stale; NEXT-4).  If the cached entry's
 * digest is `digest_prefix` (the caller's digest of the first events, i.e. the
 * old log) and it is not pinned, only the blocks whose strategy a_k matches
 * an appended event are recomputed in place (S_k of the others is unchanged,
 * Eq. 2), extraction and the request-time bias rows are redone, and the entry
 * takes `digest`; result = CLIMBER_CACHE_APPENDED, *blocks_recomputed = how
 * many of the N_b stacks ran.  Otherwise it behaves as climber_cache_acquire
 * with `digest` (*blocks_recomputed = N_b).  Scores from the updated handle
 * are bit-identical to a full encode of the new log.  Synchronises `stream`
 * once (to read which blocks changed). */
climber_status climber_cache_append(climber_ctx_t ctx, uint64_t user_key, int32_t scenario_r,
                                    uint64_t digest_prefix, uint64_t digest, const climber_events* events,
                                    int64_t n_s, climber_stream_t stream, climber_kv_t* out, int32_t* result,
                                    int32_t* blocks_recomputed);

/* Unpin a handle returned by climber_cache_acquire / climber_cache_append. */
climber_status climber_cache_release(climber_ctx_t ctx, climber_kv_t kv);

/* Entries, pinned entries, hits, misses and evictions so far (HOST int64[5]). */
climber_status climber_cache_stats(climber_ctx_t ctx, int64_t* stats);

/* ---- multi-GPU candidate sharding (latency mode) ----
 * The owner rank encodes the user, exports the handle's K/V pages into one
 * contiguous DEVICE slab, the slab is replicated with a collective of the
 * caller's process group (e.g. an NCCL broadcast over NVLink), and every other
 * rank imports it into its own page pool; each rank then scores its shard of
 * the candidates.  Slab layout: 256-byte header (int32 magic, slab version 2,
 * n_blocks, n_layers, pages per block, d, dtype, scenario r, vlen[n_blocks]
 * at int 8.., rel_bias flag at int 16) followed by the handle's pages in
 * page-table order ([2][64][d] elements each) and, for rel_bias contexts, the
 * handle's relative-bias state (token ages int32 [n_blocks][n_k], candidate-
 * row bias fp32 [n_layers][n_blocks][n_heads][n_k]).  The slab is only
 * meaningful to a ctx created with the same config. */

/* Bytes of one user's slab for this ctx's config. */
size_t climber_kv_slab_bytes(climber_ctx_t ctx);

/* Gather the handle's pages into `slab` (DEVICE, 16-byte aligned, >=
 * climber_kv_slab_bytes).  Asynchronous on `stream`.  E_INVALID_ARG for a
 * handle that holds only a block range (climber_encode_users_blocks), E_STALE
 * for a released or foreign handle. */
climber_status climber_kv_export(climber_ctx_t ctx, climber_kv_t kv, void* slab, climber_stream_t stream);

/* Allocate a handle in this ctx's pool and scatter the slab's pages into it.
 * `scenario_r` is the request scenario the slab was encoded with (host
 * state of the handle).  Asynchronous on `stream`; a slab whose header does not
 * match this ctx's config sets the device error word (E_CONFIG is returned by
 * climber_stream_status) and leaves the handle's scores NaN-free but invalid. */
climber_status climber_kv_import(climber_ctx_t ctx, const void* slab, int32_t scenario_r,
                                 climber_stream_t stream, climber_kv_t* out);

/* In-library NCCL replication of one user's K/V: collective
 * over the ctx's communicator (climber_create with world > 1 and an NCCL
 * unique id).  On `root`, *kv is the handle to replicate (unchanged); on every
 * other rank a new handle with identical pages is allocated in its pool and
 * returned in *kv.  Root exports the pages into one slab, one ncclBroadcast
 * (NVLink / NVSwitch) replicates it, the receivers import it; receivers
 * synchronise `stream` once (to read the handle's scenario from the slab
 * header).  A world-1 ctx without a communicator returns OK unchanged.
 * Every rank joins the broadcast even when the root's export fails (stale
 * handle, block-range handle): the root then sends an invalid header and
 * returns the export's error, every receiver returns E_STALE and allocates
 * nothing.  Receivers wait with a deadline (env CLIMBER_NCCL_TIMEOUT_MS,
 * default 120000); on timeout or an asynchronous NCCL error the communicator
 * is aborted (ncclCommAbort) and E_NCCL returned; later broadcasts on the
 * ctx return E_UNSUPPORTED. */
climber_status climber_kv_broadcast(climber_ctx_t ctx, climber_kv_t* kv, int32_t root,
                                    climber_stream_t stream);

/* Encode one user on `root` and replicate its K/V to every rank WHILE it is
 * being encoded ("pipelined per layer, overlapping encode of
 * layer l+1 with the broadcast of layer l").  Collective over the
 * ctx's communicator: every rank passes the same scenario_r and root; events /
 * n_s are read on root only (others may pass NULL / 0).  The root encodes as
 * climber_encode_user and, on a side stream, posts L + 1 ncclBroadcasts of
 * one slab: the header section (v_k, r, relative-bias state) as soon as
 * extraction is done, then layer l's pages of every block as soon as layer
 * l's QKV GEMM has written them; the receivers post the same broadcasts on
 * `stream` and unpack each section into their own pages right behind it.
 * Nothing synchronises the host.  On return every rank holds a handle in *out
 * (root: the encoded one); all work is ordered on `stream`.
 * Errors: E_INVALID_ARG / E_OUT_OF_RANGE (arguments, checked alike on every
 * rank), E_UNSUPPORTED (no communicator, or not the grouped bf16 tcgen05
 * path), E_CAPACITY (this rank's pool is full: it still posts its broadcasts,
 * so the others do not hang, and returns the error), root-side encode errors
 * (the root then sends a zeroed header: receivers get E_CONFIG from
 * climber_stream_status), E_NCCL (the communicator is aborted). */
climber_status climber_encode_user_bcast(climber_ctx_t ctx, const climber_events* events, int64_t n_s,
                                         int32_t scenario_r, int32_t root, climber_stream_t stream,
                                         climber_kv_t* out);

/* An NCCL unique id (128 bytes into `out`) for climber_create's nccl_uid:
 * rank 0 calls it and shares the bytes with the other ranks. */
climber_status climber_nccl_unique_id(void* out);

/* Synchronise `stream` and report the first device-side error recorded since
 * the last call (then clear it): OK, E_OUT_OF_RANGE, E_UNSORTED, E_CUDA. */
climber_status climber_stream_status(climber_ctx_t ctx, climber_stream_t stream);

/* Thread-local description of the last failure on this thread ("" if none). */
const char* climber_last_error(void);

/* ---- debug exports (synchronous; for bit-exact parity tests) ---- */

/* Canonical extraction result (G12): idx HOST int32[N_b][n_k], event indices
 * relative to the user's first event, left-padded with -1; vlen HOST int32[N_b]. */
climber_status climber_debug_extract(climber_ctx_t ctx, climber_kv_t kv, int32_t* idx, int32_t* vlen);

/* Canonical SUMI masks for M candidates, evaluated on the device from the
 * written-out visibility rule (common.cuh sumi_visible): HOST
 * uint8[N_b][(n_k+M)^2], row-major, history slots left-padded, 1 = attend
 * (SURVEY §8(c), D8).  This is the rule, not the attention kernels: what the
 * kernels actually attend is recovered by climber_debug_attn_probe. */
climber_status climber_debug_mask(climber_ctx_t ctx, climber_kv_t kv, int32_t M, uint8_t* mask);

/* Mask probe of the production attention kernels ("full-visible masks
 * between each candidate item and the entire history ... diagonal masks for
 * inter-item isolation"; G1 causal / bidirectional history; G14 self).
 * Runs the same attention kernel the encode (mode 0: history rows of layer
 * `layer`) or the score (mode 1: M candidate rows) launches for `block` of
 * handle kv, on a probe input: q = k = 0 (so every visible key gets weight
 * 1 / |visible set|) and V[j] one-hot: for head h, key j = key_off + h (d_h - 1)
 * + c (0 <= c < d_h - 1) is channel c; SUMI rows get v_self = channel d_h - 1.
 * out: HOST float [rows][d] (rows = n_k for mode 0, internal right-padded slot
 * order: slot i = i-th kept event; M for mode 1), out[row][h d_h + c] != 0 iff
 * that key (c < d_h - 1) or the self term (c = d_h - 1) is attended.  Pad rows
 * (slot >= v_k) read 0.  Covers keys [key_off, key_off + h (d_h - 1)) per call.
 * DEBUG ONLY, synchronous, not concurrent with other calls on the ctx: it
 * OVERWRITES the handle's K/V pages of (layer, block) -- release the handle
 * afterwards.  Errors: E_INVALID_ARG (mode, layer, block outside the handle's
 * blocks, M outside [1, max_candidates]), E_UNSUPPORTED (rel_bias contexts),
 * E_STALE, E_CUDA. */
climber_status climber_debug_attn_probe(climber_ctx_t ctx, climber_kv_t kv, int32_t mode, int32_t layer,
                                        int32_t block, int32_t M, int32_t key_off, float* out);

/* One layer/block of the cache, gathered from its pages in canonical order:
 * K, V HOST arrays [vlen][d] of float (dtype FP32) or uint16 bf16 bits (BF16);
 * rows = vlen[block] of the most recent extraction. */
climber_status climber_debug_kv(climber_ctx_t ctx, climber_kv_t kv, int32_t layer, int32_t block,
                                void* K, void* V);

/* The bf16 tensor-core GEMM of the path in isolation, C = sum_k A[m][k] B[n][k]
 * (fp32 accumulate) with one of the path's epilogues:
 *   epi 0: D float [M][N]  += C        (residual add)
 *   epi 1: D bf16  [M][N]   = C        (plain store)
 *   epi 2: D bf16  [M][N]   = SiLU(C)  (FFN up)
 * DEVICE pointers: A bf16 [M][K], B bf16 [N][K]; K % 64 == 0, N % 128 == 0
 * (else E_UNSUPPORTED).  use_tc = 0 runs the SIMT kernel.  Asynchronous. */
climber_status climber_debug_gemm(const void* A, const void* B, void* D, int64_t M, int32_t N, int32_t K,
                                  int32_t use_tc, int32_t epi, climber_stream_t stream);

/* ---- measurement (bench evidence) ---- */

/* Kernel classes timed by the profiler. */
typedef enum {
  CLIMBER_K_EXTRACT = 0, CLIMBER_K_EMBED = 1, CLIMBER_K_RMSNORM = 2, CLIMBER_K_GEMM_QKV = 3,
  CLIMBER_K_GEMM_O = 4, CLIMBER_K_GEMM_FFN_UP = 5, CLIMBER_K_GEMM_FFN_DOWN = 6, CLIMBER_K_GEMM_SE = 7,
  CLIMBER_K_ATTN_HIST = 8, CLIMBER_K_ATTN_SUMI = 9, CLIMBER_K_ATTN_FUSION = 10, CLIMBER_K_HEAD = 11,
  CLIMBER_K_OTHER = 12, CLIMBER_K_NUM = 13
} climber_kernel_class;

/* enable != 0: every subsequent launch is bracketed by CUDA events recorded on
 * its own stream, accumulated per kernel class.  enable == 0 stops. */
climber_status climber_profile(climber_ctx_t ctx, int32_t enable);

/* Synchronise, then for each class c write out[4*c + 0..3] = {launches,
 * total device ms, algorithmic FLOPs, algorithmic HBM bytes} accumulated since
 * the previous read, and reset.  out: HOST double[4 * CLIMBER_K_NUM].
 * FLOPs/bytes are what the operation must compute/move (GEMM 2MNK; attention
 * 4 * pairs * d with every history row valid; memory-bound kernels one read of
 * each input and one write of each output). */
climber_status climber_profile_read(climber_ctx_t ctx, double* out);

/* Number of kernel launches the library has enqueued since the ctx was
 * created (bench evidence for "gpu_launches"). */
int64_t climber_launch_count(climber_ctx_t ctx);

#ifdef __cplusplus
}
#endif
#endif /* CLIMBER_H_ */
