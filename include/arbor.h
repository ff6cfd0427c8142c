/*
 * arbor.h — C ABI of libarbor.so, the B200-native ArborKV per-step KV-eviction
 * path (arXiv 2605.22106, "ArborKV: Structure-Aware KV Cache Management for
 * Scaling Tree-based LLM Reasoning").  Citations: P:<n> = line n of the
 * paper's PAPER.md; Q<n> = a reading of the paper listed in DESIGN.md.
 *
 * Plain C: no C++ types, no exceptions cross this boundary, no torch types.
 * Pointers are either HOST (plain process memory) or DEVICE (CUDA global
 * memory on the context's device); every argument says which.
 *
 * Conventions (apply to every call):
 *  - Every call returns an arbor_status.  Arguments are validated on the host
 *    before anything is enqueued or mutated; a call that returns an error
 *    leaves library state unchanged (validate-then-mutate).  Errors detected
 *    by a kernel (e.g. a NaN score, ARBOR_ERR_INVARIANT) are latched on the
 *    device and returned by the next arbor_sync() or blocking call.
 *  - Calls are asynchronous on config.main_stream unless they have a host
 *    out-parameter (then they synchronise main_stream before returning).
 *    Stash copies run on config.side_stream; the library inserts the event
 *    dependencies between the two streams.
 *  - A context is single-threaded (one host thread at a time).
 *  - Node ids are global, dense and in creation order (parent id < child id).
 *    Token positions are absolute in one global stream (span_start = a_i).
 *  - Sharding: pools, Q, O and the score array hold only this rank's
 *    (layer, KV-head) shard; trees, budgets and node arrays are global and
 *    must be identical on every rank.  arbor_score all-reduces the per-node
 *    attention mass across ranks (one NCCL int64 all-reduce), so every rank
 *    derives bit-identical budgets and page tables.
 */
#ifndef ARBOR_H_
#define ARBOR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ARBOR_OK = 0,
  ARBOR_ERR_INVALID_ARG = 2,       /* bad config / params / tree / argument          */
  ARBOR_ERR_INFEASIBLE_BUDGET = 3, /* Σ_pinned n + Σ floors > budget (Q12)     */
  ARBOR_ERR_INVARIANT = 4,         /* NaN / negative accumulated attention, overflow  */
  ARBOR_ERR_IO = 5,                /* pinned host stash allocation failure            */
  ARBOR_ERR_OUT_OF_PAGES = 6,      /* the page pool cannot hold the request          */
  ARBOR_ERR_STATE = 7,             /* lifecycle: append to closed, close twice, ...   */
  ARBOR_ERR_CUDA = 8,              /* a CUDA runtime / launch error                   */
  ARBOR_ERR_NCCL = 9               /* an NCCL error (world_size > 1)                  */
} arbor_status;

typedef enum { ARBOR_F32 = 0, ARBOR_BF16 = 1 } arbor_dtype;

/* Allocation mode of arbor_allocate (Alg. 2). */
typedef enum {
  ARBOR_ALLOC_WATERFILL = 0,    /* budget-exact optimisation view with floors (default) */
  ARBOR_ALLOC_STATIC = 1,       /* Eqs. 2-3 directly, no budget guarantee                */
  ARBOR_ALLOC_STATIC_DRAIN = 2, /* Eqs. 2-3, then Alg. 2's Pressure drain to the budget  */
  /* f4 — the sequence-flattened StreamingLLM analogue: the single
   * active path root → ℓ is one token stream keeping its global sinks (the root's first
   * n_sinks tokens) and its most recent 𝓑 − Σ_open n − |sinks| tokens; off-path blocks get
   * k = 0; open blocks stay pinned.  Requires num_active = 1, l_tail = 0 and select_mode
   * SINKS_TAIL (the per-block selection is then exactly "sinks + the most recent k");
   * pair with no_rehydrate = 1 for the baseline's irreversible eviction. */
  ARBOR_ALLOC_STREAM = 3
} arbor_alloc_mode;

/* config.flags */
#define ARBOR_FLAG_PROFILE 1u   /* record CUDA events around every kernel (arbor_stage_times) */
/* world_size > 1 without the library's NCCL communicator: arbor_score / arbor_decode_step stop
 * after the partial node masses (a10's input, arbor_mass_buffer); the caller sums that int64
 * buffer across the ranks with its own collective (e.g. torch.distributed all_reduce, or —
 * KV-head shards on one device — a plain device sum) and calls arbor_score_finish, which runs
 * the MSVE on the reduced masses.  nccl_unique_id is then ignored. */
#define ARBOR_FLAG_EXTERNAL_REDUCE 2u
/* The library's NCCL path (a10) at any world size, including 1 (a one-rank communicator):
 * arbor_score / arbor_decode_step take the multi-rank finisher — partial node masses →
 * ncclAllReduce(int64, sum) on main_stream → the MSVE kernel — instead of the single-rank
 * fused MSVE.  Integer sums are order-free, so every result equals the single-rank path's bit
 * for bit; it lets one GPU execute the collective path (dlopen, ncclCommInitRank,
 * ncclAllReduce).  Needs nccl_unique_id; incompatible with ARBOR_FLAG_EXTERNAL_REDUCE. */
#define ARBOR_FLAG_COLLECTIVE 4u

/* Parameter bundle Π (Alg. 1 caption P:498, Alg. 2).  Host struct. */
typedef struct {
  double alpha;         /* α  > 0  global scale of Eq. 2                        */
  double gamma;         /* γ  ≥ 0  importance exponent (integer → exact powers)  */
  double lambda_d;      /* λ_d     depth decay (any sign)                        */
  double lambda_delta;  /* λ_Δ     distance-to-active-leaf decay                  */
  double eta;           /* η ∈ (0,1] off-path discount                            */
  double r_min;         /* r_min ∈ [0,1] ratio floor                              */
  int32_t k_min;        /* K_min ≥ 0 count floor (invariant (ii))          */
  int32_t l_tail;       /* L_tail ≥ 0 block tail always kept          */
  int32_t n_sinks;      /* global sinks: first n_sinks positions of the root     */
  int32_t alloc_mode;   /* arbor_alloc_mode                                       */
  double theta[4];      /* MSVE θ = (θ0 bias, θ_v, θ_u, θ_a) (Q7)     */
  /* f4 policy variants (0 = the paper's full method):            */
  int32_t select_mode;  /* arbor_select_mode: intra-block retention rule              */
  int32_t no_rehydrate; /* 1: evicted tokens never come back (P:423-428 ablation):
                         * arbor_rehydrate and Transition's rehydration are no-ops      */
  int32_t k_protect;    /* invariant (i) "k_i = n_i or a high floor k_protect":
                         * 0 (default): closed Path* blocks are pinned at k = n (Q19);
                         * > 0: they are allocated like every other block, with the floor
                         * raised to min(n, k_protect), and may be evicted down to it; the
                         * global sinks (first n_sinks positions of the root) are then kept
                         * by arbor_evict explicitly (Q22).  Open blocks stay pinned.       */
  /* Thin slice 𝓛 × 𝓗 ("aggregated over a thin slice of heads/layers"): the
   * last slice_layers layers and the first slice_kv_heads KV heads of the model (global
   * indices; 0 = all).  a_i then counts the slice rows' mass only, normalised by
   * |𝓛|·|𝓗_q| (Q4, Q6).                                                                */
  int32_t slice_layers, slice_kv_heads;
  /* 1: the paper-literal shared selection (Q1): arbor_evict ranks every block
   * once, by Â(t) = Σ_{(l,h) ∈ slice} A[l][h][t] (f32 values summed in fp64 in ascending
   * row order, rounded to f32), and every row keeps the same positions.  world_size 1. */
  int32_t select_shared;
} arbor_params;

/* Intra-block retention rule of arbor_evict (P:660-675 ablation).  The block tail
 * (L_tail) is always kept; the remaining k − |tail| slots go to the currently kept
 * non-tail positions ranked by:
 *  HEAVY      ⟨A, position⟩ descending — heavy hitters (the method);
 *  TAIL       position descending — recency only ("Tail-only");
 *  SINKS_TAIL position descending, with the global sinks first ("Sinks + Tail").
 * Global sinks 𝒮 = the first n_sinks positions of the root block (the
 * initial prompt): HEAVY and SINKS_TAIL rank them above every other candidate of the root
 * (after the tail); TAIL keeps none.  They matter only when the root can be evicted
 * (params.k_protect > 0): in the default policy the root is on Path* and pinned. */
typedef enum { ARBOR_SELECT_HEAVY = 0, ARBOR_SELECT_TAIL = 1, ARBOR_SELECT_SINKS_TAIL = 2 } arbor_select_mode;

/* Context configuration.  Host struct; device buffers are caller-owned and
 * borrowed for the lifetime of the context. */
typedef struct {
  int32_t num_layers, num_kv_heads, num_q_heads, head_dim;          /* global model shape   */
  int32_t layer_begin, layer_count, kv_head_begin, kv_head_count;   /* this rank's shard    */
  int32_t kv_dtype;        /* arbor_dtype of K/V/Q/O                                        */
  int32_t page_size;       /* P tokens per page: a power of two in 2..1024                   */
  int32_t num_pages;       /* pages in each pool                                             */
  int32_t max_nodes;       /* capacity of the node table, 1..3072 (a4 runs in one CTA's smem) */
  int32_t max_node_tokens; /* capacity of one node (≤ 32767; pos tags are int16)            */
  int32_t max_active;      /* capacity of active leaves per call                             */
  int64_t max_tokens;      /* capacity of the absolute position stream                      */
  /* DEVICE, caller-owned, [layer_count][num_pages][kv_head_count][page_size][head_dim]     */
  void *k_pool, *v_pool;
  /* DEVICE, caller-owned, [layer_count][num_pages][kv_head_count][page_size] int16:
   * within-node offset (t − a_i) of the token held by each slot                          */
  int16_t *pos_pool;
  /* DEVICE, caller-owned, zero-initialised, [layer_count][kv_head_count][max_tokens] f32:
   * accumulated attention A[l][h][t], dense by absolute position            */
  float *score;
  /* HOST pinned stash (write-through copy of closed nodes, Q20), caller-owned, or NULL to
   * let the library cudaHostAlloc it: 2 * layer_count * kv_head_count * max_tokens *
   * head_dim * sizeof(dtype) bytes, layout [2][layer_count][kv_head_count][max_tokens][d] */
  void *host_stash; size_t host_stash_bytes;
  int32_t rank, world_size;
  /* HOST, 128 bytes from arbor_nccl_unique_id() on rank 0 (ignored when world_size == 1) */
  const void *nccl_unique_id;
  /* cudaStream_t: main_stream is used as given (NULL = the legacy default stream); a NULL
   * side_stream makes the library create a non-blocking one                                */
  void *main_stream, *side_stream;
  uint32_t flags;                    /* ARBOR_FLAG_*                                        */
} arbor_config;

/* Tree snapshot.  HOST arrays, caller-owned, read during the call only. */
typedef struct {
  int32_t num_nodes;
  const int32_t *parent;        /* -1 for the root (node 0); parent < child               */
  const int64_t *span_start;    /* a_i                                                     */
  const int32_t *span_len;      /* n_i (current length for open nodes)                     */
  const uint8_t *is_open;       /* 1 while the block is still being generated             */
  const float *search_value;    /* v_i ∈ [0,1]                                      */
  const float *uncertainty;     /* u_i ∈ [0,1] (Eq. 1)                           */
  int32_t num_active;           /* ≥ 1                                                      */
  const int32_t *active;        /* active leaves ℓ* (several = DPTS frontier, Q14)  */
} arbor_tree;

typedef struct arbor_ctx arbor_ctx;

/* ---- lifecycle ---------------------------------------------------------------------- */
/* Create a context: validates config/params, allocates library-owned device state (page
 * tables, LIFO free list [num_pages-1 … 0], counters), host tables e^{-λ x} (Q9), and the
 * NCCL communicator when world_size > 1.  *out is NULL on error. */
arbor_status arbor_init(const arbor_config *cfg, const arbor_params *params, arbor_ctx **out);
void arbor_destroy(arbor_ctx *ctx);
const char *arbor_last_error(const arbor_ctx *ctx);     /* message of the last failure   */
const char *arbor_status_string(arbor_status s);
/* Rank 0 fills 128 HOST bytes; broadcast them to every rank before arbor_init. */
arbor_status arbor_nccl_unique_id(void *out128);

/* ---- node plumbing (not hot-path steps) -------------------------------------------- */
/* Register node `node` (must equal the number of known nodes) as an open block starting
 * at absolute position span_start.  Spans of all nodes must stay disjoint: opening
 * inside another span, or appending into the next node's start, is ARBOR_ERR_INVALID_ARG
 * (concurrently decoded siblings need reserved position ranges). */
arbor_status arbor_open_node(arbor_ctx *ctx, int32_t node, int64_t span_start);
/* Append ntok decoded tokens to an open node.  k, v: DEVICE [layer_count][kv_head_count]
 * [ntok][head_dim] in kv_dtype.  Pages are popped from the free list in token order, on the
 * device and asynchronously: when the pool runs out the append is skipped on the device and
 * ARBOR_ERR_OUT_OF_PAGES latches there; it is returned by the next call that syncs
 * (arbor_sync, the inspection calls, an evict with evicted_tokens_out).  Until then the
 * host's view of n (used to plan attention) is ahead of the device's: call arbor_sync after
 * appends when the pool can run dry. */
arbor_status arbor_append_kv(arbor_ctx *ctx, int32_t node, const void *k, const void *v,
                             int32_t ntok);
/* Boundary: close an open node (n_i ≥ 1), snapshot its post-close mass baseline
 * Mclose_i (Q5), reset Nq_i, and enqueue the write-through stash of its full K/V on
 * side_stream (Q20). */
arbor_status arbor_close_node(arbor_ctx *ctx, int32_t node);

/* ---- the six hot-path calls ---------------------------------------------------------- */

/* a2+a3+a10 — MSVE scoring.  For every active leaf b (index into
 * tree->active), layer l and query head g: p_t = exp(q·k_t/√d − LSE_{b,l,g}) over the
 * visible slots of Path(ℓ_b); A[l][h][a_j + pos] += Σ_g p_t; Nq_i += 1 for closed i on
 * Path(ℓ_b).  Then per closed node: Mass_i = Σ_rows round(2^24 Σ_{t∈span} A) (int64,
 * all-reduced across ranks), a_i = clamp((Mass_i − Mclose_i) 2^-24 / (Nq_i L Hq), 0, 1),
 * s_i = σ(θ0 + θ_v v_i + θ_u u_i + θ_a a_i).
 *  q:     DEVICE [num_active][layer_count][Hq_local][head_dim] kv_dtype
 *  lse:   DEVICE [num_active][layer_count][Hq_local] f32 from arbor_tree_decode_attn with the
 *         same q, or NULL (the library then computes it first).  When this call directly
 *         follows a full-range arbor_tree_decode_attn with the same q and lse buffers (and
 *         no KV-changing call in between), the logits that call produced are reused (fused
 *         a2, no K re-read); the caller must not modify q in between.
 *  s_out: DEVICE [num_nodes] f32, or NULL; open / never-scored nodes get 0.5 (Q31).
 *         The library also keeps the scores internally for arbor_allocate(s = NULL). */
arbor_status arbor_score(arbor_ctx *ctx, const arbor_tree *tree, const void *q,
                         const float *lse, float *s_out);

/* a1+a4 — tree geometry and TAE allocation (Alg. 2).
 * Pinned (Path* ∪ open) nodes get k = n; others per params.alloc_mode.  WATERFILL returns
 * Σ k = budget exactly whenever Σ n > budget (else k = n).
 *  s:     DEVICE [num_nodes] f32 scores, or NULL for the library's last scores
 *  k_out: DEVICE [num_nodes] int32 target keep counts
 *  min_feasible_out: HOST, optional; set to the smallest feasible budget when the call
 *         returns ARBOR_ERR_INFEASIBLE_BUDGET (nothing is enqueued then). */
arbor_status arbor_allocate(arbor_ctx *ctx, const arbor_tree *tree, const float *s,
                            int64_t budget_tokens, int32_t *k_out, int64_t *min_feasible_out);

/* a5+a6 — token-extractive eviction (Alg. 1, Alg. 2).
 * For every non-pinned closed node j with k_app = min(k_cur_j, max(0, k_target_j)) <
 * k_cur_j, and every row (l, h): keep the last min(L_tail, n_j) positions, plus the top
 * (k_app − tail) currently kept positions by the key ⟨f32 A, position⟩ (descending, Q3);
 * if k_app ≤ tail keep the last k_app.  Kept K/V/pos rows are compacted in place into
 * the LAST k_app of the node's k_cur valid slots (end-window hole filling, Q23*:
 * the always-kept tail already sits there): kept rows inside the window stay, the i-th
 * dropped slot of the window (ascending) receives the i-th kept row from before it
 * (ascending); every slot carries its position tag.  The window starts at page-list slot
 * c = first_slot + k_cur − k_app: the ⌊c/P⌋ leading pages are freed (all of them when
 * k_app = 0) and first_slot becomes c mod P (see arbor_read_node_offset); freed pages are
 * pushed on the LIFO free list nodes ascending, each node's run in descending list order.
 * Pinned nodes are untouched.
 *  k_target: DEVICE [num_nodes] int32 (e.g. arbor_allocate's k_out)
 *  evicted_tokens_out: HOST, optional (forces a sync): Σ_j (k_cur_j − k_app_j). */
arbor_status arbor_evict(arbor_ctx *ctx, const arbor_tree *tree, const int32_t *k_target,
                         int64_t *evicted_tokens_out);

/* a7/a8 — lazy rehydration (Alg. 2).  For each listed closed
 * node with k_cur < n (ascending id, duplicates ignored): its kept rows are the last k_cur of
 * its n list slots (Q23r); pop pages for the freed leading list entries (a node
 * evicted to 0: ⌈n/P⌉), move the kept rows within HBM to slot = position and copy ONLY the
 * n − k_cur evicted rows back from the pinned host stash (bit-exact, Q20); first_slot = 0,
 * pos = identity, k_cur = n, rehydrations += 1.  Full nodes are a no-op and are not counted.  Listing an
 * open node is ARBOR_ERR_STATE.  nodes: HOST [count] int32.
 * ARBOR_ERR_OUT_OF_PAGES is returned (state unchanged) if the pool cannot hold the worst
 * case Σ ⌈n/P⌉ − #pages of the listed nodes. */
arbor_status arbor_rehydrate(arbor_ctx *ctx, const arbor_tree *tree, const int32_t *nodes,
                             int32_t count);
/* The copy runs on side_stream and main_stream does NOT wait for it inside arbor_rehydrate:
 * the next call that reads or moves pool rows on main_stream (arbor_tree_decode_attn,
 * arbor_decode_step, arbor_score's attention, arbor_evict) waits first — "before the next
 * decoding step" — so work enqueued in between (e.g. arbor_allocate) overlaps it.
 * HOST out: 1 while the last rehydration copy is still running (no sync). */
arbor_status arbor_rehydrate_in_flight(arbor_ctx *ctx, int32_t *in_flight);

/* a9 — tree decode attention: for each active leaf b, local layer l in
 * [layer_begin, layer_begin+layer_count) and local q head g (KV head h = g / G, Q24):
 * o = Σ_t softmax_t(q·k_t/√d) v_t over the retained slots of Path(ℓ_b), root→leaf, and
 * LSE = ln Σ_t exp(q·k_t/√d).  A node shared by several active leaves is read once.
 *  q:   DEVICE [num_active][layer_count][Hq_local][head_dim] kv_dtype
 *  out: DEVICE same shape and dtype as q
 *  lse_out: DEVICE [num_active][layer_count][Hq_local] f32 (or NULL)
 *  An empty visible set gives o = 0 and LSE = -inf. */
arbor_status arbor_tree_decode_attn(arbor_ctx *ctx, const arbor_tree *tree,
                                    int32_t layer_begin, int32_t layer_count, const void *q,
                                    void *out, float *lse_out);

/* f2 — one decode step with the score fused into the attention (P:184-191,
 * "accumulated from attention weights already materialized during decoding"):
 * exactly arbor_tree_decode_attn over the full layer range followed by arbor_score with its
 * LSE — same arguments, same results up to fp32 rounding of the LSE — but as two launches:
 * the attention kernel, then one kernel that merges the split-softmax partials into out /
 * LSE and, with the LSE still on chip, accumulates A from the logits the attention kernel
 * wrote, recomputes the visible nodes' partial masses and (single rank) the MSVE scores.
 * With several ranks the int64 mass all-reduce and the MSVE launch follow, as in arbor_score.
 *  q:       DEVICE [num_active][layer_count][Hq_local][head_dim] kv_dtype
 *  out:     DEVICE same shape and dtype as q
 *  lse_out: DEVICE [num_active][layer_count][Hq_local] f32, or NULL
 *  s_out:   DEVICE [num_nodes] f32, or NULL (as arbor_score)
 *  Errors as arbor_tree_decode_attn / arbor_score; nothing is enqueued on an error. */
arbor_status arbor_decode_step(arbor_ctx *ctx, const arbor_tree *tree, const void *q, void *out,
                               float *lse_out, float *s_out);

/* f1 — event-driven controller: one policy update event (PUE) of Alg. 2 (§3
 * P:112-116).  Composes the calls above on main_stream, no host sync:
 *  ARBOR_PUE_BOUNDARY (node: a just-closed block, else ARBOR_ERR_STATE): ScoreAllocEvict of
 *    that block only (Alg. 2 l.4) — its k from Eqs. 2-3 with the library's last
 *    scores and the tree's geometry; every other node keeps its retained set.
 *  ARBOR_PUE_TRANSITION (node ignored; tree->active holds the new leaf/leaves): rehydrate
 *    every closed Path* node with k < n (lazy rehydration, Alg. 2 l.8-14), then Eqs. 2-3 for
 *    every off-path node, evicting only where the new k is smaller (Alg. 2 l.15-21).
 *  ARBOR_PUE_PRESSURE (node ignored): reallocate to `budget` — params.alloc_mode WATERFILL
 *    (budget-exact) or STATIC_DRAIN (Alg. 2 l.22-30 literally; STATIC is treated as
 *    STATIC_DRAIN) — then evict.  ARBOR_ERR_INFEASIBLE_BUDGET as arbor_allocate.
 *  k_out: DEVICE [num_nodes] int32 scratch, receives the targets that were applied. */
typedef enum { ARBOR_PUE_BOUNDARY = 0, ARBOR_PUE_TRANSITION = 1, ARBOR_PUE_PRESSURE = 2 } arbor_pue;
arbor_status arbor_policy_event(arbor_ctx *ctx, const arbor_tree *tree, int32_t kind,
                                int32_t node, int64_t budget_tokens, int32_t *k_out,
                                int64_t *min_feasible_out);
/* Alg. 2 l.31-33 waterline input: M = Σ_i k_i over every known node (open nodes count their
 * current length).  HOST out, syncs main_stream. */
arbor_status arbor_retained_tokens(arbor_ctx *ctx, int64_t *total);
/* f1 — the waterline on the device (Alg. 2 l.31-33; "M ≥ 𝓑 − δ"): enqueue, with no
 * host sync, a check of M = Σ_i k_cur_i against budget − delta and a Pressure (allocation in
 * the bundle's Pressure mode, as ARBOR_PUE_PRESSURE, then evict) that takes effect only if
 * the check fires; the Pressure is handled in the same call, so at most one is pending
 * (SPEC S:529).  k_out: DEVICE [num_nodes] scratch (k = k_cur when nothing fired).  A fired
 * check on a budget below the minimum feasible latches ARBOR_ERR_INFEASIBLE_BUDGET (reported
 * by the next synchronising call). */
arbor_status arbor_policy_waterline(arbor_ctx *ctx, const arbor_tree *tree, int64_t budget,
                                    int64_t delta, int32_t *k_out);
/* HOST out (sync): Pressures raised by arbor_policy_waterline so far. */
arbor_status arbor_pressure_events(arbor_ctx *ctx, int64_t *count);

/* f3 — Eq. 1 on the device: the MSVE uncertainty feature at a block boundary,
 * u = 1 − H/log|𝒱| with H = −Σ_w p(w) log p(w), p = softmax(logits) over the full vocabulary
 * (exact; the top-K + "other" bucket of P:140 is an optional approximation the device does not
 * need).  logits: DEVICE [batch][vocab], dtype ARBOR_F32 or ARBOR_BF16 (−inf entries are
 * masked tokens); u_out: DEVICE [batch] f32.  Asynchronous on main_stream.
 * ARBOR_ERR_INVALID_ARG for vocab < 2, batch < 1, NULL pointers or an unknown dtype. */
arbor_status arbor_boundary_uncertainty(arbor_ctx *ctx, const void *logits, int32_t dtype,
                                        int32_t batch, int32_t vocab, float *u_out);

/* f3 — MSVE θ calibration on the device ("calibrated
 * offline using hindsight interventions"; loss and optimiser from SPEC S:224-242): full-batch
 * gradient descent of L(θ) = mean_i (σ(θ₀ + θ_v v_i + θ_u u_i + θ_a a_i) − y_i)² for `epochs`
 * epochs from the given θ; a step that would raise the loss halves the rate and retries (at
 * most 20 halvings, the reduced rate is kept), so the loss never increases.
 *  phi:    DEVICE [n][3] f32 (v_i, u_i, a_i ∈ [0,1])     target: DEVICE [n] f32 y_i ∈ [0,1]
 *  theta:  HOST [4] fp64, in: start, out: fitted          loss_out: HOST [2] (initial, final) or NULL
 * Context-free and synchronous (legacy default stream).  ARBOR_ERR_INVALID_ARG for n < 1,
 * epochs < 0, lr ≤ 0, non-finite θ or NULL pointers. */
arbor_status arbor_fit_theta(const float *phi, const float *target, int32_t n, int32_t epochs,
                             double lr, double *theta, double *loss_out);

/* ---- inspection / plumbing ------------------------------------------------------------ */
arbor_status arbor_sync(arbor_ctx *ctx);   /* wait for both streams; returns latched errors */
/* HOST outs (sync): the node's k_cur, n, and live page list (pages may be NULL;
 * *num_pages in: capacity, out: ⌈(first_slot + k_cur)/P⌉ pages). */
arbor_status arbor_read_node(arbor_ctx *ctx, int32_t node, int32_t *k_cur, int32_t *n,
                             int32_t *pages, int32_t *num_pages);
/* HOST out (sync): first_slot ∈ [0, P), the slot of the node's live page list that holds
 * its valid slot 0 (valid slots: first_slot … first_slot + k_cur − 1 of the live list;
 * 0 until an eviction, Q23*). */
arbor_status arbor_read_node_offset(arbor_ctx *ctx, int32_t node, int32_t *first_slot);
/* HOST out (sync): free stack bottom→top into `pages` (capacity *count in, size out). */
arbor_status arbor_read_free_list(arbor_ctx *ctx, int32_t *pages, int32_t *count);
/* HOST outs (sync), each [num_nodes] or NULL: all-reduced Mass_i, Mclose_i (this rank's
 * partial), Nq_i, a_i, s_i as of the last arbor_score. */
arbor_status arbor_read_scores(arbor_ctx *ctx, int32_t num_nodes, int64_t *mass,
                               int64_t *mclose, int64_t *nq, float *a, float *s);
/* a10 input/output: the device buffer of this rank's per-node partial masses, int64
 * [2 * num_nodes] = [Mass_0..Mass_{N−1} | Mclose_0..Mclose_{N−1}] (units of 2^-24, Q29) as
 * of the last arbor_score / arbor_decode_step (N = that call's num_nodes).  The all-reduce
 * is an int64 SUM of this buffer across ranks, in place.  DEVICE pointer, library-owned,
 * valid for the context's lifetime; *count = 2N.  No sync. */
arbor_status arbor_mass_buffer(arbor_ctx *ctx, int64_t **dev, int32_t *count);
/* ARBOR_FLAG_EXTERNAL_REDUCE only: complete the last arbor_score / arbor_decode_step after
 * the caller's all-reduce — reduced: DEVICE int64 [2N], the summed buffer (copied into the
 * library's), or NULL when the caller reduced arbor_mass_buffer in place; then a_i, s_i
 * (MSVE) as on a single rank.  s_out: DEVICE [N] f32 or NULL.  Asynchronous on
 * main_stream.  ARBOR_ERR_STATE if no score is pending. */
arbor_status arbor_score_finish(arbor_ctx *ctx, const int64_t *reduced, float *s_out);
/* HOST out: total rehydrations performed (sync). */
arbor_status arbor_read_counters(arbor_ctx *ctx, int64_t *rehydrations, int64_t *pages_in_use);
/* Save / restore the library-owned state (page tables, free list, k_cur, counters) in a
 * device-side snapshot slot (0..3), on main_stream.  Caller-owned pools and the score
 * array are not included.  Used by benchmarks to repeat a mutating step. */
arbor_status arbor_save_state(arbor_ctx *ctx, int32_t slot);
arbor_status arbor_load_state(arbor_ctx *ctx, int32_t slot);
/* The caller wrote the accumulated-attention array directly: recompute every closed node's
 * partial mass at the next arbor_score (the library otherwise recomputes only the nodes
 * whose tokens it just scored — A changes nowhere else). */
arbor_status arbor_invalidate_masses(arbor_ctx *ctx);
/* Kernel launches issued by this context since creation (all streams). */
int64_t arbor_launch_count(const arbor_ctx *ctx);
/* 1 when arbor_tree_decode_attn / arbor_score run the tcgen05 tensor-core attention kernel
 * (bf16 KV, head_dim 128, page_size a multiple of 8 and ≤ 64, G ≤ 6, driver tensor-map
 * support; environment ARBOR_ATTN=cuda at arbor_init forces the CUDA-core kernel), 0 when
 * the CUDA-core kernel is used, −1 for a NULL context.  Both compute the same operation
 * within the north_star tolerance. */
int32_t arbor_attn_tensor_cores(const arbor_ctx *ctx);
/* With ARBOR_FLAG_PROFILE: per-stage mean device milliseconds over the launches recorded since
 * the last arbor_reset_stage_times (up to the last 128 per stage), measured with CUDA events
 * on the launching stream (HOST out [ARBOR_NUM_STAGES]; synchronises). */
#define ARBOR_NUM_STAGES 13
enum { ARBOR_ST_GEOMETRY = 0, ARBOR_ST_SCORE_ACCUM, ARBOR_ST_NODE_MASS, ARBOR_ST_MSVE,
       ARBOR_ST_ALLOCATE, ARBOR_ST_EVICT_PLAN, ARBOR_ST_SELECT_COMPACT, ARBOR_ST_REHYDRATE,
       ARBOR_ST_ATTN, ARBOR_ST_ATTN_MERGE, ARBOR_ST_ALLREDUCE, ARBOR_ST_STASH,
       ARBOR_ST_COMPACT_MOVE };
arbor_status arbor_stage_times(arbor_ctx *ctx, float *ms);
arbor_status arbor_reset_stage_times(arbor_ctx *ctx);
/* Turn the per-stage event recording of a context created with ARBOR_FLAG_PROFILE on (1) or
 * off (0).  A timing event costs the stream ~3 µs on B200, so throughput passes run with it
 * off and a separate pass measures the per-kernel durations.  ARBOR_ERR_STATE without the
 * flag. */
arbor_status arbor_set_profiling(arbor_ctx *ctx, int32_t on);

/* ---- CUDA Graph capture (SURVEY §8(d) timing protocol: eager and graph-captured steps) --
 * arbor_capture_begin: synchronises both streams, then records (does not run) the device work
 *   of the calls that follow on an internal stream in relaxed capture mode.  Only calls
 *   without a host out-parameter and without side-stream work (no stash / rehydrate) may be
 *   captured; host uploads go to pinned buffers owned by the graph.
 * arbor_capture_end: ends the capture, instantiates it, *graph_out = opaque handle (HOST).
 * arbor_graph_launch: replays it on main_stream.  A replay updates device state only (the
 *   host mirrors stay as the captured calls left them): replay from the state the capture
 *   started in, e.g. after arbor_load_state.
 * arbor_graph_destroy: synchronises the device and frees the graph and its buffers. */
arbor_status arbor_capture_begin(arbor_ctx *ctx);
arbor_status arbor_capture_end(arbor_ctx *ctx, void **graph_out);
arbor_status arbor_graph_launch(arbor_ctx *ctx, void *graph);
arbor_status arbor_graph_destroy(void *graph);

/* ---- host-only helpers (no device work; usable without a GPU) ------------------------ */
/* Validate a tree snapshot: dense ids, parent < child, spans non-overlapping along
 * every root path, closed n ≥ 1, active ids valid, n_sinks ≤ n_root.  msg may be NULL. */
arbor_status arbor_validate_tree(const arbor_tree *tree, int32_t n_sinks, char *msg,
                                 size_t msg_len);
/* Smallest feasible budget for params.alloc_mode on this tree: Σ_pinned n + Σ floors
 * (WATERFILL: f_j = min(n, max(K_min, min(L_tail, n), ⌊r_min n + 1e-9⌋)); STATIC_DRAIN:
 * min(n, K_min); STATIC: 0). */
arbor_status arbor_min_feasible_budget(const arbor_params *params, const arbor_tree *tree,
                                       int64_t *out);
/* Library version string. */
const char *arbor_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ARBOR_H_ */
