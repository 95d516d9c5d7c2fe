/*
 * cosine_verify.h — C ABI of the B200-native CoSine verification library
 * (libcosine_verify.so, sm_100a).
 *
 * What it computes: the batched parallel verification step of CoSine
 * (arXiv 2503.10325), Alg. 2 "foreach draft t in T in parallel: (V_t, R_t) <- Verify(t)"
 * (PAPER.md P:463-464), applied to drafts merged by the confidence-based token
 * fusion of Alg. 1 / Eq. 4:
 *   - target distribution o_i = softmax(l_i / T) over the full vocabulary;
 *   - per-drafter confidence c_{n,i} = q_{n,i}(X_{n,i}) and the fused token
 *     x*_i = X_{n*,i}, n* = argmax_n c_{n,i} (Eq. 4), fused distribution q_i (reading #2);
 *   - acceptance u < min(1, o_i(x*)/q_i(x*)) with counter-based Philox uniforms;
 *   - first-rejection truncation, residual resample from norm(max(0, o - q))
 *     or the bonus token x_{gamma+1} ~ o.
 * "reading #n" refers to DESIGN.md §3, where every place the paper is silent or
 * ambiguous is resolved.
 *
 * Conventions (all entry points):
 *   - extern "C", never throws; every call returns a cosine_status_t.
 *   - Device pointers unless stated otherwise.  The caller owns every I/O buffer;
 *     rows are row-major with the vocabulary innermost.  Row bases and the leading
 *     dimensions (ld * sizeof(element)) must be multiples of 16 bytes, else
 *     COSINE_ERR_UNSUPPORTED.  ld >= the context's vocabulary width.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     stream-ordered and asynchronous.  Host-side argument errors return
 *     synchronously and enqueue nothing.
 *   - Device-detected data errors are reported per request in status[b]; that request's
 *     accept_len is -1 and its out_tokens row is all -1; other requests are unaffected.
 *   - The context owns scratch memory (sized at init from the max_* fields: per (request,
 *     position) unit 16 partial records of 128 B, the decision, the tile masses, and for an
 *     unsharded context over probability drafts the SAMPLE slice sums, max_drafters floats
 *     per 256 vocabulary entries).  One context may be used by one host thread / one stream
 *     at a time.
 *   - Randomness: U(rid, node, tag) = (Philox4x32-10(ctr = {rid_lo, rid_hi, node,
 *     (step << 4) | tag}, key = {seed_lo, seed_hi}).x0 >> 8) * 2^-24 (readings #8, #9).
 *     Tags: ACCEPT = 0, SAMPLE = 1, FUSE = 2.  Results depend only on global request ids,
 *     never on batch order or on how requests are sharded across GPUs.
 */
#ifndef COSINE_VERIFY_H
#define COSINE_VERIFY_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cosine_ctx_s* cosine_ctx_t;
typedef void* cosine_stream_t; /* a cudaStream_t */

typedef enum {
  COSINE_OK = 0,
  COSINE_ERR_INVALID_ARGUMENT = 1, /* bad shape, mode, NULL pointer, out-of-range size */
  COSINE_ERR_UNSUPPORTED = 2,      /* dtype / alignment / mode combination not supported */
  COSINE_ERR_CUDA = 3,             /* a CUDA runtime call failed (see cosine_last_error) */
  COSINE_ERR_NCCL = 4,
  COSINE_ERR_OUT_OF_MEMORY = 5
} cosine_status_t;

/* Per-request status codes written to status[b] (low byte) plus info flags. */
#define COSINE_REQ_OK 0
#define COSINE_REQ_ZERO_PROB_DRAFT 1      /* a drafter's own token has q = 0          */
#define COSINE_REQ_TOKEN_OUT_OF_RANGE 2   /* draft token outside [0, V)                */
#define COSINE_REQ_NONFINITE_INPUT 3      /* NaN / +inf logit; NaN, inf or negative prob      */
#define COSINE_REQ_EMPTY_ROW 4            /* all -inf logits, or a probability row summing to 0 */
#define COSINE_REQ_BAD_DRAFT_LEN 5        /* draft_len[b] outside [1, k]                      */
#define COSINE_REQ_BAD_TREE 6             /* tree: parent order, duplicate sibling tokens, internal rows */
#define COSINE_INFO_DEGENERATE_RESIDUAL 0x100 /* Z == 0: resampled from o (reading #11) */
#define COSINE_INFO_NEAR_TIE 0x200        /* a decision margin < 1e-6 (reading #18)          */

typedef enum { COSINE_BF16 = 0, COSINE_F32 = 1 } cosine_dtype_t;
/* Drafter rows: probabilities (renormalised by their sum, reading #6) or logits (softmax at the
 * call's temperature). */
typedef enum { COSINE_DRAFT_PROBS = 0, COSINE_DRAFT_LOGITS = 1 } cosine_draft_kind_t;
/* Fused distribution q_i = sum_n w_n q_{n,i} (reading #2): CONF w_n = c_n / sum c (default),
 * WINNER w = e_{n*}, UNIFORM w = 1/N, POINT q = delta_{x*}. */
typedef enum { COSINE_W_CONF = 0, COSINE_W_WINNER = 1, COSINE_W_UNIFORM = 2, COSINE_W_POINT = 3 } cosine_weight_mode_t;
/* Fused token: Eq. 4's argmax (paper-literal) or a draw x* ~ q_i with U(rid, i+1, FUSE)
 * (distribution-exact; reading #3). */
typedef enum { COSINE_SEL_ARGMAX = 0, COSINE_SEL_SAMPLE = 1 } cosine_select_mode_t;

typedef struct {
  int32_t device;          /* CUDA device ordinal the context lives on                      */
  int64_t vocab_size;      /* global V                                                       */
  int64_t vocab_begin;     /* this rank's shard [vocab_begin, vocab_end); [0, V) unsharded    */
  int64_t vocab_end;
  int32_t max_batch;       /* largest B of any call                                          */
  int32_t max_draft_len;   /* largest k                                                      */
  int32_t max_drafters;    /* largest N (<= 8)                                               */
  int32_t max_tree_nodes;  /* largest J + 1 of cosine_verify_tree (<= 1024), 0 if unused   */
  cosine_dtype_t target_dtype;
  cosine_dtype_t draft_dtype;
  cosine_draft_kind_t draft_kind;
  uint64_t seed;           /* Philox key                                                     */
  int32_t nranks;          /* 1 = unsharded (batch sharding = independent contexts);          */
                           /* > 1 = vocabulary-sharded over nranks GPUs (<= 32), see below    */
  int32_t rank;            /* this rank, in [0, nranks); shards concatenate in rank order     */
  const void* nccl_unique_id; /* nranks > 1: COSINE_NCCL_UNIQUE_ID_BYTES from rank 0's        */
                           /* cosine_nccl_unique_id(), identical on every rank (the caller    */
                           /* broadcasts it); the context owns the NCCL communicator          */
  int32_t cluster_size;    /* 0 = automatic; else 1, 2, 4, 8 or 16 CTAs per (request,        */
                           /* position) of the statistics pass (fixed: no one-launch path)    */
  int32_t exchange;        /* sharded contexts: 0 = in-kernel peer writes when every rank can  */
                           /* map the others' memory, else NCCL; 1 = NCCL all-gathers only    */
} cosine_config_t;

/* Optional per-unit diagnostics of cosine_verify_batch (any member may be NULL). */
typedef struct {
  float* p_x;           /* [B][k]  o_i(x*_i)                                                 */
  float* q_x;           /* [B][k]  q_i(x*_i)                                                 */
  float* accept_u;      /* [B][k]  U(rid, i+1, ACCEPT)                                        */
  float* row_max;       /* [B][k+1] M = max_v l(v) (raw logit; T = 0: the max)               */
  float* row_sumexp;    /* [B][k+1] S = sum_v exp((l(v) - M) / T)  (T = 0: 0)                 */
  float* draft_norm;    /* [B][k][N] sigma (PROBS: row sum; LOGITS: sum exp((d - max)/T))   */
  float* conf;          /* [B][k][N] c_{n,i}                                                 */
  float* weights;       /* [B][k][N] w_{n,i}                                                 */
  int32_t* fused_tokens;/* [B][k]  x*_i                                                      */
  float* residual_mass; /* [B] Z of the final sample in probability units (bonus: 1)         */
  float* tie_margin;    /* [B] smallest decision margin the GPU saw for the realised path     */
} cosine_debug_t;

/* Create a context on cfg->device (allocates scratch).  *out = NULL on failure. */
cosine_status_t cosine_verify_init(const cosine_config_t* cfg, cosine_ctx_t* out);
/* Free the context (synchronises its device).  NULL is a no-op. */
cosine_status_t cosine_verify_destroy(cosine_ctx_t ctx);
/* Last error message of ctx (or of the calling thread's last failed init if ctx is NULL). */
const char* cosine_last_error(cosine_ctx_t ctx);

/*
 * Vocabulary-sharded mode (SURVEY §8(e) "Vocab", config c5; logits from a tensor-parallel LM
 * head).  Rank g's context has [vocab_begin, vocab_end) = its column shard; the
 * shards of ranks 0..nranks-1 must tile [0, vocab_size) in rank order.  Every rank calls
 * cosine_verify_batch collectively (same B, k, N, draft_tokens, draft_len, request_ids, step,
 * modes, temperature) with ITS columns of every row (ld >= the shard width; token ids stay
 * global); the outputs are identical on every rank and equal to the unsharded call on the full
 * rows up to flagged near-ties.  Three exchanges: per-(request, position) row statistics and
 * candidate gathers (~N^2 + 4N + 8 words), the local masses of the final draw (B doubles), the
 * owner's token (B x 16 bytes).  With <= 8 ranks whose GPUs can map each other's memory (CUDA
 * IPC over NVLink, set up collectively at init) the producing kernels write them straight into
 * every rank's gather buffer and count them on per-rank arrival counters that the consuming
 * kernels wait on (no collective launches; a wait gives up after ~5 s instead of hanging);
 * otherwise three NCCL all-gathers on `stream`.  ARGMAX selection only;
 * cosine_fuse_drafts / cosine_sample_residual / cosine_verify_tree return COSINE_ERR_UNSUPPORTED
 * on a sharded context.
 *
 * cosine_nccl_unique_id — write a fresh NCCL unique id (COSINE_NCCL_UNIQUE_ID_BYTES bytes, host
 * memory) to `out`; call on rank 0 and broadcast.  capacity < the id size ->
 * COSINE_ERR_INVALID_ARGUMENT; NCCL failure -> COSINE_ERR_NCCL.
 */
#define COSINE_NCCL_UNIQUE_ID_BYTES 128
cosine_status_t cosine_nccl_unique_id(void* out, int64_t capacity);

/*
 * Virtual group (TEST / DIAGNOSTIC) — the vocabulary-sharded call of G ranks inside ONE process
 * on ONE device, for checking the sharded kernels without G GPUs.
 * cosine_verify_init_vgroup: cfgs[g] is rank g of G (nranks = G, rank = g, shards tiling
 *   [0, vocab_size) in rank order, every other field equal; nccl_unique_id ignored); creates G
 *   contexts (out[g]) that own no NCCL communicator.  On failure every created context is freed.
 * cosine_verify_batch_vgroup: the collective cosine_verify_batch of the G contexts (ARGMAX
 *   selection, no diagnostics), run phase by phase on `stream`: exactly the kernels and record
 *   layouts of the NCCL path, with each all-gather replaced by device copies
 *   of every rank's send buffer into every rank's gather buffer in rank order.
 *   target_logits[g] / draft[g]: rank g's column shard ([B][k+1][ld_t] / [B][k][N][ld_q], one ld
 *   for all ranks); accept_len[g] / out_tokens[g] / status[g]: rank g's (replicated) outputs.
 *   exchange: 0 = device copies between the phases (the layout of the NCCL all-gathers);
 *   1 = the in-kernel peer-memory exchange of multi-GPU calls (G <= 8), the peers being the
 *   other contexts' gather blocks.
 *   Errors as cosine_verify_batch; a vgroup context passed to cosine_verify_batch returns
 *   COSINE_ERR_UNSUPPORTED.
 */
cosine_status_t cosine_verify_init_vgroup(const cosine_config_t* cfgs, int32_t G, cosine_ctx_t* out);
cosine_status_t cosine_verify_batch_vgroup(const cosine_ctx_t* ctxs, int32_t G, cosine_stream_t stream, int32_t B,
                                           int32_t k, int32_t N, const void* const* target_logits, int64_t ld_t,
                                           float temperature, const void* const* draft, int64_t ld_q,
                                           const int32_t* draft_tokens, const int32_t* draft_len,
                                           const uint64_t* request_ids, uint32_t step,
                                           cosine_weight_mode_t weight_mode, int32_t* const* accept_len,
                                           int32_t* const* out_tokens, int32_t* const* status, int32_t exchange);

/*
 * cosine_fuse_drafts — Eq. 4 token fusion only (Alg. 1 TokenFusion P:376-381).
 *   draft        [B][k][N][ld_q] drafter rows (config draft_dtype / draft_kind)
 *   draft_tokens [B][k][N] int32 X_{n,i};  request_ids [B] uint64 (global ids);  step
 *   temperature  used only for COSINE_DRAFT_LOGITS (must be > 0 then)
 * Outputs: fused_tokens [B][k] (x*_i), weights [B][k][N] (w_{n,i}), draft_norm [B][k][N]
 *   (sigma), fused_q [B][k][ld_fq] fp32 q_i(v) for v < V (NULL = not materialised), status [B].
 *   weights / draft_norm may be NULL.  A request with an error has all fused_tokens = -1.
 */
cosine_status_t cosine_fuse_drafts(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t k,
                                   int32_t N, const void* draft, int64_t ld_q,
                                   const int32_t* draft_tokens, const uint64_t* request_ids,
                                   uint32_t step, float temperature,
                                   cosine_weight_mode_t weight_mode, cosine_select_mode_t select_mode,
                                   int32_t* fused_tokens, float* weights, float* draft_norm,
                                   float* fused_q, int64_t ld_fq, int32_t* status);

/*
 * cosine_verify_batch — the whole verification step for B independent requests.
 *   target_logits [B][k+1][ld_t]: row i is the target's next-token logits after the prefix and
 *                 x*_0..x*_{i-1}; row gamma_b is the bonus row (reading #14).
 *   temperature   T > 0 samples; T == 0 is greedy (lowest-index argmax, reading #7).
 *   draft         [B][k][N][ld_q] drafter rows at the fused-path positions (Eq. 4).
 *   draft_tokens  [B][k][N] int32;  draft_len [B] int32 gamma_b in [1, k] or NULL (= k) (Alg. 2
 *                 AdaptiveSpeculation; reading #15).
 *   request_ids   [B] uint64 global ids;  step = decoding step (Philox counter word).
 * Outputs: accept_len [B] = L_b (-1 on a per-request error); out_tokens [B][k+1] = x*_0 ..
 *   x*_{L-1}, y, then -1; status [B].  debug may be NULL.
 * Rows after gamma_b are never read.  All rows 0..gamma_b are read and validated.
 * One GPU: three launches on `stream` — the row statistics (every input byte read once), the
 * decisions (a warp per position; SAMPLE over probability drafts draws x* ~ q from the chunk
 * records and the 32-group slice sums the statistics keep, reading #26; over logit drafts a CTA
 * per position scans the crossing chunk) and the final draws (the rows at L re-read once) — the
 * latter two as programmatic dependents waiting on device counters.  When the batch's (position,
 * chunk) grid fits one wave (small batches, ARGMAX), the three steps run as ONE cooperative
 * launch instead (cosine_last_launch_count reports 1).
 */
cosine_status_t cosine_verify_batch(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t k,
                                    int32_t N, const void* target_logits, int64_t ld_t,
                                    float temperature, const void* draft, int64_t ld_q,
                                    const int32_t* draft_tokens, const int32_t* draft_len,
                                    const uint64_t* request_ids, uint32_t step,
                                    cosine_weight_mode_t weight_mode,
                                    cosine_select_mode_t select_mode, int32_t* accept_len,
                                    int32_t* out_tokens, int32_t* status,
                                    const cosine_debug_t* debug);

/*
 * cosine_verify_batch_lazy — the same verification with early exit: rows
 * are streamed position by position, i = 0, 1, ..., and a request stops reading at its first
 * rejection (the rows after it are discarded anyway), at an error, or at its bonus row.
 * Each round streams the next 2 positions of the requests still verifying and decides them in
 * order; then the final draws: 2 ceil((k + 1) / 2) + 1 kernel launches.  Rows after the round
 * holding L_b are never read (at most one speculative position per request), so the realised
 * bytes are ~ sum_b (L_b + 2) rows (+ the resample pass).
 * Arguments and outputs as cosine_verify_batch (ARGMAX selection; unsharded contexts only).
 * Outputs are identical to cosine_verify_batch (counter-based Philox, reading #8) for every
 * request whose rows 0..L_b are valid; a data error in a row after L_b is NOT detected (that
 * request gets its normal result instead of an error status).  debug: per-position arrays are
 * written for positions <= L_b only.
 */
cosine_status_t cosine_verify_batch_lazy(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t k,
                                         int32_t N, const void* target_logits, int64_t ld_t,
                                         float temperature, const void* draft, int64_t ld_q,
                                         const int32_t* draft_tokens, const int32_t* draft_len,
                                         const uint64_t* request_ids, uint32_t step,
                                         cosine_weight_mode_t weight_mode, int32_t* accept_len,
                                         int32_t* out_tokens, int32_t* status,
                                         const cosine_debug_t* debug);

/*
 * cosine_fuse_step — drafter-side token fusion of ONE drafting iteration (
 * Alg. 1 Fuse P:376-381, Eq. 4 first line P:406-408, greedy drafting P:681): the central node's
 * step between the drafters' LM heads and the next iteration.
 *   logits [B][N][ld] the N drafters' LM-head outputs for request b (config draft_dtype;
 *          ld >= V, 16-byte aligned rows);  temperature > 0 (softmax of l / T)
 * Outputs: own_tokens [B][N] X_n = argmax_v l_n(v) (lowest index on ties); conf [B][N]
 *   c_n = softmax(l_n / T)(X_n); fused_token [B] x* = X_{n*}; winner [B] n* = argmax_n c_n
 *   (lowest n on ties); status [B] (NaN / +inf logit -> NONFINITE_INPUT, all -inf -> EMPTY_ROW;
 *   the first erroring drafter decides; tokens -1).  Needs B * N <= max_batch * (max_draft_len + 1)
 *   (context scratch).  Two launches (one streaming pass over the rows, one combine).
 */
cosine_status_t cosine_fuse_step(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t N,
                                 const void* logits, int64_t ld, float temperature, int32_t* own_tokens,
                                 float* conf, int32_t* fused_token, int32_t* winner, int32_t* status);

/*
 * cosine_route_update — routing feedback after verification (Alg. 1 "Update
 * routing matrix"; Eq. 1, Eq. 2; decay of non-participating nodes S:315).
 *   draft_tokens [B][N][K] int32 X_{n,i} (node n's own draft);  conf [B][N][K] fp32 c_{n,i}
 *   accepted [B][acc_stride] int32 (e.g. out_tokens, acc_stride = k + 1);  accept_len [B] L_b
 *     (< 0: the request failed verification -> no update)
 *   emb [V][ld_e] embedding rows H(.) (bf16 / fp32, hidden % 8 == 0, 16-byte aligned rows)
 *   participating [B][N] uint8 or NULL (= all);  decay in [0, 1]
 *   M [B][N] fp32 routing scores, updated in place:  m_n = (1/K) sum_i c d / (c d + (1-c)(1-d))
 *     with d_{n,i} = cos(H(x_i), H(X_{n,i})) for i < L_b else 0, c and d clamped to
 *     [1e-6, 1 - 1e-6] (reading #24); non-participating: M = 0.5 + decay (M - 0.5)
 *   d_out [B][N][K] fp32 or NULL;  status [B]: 2 if a token is outside [0, vocab_size) (M kept).
 * One launch (CTA per request, warp per node).  V = the context's vocab_size.
 */
cosine_status_t cosine_route_update(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t N, int32_t K,
                                    const int32_t* draft_tokens, const float* conf, const int32_t* accepted,
                                    int64_t acc_stride, const int32_t* accept_len, const void* emb,
                                    int64_t hidden, int64_t ld_e, cosine_dtype_t emb_dtype,
                                    const uint8_t* participating, float decay, float* M, float* d_out,
                                    int32_t* status);

/*
 * cosine_tree_select — TreeSelection (Alg. 1 "TreeSelection" P:372; the paper
 * does not define it: SPEC S:303-311's construction, reading #25).  Per request, S branch
 * sequences (each drafter's own and fused branch) of K tokens with their confidences:
 *   tokens [B][S][K] int32 (< 0 ends a branch), conf [B][S][K] fp32, budget = non-root nodes kept.
 * The branches are merged into a prefix tree rooted at the last verified token (node 0); a node's
 * score is the largest product of confidences along a branch reaching it; the `budget` best nodes
 * (score desc, depth asc, creation order) are kept — a prefix-closed set — and renumbered
 * breadth-first with siblings by (score desc, creation), ready for cosine_verify_tree.
 * Outputs [B][budget + 1]: parent (-1 root / padding), token (-1 root / padding), score, depth;
 * n_nodes [B] = kept + 1.  S * K + 1 <= 1024.  One launch (CTA per request).
 */
cosine_status_t cosine_tree_select(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t S, int32_t K,
                                   const int32_t* tokens, const float* conf, int32_t budget, int32_t* n_nodes,
                                   int32_t* parent, int32_t* token, float* score, int32_t* depth);

/*
 * cosine_sample_residual — the final-token sample of one row group per request,
 * for callers that verify elsewhere.
 *   target_rows [B][ld_t] logits of the row at L_b;  temperature (0 = argmax)
 *   row_max, row_sumexp [B] fp32 M = max l and S = sum exp((l - M)/T), or both NULL (recompute)
 *   draft_rows [B][N][ld_q] drafter PROBS rows at L_b, or NULL => bonus sample y ~ o
 *   weights, draft_norm [B][N] fp32 w_n and sigma_n (e.g. from cosine_fuse_drafts)
 *   node_ids [B] uint32 Philox node (= L_b);  request_ids [B];  step
 * Output: out_token [B] y (-1 on error), status [B].
 * y = smallest v with C(v) > U(rid, node, SAMPLE) * Z over r(v) = max(0, o(v) - q(v))
 * (q = sum_n w_n d_n(v) / sigma_n) — or over o itself for the bonus and when Z == 0.
 */
cosine_status_t cosine_sample_residual(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B,
                                       const void* target_rows, int64_t ld_t, float temperature,
                                       const float* row_max, const float* row_sumexp,
                                       const void* draft_rows, int64_t ld_q, const float* weights,
                                       const float* draft_norm, int32_t N,
                                       const uint32_t* node_ids, const uint64_t* request_ids,
                                       uint32_t step, int32_t* out_token, int32_t* status);

/*
 * cosine_verify_tree — tree-shaped drafts ("merge them into a tree topology", P:414-415;
 * the algorithm is DESIGN.md reading #13, the paper does not give it): multi-candidate recursive
 * rejection.  One tree per request with J+1 nodes, node 0 = the root (last verified token).
 *   parent [B][J+1] int32 (parent[0] = -1, 0 <= parent[j] < j; children of a node are visited in
 *                  ascending node id = draw order);  node_token [B][J+1] int32 (root ignored)
 *   internal_row [B][J+1] int32: row of `draft` holding node j's drafter distributions, -1 iff j
 *                  is a leaf;  target [B][J+1][ld_t]: row j = the target's logits after the path
 *                  to node j;  draft [B][I][N][ld_q];  node_draft_tokens [B][I][N] (the drafters'
 *                  own tokens at each internal node, for Eq. 4 confidences)
 *   temperature > 0;  weight_mode CONF / WINNER / UNIFORM (POINT is undefined for several children)
 * Outputs: accept_len [B] = depth of the accepted path (-1 on error); accepted_nodes [B][J+1] node
 *   ids of the accepted path, -1 padded; out_tokens [B][J+1] = tokens of the path then the final
 *   token, -1 padded; status [B].  Requires cfg.max_tree_nodes >= J + 1.
 * Every node's rows are read once; each rejection costs one more pass over its node's rows.
 */
cosine_status_t cosine_verify_tree(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t J,
                                   int32_t I, int32_t N, const int32_t* parent,
                                   const int32_t* node_token, const int32_t* internal_row,
                                   const void* target, int64_t ld_t, float temperature,
                                   const void* draft, int64_t ld_q,
                                   const int32_t* node_draft_tokens, const uint64_t* request_ids,
                                   uint32_t step, cosine_weight_mode_t weight_mode,
                                   int32_t* accept_len, int32_t* accepted_nodes,
                                   int32_t* out_tokens, int32_t* status);

/*
 * cosine_verify_tree_lazy — the tree walk with early exit: instead of
 * reading every node's rows up front, the walk kernel computes the statistics of each node it
 * visits (one pass over that node's rows, then the node's Eq. 4 fusion and its children's
 * o / q) — path-only bytes, one kernel launch.  Arguments and outputs as cosine_verify_tree.
 * Outputs are identical to cosine_verify_tree for every request whose visited nodes are valid;
 * a data error in a node the walk does not visit is not detected (reading #23);
 * structure errors (parent order, siblings, internal rows) are checked for the whole tree.
 */
cosine_status_t cosine_verify_tree_lazy(cosine_ctx_t ctx, cosine_stream_t stream, int32_t B, int32_t J,
                                   int32_t I, int32_t N, const int32_t* parent,
                                   const int32_t* node_token, const int32_t* internal_row,
                                   const void* target, int64_t ld_t, float temperature,
                                   const void* draft, int64_t ld_q,
                                   const int32_t* node_draft_tokens, const uint64_t* request_ids,
                                   uint32_t step, cosine_weight_mode_t weight_mode,
                                   int32_t* accept_len, int32_t* accepted_nodes,
                                   int32_t* out_tokens, int32_t* status);

/* Number of kernels the last successful call on ctx enqueued (for launch accounting). */
int32_t cosine_last_launch_count(cosine_ctx_t ctx);
/* How a sharded context exchanges: 0 unsharded, 1 NCCL all-gathers, 2 in-kernel writes into the
 * peers' memory (CUDA IPC over NVLink), 3 a virtual group (cosine_verify_init_vgroup). */
int32_t cosine_exchange_mode(cosine_ctx_t ctx);

/* Live timing of the dominant kernel (the streaming statistics kernel of cosine_verify_batch):
 * when enabled, every verify call brackets it with CUDA events on the caller's stream.
 * cosine_profile_read synchronises on them, returns the summed duration (ms) and the number of
 * bracketed launches since the last read / enable, and resets the accumulator. */
cosine_status_t cosine_profile_enable(cosine_ctx_t ctx, int32_t enable);
cosine_status_t cosine_profile_read(cosine_ctx_t ctx, double* total_ms, int32_t* launches);


#ifdef __cplusplus
}
#endif
#endif /* COSINE_VERIFY_H */
