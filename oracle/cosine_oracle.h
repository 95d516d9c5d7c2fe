/*
 * cosine_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU oracle for the batched verification step of CoSine
 * (arXiv 2503.10325).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or helper with the CUDA path (paper_2503_10325_b200/csrc).
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * "reading #n" = DESIGN.md §3 (the readings of the paper this oracle follows).
 *
 * All floating point inputs are fp64 copies of the (bf16 / fp32) values the
 * GPU path receives; all arithmetic is fp64, sums are sequential in
 * ascending vocabulary index.  No blocking, fusion or reordering.
 */
#ifndef COSINE_ORACLE_H
#define COSINE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Philox tags (reading #8). */
enum { ORC_TAG_ACCEPT = 0, ORC_TAG_SAMPLE = 1, ORC_TAG_FUSE = 2, ORC_TAG_TREE_GEN = 3 };
/* weight modes (reading #2) */
enum { ORC_W_CONF = 0, ORC_W_WINNER = 1, ORC_W_UNIFORM = 2, ORC_W_POINT = 3 };
/* select modes (Eq. 4 literal ARGMAX, or SAMPLE x* ~ fused q; reading #3) */
enum { ORC_SEL_ARGMAX = 0, ORC_SEL_SAMPLE = 1 };
/* draft kinds */
enum { ORC_DRAFT_PROBS = 0, ORC_DRAFT_LOGITS = 1 };
/* per-request status codes (low byte) and info flags */
enum {
  ORC_ST_OK = 0, ORC_ST_ZERO_PROB_DRAFT = 1, ORC_ST_TOKEN_OUT_OF_RANGE = 2,
  ORC_ST_NONFINITE_OR_NEGATIVE = 3, ORC_ST_EMPTY_ROW = 4, ORC_ST_BAD_DRAFT_LEN = 5,
  ORC_ST_BAD_TREE = 6,
  ORC_INFO_DEGENERATE_RESIDUAL = 0x100
};

/* Philox4x32-10, one block: out[4] = philox(ctr[4], key[2]). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* U(rid, node, tag) in [0, 1 - 2^-24] (reading #8, #9). */
double orc_uniform(uint64_t seed, uint64_t request_id, uint32_t node, uint32_t step, uint32_t tag);

/* Inverse CDF: smallest v with sum_{w'<=v} w > u * sum(w); if none, last v with w > 0;
 * -1 if all weights are zero.  *margin (may be NULL) = distance of t to the chosen
 * bin's edges divided by sum(w) (reading #10). */
int64_t orc_invcdf(const double* w, int64_t V, double u, double* margin);

/* Target softmax at temperature T > 0 (reading #1).
 * Returns 0, or a status code (NONFINITE / EMPTY_ROW).  M = max_v l(v)/T, S = sum exp(l/T - M). */
int orc_softmax(const double* l, int64_t V, double T, double* p, double* M, double* S);

/* Residual norm(max(0, o - q)); returns 1 if degenerate (all zero), in which
 * case r is left as the zero vector. */
int orc_residual(const double* o, const double* q, int64_t V, double* r);

/* Linear verification of a batch (§8(c) steps 1-7).  Returns 0 or 1 (invalid argument).
 * Debug outputs may be NULL.  tie_margin[b] = smallest decision margin (see reading #18). */
int orc_verify_batch(int32_t B, int32_t k, int32_t N, int64_t V,
                     const double* target, double temperature,
                     const double* draft, int32_t draft_kind,
                     const int32_t* draft_tokens, const int32_t* draft_len,
                     const uint64_t* request_ids, uint64_t seed, uint32_t step,
                     int32_t weight_mode, int32_t select_mode,
                     int32_t* accept_len, int32_t* out_tokens, int32_t* status,
                     double* dbg_p_x, double* dbg_q_x, double* dbg_M, double* dbg_S,
                     double* dbg_sigma, double* dbg_conf, double* dbg_w, int32_t* dbg_fused,
                     double* dbg_u, double* dbg_Z, double* tie_margin);

/* Fusion only (Eq. 4): fused tokens, weights, draft normalisers and
 * (optionally) the fused q rows.  Returns 0 or 1. */
int orc_fuse_drafts(int32_t B, int32_t k, int32_t N, int64_t V,
                    const double* draft, int32_t draft_kind, double temperature,
                    const int32_t* draft_tokens, const uint64_t* request_ids,
                    uint64_t seed, uint32_t step, int32_t weight_mode, int32_t select_mode,
                    int32_t* fused_tokens, double* weights, double* draft_norm,
                    double* fused_q, int32_t* status, double* tie_margin);

/* Residual / bonus sample for one row group per request.
 * target [B][V] logits; row_max/row_sumexp NULL => recompute.  draft [B][N][V] PROBS or NULL
 * (=> bonus from the target).  weights / draft_norm [B][N]. */
int orc_sample_residual(int32_t B, int64_t V, const double* target, double temperature,
                        const double* row_max, const double* row_sumexp,
                        const double* draft, int32_t N, const double* weights,
                        const double* draft_norm, const uint32_t* node_ids,
                        const uint64_t* request_ids, uint64_t seed, uint32_t step,
                        int32_t* out_token, int32_t* status, double* dbg_Z, double* tie_margin);

/* Tree verification (reading #13).  One tree per request with J+1 nodes
 * (node 0 = root = last verified token).  parent[B][J+1] (parent[0] = -1, parent[j] < j),
 * node_token[B][J+1] (root token ignored), target [B][J+1][V] (row j = target distribution
 * after the path to node j), internal_row[B][J+1] (row index into draft for nodes with
 * children, -1 for leaves), draft [B][I][N][V], node_draft_tokens [B][I][N].
 * accepted_nodes[B][J+1] = node ids of the accepted path (root excluded), -1 padded;
 * out_tokens[B][J+1] = tokens of the accepted path then the final token, -1 padded. */
int orc_verify_tree(int32_t B, int32_t J, int32_t I, int32_t N, int64_t V,
                    const int32_t* parent, const int32_t* node_token, const int32_t* internal_row,
                    const double* target, double temperature,
                    const double* draft, int32_t draft_kind, const int32_t* node_draft_tokens,
                    const uint64_t* request_ids, uint64_t seed, uint32_t step, int32_t weight_mode,
                    int32_t* accept_len, int32_t* accepted_nodes, int32_t* out_tokens,
                    int32_t* status, double* tie_margin);

/* Drafter-side token fusion of one drafting iteration (Alg. 1 Fuse,
 * P:376-381, Eq. 4 first line P:406-408, greedy drafting P:681): logits[B][N][V] are the N
 * drafters' LM-head outputs for request b at iteration i.  Per drafter: its own token
 * X_n = argmax_v l_n(v) (lowest index on ties) and its probability c_n = softmax(l_n / T)(X_n)
 * = 1 / sum_v exp(l_n(v)/T - max/T); then x* = X_{n*}, n* = argmax_n c_n (lowest n on ties).
 * Outputs own_tokens[B][N], conf[B][N], fused_token[B], winner[B], status[B] (per request: the
 * first drafter row with an error decides it; -1 tokens), conf_gap[B] = (c_(1) - c_(2)) / c_(1)
 * (the tie margin, reading #18; +inf for N = 1).  Returns 0, or 1 on a bad argument. */
int orc_fuse_step(int32_t B, int32_t N, int64_t V, const double* logits, double temperature,
                  int32_t* own_tokens, double* conf, int32_t* fused_token, int32_t* winner,
                  int32_t* status, double* conf_gap);

/* Routing feedback after verification (Alg. 1 "Update routing matrix",
 * Eq. 1 P:318-327 and Eq. 2).  Per request b and node n:
 *   d_{n,i} = cos(H(x_i), H(X_{n,i})) for i < L_b (x_i = accepted token i, H = embedding rows
 *             emb[V][Hd]), else 0                                              (Eq. 1)
 *   m_n = (1/K) sum_i c d / (c d + (1 - c)(1 - d)), c and d clamped to [eps, 1 - eps]  (Eq. 2)
 * participating[b][n] != 0: M[b][n] = m_n; else M[b][n] = 0.5 + decay (M[b][n] - 0.5)
 * (S:315).  draft_tokens [B][N][K], conf [B][N][K], accepted [B][K] (or longer rows, stride
 * acc_stride), accept_len [B] (< 0: request skipped), M [B][N] in/out, d_out [B][N][K] or NULL.
 * A token outside [0, V) makes that request's status 2 (M unchanged).  Returns 0 / 1 (bad arg). */
int orc_route_update(int32_t B, int32_t N, int32_t K, int64_t V, int64_t Hd, const int32_t* draft_tokens,
                     const double* conf, const int32_t* accepted, int64_t acc_stride, const int32_t* accept_len,
                     const double* emb, const uint8_t* participating, double decay, double eps, double* M,
                     double* d_out, int32_t* status);

/* TreeSelection (Alg. 1 "TreeSelection" P:372, not defined by the paper —
 * SPEC S:303-311's construction, reading #25).  Per request: S branches (each node's own
 * and fused branch) of K tokens with confidences are merged into a prefix tree rooted at the last
 * verified token (node 0); a node's score is the largest product of confidences along any branch
 * reaching it; the `budget` best non-root nodes are kept (score desc, then depth asc, then creation
 * order), which is prefix-closed; the kept nodes are renumbered breadth-first with siblings in
 * (score desc, creation) order, so parent[j] < j and children are in slot order.
 * Outputs [B][budget + 1]: parent (-1 root / padding), token (-1 root / padding), score, depth;
 * n_nodes[B] = kept + 1.  tokens < 0 end a branch.  Returns 0 / 1 (bad argument). */
int orc_tree_select(int32_t B, int32_t S, int32_t K, const int32_t* tokens, const double* conf, int32_t budget,
                    int32_t* n_nodes, int32_t* parent, int32_t* token, double* score, int32_t* depth);

#ifdef __cplusplus
}
#endif
#endif
