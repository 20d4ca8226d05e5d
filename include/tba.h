/*
 * tba.h — C ABI of libtba.so: the VarGrad trajectory-balance loss head of
 * "Trajectory Balance with Asynchrony" (TBA, arXiv 2503.18929), hand-written CUDA for
 * B200 (sm_100a).
 *
 * Citations: P:L = PAPER.md line L (the paper's LaTeX source), S:L = SPEC.md line L.
 *   Eq. 4  (eq:logZ,    P:122-130)  log Z(x_i) = 1/K sum_j (log pi_ref - log pi_theta + r_phi/beta)
 *   Eq. 5  (eq:vargrad)  L = 1/(BK) sum_ij (SG[log Z_i] + log pi_theta - log pi_ref - r_phi/beta)^2
 *   App. A              grad L = 1/(BK) sum_ij -2(...) grad log pi_theta
 *   log pi_theta(y|x) = sum_t log softmax(z_t)[y_t]  ("parallel likelihood evaluation of an
 *   entire sequence through a single forward pass")
 *
 * Layout. N = n_seq sequences, group-major: sequence s = i*K + j is sample j
 * of prompt i (the paper's B queries x K responses). Row (s, t) = s*seq_len + t.
 *   logits  : row (s,t) starts at logits + ((s*seq_len + t) * row_stride) elements;
 *             elements [0, vocab) are read, the padding [vocab, row_stride) never is.
 *   tokens  : int64 [N, seq_len], the sampled token y_{s,t}; ignored where mask == 0
 *             (may hold -1 / -100 / garbage there).
 *   mask    : uint8 [N, seq_len], 0/1 response mask mu_{s,t}.
 * All pointers are caller-owned DEVICE memory unless stated otherwise; the library never
 * allocates, frees or synchronises. Every call is stream-ordered on `stream` (NULL = the
 * legacy default stream) and reentrant (no global mutable state; "pure functions").
 *
 * Errors. Host-side validation happens before any CUDA call and returns synchronously:
 *   TBA_ERR_INVALID_ARG    null pointer, negative size, row_stride < vocab, n_seq % K != 0,
 *                          unknown dtype, misaligned pointer, 64-bit size overflow;
 *   TBA_ERR_INVALID_CONFIG beta <= 0 or non-finite, K < 2, bad IS mode or
 *                          temperature;
 *   TBA_ERR_CUDA           a launch failed (cudaGetLastError()).
 * Device-side conditions are reported asynchronously by atomicOr into *dev_status
 * (nullable): TBA_DEV_TOKEN_RANGE — a token outside [0, vocab) at a valid position (S:50
 * invalid-input; that row's log-prob becomes NaN); TBA_DEV_NONFINITE_ROW — a valid row with
 * no finite maximum or a non-finite sum (e.g. all -inf, +inf or NaN logits).
 */
#ifndef TBA_H
#define TBA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* tba_stream_t; /* == cudaStream_t */

enum tba_status { TBA_OK = 0, TBA_ERR_INVALID_ARG = 1, TBA_ERR_INVALID_CONFIG = 2, TBA_ERR_CUDA = 3 };
enum tba_dev_status { TBA_DEV_TOKEN_RANGE = 1, TBA_DEV_NONFINITE_ROW = 2 };
enum tba_dtype { TBA_BF16 = 0, TBA_FP32 = 1 };

#define TBA_ABI_VERSION 1

/* The rows the head reads. All fields describe caller-owned device memory. */
typedef struct tba_rows {
  const void*    logits;      /* [n_seq, seq_len, row_stride] of `dtype`; 2-byte (bf16) / 4-byte aligned */
  int32_t        dtype;       /* TBA_BF16 or TBA_FP32 */
  int32_t        _pad;
  int64_t        n_seq;       /* N >= 0 */
  int64_t        seq_len;     /* T >= 0 */
  int64_t        vocab;       /* V >= 1 */
  int64_t        row_stride;  /* elements between consecutive rows, >= V */
  const int64_t* tokens;      /* [n_seq, seq_len] */
  const uint8_t* mask;        /* [n_seq, seq_len] */
} tba_rows;

int         tba_abi_version(void);
const char* tba_status_string(int code);

/* Bytes of device workspace the calls below need for N sequences of T rows: per-row
 * statistics (log2-domain max and log2 of the partition sum, 8 B), per-row log-prob (8 B),
 * per-group scratch (8 B/sequence) and a counter. Caller allocates; contents need not be
 * initialised; it must stay alive and unmodified from tba_vargrad_tb_loss_fwd until the
 * matching tba_vargrad_tb_loss_bwd. 256-byte aligned base required. */
size_t tba_workspace_bytes(int64_t n_seq, int64_t seq_len);

/* log pi(y_s | x) for every sequence (steps a1+a2; used for pi_theta and for pi_ref).
 *   seq_logp[s] = sum_{t: mask=1} log softmax(z_{s,t})[y_{s,t}]   (fp64, [N])
 *   n_tokens[s] = sum_t mask[s,t]                                  (int32, [N])
 * An all-zero mask row gives 0 and 0 (legal; reading R6). Logits are read once
 * (2V or 4V bytes per valid row; masked rows are not read). dev_status nullable. */
int tba_seq_logprob(const tba_rows* x, void* workspace, double* seq_logp, int32_t* n_tokens,
                    int32_t* dev_status, tba_stream_t stream);

/* Per-token log-probs (step a1 alone; SPEC's logprob per_token):
 *   tok_logp[s,t] = mask ? log softmax(inv_temp * z_{s,t})[y_{s,t}] : 0   (fp64, [N, T])
 * e.g. to record pi_gen log-probs for TBA' or per-token KL terms. inv_temp finite and > 0. */
int tba_token_logprob(const tba_rows* x, double inv_temp, void* workspace, double* tok_logp,
                      int32_t* dev_status, tba_stream_t stream);

/* Forward of the VarGrad TB loss over this call's groups (steps a1-a3), Eqs. 4-5.
 *   ref_logp[s]   = log pi_ref(y_s|x)  (fp64, [N]; e.g. from tba_seq_logprob on pi_ref logits)
 *   log_reward[s] = r_phi(y_s; x)       (fp64, [N]; the paper's r_phi, divided by beta here)
 *   beta > 0, K >= 2, n_seq % K == 0; n_seq_global = BK of the WHOLE batch (>= n_seq) —
 *   the 1/(BK) of Eq. 5, so that shards of one batch compose exactly.
 * Outputs (device, fp64 unless noted):
 *   seq_logp [N], n_tokens [N] (int32)   as tba_seq_logprob
 *   log_z    [N/K]  Eq. 4 (detached: STOP-GRAD)
 *   resid    [N]    eps_s = log_z_i + seq_logp_s - ref_logp_s - log_reward_s/beta (Eq. 5 bracket)
 *   partial  [3]    { sum_s eps_s^2 / n_seq_global, n_seq, n_seq/K }  — sum over ranks
 *                   (one allreduce) gives { L, N_global, B_global }.
 * Deterministic (fixed-order fp64 reductions, no float atomics). */
int tba_vargrad_tb_loss_fwd(const tba_rows* x, const double* ref_logp, const double* log_reward,
                            double beta, int32_t K, double n_seq_global, void* workspace,
                            double* seq_logp, int32_t* n_tokens, double* log_z, double* resid,
                            double* partial, int32_t* dev_status, tba_stream_t stream);

/* Backward (step a5): dlogits = dL/dz for L of Eq. 5, App. A:
 *   dz_{s,t,v} = mu_{s,t} * grad_scale * g * resid_s * (1[v = y_{s,t}] - softmax(z_{s,t})_v)
 * with g = *grad_out (device fp64 scalar; NULL means 1) and grad_scale = 2 / n_seq_global
 * (host scalar). Reads the row statistics the matching fwd left in `workspace`. Masked rows
 * are written with +0 and their logits are not read. Columns [vocab, dlogits_row_stride)
 * are not written. dlogits may alias logits exactly (same pointer, dtype and stride):
 * every element is read before it is written by the same thread.
 * dlogits_dtype TBA_BF16 (round-to-nearest-even) or TBA_FP32. */
int tba_vargrad_tb_loss_bwd(const tba_rows* x, const void* workspace, const double* resid,
                            double grad_scale, const double* grad_out, void* dlogits,
                            int32_t dlogits_dtype, int64_t dlogits_row_stride, tba_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Trajectory-balance head variants. The two calls above are these with
 * opts = NULL (VarGrad estimate, inv_temp = 1).
 *   log_z_param = NULL : log Z_i is the VarGrad K-sample estimate of Eq. 4, detached;
 *   log_z_param != NULL: log Z_i is a learned per-prompt scalar, Eq. 3 (the RT
 *                        trainer lineage of Lee et al.); resid uses it, log_z echoes it,
 *                        and tba_tb_loss_bwd returns dL/dlog Z_i = grad_scale * g * sum_j eps.
 *   inv_temp           : log pi = log softmax(inv_temp * z) (temperature-scaled policy; the
 *                        generation temperatures of P:511); must be finite and > 0, and
 *                        the same in the fwd and the matching bwd. 1.0 = the policy itself. */
typedef struct tba_tb_opts {
  double        inv_temp;
  const double* log_z_param; /* [n_seq/K] device fp64 or NULL */
} tba_tb_opts;

int tba_tb_loss_fwd(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp,
                    const double* log_reward, double beta, int32_t K, double n_seq_global,
                    void* workspace, double* seq_logp, int32_t* n_tokens, double* log_z,
                    double* resid, double* partial, int32_t* dev_status, tba_stream_t stream);

/* dz = mu * grad_scale * g * inv_temp * resid_s * (1[v=y] - softmax(inv_temp z)_v); d_log_z
 * (nullable, [n_seq/K]) receives dL/dlog Z for a learned log Z (K needed only then). */
int tba_tb_loss_bwd(const tba_rows* x, const tba_tb_opts* opts, const void* workspace,
                    const double* resid, double grad_scale, const double* grad_out, void* dlogits,
                    int32_t dlogits_dtype, int64_t dlogits_row_stride, double* d_log_z, int32_t K,
                    tba_stream_t stream);

/* One-launch forward + backward: the outputs of tba_tb_loss_fwd followed
 * by tba_tb_loss_bwd with grad_scale = 2 g / n_seq_global fixed at call time (g = 1 when the
 * loss is the training objective). A persistent kernel schedules forward rows, group heads and
 * gradient rows from one work counter, the backward of group i after the forward of group i+D;
 * when D groups of logits fit in L2 the backward re-read hits L2. Same results as the two-call
 * path (bitwise for resid/loss; dlogits identical). d_log_z as in tba_tb_loss_bwd. dlogits may
 * alias logits. */
int tba_tb_loss_fused(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp,
                      const double* log_reward, double beta, int32_t K, double n_seq_global,
                      double grad_scale, void* workspace, double* seq_logp, int32_t* n_tokens,
                      double* log_z, double* resid, double* partial, void* dlogits,
                      int32_t dlogits_dtype, int64_t dlogits_row_stride, double* d_log_z,
                      int32_t* dev_status, tba_stream_t stream);

/* Group-chunked, two-stream forward + backward (stream-level form):
 * the same outputs as tba_tb_loss_fwd + tba_tb_loss_bwd (bitwise: every row, head and the
 * final fixed-order reduction run the same arithmetic), scheduled in chunks of
 * groups_per_chunk whole groups (<= 0: as many groups as fit in ~1/4 of L2, at least 1).
 * For chunk c, `stream` runs the forward rows and the Eq. 4/5 head of c while `aux_stream`
 * runs the gradient writer of chunk c-1; the forward of chunk c+1 waits for the writer of
 * chunk c-1. When a chunk fits in L2, the writer's re-read of its logits hits L2 (4V instead
 * of 6V HBM bytes per token for groups of <= ~30 MB: the Pythia and red-teaming shapes).
 * Measured on B200 it is not faster than the two calls: small chunks pay
 * ~10 us of launch + cross-stream latency per chunk, large ones gain no reuse.
 * On return all work, including aux_stream's, is ordered before later work on `stream`
 * (capturable in a CUDA graph). aux_stream may equal stream (no overlap). d_log_z as in
 * tba_tb_loss_bwd (learned log Z only). dlogits may alias logits element-for-element (the
 * writer of chunk c-1 and the forward of chunk c touch disjoint rows). */
int tba_tb_loss_pipelined(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp,
                          const double* log_reward, double beta, int32_t K, double n_seq_global,
                          double grad_scale, int32_t groups_per_chunk, void* workspace, double* seq_logp,
                          int32_t* n_tokens, double* log_z, double* resid, double* partial, void* dlogits,
                          int32_t dlogits_dtype, int64_t dlogits_row_stride, double* d_log_z,
                          int32_t* dev_status, tba_stream_t stream, tba_stream_t aux_stream);

/* Deferred-scale forward: everything tba_tb_loss_fwd returns, plus
 * the UNSCALED gradient written in the same pass over the logits:
 *   grad_unscaled[s,t,v] = mu_{s,t} * inv_temp * (1[v = y] - softmax(inv_temp z)_v)
 * so that dL/dz = grad_scale * g * resid_s * grad_unscaled with grad_scale = 2 / n_seq_global.
 * The consumer (the LM-head backward) applies that per-sequence factor as a row scale. Each
 * valid row is read from HBM once and re-read on chip: one CTA per row, two per SM, the row's
 * first 96 KB kept in shared memory and the rest re-read from L2 (rows <= 128 KB: four CTAs per
 * SM, all from L2): 4V HBM bytes per token instead of 6V, plus the re-reads that miss L2
 * (DESIGN.md §5.4). grad_unscaled must not overlap logits at all (TBA_ERR_INVALID_ARG). */
int tba_tb_loss_fwd_deferred(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp,
                             const double* log_reward, double beta, int32_t K, double n_seq_global,
                             void* workspace, double* seq_logp, int32_t* n_tokens, double* log_z,
                             double* resid, double* partial, void* grad_unscaled, int32_t g_dtype,
                             int64_t g_row_stride, int32_t* dev_status, tba_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * TBA' token-level update: Eq. 16 (eq:tbaGrad), the rule
 * the paper scales to Qwen2.5-7B with PRIME-RL (§6; Table 5):
 *   grad J = sum_j sum_t sg( w(lambda_t) (r_j - rbar - beta (log Lambda_j - mean log Lambda)) )
 *            grad log pi_theta(y_t | x, y_<t)
 *   lambda_t = pi_theta(y_t)/pi_gen(y_t) = exp(lp_t - gen_logp_t)      (per token)
 *   log Lambda_j = log pi_theta(y_j|x) - log pi_ref(y_j|x) = seq_logp_j - ref_logp_j
 * IS weight w (is_mode): TBA_IS_NONE w = 1; TBA_IS_CLIP w = clamp(lambda, is_lo, is_hi)
 * (CISPO bounds 0/8, Table 5); TBA_IS_ICEPOP w = lambda inside [is_lo, is_hi], else 0
 * (masking; reading R14). Normalisation (the paper's "GRPO-style",
 * P:708): by the global number of valid tokens n_tok_global (reading R15). The value
 * returned is the surrogate loss whose gradient is -grad J / n_tok_global:
 *   partial = { -(1/n_tok_global) sum_{valid t} coef_t * lp_t, n_tok (this call), n_seq }
 * Outputs: seq_logp [N], n_tokens [N], adv [N] (the bracket A_j), coef [N, T] fp32
 * (w * A_j, 0 where masked). beta >= 0 (beta = 0 is Dr. GRPO); K >= 2. */
enum tba_is_mode { TBA_IS_NONE = 0, TBA_IS_CLIP = 1, TBA_IS_ICEPOP = 2 };

int tba_tbap_loss_fwd(const tba_rows* x, const float* gen_logp /* [N, T] fp32, pi_gen log-probs */,
                      const double* ref_logp, const double* log_reward, double beta, int32_t K, int32_t is_mode,
                      double is_lo, double is_hi, double n_tok_global, void* workspace, double* seq_logp,
                      int32_t* n_tokens, double* adv, float* coef, double* partial, int32_t* dev_status,
                      tba_stream_t stream);

/* TBA' with the deferred-scale row pass (as tba_tb_loss_fwd_deferred): also writes
 * grad_unscaled = mu (1[v=y] - softmax) in the same pass; dL'/dz = -(coef_{s,t} / n_tok_global) *
 * g * grad_unscaled (a per-token row scale applied by the consumer). */
int tba_tbap_loss_fwd_deferred(const tba_rows* x, const float* gen_logp, const double* ref_logp,
                               const double* log_reward, double beta, int32_t K, int32_t is_mode,
                               double is_lo, double is_hi, double n_tok_global, void* workspace,
                               double* seq_logp, int32_t* n_tokens, double* adv, float* coef,
                               double* partial, void* grad_unscaled, int32_t g_dtype,
                               int64_t g_row_stride, int32_t* dev_status, tba_stream_t stream);

/* dlogits for the TBA' surrogate: dz_{s,t,v} = mu * grad_scale * g * coef_{s,t} (1[v=y] - softmax_v)
 * with grad_scale = -1 / n_tok_global; otherwise as tba_vargrad_tb_loss_bwd. */
int tba_tbap_loss_bwd(const tba_rows* x, const void* workspace, const float* coef, double grad_scale,
                      const double* grad_out, void* dlogits, int32_t dlogits_dtype, int64_t dlogits_row_stride,
                      tba_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * LM-head-fused head, forward: the same log pi(y|x) and Eq. 4/5
 * outputs, computed from the final hidden states and the LM-head weight WITHOUT writing
 * the logits. "Parallel likelihood evaluation of an entire sequence through a single
 * forward pass" ends in z_{s,t} = W h_{s,t}; here that contraction runs on the
 * tcgen05 tensor cores (bf16 operands, fp32 accumulation in TMEM) and its epilogue folds
 * each 128 x 256 logit tile into the row's online log-sum-exp and gathers z[y], so the
 * [N, T, V] logits (20 GB at the Qwen shard) never reach HBM.
 *   hidden : bf16, row (s, t) at hidden + (s*seq_len + t) * hidden_stride elements, d used
 *   weight : bf16 [vocab, d], row v at weight + v * weight_stride elements (no bias)
 *   z_{s,t,v} = sum_i hidden[s,t,i] * weight[v,i]   (fp32 accumulation, any order)
 * Requirements (TBA_ERR_INVALID_ARG otherwise): d >= 8, d and both strides multiples of 8
 * elements, hidden/weight 16-byte aligned, n_seq*seq_len <= 2^31 - 1, vocab <= 2^31 - 1.
 * tokens / mask as in tba_rows. Numerics: the logits carry the fp32 accumulation error of
 * a d-term dot product; the softmax epilogue is as accurate as the row
 * kernels'. The backward through the head (dL/dhidden, dL/dW) is tba_lmhead_tb_loss_bwd /
 * tba_lmhead_tbap_loss_bwd below. */
typedef struct tba_lmhead {
  const void*    hidden;         /* bf16 */
  const void*    weight;         /* bf16 */
  int64_t        n_seq;          /* N >= 0 */
  int64_t        seq_len;        /* T >= 0 */
  int64_t        d;              /* hidden size */
  int64_t        vocab;          /* V >= 1 */
  int64_t        hidden_stride;  /* elements between consecutive hidden rows, >= d */
  int64_t        weight_stride;  /* elements between consecutive weight rows, >= d */
  const int64_t* tokens;         /* [n_seq, seq_len] */
  const uint8_t* mask;           /* [n_seq, seq_len] */
} tba_lmhead;

/* Workspace for the two calls below: tba_workspace_bytes(n_seq, seq_len) plus the per-(row,
 * vocab group of 1024) partial {max, sum} and the gathered logit (256-B aligned base). */
size_t tba_lmhead_workspace_bytes(int64_t n_seq, int64_t seq_len, int64_t vocab);

/* tba_seq_logprob from hidden states: seq_logp[s] = sum_t mask * log softmax(inv_temp z)[y]. */
int tba_lmhead_seq_logprob(const tba_lmhead* x, double inv_temp, void* workspace, double* seq_logp,
                           int32_t* n_tokens, int32_t* dev_status, tba_stream_t stream);

/* tba_token_logprob from hidden states: tok_logp[s,t] = mask ? log softmax(inv_temp z)[y] : 0. */
int tba_lmhead_token_logprob(const tba_lmhead* x, double inv_temp, void* workspace, double* tok_logp,
                             int32_t* dev_status, tba_stream_t stream);

/* tba_tbap_loss_fwd (TBA', Eq. 16) from hidden states: same outputs; gen_logp [N, T] fp32. */
int tba_lmhead_tbap_loss_fwd(const tba_lmhead* x, const float* gen_logp, const double* ref_logp,
                             const double* log_reward, double beta, int32_t K, int32_t is_mode, double is_lo,
                             double is_hi, double n_tok_global, void* workspace, double* seq_logp,
                             int32_t* n_tokens, double* adv, float* coef, double* partial, int32_t* dev_status,
                             tba_stream_t stream);

/* tba_tb_loss_fwd from hidden states (Eqs. 4-5 / Eq. 3; opts as there). */
int tba_lmhead_tb_loss_fwd(const tba_lmhead* x, const tba_tb_opts* opts, const double* ref_logp,
                           const double* log_reward, double beta, int32_t K, double n_seq_global,
                           void* workspace, double* seq_logp, int32_t* n_tokens, double* log_z,
                           double* resid, double* partial, int32_t* dev_status, tba_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * LM-head-fused backward: the gradient of the TB / TBA' loss with
 * respect to the hidden states and the LM-head weight, by the chain rule through z = W h
 * applied to App. A:
 *   dz_{r,v}   = c_r (1[v = y_r] - softmax(inv_temp z_r)_v)       (0 where mask == 0)
 *   dhidden_r  = sum_v dz_{r,v} W_v          (bf16 or fp32, [n_seq, seq_len] rows of d)
 *   dweight_v  = sum_r dz_{r,v} hidden_r     (fp32 [vocab] rows of d)
 * with c_r = grad_scale * g * inv_temp * resid_s (TB: the matching tba_lmhead_tb_loss_fwd's
 * resid, s = r / seq_len) or grad_scale * g * coef_r (TBA': tba_lmhead_tbap_loss_fwd's coef),
 * g = *grad_out (NULL = 1). The logits are recomputed on the tensor cores tile by tile from
 * the forward's row statistics (`workspace` of the matching forward, unmodified since); dz
 * is formed in bf16 (round-to-nearest-even) for the two gradient GEMMs, which accumulate in
 * fp32. Valid rows are processed in compacted chunks of chunk_rows (<= 0: 16384; rounded
 * up to a multiple of 128), so the per-call memory is bwd_workspace, not [rows, V].
 *   dhidden / dweight: either may be NULL (that gradient is skipped). Row strides in elements
 *   (>= d). dhidden must not alias hidden. accumulate = 0 overwrites (masked rows of dhidden
 *   are written with 0), accumulate = 1 adds into the existing contents (micro-batching).
 *   d_log_z (TB only, nullable): dL/dlog Z_i for a learned log Z, as in tba_tb_loss_bwd.
 * dhidden may be summed over up to 4 slices of the vocabulary (split-K: fixed slice bounds that
 * depend on d, vocab and the SM count only, added in slice order).
 * Deterministic: fixed tile order, no atomics. bwd_workspace: 256-byte aligned, of
 * tba_lmhead_bwd_workspace_bytes(n_seq, seq_len, d, vocab, chunk_rows) bytes. */
size_t tba_lmhead_bwd_workspace_bytes(int64_t n_seq, int64_t seq_len, int64_t d, int64_t vocab,
                                      int64_t chunk_rows);

int tba_lmhead_tb_loss_bwd(const tba_lmhead* x, const tba_tb_opts* opts, const void* workspace,
                           const double* resid, double grad_scale, const double* grad_out, void* dhidden,
                           int32_t dhidden_dtype, int64_t dhidden_row_stride, float* dweight,
                           int64_t dweight_row_stride, int32_t accumulate, double* d_log_z, int32_t K,
                           int64_t chunk_rows, void* bwd_workspace, tba_stream_t stream);

int tba_lmhead_tbap_loss_bwd(const tba_lmhead* x, const void* workspace, const float* coef, double grad_scale,
                             const double* grad_out, void* dhidden, int32_t dhidden_dtype,
                             int64_t dhidden_row_stride, float* dweight, int64_t dweight_row_stride,
                             int32_t accumulate, int64_t chunk_rows, void* bwd_workspace, tba_stream_t stream);

/* One-call forward + backward from hidden states: the outputs of
 * tba_lmhead_tb_loss_fwd followed by tba_lmhead_tb_loss_bwd with grad_scale = 2 g / n_seq_global
 * fixed at call time, scheduled over chunks of groups_per_chunk WHOLE groups (<= 0: as many as
 * fit in 16384 rows, at least 1). Eq. 4 couples only the K samples of one prompt, so once a
 * chunk's forward and head are done its gradient is final: the forward's epilogue also stores
 * the chunk's logits in fp32 (bwd_workspace), and the gradient pass forms dz from them instead
 * of recomputing z = W h (one GEMM of three fewer than the two calls). Same results as the two
 * calls (seq_logp, resid, log_z, loss bitwise; the logits the gradient uses are the same fp32
 * tensor-core values). bwd_workspace: tba_lmhead_fwd_bwd_workspace_bytes(...) bytes (256-B
 * aligned); workspace: tba_lmhead_workspace_bytes(...) as for the forward. */
size_t tba_lmhead_fwd_bwd_workspace_bytes(int64_t n_seq, int64_t seq_len, int64_t d, int64_t vocab, int32_t K,
                                          int32_t groups_per_chunk);

int tba_lmhead_tb_loss_fwd_bwd(const tba_lmhead* x, const tba_tb_opts* opts, const double* ref_logp,
                               const double* log_reward, double beta, int32_t K, double n_seq_global,
                               double grad_scale, int32_t groups_per_chunk, void* workspace, double* seq_logp,
                               int32_t* n_tokens, double* log_z, double* resid, double* partial, void* dhidden,
                               int32_t dhidden_dtype, int64_t dhidden_row_stride, float* dweight,
                               int64_t dweight_row_stride, int32_t accumulate, double* d_log_z,
                               void* bwd_workspace, int32_t* dev_status, tba_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* TBA_H */
