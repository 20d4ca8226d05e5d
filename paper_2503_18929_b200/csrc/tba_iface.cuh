// libtba.so — the trajectory-balance loss head of TBA (arXiv 2503.18929) for B200 (sm_100a).
//
// Internal interface between the translation units of the library (one TU per kernel family,
// compiled in parallel; abi.cu holds the extern "C" entry points of include/tba.h and launches
// nothing itself). Kernels:
//   fwd.cu       row_fwd_rows  a1   stream each valid logits row from HBM once (TPR threads per
//                                   row, 128-bit loads): online max + sum of 2^(z*sc - R2), one
//                                   ex2 per element (packed FFMA2/FADD2; 1 of 4 pairs on the FMA
//                                   pipe), gather z[y]; the token's own term kept out of the
//                                   sum; writes per-row (M2, log2 S), 1 - p_y and the token
//                                   log-prob (fp64). PDL-chained to seq_head and row_bwd.
//   head.cu      seq_head      a2+a3 per-sequence fixed-order fp64 sums of token log-probs
//                                   (log pi(y|x)) and token counts; per group Eq. 4 log Z (or a
//                                   learned log Z, Eq. 3) and the Eq. 5 residuals; the last CTA
//                                   reduces the per-group sums of squares.
//                tbap_head     a2+a3' TBA' (Eq. 16): per-group advantages, per-token IS-weighted
//                                   coefficients.
//   bwd.cu       row_bwd       a5   stream each valid row again: dz = c (1[v=y] - softmax); c per
//                                   sequence (TB) or per token (TBA'); masked rows zero-filled.
//   fused.cu     tb_fused      a1-a5 in one persistent launch (NEXT 2 (i)).
//   deferred.cu  row_single1   a1 + unscaled a5 in one pass per row (NEXT 2 (ii)): pass 1 from HBM
//                                   (long rows: the first 96 KB into shared memory by cp.async), pass 2
//                                   from shared memory and L2.
//   lmhead*.cu   NEXT 3: the tcgen05 LM-head GEMMs (forward with the softmax epilogue, dz / dH / dW).
// No float atomics: every output is bitwise reproducible run to run.
#pragma once
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "../../include/tba.h"

namespace tba {

constexpr float kL2E = 1.4426950408889634f;  // fp32(log2 e)
constexpr double kLN2 = 0.69314718055994530942;
constexpr float kSlack = 6.0f;  // nats a chunk max may exceed the running reference before a re-base
constexpr int kFusedU = 4;
constexpr int kU = 4;
constexpr int64_t kSmallRowBytes = 8192;  // rows up to 8 KB: one warp per row in the backward

// Row scaling: rows are soft-maxed as 2^(z * sc) with sc = fl(kL2E * inv_temp); slack is kSlack in
// logit units (kSlack / inv_temp); inv_temp enters the log-prob and the gradient exactly (fp64).
struct RowScale {
  float sc, slack;
  double inv_temp;
};

// Arguments of the per-sequence sums and the Eq. 4/5 group head (seq_head).
struct HeadArgs {
  int64_t T;
  int K;             // sequences per unit (1 = log-probs only)
  int head;          // 1 = TB head per group
  int64_t n_seq;
  const double* ref_logp;
  const double* log_reward;
  const double* log_z_param;
  double inv_beta, inv_n_global;
  double* seq_logp;
  int32_t* n_tokens;
  double* log_z;
  double* resid;
  double* group_sq;
  double* partial;
};

// One persistent launch for the whole VarGrad TB step: forward rows, the group head and the
// gradient writer, scheduled from one atomic work counter over an item stream in which the
// forward items of group g+D precede the backward items of group g. The CTA finishing the
// last forward row of a group computes its head (Eq. 4/5) and publishes a ready flag; backward
// items of that group wait on it. When D groups of logits fit in L2, the backward re-read of a
// group hits L2 (6V -> ~4V HBM bytes per token for short-response shapes: Pythia, red-teaming);
// for large groups (Qwen) it is a single-launch schedule with fwd/bwd overlap.
struct FusedArgs {
  const void* logits;
  void* dlogits;
  const int64_t* tokens;
  const uint8_t* mask;
  const double* ref_logp;
  const double* log_reward;
  const double* log_z_param;
  float2* stats;
  float* qy;
  double* lp;
  double* seq_logp;
  int32_t* n_tokens;
  double* log_z;
  double* resid;
  double* group_sq;
  double* partial;
  int32_t* dev_status;
  unsigned int* work;        // [1] item counter
  unsigned int* groups_done; // [1]
  unsigned int* rows_done;   // [groups]
  unsigned int* ready;       // [groups]
  int64_t rows, T, V, stride, ostride, n_seq;
  int K, groups, D, nF, nB, RF, RB;
  double inv_beta, inv_n_global, grad_scale;
  RowScale rs;
};

// ------------------------------------------------------------------------------ host helpers
inline RowScale make_scale(double inv_temp) {
  RowScale r;
  r.sc = (float)((double)kL2E * inv_temp);
  r.slack = (float)((double)kSlack / inv_temp);
  r.inv_temp = inv_temp;
  return r;
}

// Workspace (tba_workspace_bytes): per-row stats, per-row fp64 log-probs, per-group sums of
// squares, the last-CTA counter, and the fused/fused-head counters; each block 256-byte aligned.
struct WsLayout {
  float2* stats;
  double* lp;
  double* group_sq;
  unsigned int* counter;
  unsigned int* fused;
  float* qy;  // per row: 1 - p_y (the token's complement probability, exact when p_y -> 1)
};

inline size_t fused_counter_bytes(int64_t n_seq) { return (size_t)(2 + 2 * n_seq) * sizeof(unsigned int); }

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

inline WsLayout ws_layout(void* ws, int64_t n_seq, int64_t T) {
  const size_t rows = (size_t)n_seq * (size_t)T;
  char* p = static_cast<char*>(ws);
  WsLayout l;
  size_t off = 0;
  l.stats = reinterpret_cast<float2*>(p + off);
  off = align_up(off + rows * sizeof(float2), 256);
  l.lp = reinterpret_cast<double*>(p + off);
  off = align_up(off + rows * sizeof(double), 256);
  l.group_sq = reinterpret_cast<double*>(p + off);
  off = align_up(off + (size_t)n_seq * sizeof(double), 256);
  l.counter = reinterpret_cast<unsigned int*>(p + off);
  off = align_up(off + 4 * sizeof(unsigned int), 256);
  l.fused = reinterpret_cast<unsigned int*>(p + off);  // work, groups_done, rows_done[n_seq], ready[n_seq]
  off = align_up(off + fused_counter_bytes(n_seq), 256);
  l.qy = reinterpret_cast<float*>(p + off);
  return l;
}

inline size_t ws_bytes(int64_t n_seq, int64_t T) {
  const size_t rows = (size_t)n_seq * (size_t)T;
  return align_up(rows * sizeof(float2), 256) + align_up(rows * sizeof(double), 256) +
         align_up((size_t)n_seq * sizeof(double), 256) + 256 + align_up(fused_counter_bytes(n_seq), 256) +
         align_up(rows * sizeof(float), 256);
}

inline int validate_rows(const tba_rows* x) {
  if (!x) return TBA_ERR_INVALID_ARG;
  if (x->dtype != TBA_BF16 && x->dtype != TBA_FP32) return TBA_ERR_INVALID_ARG;
  if (x->n_seq < 0 || x->seq_len < 0 || x->vocab < 1 || x->row_stride < x->vocab) return TBA_ERR_INVALID_ARG;
  const int64_t esz = x->dtype == TBA_BF16 ? 2 : 4;
  const int64_t lim = INT64_MAX / 8;
  if (x->n_seq > 0 && x->seq_len > lim / x->n_seq) return TBA_ERR_INVALID_ARG;
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows > 0 && x->row_stride > lim / esz / rows) return TBA_ERR_INVALID_ARG;
  if (rows > (int64_t)INT32_MAX / 4) return TBA_ERR_INVALID_ARG;  // grid.x limit (up to 4 CTAs per row)
  if (rows > 0) {
    if (!x->logits || !x->tokens || !x->mask) return TBA_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(x->logits) % esz) return TBA_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(x->tokens) % 8) return TBA_ERR_INVALID_ARG;
  }
  return TBA_OK;
}

inline int64_t esz_of(int32_t dt) { return dt == TBA_BF16 ? 2 : 4; }

// Do [a, a + span_a) and [b, b + span_b) intersect, each the bytes of `rows` rows of `vocab`
// elements at the given row stride (the last row ends at its vocab-th element)?
inline bool ranges_overlap(const void* a, int64_t rows, int64_t a_stride, int64_t vocab, int64_t a_esz, const void* b,
                           int64_t b_stride, int64_t b_esz) {
  if (rows <= 0) return false;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  const uintptr_t a1 = a0 + (uintptr_t)(((rows - 1) * a_stride + vocab) * a_esz);
  const uintptr_t b1 = b0 + (uintptr_t)(((rows - 1) * b_stride + vocab) * b_esz);
  return a0 < b1 && b0 < a1;
}

inline int validate_out(const tba_rows* x, const void* dlogits, int32_t odt, int64_t ostride) {
  if (odt != TBA_BF16 && odt != TBA_FP32) return TBA_ERR_INVALID_ARG;
  if (ostride < x->vocab) return TBA_ERR_INVALID_ARG;
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows == 0) return TBA_OK;
  const int64_t oesz = odt == TBA_BF16 ? 2 : 4;
  if (ostride > INT64_MAX / 8 / oesz / rows) return TBA_ERR_INVALID_ARG;
  if (!dlogits || reinterpret_cast<uintptr_t>(dlogits) % oesz) return TBA_ERR_INVALID_ARG;
  // Aliasing: only element-for-element (same base, dtype and row stride); any other overlap of the
  // two byte ranges would let one row's writes clobber logits another thread still reads.
  if (dlogits == x->logits) {
    if (odt != x->dtype || ostride != x->row_stride) return TBA_ERR_INVALID_ARG;
  } else if (ranges_overlap(x->logits, rows, x->row_stride, x->vocab, esz_of(x->dtype), dlogits, ostride, oesz)) {
    return TBA_ERR_INVALID_ARG;
  }
  return TBA_OK;
}

// The output of a row pass that re-reads its rows (deferred scale) may not overlap them at all.
inline bool out_overlaps_rows(const tba_rows* x, const void* out, int64_t ostride, int32_t odt) {
  const int64_t rows = x->n_seq * x->seq_len;
  return rows > 0 && ranges_overlap(x->logits, rows, x->row_stride, x->vocab, esz_of(x->dtype), out, ostride,
                                    odt == TBA_BF16 ? 2 : 4);
}

inline int device_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  static int cache[64] = {0};
  if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cache[dev] = n;
  return n;
}

// Environment overrides of the two non-default schedules' chunking (tba_tb_loss_fused's lookahead,
// tba_tb_loss_pipelined's default chunk), read ONCE per process; never consulted by the default
// two-call path.
inline int env_once(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Forward threads per row, measured on B200: one warp per row (8 rows per CTA) for
// rows under 128 KB (Pythia, red-teaming, the GSM8K / RhoMath presets: forward 1-3 % faster with the
// polynomial offload), 64 threads (4 rows per CTA) for the 304 KB Qwen rows.
inline int fwd_tpr(int64_t V, int64_t esz) { return (V * esz / 16) < 8192 ? 32 : 64; }

// Backward threads per row: one CTA per long row, one warp per short row.
inline int bwd_tpr(int64_t V, int64_t esz) { return V * esz <= kSmallRowBytes ? 32 : 256; }

// Groups of look-ahead in the fused schedule: as many groups of logits as fit in ~35 % of L2.
inline int fused_lookahead(int64_t group_bytes, int groups) {
  static const int env = env_once("TBA_FUSED_D", -1);
  int d;
  if (env >= 0) {
    d = env;
  } else {
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess || l2 <= 0) l2 = 126 << 20;
    d = (int)(0.35 * (double)l2 / (double)(group_bytes > 0 ? group_bytes : 1));
  }
  if (d < 1) d = 1;
  if (d > groups) d = groups;
  return d;
}

// Groups per chunk of the pipelined schedule: chunks of <= ~1/4 of L2, so that chunk c (being
// re-read by the gradient writer) and chunk c+1 (being read by the forward) both stay resident.
inline int pipe_groups(int64_t group_bytes, int64_t groups) {
  static const int env = env_once("TBA_PIPE_GROUPS", 0);
  int d = env;
  if (d <= 0) {
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess || l2 <= 0) l2 = 126 << 20;
    d = (int)(0.25 * (double)l2 / (double)(group_bytes > 0 ? group_bytes : 1));
  }
  if (d < 1) d = 1;
  if (d > groups) d = (int)groups;
  return d;
}

// tba_lmhead: sizes, strides and alignment the TMA tensor maps need (16-byte strides, int32
// coordinates), and the row-count limit shared with tba_rows.
inline int validate_lmhead(const tba_lmhead* x) {
  if (!x) return TBA_ERR_INVALID_ARG;
  if (x->n_seq < 0 || x->seq_len < 0 || x->vocab < 1 || x->vocab > (int64_t)INT32_MAX) return TBA_ERR_INVALID_ARG;
  if (x->d < 8 || x->d % 8 || x->hidden_stride < x->d || x->hidden_stride % 8 || x->weight_stride < x->d ||
      x->weight_stride % 8 || x->d > (int64_t)1 << 24)
    return TBA_ERR_INVALID_ARG;
  if (x->n_seq > 0 && x->seq_len > (int64_t)INT32_MAX / x->n_seq) return TBA_ERR_INVALID_ARG;
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows > 0) {
    if (!x->hidden || !x->weight || !x->tokens || !x->mask) return TBA_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(x->hidden) % 16 || reinterpret_cast<uintptr_t>(x->weight) % 16 ||
        reinterpret_cast<uintptr_t>(x->tokens) % 8)
      return TBA_ERR_INVALID_ARG;
  }
  return TBA_OK;
}

inline int check_opts(const tba_tb_opts* o) {
  if (!o) return TBA_OK;
  if (!(std::isfinite(o->inv_temp) && o->inv_temp > 0.0)) return TBA_ERR_INVALID_CONFIG;
  return TBA_OK;
}

inline double opt_inv_temp(const tba_tb_opts* o) { return o ? o->inv_temp : 1.0; }

inline int launch_status() { return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA; }

// Launch with programmatic dependent launch (see pdl_trigger / pdl_wait in tba_device.cuh): the
// kernel may be scheduled before the previous kernel in `s` finishes and waits for it on the device.
template <class... KArgs, class... Args>
inline int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
#ifdef TBA_AB_NO_PDL
  cfg.numAttrs = 0;
#else
  cfg.numAttrs = 1;
#endif
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

// ------------------------------------------------------------------------------ launchers
// Defined in the kernel TUs; each returns a TBA_* status (launch errors included).

// fwd.cu — a1 over every row of x: per-row stats + fp64 token log-probs into the workspace.
int launch_fwd_rows(const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status, cudaStream_t s);

// head.cu
// seq_head: HEAD = false -> log pi(y|x) and counts only (ha.K ignored); true -> + Eq. 4/5 head.
int launch_seq_head(bool head, const WsLayout& w, const uint8_t* mask, const HeadArgs& ha, cudaStream_t s);
int launch_tbap_head(const WsLayout& w, const uint8_t* mask, const float* gen_logp, int64_t n_seq, int64_t T, int K,
                     const double* ref_logp, const double* log_reward, double beta, int is_mode, double is_lo,
                     double is_hi, double neg_inv_ntok, double* seq_logp, int32_t* n_tokens, double* adv,
                     float* coef, double* partial, cudaStream_t s);
int launch_token_lp(const WsLayout& w, const uint8_t* mask, int64_t rows, double* tok_logp, cudaStream_t s);
// The final fixed-order loss reduction over group_sq[0, groups) (a chunked step's tail).
int launch_tb_finish(const double* group_sq, int64_t groups, int64_t n_seq, double inv_n_global, double* partial,
                     cudaStream_t s);
int launch_dlogz(const double* resid, int64_t groups, int K, double grad_scale, const double* grad_out,
                 double* d_log_z, cudaStream_t s);

// bwd.cu — a5: per_row = false: c = resid[s] (TB); true: c = coef[row] (TBA').
int launch_bwd(bool per_row, const tba_rows* x, const float2* stats, const float* qy, const double* resid,
               const float* coef,
               double gs, const double* go, const RowScale& rs, void* dlogits, int32_t odt, int64_t ostride,
               cudaStream_t s);

// fused.cu — the whole VarGrad TB step (a.* filled except nF/nB/RF/RB, set here).
int launch_fused(FusedArgs& a, int32_t in_dtype, int32_t out_dtype, int tpr_f, int tpr_b, cudaStream_t s);

// lmhead.cu — a1 from hidden states: tcgen05 LM-head GEMM with the online log-softmax in its
// epilogue + the fixed-order group combine; writes w.stats / w.lp like launch_fwd_rows.
size_t lmhead_partial_bytes(int64_t rows, int64_t V);
// zst (nullable): also store the fp32 logits, row r at zst + r * zst_ld (16-byte aligned rows).
int launch_lmhead_rows(const tba_lmhead* x, void* part_ws, const WsLayout& w, const RowScale& rs, int32_t* dev_status,
                       cudaStream_t s, float* zst = nullptr, int64_t zst_ld = 0);

// lmhead_bwd.cu — backward through the LM head (dz recomputed on the tensor cores, dH = dZ W,
// dW (+)= dZ^T H) over compacted chunks of valid rows. Per-row coefficient c_r = gs * g *
// (coef ? coef[r] : resid[r / T]); sc = fl(log2(e) inv_temp).
int64_t lmhead_bwd_chunk(int64_t rows, int64_t chunk_rows);
size_t lmhead_bwd_ws_bytes(int64_t rows, int64_t d, int64_t V, int64_t chunk_rows);
int launch_lmhead_bwd(const tba_lmhead* x, const float2* stats, const double* resid, const float* coef, double gs,
                      const double* grad_out, float sc, void* dh, int32_t dh_dt, int64_t dh_stride, float* dw,
                      int64_t dw_stride, bool accumulate, int64_t chunk_rows, void* bws, cudaStream_t s);
// One-call forward + backward from hidden states over chunks of whole groups: per chunk the forward
// (logits also stored in fp32), the Eq. 4/5 head, dz from the stored logits, dH and dW; then the
// fixed-order loss reduction into ha0.partial. ha0 = tb_head_args of the whole call.
size_t lmhead_fb_ws_bytes(int64_t n_seq, int64_t T, int64_t d, int64_t V, int32_t K, int32_t groups_per_chunk);
int launch_lmhead_fwd_bwd(const tba_lmhead* x, const RowScale& rs, const WsLayout& w, const HeadArgs& ha0, int32_t K,
                          double grad_scale, double inv_n_global, void* dh, int32_t dh_dt, int64_t dh_stride, float* dw,
                          int64_t dw_stride, bool accumulate, int32_t groups_per_chunk, void* bws,
                          int32_t* dev_status, cudaStream_t s);

// deferred.cu — a1 + the unscaled gradient in one pass per row.
int launch_single(const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status,
                  void* grad_unscaled, int32_t g_dtype, int64_t g_row_stride, cudaStream_t s);

}  // namespace tba
