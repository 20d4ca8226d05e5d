// The C ABI of libtba.so (include/tba.h): argument validation, workspace carving and launch
// order. Every step of the path runs in the kernels of fwd.cu / head.cu / bwd.cu / fused.cu /
// deferred.cu; nothing here computes on the host.
#include "tba_iface.cuh"

using namespace tba;

namespace {

// The Eq. 4/5 group-head arguments shared by the two-call and deferred forwards.
HeadArgs tb_head_args(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp, const double* log_reward,
                      double beta, int32_t K, double n_seq_global, const WsLayout& w, double* seq_logp,
                      int32_t* n_tokens, double* log_z, double* resid, double* partial) {
  HeadArgs ha{};
  ha.T = x->seq_len;
  ha.K = K;
  ha.head = 1;
  ha.n_seq = x->n_seq;
  ha.ref_logp = ref_logp;
  ha.log_reward = log_reward;
  ha.log_z_param = opts ? opts->log_z_param : nullptr;
  ha.inv_beta = 1.0 / beta;
  ha.inv_n_global = 1.0 / n_seq_global;
  ha.seq_logp = seq_logp;
  ha.n_tokens = n_tokens;
  ha.log_z = log_z;
  ha.resid = resid;
  ha.group_sq = w.group_sq;
  ha.partial = partial;
  return ha;
}

// Four timing-free events per (host thread, device) for the pipelined schedule, created on first
// use and reused: a wait always refers to the latest record issued before it, so reuse across
// calls is safe, and thread-local storage keeps concurrent callers on other threads apart.
cudaEvent_t* pipe_events() {
  thread_local cudaEvent_t ev[64][4] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!ev[dev][0])
    for (int i = 0; i < 4; ++i)
      if (cudaEventCreateWithFlags(&ev[dev][i], cudaEventDisableTiming) != cudaSuccess) return nullptr;
  return ev[dev];
}

// Any byte overlap between the LM-head backward's outputs (dhidden, dweight) and its inputs (hidden,
// weight, both re-read chunk by chunk) or each other.
bool lm_outputs_overlap(const tba_lmhead* x, const void* dh, int64_t dh_stride, int32_t dh_dt, const float* dw,
                        int64_t dw_stride) {
  const int64_t rows = x->n_seq * x->seq_len, d = x->d, V = x->vocab, dhe = esz_of(dh_dt);
  auto span_hit = [](const void* a, int64_t na, int64_t sa, int64_t ea, const void* b, int64_t nb, int64_t sb,
                     int64_t eb, int64_t cols) {
    if (!a || !b || na <= 0 || nb <= 0) return false;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
    const uintptr_t a1 = a0 + (uintptr_t)(((na - 1) * sa + cols) * ea), b1 = b0 + (uintptr_t)(((nb - 1) * sb + cols) * eb);
    return a0 < b1 && b0 < a1;
  };
  return span_hit(dh, rows, dh_stride, dhe, x->hidden, rows, x->hidden_stride, 2, d) ||
         span_hit(dh, rows, dh_stride, dhe, x->weight, V, x->weight_stride, 2, d) ||
         span_hit(dw, V, dw_stride, 4, x->hidden, rows, x->hidden_stride, 2, d) ||
         span_hit(dw, V, dw_stride, 4, x->weight, V, x->weight_stride, 2, d) ||
         span_hit(dh, rows, dh_stride, dhe, dw, V, dw_stride, 4, d);
}

}  // namespace

// ================================================================================ C ABI
extern "C" {

int tba_abi_version(void) { return TBA_ABI_VERSION; }

const char* tba_status_string(int code) {
  switch (code) {
    case TBA_OK: return "TBA_OK";
    case TBA_ERR_INVALID_ARG: return "TBA_ERR_INVALID_ARG: invalid argument (null pointer, size, stride, alignment or N % K)";
    case TBA_ERR_INVALID_CONFIG: return "TBA_ERR_INVALID_CONFIG: invalid configuration (beta, K, IS mode or temperature)";
    case TBA_ERR_CUDA: return "TBA_ERR_CUDA: CUDA launch failed";
    default: return "TBA: unknown status";
  }
}

size_t tba_workspace_bytes(int64_t n_seq, int64_t seq_len) {
  if (n_seq < 0 || seq_len < 0) return 0;
  return ws_bytes(n_seq, seq_len);
}

int tba_seq_logprob(const tba_rows* x, void* workspace, double* seq_logp, int32_t* n_tokens, int32_t* dev_status,
                    tba_stream_t stream) {
  int rc = validate_rows(x);
  if (rc) return rc;
  if (x->n_seq == 0) return TBA_OK;
  if (!workspace || !seq_logp || !n_tokens) return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  HeadArgs ha{};
  ha.T = x->seq_len;
  ha.K = 1;
  ha.head = 0;
  ha.n_seq = x->n_seq;
  ha.seq_logp = seq_logp;
  ha.n_tokens = n_tokens;
  rc = launch_fwd_rows(x, w, make_scale(1.0), dev_status, s);
  if (rc) return rc;
  return launch_seq_head(false, w, x->mask, ha, s);
}

int tba_token_logprob(const tba_rows* x, double inv_temp, void* workspace, double* tok_logp, int32_t* dev_status,
                      tba_stream_t stream) {
  int rc = validate_rows(x);
  if (rc) return rc;
  if (!(std::isfinite(inv_temp) && inv_temp > 0.0)) return TBA_ERR_INVALID_CONFIG;
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows == 0) return TBA_OK;
  if (!workspace || !tok_logp || reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  rc = launch_fwd_rows(x, w, make_scale(inv_temp), dev_status, s);
  if (rc) return rc;
  return launch_token_lp(w, x->mask, rows, tok_logp, s);
}

int tba_tb_loss_fwd(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp, const double* log_reward,
                    double beta, int32_t K, double n_seq_global, void* workspace, double* seq_logp, int32_t* n_tokens,
                    double* log_z, double* resid, double* partial, int32_t* dev_status, tba_stream_t stream) {
  if (!(std::isfinite(beta) && beta > 0.0)) return TBA_ERR_INVALID_CONFIG;
  if (K < 2) return TBA_ERR_INVALID_CONFIG;
  int rc = check_opts(opts);
  if (rc) return rc;
  rc = validate_rows(x);
  if (rc) return rc;
  if (x->n_seq % K) return TBA_ERR_INVALID_ARG;
  if (!(std::isfinite(n_seq_global) && n_seq_global >= (double)x->n_seq && n_seq_global > 0.0))
    return TBA_ERR_INVALID_ARG;
  if (!partial) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (x->n_seq == 0)  // a rank with zero groups contributes zero partials
    return cudaMemsetAsync(partial, 0, 3 * sizeof(double), s) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
  if (!workspace || !ref_logp || !log_reward || !seq_logp || !n_tokens || !log_z || !resid)
    return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  const RowScale rs = make_scale(opt_inv_temp(opts));
  const HeadArgs ha = tb_head_args(x, opts, ref_logp, log_reward, beta, K, n_seq_global, w, seq_logp, n_tokens,
                                   log_z, resid, partial);
  // the head's counter is zeroed by the forward kernel (no memset node between the PDL-chained kernels)
  if (x->seq_len == 0 && cudaMemsetAsync(w.counter, 0, sizeof(unsigned int), s) != cudaSuccess) return TBA_ERR_CUDA;
  rc = launch_fwd_rows(x, w, rs, dev_status, s);
  if (rc) return rc;
  return launch_seq_head(true, w, x->mask, ha, s);
}

int tba_tb_loss_bwd(const tba_rows* x, const tba_tb_opts* opts, const void* workspace, const double* resid,
                    double grad_scale, const double* grad_out, void* dlogits, int32_t dlogits_dtype,
                    int64_t dlogits_row_stride, double* d_log_z, int32_t K, tba_stream_t stream) {
  int rc = check_opts(opts);
  if (rc) return rc;
  rc = validate_rows(x);
  if (rc) return rc;
  rc = validate_out(x, dlogits, dlogits_dtype, dlogits_row_stride);
  if (rc) return rc;
  if (!std::isfinite(grad_scale)) return TBA_ERR_INVALID_ARG;
  if (d_log_z && (K < 1 || x->n_seq % K)) return TBA_ERR_INVALID_ARG;
  if (x->n_seq == 0) return TBA_OK;
  if (!resid) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (d_log_z) {
    const int64_t groups = x->n_seq / K;
    rc = launch_dlogz(resid, groups, K, grad_scale, grad_out, d_log_z, s);
    if (rc) return rc;
  }
  if (x->seq_len == 0) return TBA_OK;
  if (!workspace || reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  const WsLayout w = ws_layout(const_cast<void*>(workspace), x->n_seq, x->seq_len);
  return launch_bwd(false, x, w.stats, w.qy, resid, nullptr, grad_scale, grad_out, make_scale(opt_inv_temp(opts)),
                    dlogits, dlogits_dtype, dlogits_row_stride, s);
}

int tba_tb_loss_fused(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp, const double* log_reward,
                      double beta, int32_t K, double n_seq_global, double grad_scale, void* workspace,
                      double* seq_logp, int32_t* n_tokens, double* log_z, double* resid, double* partial,
                      void* dlogits, int32_t dlogits_dtype, int64_t dlogits_row_stride, double* d_log_z,
                      int32_t* dev_status, tba_stream_t stream) {
  if (!(std::isfinite(beta) && beta > 0.0)) return TBA_ERR_INVALID_CONFIG;
  if (K < 2) return TBA_ERR_INVALID_CONFIG;
  int rc = check_opts(opts);
  if (rc) return rc;
  rc = validate_rows(x);
  if (rc) return rc;
  if (x->n_seq % K) return TBA_ERR_INVALID_ARG;
  if (!(std::isfinite(n_seq_global) && n_seq_global >= (double)x->n_seq && n_seq_global > 0.0))
    return TBA_ERR_INVALID_ARG;
  if (!std::isfinite(grad_scale)) return TBA_ERR_INVALID_ARG;
  if (!partial) return TBA_ERR_INVALID_ARG;
  rc = validate_out(x, dlogits, dlogits_dtype, dlogits_row_stride);
  if (rc) return rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (x->n_seq == 0)
    return cudaMemsetAsync(partial, 0, 3 * sizeof(double), s) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
  if (x->seq_len == 0) {  // no rows: the separate calls already handle this shape
    rc = tba_tb_loss_fwd(x, opts, ref_logp, log_reward, beta, K, n_seq_global, workspace, seq_logp, n_tokens, log_z,
                         resid, partial, dev_status, stream);
    if (rc) return rc;
    return tba_tb_loss_bwd(x, opts, workspace, resid, grad_scale, nullptr, dlogits, dlogits_dtype,
                           dlogits_row_stride, d_log_z, K, stream);
  }
  if (!workspace || !ref_logp || !log_reward || !seq_logp || !n_tokens || !log_z || !resid)
    return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  if (cudaMemsetAsync(w.fused, 0, fused_counter_bytes(x->n_seq), s) != cudaSuccess) return TBA_ERR_CUDA;
  const int64_t groups = x->n_seq / K;
  const int64_t esz = x->dtype == TBA_BF16 ? 2 : 4;
  FusedArgs a;
  a.logits = x->logits;
  a.dlogits = dlogits;
  a.tokens = x->tokens;
  a.mask = x->mask;
  a.ref_logp = ref_logp;
  a.log_reward = log_reward;
  a.log_z_param = opts ? opts->log_z_param : nullptr;
  a.stats = w.stats;
  a.qy = w.qy;
  a.lp = w.lp;
  a.seq_logp = seq_logp;
  a.n_tokens = n_tokens;
  a.log_z = log_z;
  a.resid = resid;
  a.group_sq = w.group_sq;
  a.partial = partial;
  a.dev_status = dev_status;
  a.work = w.fused;
  a.groups_done = w.fused + 1;
  a.rows_done = w.fused + 2;
  a.ready = w.fused + 2 + groups;
  a.rows = x->n_seq * x->seq_len;
  a.T = x->seq_len;
  a.V = x->vocab;
  a.stride = x->row_stride;
  a.ostride = dlogits_row_stride;
  a.n_seq = x->n_seq;
  a.K = K;
  a.groups = (int)groups;
  a.D = fused_lookahead((int64_t)K * x->seq_len * x->vocab * esz, (int)groups);
  a.inv_beta = 1.0 / beta;
  a.inv_n_global = 1.0 / n_seq_global;
  a.grad_scale = grad_scale;
  a.rs = make_scale(opt_inv_temp(opts));
  const int tf = fwd_tpr(x->vocab, esz) == 32 ? 32 : 64;
  const int tb = bwd_tpr(x->vocab, esz) == 32 ? 32 : 256;
  rc = launch_fused(a, x->dtype, dlogits_dtype, tf, tb, s);
  if (rc) return rc;
  if (d_log_z && a.log_z_param) return launch_dlogz(resid, groups, K, grad_scale, nullptr, d_log_z, s);
  return TBA_OK;
}

int tba_tb_loss_pipelined(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp,
                          const double* log_reward, double beta, int32_t K, double n_seq_global,
                          double grad_scale, int32_t groups_per_chunk, void* workspace, double* seq_logp,
                          int32_t* n_tokens, double* log_z, double* resid, double* partial, void* dlogits,
                          int32_t dlogits_dtype, int64_t dlogits_row_stride, double* d_log_z,
                          int32_t* dev_status, tba_stream_t stream, tba_stream_t aux_stream) {
  if (!(std::isfinite(beta) && beta > 0.0)) return TBA_ERR_INVALID_CONFIG;
  if (K < 2) return TBA_ERR_INVALID_CONFIG;
  int rc = check_opts(opts);
  if (rc) return rc;
  rc = validate_rows(x);
  if (rc) return rc;
  if (x->n_seq % K) return TBA_ERR_INVALID_ARG;
  if (!(std::isfinite(n_seq_global) && n_seq_global >= (double)x->n_seq && n_seq_global > 0.0))
    return TBA_ERR_INVALID_ARG;
  if (!std::isfinite(grad_scale)) return TBA_ERR_INVALID_ARG;
  if (!partial) return TBA_ERR_INVALID_ARG;
  rc = validate_out(x, dlogits, dlogits_dtype, dlogits_row_stride);
  if (rc) return rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaStream_t sb = reinterpret_cast<cudaStream_t>(aux_stream);
  if (x->n_seq == 0)
    return cudaMemsetAsync(partial, 0, 3 * sizeof(double), s) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
  if (x->seq_len == 0) {  // no rows: the separate calls already handle this shape
    rc = tba_tb_loss_fwd(x, opts, ref_logp, log_reward, beta, K, n_seq_global, workspace, seq_logp, n_tokens, log_z,
                         resid, partial, dev_status, stream);
    if (rc) return rc;
    return tba_tb_loss_bwd(x, opts, workspace, resid, grad_scale, nullptr, dlogits, dlogits_dtype,
                           dlogits_row_stride, d_log_z, K, stream);
  }
  if (!workspace || !ref_logp || !log_reward || !seq_logp || !n_tokens || !log_z || !resid)
    return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  const WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  const RowScale rs = make_scale(opt_inv_temp(opts));
  const int64_t groups = x->n_seq / K, T = x->seq_len;
  const int64_t esz = x->dtype == TBA_BF16 ? 2 : 4, oesz = dlogits_dtype == TBA_BF16 ? 2 : 4;
  const int64_t gpc = groups_per_chunk > 0 ? (groups_per_chunk < groups ? groups_per_chunk : groups)
                                           : pipe_groups((int64_t)K * T * x->vocab * esz, groups);
  const int64_t nchunks = (groups + gpc - 1) / gpc;
  const bool two = sb != s;
  cudaEvent_t* ev = two ? pipe_events() : nullptr;
  if (two && !ev) return TBA_ERR_CUDA;
  cudaEvent_t* evF = two ? ev : nullptr;
  cudaEvent_t* evB = two ? ev + 2 : nullptr;
  for (int64_t c = 0; c < nchunks && rc == TBA_OK; ++c) {
    const int64_t g0 = c * gpc, gc = (g0 + gpc <= groups) ? gpc : groups - g0;
    const int64_t s0 = g0 * K, r0 = s0 * T;
    tba_rows xc = *x;
    xc.logits = static_cast<const char*>(x->logits) + r0 * x->row_stride * esz;
    xc.tokens = x->tokens + r0;
    xc.mask = x->mask + r0;
    xc.n_seq = gc * K;
    const WsLayout wc{w.stats + r0, w.lp + r0, w.group_sq + g0, nullptr, nullptr, w.qy + r0};
    // forward of chunk c after the writer of chunk c-2: at most two chunks of logits live in L2
    if (two && c >= 2 && cudaStreamWaitEvent(s, evB[c % 2], 0) != cudaSuccess) rc = TBA_ERR_CUDA;
    if (!rc) rc = launch_fwd_rows(&xc, wc, rs, dev_status, s);
    if (rc) break;
    HeadArgs ha = tb_head_args(&xc, opts, ref_logp + s0, log_reward + s0, beta, K, n_seq_global, wc, seq_logp + s0,
                               n_tokens + s0, log_z + g0, resid + s0, partial);
    if (ha.log_z_param) ha.log_z_param += g0;
    rc = launch_seq_head(true, wc, xc.mask, ha, s);  // wc.counter == NULL: no per-chunk reduction
    if (rc) break;
    if (two && (cudaEventRecord(evF[c % 2], s) != cudaSuccess || cudaStreamWaitEvent(sb, evF[c % 2], 0) != cudaSuccess))
      rc = TBA_ERR_CUDA;
    if (!rc)
      rc = launch_bwd(false, &xc, wc.stats, wc.qy, resid + s0, nullptr, grad_scale, nullptr, rs,
                      static_cast<char*>(dlogits) + r0 * dlogits_row_stride * oesz, dlogits_dtype, dlogits_row_stride,
                      two ? sb : s);
    if (!rc && two && cudaEventRecord(evB[c % 2], sb) != cudaSuccess) rc = TBA_ERR_CUDA;
  }
  // join: the aux stream's last writer (and, in stream order, all before it) precedes the tail
  if (two && cudaStreamWaitEvent(s, evB[(nchunks - 1) % 2], 0) != cudaSuccess && !rc) rc = TBA_ERR_CUDA;
  if (!rc) rc = launch_tb_finish(w.group_sq, groups, x->n_seq, 1.0 / n_seq_global, partial, s);
  if (!rc && d_log_z && opts && opts->log_z_param) rc = launch_dlogz(resid, groups, K, grad_scale, nullptr, d_log_z, s);
  return rc;
}

int tba_tb_loss_fwd_deferred(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp,
                             const double* log_reward, double beta, int32_t K, double n_seq_global, void* workspace,
                             double* seq_logp, int32_t* n_tokens, double* log_z, double* resid, double* partial,
                             void* grad_unscaled, int32_t g_dtype, int64_t g_row_stride, int32_t* dev_status,
                             tba_stream_t stream) {
  if (!(std::isfinite(beta) && beta > 0.0)) return TBA_ERR_INVALID_CONFIG;
  if (K < 2) return TBA_ERR_INVALID_CONFIG;
  int rc = check_opts(opts);
  if (rc) return rc;
  rc = validate_rows(x);
  if (rc) return rc;
  if (x->n_seq % K) return TBA_ERR_INVALID_ARG;
  if (!(std::isfinite(n_seq_global) && n_seq_global >= (double)x->n_seq && n_seq_global > 0.0))
    return TBA_ERR_INVALID_ARG;
  if (!partial) return TBA_ERR_INVALID_ARG;
  rc = validate_out(x, grad_unscaled, g_dtype, g_row_stride);
  if (rc) return rc;
  if (grad_unscaled && out_overlaps_rows(x, grad_unscaled, g_row_stride, g_dtype))
    return TBA_ERR_INVALID_ARG;  // pass 2 re-reads the row
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (x->n_seq == 0)
    return cudaMemsetAsync(partial, 0, 3 * sizeof(double), s) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
  if (!workspace || !ref_logp || !log_reward || !seq_logp || !n_tokens || !log_z || !resid)
    return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  if (cudaMemsetAsync(w.counter, 0, sizeof(unsigned int), s) != cudaSuccess) return TBA_ERR_CUDA;
  rc = launch_single(x, w, make_scale(opt_inv_temp(opts)), dev_status, grad_unscaled, g_dtype, g_row_stride, s);
  if (rc) return rc;
  const HeadArgs ha = tb_head_args(x, opts, ref_logp, log_reward, beta, K, n_seq_global, w, seq_logp, n_tokens,
                                   log_z, resid, partial);
  return launch_seq_head(true, w, x->mask, ha, s);
}

int tba_vargrad_tb_loss_fwd(const tba_rows* x, const double* ref_logp, const double* log_reward, double beta,
                            int32_t K, double n_seq_global, void* workspace, double* seq_logp, int32_t* n_tokens,
                            double* log_z, double* resid, double* partial, int32_t* dev_status,
                            tba_stream_t stream) {
  return tba_tb_loss_fwd(x, nullptr, ref_logp, log_reward, beta, K, n_seq_global, workspace, seq_logp, n_tokens,
                         log_z, resid, partial, dev_status, stream);
}

int tba_vargrad_tb_loss_bwd(const tba_rows* x, const void* workspace, const double* resid, double grad_scale,
                            const double* grad_out, void* dlogits, int32_t dlogits_dtype, int64_t dlogits_row_stride,
                            tba_stream_t stream) {
  return tba_tb_loss_bwd(x, nullptr, workspace, resid, grad_scale, grad_out, dlogits, dlogits_dtype,
                         dlogits_row_stride, nullptr, 0, stream);
}

static int check_tbap_config(double beta, int32_t K, int32_t is_mode, double is_lo, double is_hi) {
  if (!(std::isfinite(beta) && beta >= 0.0)) return TBA_ERR_INVALID_CONFIG;  // beta = 0 is Dr. GRPO
  if (K < 2) return TBA_ERR_INVALID_CONFIG;
  if (is_mode != TBA_IS_NONE && is_mode != TBA_IS_CLIP && is_mode != TBA_IS_ICEPOP) return TBA_ERR_INVALID_CONFIG;
  if (is_mode != TBA_IS_NONE && !(is_lo >= 0.0 && is_hi >= is_lo && !std::isnan(is_hi)))
    return TBA_ERR_INVALID_CONFIG;
  return TBA_OK;
}

static int tbap_fwd_impl(const tba_rows* x, const float* gen_logp, const double* ref_logp, const double* log_reward,
                         double beta, int32_t K, int32_t is_mode, double is_lo, double is_hi, double n_tok_global,
                         void* workspace, double* seq_logp, int32_t* n_tokens, double* adv, float* coef,
                         double* partial, int32_t* dev_status, void* grad_unscaled, int32_t g_dtype,
                         int64_t g_row_stride, tba_stream_t stream) {
  int rc = check_tbap_config(beta, K, is_mode, is_lo, is_hi);
  if (rc) return rc;
  rc = validate_rows(x);
  if (rc) return rc;
  if (x->n_seq % K) return TBA_ERR_INVALID_ARG;
  if (!(std::isfinite(n_tok_global) && n_tok_global > 0.0)) return TBA_ERR_INVALID_ARG;
  if (!partial) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (x->n_seq == 0)  // a rank with zero groups contributes zero partials
    return cudaMemsetAsync(partial, 0, 3 * sizeof(double), s) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
  // gen_logp and coef are [N, T]: null is legal when T == 0 (an empty tensor has no storage)
  if (!workspace || !ref_logp || !log_reward || !seq_logp || !n_tokens || !adv ||
      (x->seq_len > 0 && (!gen_logp || !coef)))
    return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256 || reinterpret_cast<uintptr_t>(gen_logp) % 4 ||
      reinterpret_cast<uintptr_t>(coef) % 4)
    return TBA_ERR_INVALID_ARG;
  WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  if (cudaMemsetAsync(w.counter, 0, sizeof(unsigned int), s) != cudaSuccess) return TBA_ERR_CUDA;
  if (grad_unscaled) {
    rc = validate_out(x, grad_unscaled, g_dtype, g_row_stride);
    if (rc) return rc;
    if (out_overlaps_rows(x, grad_unscaled, g_row_stride, g_dtype)) return TBA_ERR_INVALID_ARG;
    rc = launch_single(x, w, make_scale(1.0), dev_status, grad_unscaled, g_dtype, g_row_stride, s);
  } else {
    rc = launch_fwd_rows(x, w, make_scale(1.0), dev_status, s);
  }
  if (rc) return rc;
  return launch_tbap_head(w, x->mask, gen_logp, x->n_seq, x->seq_len, K, ref_logp, log_reward, beta, is_mode, is_lo,
                          is_hi, -1.0 / n_tok_global, seq_logp, n_tokens, adv, coef, partial, s);
}

int tba_tbap_loss_fwd(const tba_rows* x, const float* gen_logp, const double* ref_logp, const double* log_reward,
                      double beta, int32_t K, int32_t is_mode, double is_lo, double is_hi, double n_tok_global,
                      void* workspace, double* seq_logp, int32_t* n_tokens, double* adv, float* coef, double* partial,
                      int32_t* dev_status, tba_stream_t stream) {
  return tbap_fwd_impl(x, gen_logp, ref_logp, log_reward, beta, K, is_mode, is_lo, is_hi, n_tok_global, workspace,
                       seq_logp, n_tokens, adv, coef, partial, dev_status, nullptr, TBA_BF16, 0, stream);
}

int tba_tbap_loss_fwd_deferred(const tba_rows* x, const float* gen_logp, const double* ref_logp,
                               const double* log_reward, double beta, int32_t K, int32_t is_mode, double is_lo,
                               double is_hi, double n_tok_global, void* workspace, double* seq_logp,
                               int32_t* n_tokens, double* adv, float* coef, double* partial, void* grad_unscaled,
                               int32_t g_dtype, int64_t g_row_stride, int32_t* dev_status, tba_stream_t stream) {
  if (!grad_unscaled && x && x->n_seq * x->seq_len > 0) return TBA_ERR_INVALID_ARG;
  return tbap_fwd_impl(x, gen_logp, ref_logp, log_reward, beta, K, is_mode, is_lo, is_hi, n_tok_global, workspace,
                       seq_logp, n_tokens, adv, coef, partial, dev_status, grad_unscaled, g_dtype, g_row_stride,
                       stream);
}

int tba_tbap_loss_bwd(const tba_rows* x, const void* workspace, const float* coef, double grad_scale,
                      const double* grad_out, void* dlogits, int32_t dlogits_dtype, int64_t dlogits_row_stride,
                      tba_stream_t stream) {
  int rc = validate_rows(x);
  if (rc) return rc;
  rc = validate_out(x, dlogits, dlogits_dtype, dlogits_row_stride);
  if (rc) return rc;
  if (!std::isfinite(grad_scale)) return TBA_ERR_INVALID_ARG;
  if (x->n_seq * x->seq_len == 0) return TBA_OK;
  if (!workspace || !coef) return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  const WsLayout w = ws_layout(const_cast<void*>(workspace), x->n_seq, x->seq_len);
  return launch_bwd(true, x, w.stats, w.qy, nullptr, coef, grad_scale, grad_out, make_scale(1.0), dlogits, dlogits_dtype,
                    dlogits_row_stride, reinterpret_cast<cudaStream_t>(stream));
}

// ---- LM-head-fused head (NEXT 3)
size_t tba_lmhead_workspace_bytes(int64_t n_seq, int64_t seq_len, int64_t vocab) {
  if (n_seq < 0 || seq_len < 0 || vocab < 1) return 0;
  return ws_bytes(n_seq, seq_len) + lmhead_partial_bytes(n_seq * seq_len, vocab);
}

int tba_lmhead_seq_logprob(const tba_lmhead* x, double inv_temp, void* workspace, double* seq_logp,
                           int32_t* n_tokens, int32_t* dev_status, tba_stream_t stream) {
  int rc = validate_lmhead(x);
  if (rc) return rc;
  if (!(std::isfinite(inv_temp) && inv_temp > 0.0)) return TBA_ERR_INVALID_CONFIG;
  if (x->n_seq == 0) return TBA_OK;
  if (!workspace || !seq_logp || !n_tokens || reinterpret_cast<uintptr_t>(workspace) % 256)
    return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  rc = launch_lmhead_rows(x, static_cast<char*>(workspace) + ws_bytes(x->n_seq, x->seq_len), w,
                          make_scale(inv_temp), dev_status, s);
  if (rc) return rc;
  HeadArgs ha{};
  ha.T = x->seq_len;
  ha.K = 1;
  ha.n_seq = x->n_seq;
  ha.seq_logp = seq_logp;
  ha.n_tokens = n_tokens;
  return launch_seq_head(false, w, x->mask, ha, s);
}

int tba_lmhead_token_logprob(const tba_lmhead* x, double inv_temp, void* workspace, double* tok_logp,
                             int32_t* dev_status, tba_stream_t stream) {
  int rc = validate_lmhead(x);
  if (rc) return rc;
  if (!(std::isfinite(inv_temp) && inv_temp > 0.0)) return TBA_ERR_INVALID_CONFIG;
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows == 0) return TBA_OK;
  if (!workspace || !tok_logp || reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  rc = launch_lmhead_rows(x, static_cast<char*>(workspace) + ws_bytes(x->n_seq, x->seq_len), w,
                          make_scale(inv_temp), dev_status, s);
  if (rc) return rc;
  return launch_token_lp(w, x->mask, rows, tok_logp, s);
}

int tba_lmhead_tbap_loss_fwd(const tba_lmhead* x, const float* gen_logp, const double* ref_logp,
                             const double* log_reward, double beta, int32_t K, int32_t is_mode, double is_lo,
                             double is_hi, double n_tok_global, void* workspace, double* seq_logp,
                             int32_t* n_tokens, double* adv, float* coef, double* partial, int32_t* dev_status,
                             tba_stream_t stream) {
  int rc = check_tbap_config(beta, K, is_mode, is_lo, is_hi);
  if (rc) return rc;
  rc = validate_lmhead(x);
  if (rc) return rc;
  if (x->n_seq % K) return TBA_ERR_INVALID_ARG;
  if (!(std::isfinite(n_tok_global) && n_tok_global > 0.0)) return TBA_ERR_INVALID_ARG;
  if (!partial) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (x->n_seq == 0)
    return cudaMemsetAsync(partial, 0, 3 * sizeof(double), s) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
  // gen_logp and coef are [N, T]: null is legal when T == 0 (an empty tensor has no storage)
  if (!workspace || !ref_logp || !log_reward || !seq_logp || !n_tokens || !adv ||
      (x->seq_len > 0 && (!gen_logp || !coef)))
    return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256 || reinterpret_cast<uintptr_t>(gen_logp) % 4 ||
      reinterpret_cast<uintptr_t>(coef) % 4)
    return TBA_ERR_INVALID_ARG;
  const WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  if (cudaMemsetAsync(w.counter, 0, sizeof(unsigned int), s) != cudaSuccess) return TBA_ERR_CUDA;
  rc = launch_lmhead_rows(x, static_cast<char*>(workspace) + ws_bytes(x->n_seq, x->seq_len), w, make_scale(1.0),
                          dev_status, s);
  if (rc) return rc;
  return launch_tbap_head(w, x->mask, gen_logp, x->n_seq, x->seq_len, K, ref_logp, log_reward, beta, is_mode, is_lo,
                          is_hi, -1.0 / n_tok_global, seq_logp, n_tokens, adv, coef, partial, s);
}

int tba_lmhead_tb_loss_fwd(const tba_lmhead* x, const tba_tb_opts* opts, const double* ref_logp,
                           const double* log_reward, double beta, int32_t K, double n_seq_global,
                           void* workspace, double* seq_logp, int32_t* n_tokens, double* log_z,
                           double* resid, double* partial, int32_t* dev_status, tba_stream_t stream) {
  if (!(std::isfinite(beta) && beta > 0.0)) return TBA_ERR_INVALID_CONFIG;
  if (K < 2) return TBA_ERR_INVALID_CONFIG;
  int rc = check_opts(opts);
  if (rc) return rc;
  rc = validate_lmhead(x);
  if (rc) return rc;
  if (x->n_seq % K) return TBA_ERR_INVALID_ARG;
  if (!(std::isfinite(n_seq_global) && n_seq_global >= (double)x->n_seq && n_seq_global > 0.0))
    return TBA_ERR_INVALID_ARG;
  if (!partial) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (x->n_seq == 0)
    return cudaMemsetAsync(partial, 0, 3 * sizeof(double), s) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
  if (!workspace || !ref_logp || !log_reward || !seq_logp || !n_tokens || !log_z || !resid)
    return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  const WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  if (cudaMemsetAsync(w.counter, 0, sizeof(unsigned int), s) != cudaSuccess) return TBA_ERR_CUDA;
  rc = launch_lmhead_rows(x, static_cast<char*>(workspace) + ws_bytes(x->n_seq, x->seq_len), w,
                          make_scale(opt_inv_temp(opts)), dev_status, s);
  if (rc) return rc;
  tba_rows xr{};
  xr.n_seq = x->n_seq;
  xr.seq_len = x->seq_len;
  const HeadArgs ha = tb_head_args(&xr, opts, ref_logp, log_reward, beta, K, n_seq_global, w, seq_logp, n_tokens,
                                   log_z, resid, partial);
  return launch_seq_head(true, w, x->mask, ha, s);
}

// ---- LM-head-fused head (NEXT 3), backward
size_t tba_lmhead_bwd_workspace_bytes(int64_t n_seq, int64_t seq_len, int64_t d, int64_t vocab,
                                      int64_t chunk_rows) {
  if (n_seq < 0 || seq_len < 0 || d < 1 || vocab < 1) return 0;
  if (n_seq > 0 && seq_len > (int64_t)INT32_MAX / n_seq) return 0;
  return lmhead_bwd_ws_bytes(n_seq * seq_len, d, vocab, chunk_rows);
}

static int lmhead_bwd_impl(const tba_lmhead* x, const void* workspace, const double* resid, const float* coef,
                           double gs, const double* grad_out, float sc, void* dhidden, int32_t dh_dtype,
                           int64_t dh_stride, float* dweight, int64_t dw_stride, int32_t accumulate,
                           int64_t chunk_rows, void* bwd_workspace, cudaStream_t s) {
  int rc = validate_lmhead(x);
  if (rc) return rc;
  if (!std::isfinite(gs)) return TBA_ERR_INVALID_ARG;
  if (dhidden) {
    if (dh_dtype != TBA_BF16 && dh_dtype != TBA_FP32) return TBA_ERR_INVALID_ARG;
    if (dh_stride < x->d || reinterpret_cast<uintptr_t>(dhidden) % (dh_dtype == TBA_BF16 ? 2 : 4))
      return TBA_ERR_INVALID_ARG;
  }
  if (dweight && (dw_stride < x->d || reinterpret_cast<uintptr_t>(dweight) % 4)) return TBA_ERR_INVALID_ARG;
  if (lm_outputs_overlap(x, dhidden, dh_stride, dh_dtype, dweight, dw_stride))
    return TBA_ERR_INVALID_ARG;  // hidden and the weight are re-read chunk by chunk
  const int64_t rows = x->n_seq * x->seq_len;
  if (!dhidden && !dweight) return TBA_OK;
  if (rows > 0) {
    if (!workspace || !bwd_workspace || reinterpret_cast<uintptr_t>(workspace) % 256 ||
        reinterpret_cast<uintptr_t>(bwd_workspace) % 256)
      return TBA_ERR_INVALID_ARG;
    if (!resid && !coef) return TBA_ERR_INVALID_ARG;
  }
  const WsLayout w = ws_layout(const_cast<void*>(workspace), x->n_seq, x->seq_len);
  return launch_lmhead_bwd(x, rows > 0 ? w.stats : nullptr, resid, coef, gs, grad_out, sc, dhidden, dh_dtype,
                           dh_stride, dweight, dw_stride, accumulate != 0, chunk_rows, bwd_workspace, s);
}

int tba_lmhead_tb_loss_bwd(const tba_lmhead* x, const tba_tb_opts* opts, const void* workspace,
                           const double* resid, double grad_scale, const double* grad_out, void* dhidden,
                           int32_t dhidden_dtype, int64_t dhidden_row_stride, float* dweight,
                           int64_t dweight_row_stride, int32_t accumulate, double* d_log_z, int32_t K,
                           int64_t chunk_rows, void* bwd_workspace, tba_stream_t stream) {
  int rc = check_opts(opts);
  if (rc) return rc;
  rc = validate_lmhead(x);
  if (rc) return rc;
  if (d_log_z && (K < 1 || x->n_seq % K)) return TBA_ERR_INVALID_ARG;
  if (!std::isfinite(grad_scale)) return TBA_ERR_INVALID_ARG;
  if (x->n_seq > 0 && !resid) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (d_log_z && x->n_seq > 0) {
    rc = launch_dlogz(resid, x->n_seq / K, K, grad_scale, grad_out, d_log_z, s);
    if (rc) return rc;
  }
  const RowScale rs = make_scale(opt_inv_temp(opts));
  return lmhead_bwd_impl(x, workspace, resid, nullptr, grad_scale * rs.inv_temp, grad_out, rs.sc, dhidden,
                         dhidden_dtype, dhidden_row_stride, dweight, dweight_row_stride, accumulate, chunk_rows,
                         bwd_workspace, s);
}

int tba_lmhead_tbap_loss_bwd(const tba_lmhead* x, const void* workspace, const float* coef, double grad_scale,
                             const double* grad_out, void* dhidden, int32_t dhidden_dtype,
                             int64_t dhidden_row_stride, float* dweight, int64_t dweight_row_stride,
                             int32_t accumulate, int64_t chunk_rows, void* bwd_workspace, tba_stream_t stream) {
  int rc = validate_lmhead(x);
  if (rc) return rc;
  if (x->n_seq * x->seq_len > 0 && (!coef || reinterpret_cast<uintptr_t>(coef) % 4)) return TBA_ERR_INVALID_ARG;
  return lmhead_bwd_impl(x, workspace, nullptr, coef, grad_scale, grad_out, make_scale(1.0).sc, dhidden,
                         dhidden_dtype, dhidden_row_stride, dweight, dweight_row_stride, accumulate, chunk_rows,
                         bwd_workspace, reinterpret_cast<cudaStream_t>(stream));
}

size_t tba_lmhead_fwd_bwd_workspace_bytes(int64_t n_seq, int64_t seq_len, int64_t d, int64_t vocab, int32_t K,
                                          int32_t groups_per_chunk) {
  if (n_seq < 0 || seq_len < 0 || d < 1 || vocab < 1 || K < 1 || n_seq % K) return 0;
  if (n_seq > 0 && seq_len > (int64_t)INT32_MAX / n_seq) return 0;
  if (n_seq == 0 || seq_len == 0) return 256;
  return lmhead_fb_ws_bytes(n_seq, seq_len, d, vocab, K, groups_per_chunk);
}

int tba_lmhead_tb_loss_fwd_bwd(const tba_lmhead* x, const tba_tb_opts* opts, const double* ref_logp,
                               const double* log_reward, double beta, int32_t K, double n_seq_global,
                               double grad_scale, int32_t groups_per_chunk, void* workspace, double* seq_logp,
                               int32_t* n_tokens, double* log_z, double* resid, double* partial, void* dhidden,
                               int32_t dhidden_dtype, int64_t dhidden_row_stride, float* dweight,
                               int64_t dweight_row_stride, int32_t accumulate, double* d_log_z,
                               void* bwd_workspace, int32_t* dev_status, tba_stream_t stream) {
  if (!(std::isfinite(beta) && beta > 0.0)) return TBA_ERR_INVALID_CONFIG;
  if (K < 2) return TBA_ERR_INVALID_CONFIG;
  int rc = check_opts(opts);
  if (rc) return rc;
  rc = validate_lmhead(x);
  if (rc) return rc;
  if (x->n_seq % K) return TBA_ERR_INVALID_ARG;
  if (!(std::isfinite(n_seq_global) && n_seq_global >= (double)x->n_seq && n_seq_global > 0.0))
    return TBA_ERR_INVALID_ARG;
  if (!std::isfinite(grad_scale) || !partial) return TBA_ERR_INVALID_ARG;
  if (dhidden) {
    if (dhidden_dtype != TBA_BF16 && dhidden_dtype != TBA_FP32) return TBA_ERR_INVALID_ARG;
    if (dhidden_row_stride < x->d || reinterpret_cast<uintptr_t>(dhidden) % (dhidden_dtype == TBA_BF16 ? 2 : 4))
      return TBA_ERR_INVALID_ARG;
  }
  if (dweight && (dweight_row_stride < x->d || reinterpret_cast<uintptr_t>(dweight) % 4)) return TBA_ERR_INVALID_ARG;
  if (lm_outputs_overlap(x, dhidden, dhidden_row_stride, dhidden_dtype, dweight, dweight_row_stride))
    return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (x->n_seq == 0 || x->seq_len == 0) {  // no rows: the two calls handle these shapes
    rc = tba_lmhead_tb_loss_fwd(x, opts, ref_logp, log_reward, beta, K, n_seq_global, workspace, seq_logp, n_tokens,
                                log_z, resid, partial, dev_status, stream);
    if (rc) return rc;
    return lmhead_bwd_impl(x, workspace, resid, nullptr, grad_scale * opt_inv_temp(opts), nullptr,
                           make_scale(opt_inv_temp(opts)).sc, dhidden, dhidden_dtype, dhidden_row_stride, dweight,
                           dweight_row_stride, accumulate, 0, bwd_workspace, s);
  }
  if (!workspace || !bwd_workspace || !ref_logp || !log_reward || !seq_logp || !n_tokens || !log_z || !resid)
    return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256 || reinterpret_cast<uintptr_t>(bwd_workspace) % 256)
    return TBA_ERR_INVALID_ARG;
  const WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  const RowScale rs = make_scale(opt_inv_temp(opts));
  tba_rows xr{};
  xr.n_seq = x->n_seq;
  xr.seq_len = x->seq_len;
  const HeadArgs ha = tb_head_args(&xr, opts, ref_logp, log_reward, beta, K, n_seq_global, w, seq_logp, n_tokens,
                                   log_z, resid, partial);
  rc = launch_lmhead_fwd_bwd(x, rs, w, ha, K, grad_scale, 1.0 / n_seq_global, dhidden, dhidden_dtype,
                             dhidden_row_stride, dweight, dweight_row_stride, accumulate != 0, groups_per_chunk,
                             bwd_workspace, dev_status, s);
  if (!rc && d_log_z && opts && opts->log_z_param)
    rc = launch_dlogz(resid, x->n_seq / K, K, grad_scale, nullptr, d_log_z, s);
  return rc;
}

}  // extern "C"


