// a2 + a3: per-sequence sums and the group heads (VarGrad TB, Eqs. 4-5; TBA', Eq. 16) and the
// small helper kernels.
#include "tba_device.cuh"

namespace tba {
namespace {
// One CTA per group of K sequences (HEAD), or per 8 sequences (log-probs only).
// Eq. 4: log Z_i = 1/K sum_j delta_j (delta = rho - ell + r/beta), or the learned log Z_i of
// Eq. 3 when log_z_param != NULL; Eq. 5 residual eps = log Z_i - delta. The last CTA (counter)
// reduces the per-group sums of squares in group order.
template <bool HEAD>
__global__ void __launch_bounds__(1024) seq_head(const double* __restrict__ lp, const uint8_t* __restrict__ mask,
                                                int64_t n_seq, int64_t T, int K, const double* __restrict__ ref_logp,
                                                const double* __restrict__ log_reward,
                                                const double* __restrict__ log_z_param, double inv_beta,
                                                double inv_n_global, double* __restrict__ seq_logp,
                                                int32_t* __restrict__ n_tokens, double* __restrict__ log_z,
                                                double* __restrict__ resid, double* __restrict__ group_sq,
                                                double* __restrict__ partial, unsigned int* counter) {
  const int per = HEAD ? K : 8;
  const int64_t s0 = (int64_t)blockIdx.x * per;
  pdl_trigger();
  pdl_wait();
  seq_sums(lp, mask, n_seq, T, s0, per, seq_logp, n_tokens, nullptr);
  if (!HEAD) return;
  __syncthreads();
  __shared__ bool am_last;
  if (threadIdx.x < 32) {  // warp 0: the group head
    tb_group_head((int64_t)blockIdx.x, K, ref_logp, log_reward, log_z_param, inv_beta, seq_logp, log_z, resid,
                  group_sq, (int)threadIdx.x);
    __threadfence();  // every lane's residuals before the counter moves
    __syncwarp();
    if (threadIdx.x == 0) {
      am_last = false;
      if (counter)  // counter == NULL: a chunk of a larger batch; tb_finish_kernel reduces later
        am_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (am_last && threadIdx.x == 0) {
    __threadfence();
    *counter = 0u;
    tb_finish(group_sq, (int64_t)gridDim.x, n_seq, inv_n_global, partial);
  }
}


// ------------------------------------------------------------------------------ TBA' head (Eq. 16)
// One CTA per group: sequence sums as seq_head; thread 0 forms A_j = (r_j - rbar) -
// beta (log Lambda_j - mean log Lambda) with log Lambda_j = ell_j - rho_j; every thread then
// walks the group's rows: lambda_t = exp(lp_t - gen_t), IS weight w, coef_t = w * A_j (a
// stop-gradient constant) and the surrogate term coef_t * lp_t, in a fixed order.
__global__ void __launch_bounds__(256) tbap_head(const double* __restrict__ lp, const uint8_t* __restrict__ mask,
                                                 const float* __restrict__ gen_logp, int64_t n_seq, int64_t T, int K,
                                                 const double* __restrict__ ref_logp,
                                                 const double* __restrict__ log_reward, double beta, int is_mode,
                                                 double is_lo, double is_hi, double neg_inv_ntok,
                                                 double* __restrict__ seq_logp, int32_t* __restrict__ n_tokens,
                                                 double* __restrict__ adv, float* __restrict__ coef,
                                                 double* __restrict__ group_acc, double* __restrict__ partial,
                                                 unsigned int* counter) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s0 = (int64_t)blockIdx.x * K;
  __shared__ int sm_cnt[8];
  int my_cnt = 0;
  seq_sums(lp, mask, n_seq, T, s0, K, seq_logp, n_tokens, &my_cnt);
  if (lane == 0) sm_cnt[warp] = my_cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    double rbar = 0.0, lbar = 0.0;
    for (int j = 0; j < K; ++j) {
      rbar += log_reward[s0 + j];
      lbar += seq_logp[s0 + j] - ref_logp[s0 + j];
    }
    rbar /= (double)K;
    lbar /= (double)K;
    for (int j = 0; j < K; ++j)
      adv[s0 + j] = (log_reward[s0 + j] - rbar) - beta * ((seq_logp[s0 + j] - ref_logp[s0 + j]) - lbar);
  }
  __syncthreads();
  double acc = 0.0;
  const int64_t nr = (int64_t)K * T, r0 = s0 * T;
  for (int64_t i = threadIdx.x; i < nr; i += 256) {
    const int64_t r = r0 + i;
    float cf = 0.f;
    if (mask[r]) {
      const double l = lp[r];
      const double lam = exp(l - (double)gen_logp[r]);
      double wgt = 1.0;
      if (is_mode == TBA_IS_CLIP) wgt = fmin(fmax(lam, is_lo), is_hi);
      else if (is_mode == TBA_IS_ICEPOP) wgt = (lam >= is_lo && lam <= is_hi) ? lam : 0.0;
      const double c = wgt * adv[r / T];
      cf = (float)c;
      acc += c * l;
    }
    coef[r] = cf;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double sm_acc[8];
  __shared__ bool am_last;
  if (lane == 0) sm_acc[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double g = 0.0;
    int n = 0;
    for (int w = 0; w < 8; ++w) {
      g += sm_acc[w];
      n += sm_cnt[w];
    }
    group_acc[2 * blockIdx.x] = g;
    group_acc[2 * blockIdx.x + 1] = (double)n;
    __threadfence();
    am_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (am_last && threadIdx.x == 0) {
    __threadfence();
    const volatile double* ga = group_acc;
    double tot = 0.0, ntok = 0.0;
    for (unsigned i = 0; i < gridDim.x; ++i) {
      tot += ga[2 * i];
      ntok += ga[2 * i + 1];
    }
    partial[0] = tot * neg_inv_ntok;
    partial[1] = ntok;
    partial[2] = (double)n_seq;
    *counter = 0u;
  }
}

// Per-token log-probs out of the workspace: tok_logp[r] = mask ? lp[r] : 0.
__global__ void token_lp_kernel(const double* __restrict__ lp, const uint8_t* __restrict__ mask, int64_t rows,
                                double* __restrict__ out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    out[r] = mask[r] ? lp[r] : 0.0;
}

// dL/d log Z_i for a learned log Z (Eq. 3): grad_scale * g * sum_j eps_{iK+j}.
__global__ void dlogz_kernel(const double* __restrict__ resid, int64_t groups, int K, double grad_scale,
                             const double* __restrict__ grad_out, double* __restrict__ d_log_z) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= groups) return;
  double s = 0.0;
  for (int j = 0; j < K; ++j) s += resid[i * K + j];
  d_log_z[i] = grad_scale * (grad_out ? *grad_out : 1.0) * s;
}


// The final fixed-order reduction of a chunked step (tba_tb_loss_pipelined): the same
// arithmetic as seq_head's last CTA over all groups of the call.
__global__ void tb_finish_kernel(const double* __restrict__ group_sq, int64_t groups, int64_t n_seq,
                                 double inv_n_global, double* __restrict__ partial) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    tb_finish(group_sq, groups, n_seq, inv_n_global, partial);
}

// ------------------------------------------------------------------------------ launch
}  // namespace

int launch_seq_head(bool head, const WsLayout& w, const uint8_t* mask, const HeadArgs& ha, cudaStream_t s) {
  if (head) {
    // one warp per sequence of the group (K > 8: more than one round of 8 warps otherwise)
    const int threads = ha.K <= 8 ? 256 : (ha.K >= 32 ? 1024 : 32 * ha.K);
    return launch_pdl(seq_head<true>, dim3((unsigned)(ha.n_seq / ha.K)), dim3(threads), 0, s, w.lp, mask, ha.n_seq,
                      ha.T, ha.K, ha.ref_logp, ha.log_reward, ha.log_z_param, ha.inv_beta, ha.inv_n_global,
                      ha.seq_logp, ha.n_tokens, ha.log_z, ha.resid, w.group_sq, ha.partial, w.counter);
  }
  return launch_pdl(seq_head<false>, dim3((unsigned)((ha.n_seq + 7) / 8)), dim3(256), 0, s, w.lp, mask, ha.n_seq,
                    ha.T, 8, (const double*)nullptr, (const double*)nullptr, (const double*)nullptr, 0.0, 0.0,
                    ha.seq_logp, ha.n_tokens, (double*)nullptr, (double*)nullptr, (double*)nullptr, (double*)nullptr,
                    (unsigned int*)nullptr);
}

int launch_tbap_head(const WsLayout& w, const uint8_t* mask, const float* gen_logp, int64_t n_seq, int64_t T, int K,
                     const double* ref_logp, const double* log_reward, double beta, int is_mode, double is_lo,
                     double is_hi, double neg_inv_ntok, double* seq_logp, int32_t* n_tokens, double* adv,
                     float* coef, double* partial, cudaStream_t s) {
  tbap_head<<<(unsigned)(n_seq / K), 256, 0, s>>>(w.lp, mask, gen_logp, n_seq, T, K, ref_logp, log_reward, beta,
                                                  is_mode, is_lo, is_hi, neg_inv_ntok, seq_logp, n_tokens, adv, coef,
                                                  w.group_sq, partial, w.counter);
  return launch_status();
}

int launch_token_lp(const WsLayout& w, const uint8_t* mask, int64_t rows, double* tok_logp, cudaStream_t s) {
  const int64_t blocks = (rows + 255) / 256 < 4096 ? (rows + 255) / 256 : 4096;
  token_lp_kernel<<<(unsigned)blocks, 256, 0, s>>>(w.lp, mask, rows, tok_logp);
  return launch_status();
}

int launch_dlogz(const double* resid, int64_t groups, int K, double grad_scale, const double* grad_out,
                 double* d_log_z, cudaStream_t s) {
  dlogz_kernel<<<(unsigned)((groups + 127) / 128), 128, 0, s>>>(resid, groups, K, grad_scale, grad_out, d_log_z);
  return launch_status();
}

int launch_tb_finish(const double* group_sq, int64_t groups, int64_t n_seq, double inv_n_global, double* partial,
                     cudaStream_t s) {
  tb_finish_kernel<<<1, 32, 0, s>>>(group_sq, groups, n_seq, inv_n_global, partial);
  return launch_status();
}

}  // namespace tba
