// a5: the gradient writer (one streaming pass per valid row; masked rows zero-filled).
#include "tba_device.cuh"

namespace tba {
namespace {
// TPR threads per row, 256/TPR rows per CTA. Row coefficient c = grad_scale * g * inv_temp *
// (resid[s] for the TB losses, per sequence | coef[row] for per-token rules such as TBA').
template <class T, class TO, int TPR, int U, bool PER_ROW>
__global__ void __launch_bounds__(256, TPR == 32 ? 4 : 6) row_bwd(const T* __restrict__ logits, int64_t rows, int64_t T_len, int64_t V,
                                               int64_t stride, const int64_t* __restrict__ tokens,
                                               const uint8_t* __restrict__ mask, const float2* __restrict__ stats,
                                               const float* __restrict__ qy_in, const double* __restrict__ resid,
                                               const float* __restrict__ coef,
                                               double grad_scale, const double* __restrict__ grad_out, RowScale rs,
                                               TO* __restrict__ dlogits, int64_t ostride) {
  constexpr int RPC = 256 / TPR;
  pdl_trigger();
  pdl_wait();
  const int64_t row = (int64_t)blockIdx.x * RPC + threadIdx.x / TPR;
  if (row >= rows) return;
  const int tid = threadIdx.x % TPR;
  const bool valid = mask[row] != 0;
  float M2 = 0.f, L2S = 0.f, c = 0.f, qy = 0.f;
  int64_t y = -1;
  if (valid) {
    const float2 st = stats[row];
    M2 = st.x;
    L2S = st.y;
    qy = qy_in[row];
    const double g = (grad_out ? *grad_out : 1.0) * grad_scale * rs.inv_temp;
    c = PER_ROW ? (float)(g * (double)coef[row]) : (float)(g * resid[row / T_len]);
    y = tokens[row];
  }
  bwd_row<T, TO, U>(logits + row * stride, dlogits + row * ostride, V, tid, TPR, valid, rs.sc, M2, L2S, c, y, qy);
}


// ------------------------------------------------------------------------------ launch
template <class T, class TO, bool PER_ROW>
int launch_bwd_t(const tba_rows* x, const float2* stats, const float* qy, const double* resid, const float* coef,
                  double gs,
                  const double* go, const RowScale& rs, TO* out, int64_t ostride, cudaStream_t s) {
  const int64_t rows = x->n_seq * x->seq_len;
  const int tpr = bwd_tpr(x->vocab, (int64_t)sizeof(T));
  const int64_t rpc = 256 / tpr;
  const unsigned grid = (unsigned)((rows + rpc - 1) / rpc);
  auto lg = static_cast<const T*>(x->logits);
#define TBA_BWD(TPR_)                                                                                             \
  return launch_pdl(row_bwd<T, TO, TPR_, kU, PER_ROW>, dim3(grid), dim3(256), 0, s, lg, rows, x->seq_len, x->vocab, \
                    x->row_stride, x->tokens, x->mask, stats, qy, resid, coef, gs, go, rs, out, ostride)
  if (tpr == 32) TBA_BWD(32);
  else TBA_BWD(256);
#undef TBA_BWD
}

template <bool PER_ROW>
int launch_bwd_dt(const tba_rows* x, const float2* stats, const float* qy, const double* resid, const float* coef,
                  double gs,
                  const double* go, const RowScale& rs, void* dlogits, int32_t odt, int64_t ostride, cudaStream_t s) {
  if (x->n_seq * x->seq_len == 0) return TBA_OK;
  if (x->dtype == TBA_BF16) {
    if (odt == TBA_BF16)
      return launch_bwd_t<uint16_t, uint16_t, PER_ROW>(x, stats, qy, resid, coef, gs, go, rs,
                                                       static_cast<uint16_t*>(dlogits), ostride, s);
    return launch_bwd_t<uint16_t, float, PER_ROW>(x, stats, qy, resid, coef, gs, go, rs, static_cast<float*>(dlogits),
                                                  ostride, s);
  }
  if (odt == TBA_BF16)
    return launch_bwd_t<float, uint16_t, PER_ROW>(x, stats, qy, resid, coef, gs, go, rs, static_cast<uint16_t*>(dlogits),
                                                  ostride, s);
  return launch_bwd_t<float, float, PER_ROW>(x, stats, qy, resid, coef, gs, go, rs, static_cast<float*>(dlogits),
                                             ostride, s);
}

}  // namespace

int launch_bwd(bool per_row, const tba_rows* x, const float2* stats, const float* qy, const double* resid,
               const float* coef, double gs, const double* go, const RowScale& rs, void* dlogits, int32_t odt, int64_t ostride,
               cudaStream_t s) {
  return per_row ? launch_bwd_dt<true>(x, stats, qy, resid, coef, gs, go, rs, dlogits, odt, ostride, s)
                 : launch_bwd_dt<false>(x, stats, qy, resid, coef, gs, go, rs, dlogits, odt, ostride, s);
}

}  // namespace tba
