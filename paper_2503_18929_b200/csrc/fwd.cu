// a1: the row forward kernels (log-softmax statistics + gathered token log-prob per row).
#include "tba_device.cuh"

namespace tba {
namespace {
#ifdef TBA_AB_FWD_TRACE
// per row [smid, globaltimer at the group's start, at its end] (A/B build only,
// scripts/microbench/fwd_trace.py)
constexpr int FTR_ROWS = 1 << 19;
__device__ unsigned long long g_ftrace[FTR_ROWS * 3];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c));
  return c;
}
#endif
// TPR threads per row, 256/TPR rows per CTA (TPR = 32 ... 256). Each row group meets on its own
// named barrier (ids 1..8); a masked row's group exits as a whole.
template <class T, int TPR, int U, int NP = 0>
__global__ void __launch_bounds__(256, 4) row_fwd_rows(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                     int64_t stride, const int64_t* __restrict__ tokens,
                                                     const uint8_t* __restrict__ mask, RowScale rs,
                                                     float2* __restrict__ stats, float* __restrict__ qy,
                                                     double* __restrict__ lp, int32_t* dev_status,
                                                     unsigned int* zero_counter) {
  constexpr int RPC = 256 / TPR, WPRS = TPR / 32 > 0 ? TPR / 32 : 1;
  __shared__ float sm_m[RPC][WPRS], sm_M2[RPC][WPRS];
  __shared__ double sm_s[RPC][WPRS];
  pdl_trigger();
  pdl_wait();
  // the head's last-CTA counter (read only by the next kernel, after this grid completes)
  if (zero_counter && blockIdx.x == 0 && threadIdx.x == 0) *zero_counter = 0u;
  const int grp = threadIdx.x / TPR, gt = threadIdx.x % TPR;
  const int64_t row = (int64_t)blockIdx.x * RPC + grp;
  if (row >= rows || mask[row] == 0) return;
#ifdef TBA_AB_FWD_TRACE
  if (gt == 0 && row < FTR_ROWS) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_ftrace[row * 3] = sm;
    g_ftrace[row * 3 + 1] = gtimer();
  }
#endif
  fwd_row_group<T, TPR, U, NP>(logits, row, V, stride, tokens, rs, stats, qy, lp, dev_status, sm_m, sm_M2, sm_s, grp,
                               gt);
#ifdef TBA_AB_FWD_TRACE
  if (gt == 0 && row < FTR_ROWS) g_ftrace[row * 3 + 2] = gtimer();
#endif
}

template <class T>
int launch_fwd_rows_t(const T* lg, const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status,
                       cudaStream_t s, int tpr) {
  const int64_t rows = x->n_seq * x->seq_len;
  const int64_t rpc = 256 / tpr;
  const unsigned grid = (unsigned)((rows + rpc - 1) / rpc);
#define TBA_ROWS(TPR_, NP_)                                                                                     \
  return launch_pdl(row_fwd_rows<T, TPR_, kU, NP_>, dim3(grid), dim3(256), 0, s, lg, rows, x->vocab, x->row_stride, \
                    x->tokens, x->mask, rs, w.stats, w.qy, w.lp, dev_status, w.counter)
  // 1 of the 4 element pairs per 16-byte vector (1 of 2 for fp32 rows) takes the FMA-pipe exp2
  // (exp2_poly2) instead of MUFU — relieves the XU pipe (75 % busy), +1-3 % forward bandwidth on
  // every BASELINE shape; 2 of 4 over-loads the FMA/ALU pipes.
  // (the 304 KB Qwen rows: 1 of 8 pairs, NP = -1 — 1.3 % faster than 1 of 4 there)
  if (tpr == 64) TBA_ROWS(64, -1);
  TBA_ROWS(32, 1);  // (1 of 8 measured equal on the < 128 KB rows)
#undef TBA_ROWS
}

}  // namespace

int launch_fwd_rows(const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status, cudaStream_t s) {
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows == 0) return TBA_OK;
  const int64_t esz = x->dtype == TBA_BF16 ? 2 : 4;
  const int tpr = fwd_tpr(x->vocab, esz);
  return x->dtype == TBA_BF16
             ? launch_fwd_rows_t<uint16_t>(static_cast<const uint16_t*>(x->logits), x, w, rs, dev_status, s, tpr)
             : launch_fwd_rows_t<float>(static_cast<const float*>(x->logits), x, w, rs, dev_status, s, tpr);
}

}  // namespace tba

#ifdef TBA_AB_FWD_TRACE
extern "C" int tba_debug_fwd_trace(void* host, long long n) {
  if (n > (long long)tba::FTR_ROWS * 3) n = (long long)tba::FTR_ROWS * 3;
  return cudaMemcpyFromSymbol(host, tba::g_ftrace, (size_t)n * 8) == cudaSuccess ? 0 : 3;
}
#endif
