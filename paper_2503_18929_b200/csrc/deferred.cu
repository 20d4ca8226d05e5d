// Deferred-scale row pass (NEXT 2 (ii)).
#include "tba_device.cuh"

namespace tba {
namespace {
// A cluster of CS CTAs (NT threads each) per valid row: pass 1 streams the row from HBM with an
// L2 evict_last policy (online max/sum); the CTAs of the cluster exchange their (max, sum)
// partials through distributed shared memory; pass 2 re-reads the row — an L2 hit, because the
// grid keeps only ~40-60 MB of rows in flight (CS and NT are chosen per row size) — and writes
// the UNSCALED gradient G = inv_temp (1[v=y] - softmax) once. HBM bytes: 2V read + 2V write per
// valid row (the 4V floor); the per-sequence factor grad_scale * g * eps_s is applied by the
// consumer (the LM-head backward, as a row scale), SURVEY §8(f) NEXT 2.
template <class T, class TO, int NT, int CS, int U2 = 4, bool REV = false>
__device__ __forceinline__ void row_single_body(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                int64_t stride, const int64_t* __restrict__ tokens,
                                                const uint8_t* __restrict__ mask, RowScale rs,
                                                float2* __restrict__ stats, float* __restrict__ qy,
                                                double* __restrict__ lp, int32_t* dev_status,
                                                TO* __restrict__ g_out, int64_t ostride) {
  namespace cg = cooperative_groups;
  constexpr int NW = NT / 32;
  const int rank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int64_t row = (int64_t)blockIdx.x / CS;
  const int gt = rank * NT + (int)threadIdx.x;  // thread index within the row's cluster
  __shared__ float sm_m[NW], sm_M2[NW];
  __shared__ double sm_s[NW];
  __shared__ float part_m, part_M2;  // this CTA's partial, read by the cluster through DSMEM
  __shared__ double part_s;
  __shared__ float sh_M2, sh_L2S, sh_qy;
  __shared__ int64_t sh_y;
  const bool live = row < rows;
  const bool valid = live && mask[row] != 0;  // uniform over the cluster
  const T* rp = logits + (live ? row : 0) * stride;
  TO* op = g_out + (live ? row : 0) * ostride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float M = -INFINITY, M2 = 0.f;
  double S = 0.0;
  if (valid) {
    const int64_t yt = tokens[row];
    if (threadIdx.x == 0) sh_y = yt;
    OnlineState st;
    st.init(rs);
    fwd_accumulate<T, 4, true>(rp, V, gt, CS * NT, st, (yt >= 0 && yt < V) ? yt : -1, make_policy(true));
    combine_lanes(st.m, st.R2, st.s, true, rs.sc, M, M2, S);
    if (lane == 0) {
      sm_m[warp] = M;
      sm_M2[warp] = M2;
      sm_s[warp] = S;
    }
    __syncthreads();
    if (warp == 0) {
      const bool act = lane < NW;
      combine_lanes(act ? sm_m[lane] : -INFINITY, act ? sm_M2[lane] : 0.f, act ? sm_s[lane] : 0.0, act, rs.sc, M,
                    M2, S);
      if (lane == 0) {
        part_m = M;
        part_M2 = M2;
        part_s = S;
      }
    }
  }
  if constexpr (CS > 1) {
    cg::cluster_group cl = cg::this_cluster();
    // phase 1: every CTA's partial is visible cluster-wide (release/acquire)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (valid && warp == 0) {
      const bool act = lane < CS;
      float pm = -INFINITY, pm2 = 0.f;
      double ps = 0.0;
      if (act) {
        pm = *cl.map_shared_rank(&part_m, lane);
        pm2 = *cl.map_shared_rank(&part_M2, lane);
        ps = *cl.map_shared_rank(&part_s, lane);
      }
      combine_lanes(pm, pm2, ps, act, rs.sc, M, M2, S);
    }
    // phase 2 (split): "done reading peers" now, wait only before exiting, so that no CTA's
    // shared memory disappears while a peer reads it and the barrier latency hides behind pass 2
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  }
  if (!live) {
    if constexpr (CS > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    return;
  }
  if (!valid) {
    bwd_row<T, TO, 4>(rp, op, V, gt, CS * NT, false, 0.f, 0.f, 0.f, 0.f, -1, 0.f);
    if constexpr (CS > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    return;
  }
  if (threadIdx.x == 0) {
    const int64_t y = sh_y;
    const bool ok = (y >= 0 && y < V);
    const float zy = ok ? Elem<T>::load1(rp + y) : 0.f;
    finalize_row(M, M2, S, zy, ok, row, rs, stats, qy, lp, dev_status);  // CS == 1: this CTA owns the row
    const float2 st2 = stats[row];  // written just above by this thread
    sh_M2 = st2.x;
    sh_L2S = st2.y;
    sh_qy = qy[row];
  }
  __syncthreads();
  bwd_row<T, TO, U2, true, REV>(rp, op, V, gt, CS * NT, true, rs.sc, sh_M2, sh_L2S, (float)rs.inv_temp, sh_y, sh_qy,
                                make_policy(false));
  if constexpr (CS > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

template <class T, class TO, int NT, int U2 = 4, bool REV = false>
__global__ void __launch_bounds__(NT) row_single1(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                  int64_t stride, const int64_t* __restrict__ tokens,
                                                  const uint8_t* __restrict__ mask, RowScale rs,
                                                  float2* __restrict__ stats, float* __restrict__ qy,
                                                  double* __restrict__ lp, int32_t* dev_status,
                                                  TO* __restrict__ g_out, int64_t ostride) {
  row_single_body<T, TO, NT, 1, U2, REV>(logits, rows, V, stride, tokens, mask, rs, stats, qy, lp, dev_status, g_out,
                                         ostride);
}

// ------------------------------------------------------------------------------ launch
}  // namespace

// deferred-scale row pass (row_single*): configuration by row length, see DESIGN.md §5.4
int launch_single(const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status,
                  void* grad_unscaled, int32_t g_dtype, int64_t g_row_stride, cudaStream_t s) {
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows > 0) {
    // Rows in flight x row bytes must stay inside L2 for pass 2 to hit it. Measured:
    // rows <= 128 KB: 256 threads per row (4 CTAs/SM); longer rows: 512 threads (2 CTAs/SM) with 8
    // vectors per thread in pass 2 — it keeps ~70 % of the re-reads in L2 and overlaps the two passes
    // across the SM's CTAs, which beats the exact-4V 2-CTA cluster variants (cfg 2/3/5/6). Pass 2
    // sweeps the row backwards (cfg 8 / 9 = cfg 4 / 0 reversed): the row's most recently streamed
    // vectors are re-read first, while still in L2 (Qwen 8.13 -> 7.96 ms, scripts/gpu_ab_rev.sh).
    const int64_t rb = x->vocab * (x->dtype == TBA_BF16 ? 2 : 4);
    const bool small = rb <= 128 * 1024;
#define TBA_SINGLE1(T_, TO_, NT_, U2_)                                                                          \
  row_single1<T_, TO_, NT_, U2_, true><<<(unsigned)rows, NT_, 0, s>>>(                                         \
      static_cast<const T_*>(x->logits), rows, x->vocab, x->row_stride, x->tokens, x->mask, rs, w.stats, w.qy, w.lp, \
      dev_status, static_cast<TO_*>(grad_unscaled), g_row_stride)
#define TBA_SINGLE(T_, TO_)                   \
  do {                                        \
    if (small) TBA_SINGLE1(T_, TO_, 256, 4);  \
    else TBA_SINGLE1(T_, TO_, 512, 8);        \
  } while (0)
    if (x->dtype == TBA_BF16) {
      if (g_dtype == TBA_BF16) TBA_SINGLE(uint16_t, uint16_t);
      else TBA_SINGLE(uint16_t, float);
    } else {
      if (g_dtype == TBA_BF16) TBA_SINGLE(float, uint16_t);
      else TBA_SINGLE(float, float);
    }
#undef TBA_SINGLE
#undef TBA_SINGLE1
    if (cudaGetLastError() != cudaSuccess) return TBA_ERR_CUDA;
  }
  return TBA_OK;
}


}  // namespace tba
