// a1-a5 in one persistent launch (NEXT 2 (i)).
#include "tba_device.cuh"

namespace tba {
namespace {
__device__ __forceinline__ void decode_item(const FusedArgs& a, int64_t i, bool& bwd, int& g, int& j) {
  const int64_t pre = (int64_t)a.D * a.nF;
  if (i < pre) {
    bwd = false;
    g = (int)(i / a.nF);
    j = (int)(i % a.nF);
    return;
  }
  i -= pre;
  const int64_t blk = a.nF + a.nB, nfull = a.groups - a.D;
  if (i < nfull * blk) {
    const int k = (int)(i / blk), r = (int)(i % blk);
    if (r < a.nF) {
      bwd = false;
      g = k + a.D;
      j = r;
    } else {
      bwd = true;
      g = k;
      j = r - a.nF;
    }
    return;
  }
  i -= nfull * blk;
  bwd = true;
  g = (int)(nfull + i / a.nB);
  j = (int)(i % a.nB);
}

template <class T, class TO, int TPR_F, int TPR_B>
__global__ void __launch_bounds__(256) tb_fused(FusedArgs a) {
  constexpr int RF = 256 / TPR_F, WPR = TPR_F / 32, RB = 256 / TPR_B;
  __shared__ int sh_item;
  __shared__ bool sh_head;
  __shared__ float sm_m[RF][WPR], sm_M2[RF][WPR];
  __shared__ double sm_s[RF][WPR];
  const int64_t n_items = (int64_t)a.groups * (a.nF + a.nB);
  const int64_t rows_per_group = (int64_t)a.K * a.T;
  const T* logits = static_cast<const T*>(a.logits);
  TO* dlogits = static_cast<TO*>(a.dlogits);
  const int lane = threadIdx.x & 31;
  for (;;) {
    if (threadIdx.x == 0) sh_item = (int)atomicAdd(a.work, 1u);
    __syncthreads();
    const int64_t item = sh_item;
    __syncthreads();
    if (item >= n_items) break;
    bool bwd;
    int g, j;
    decode_item(a, item, bwd, g, j);
    const int64_t gr0 = (int64_t)g * rows_per_group;
    if (!bwd) {
      // ---- forward rows [gr0 + j*RF, +RF) of group g, TPR_F threads per row
      const int grp = threadIdx.x / TPR_F, gt = threadIdx.x % TPR_F, wig = gt >> 5;
      const int64_t rin = (int64_t)j * RF + grp;  // row within the group
      const int64_t row = gr0 + rin;
      if (rin < rows_per_group && a.mask[row]) {
        const T* rp = logits + row * a.stride;
        const int64_t y = a.tokens[row];
        const bool ok = (y >= 0 && y < a.V);
        float zy = 0.f;
        if (gt == 0 && ok) zy = Elem<T>::load1(rp + y);
        OnlineState st;
        st.init(a.rs);
        fwd_accumulate<T, kFusedU, false, (TPR_F == 64 ? -1 : 1)>(rp, a.V, gt, TPR_F, st, ok ? y : -1);  // as two-call
        float M, M2;
        double S;
        combine_lanes(st.m, st.R2, st.s, true, a.rs.sc, M, M2, S);
        if (WPR == 1) {
          if (lane == 0) finalize_row(M, M2, S, zy, ok, row, a.rs, a.stats, a.qy, a.lp, a.dev_status);
        } else {
          if (lane == 0) {
            sm_m[grp][wig] = M;
            sm_M2[grp][wig] = M2;
            sm_s[grp][wig] = S;
          }
          asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(TPR_F) : "memory");
          if (wig == 0) {
            const bool act = lane < WPR;
            combine_lanes(act ? sm_m[grp][lane] : -INFINITY, act ? sm_M2[grp][lane] : 0.f,
                          act ? sm_s[grp][lane] : 0.0, act, a.rs.sc, M, M2, S);
            if (lane == 0) finalize_row(M, M2, S, zy, ok, row, a.rs, a.stats, a.qy, a.lp, a.dev_status);
          }
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int64_t n = rows_per_group - (int64_t)j * RF;
        n = n < RF ? n : RF;
        __threadfence();
        const unsigned prev = atomicAdd(&a.rows_done[g], (unsigned)n);
        sh_head = (prev + (unsigned)n == (unsigned)rows_per_group);
        if (sh_head) __threadfence();
      }
      __syncthreads();
      if (sh_head) {
        // ---- group head (Eq. 4 / Eq. 3 and Eq. 5) by the CTA that finished the group's last row
        const int64_t s0 = (int64_t)g * a.K;
        seq_sums(a.lp, a.mask, a.n_seq, a.T, s0, a.K, a.seq_logp, a.n_tokens, nullptr);
        __syncthreads();
        if (threadIdx.x < 32) {  // warp 0: the group head, as seq_head
          tb_group_head((int64_t)g, a.K, a.ref_logp, a.log_reward, a.log_z_param, a.inv_beta, a.seq_logp, a.log_z,
                        a.resid, a.group_sq, (int)threadIdx.x);
          __threadfence();
          __syncwarp();
        }
        if (threadIdx.x == 0) {
          __threadfence();
          st_release(&a.ready[g], 1u);
          if (atomicAdd(a.groups_done, 1u) == (unsigned)a.groups - 1) {
            __threadfence();
            double tot = 0.0;
            for (int q = 0; q < a.groups; ++q) tot += __ldcg(a.group_sq + q);
            a.partial[0] = tot * a.inv_n_global;
            a.partial[1] = (double)a.n_seq;
            a.partial[2] = (double)a.groups;
          }
        }
      }
    } else {
      // ---- backward rows [gr0 + j*RB, +RB) of group g, TPR_B threads per row
      if (threadIdx.x == 0) {
        unsigned ns = 32;
        while (ld_acquire(&a.ready[g]) == 0u) {
          __nanosleep(ns);
          ns = ns < 2048 ? 2 * ns : ns;
        }
      }
      __syncthreads();
      const int grp = threadIdx.x / TPR_B, tid = threadIdx.x % TPR_B;
      const int64_t rin = (int64_t)j * RB + grp;
      if (rin < rows_per_group) {
        const int64_t row = gr0 + rin;
        const bool valid = a.mask[row] != 0;
        float M2 = 0.f, L2S = 0.f, c = 0.f, qy = 0.f;
        int64_t y = -1;
        if (valid) {
          const float2 stt = __ldcg(a.stats + row);
          M2 = stt.x;
          L2S = stt.y;
          qy = __ldcg(a.qy + row);
          c = (float)(a.grad_scale * a.rs.inv_temp * __ldcg(a.resid + row / a.T));
          y = a.tokens[row];
        }
        bwd_row<T, TO, 4>(logits + row * a.stride, dlogits + row * a.ostride, a.V, tid, TPR_B, valid, a.rs.sc, M2,
                          L2S, c, y, qy);
      }
    }
  }
}


// ------------------------------------------------------------------------------ launch
template <class T, class TO, int TPR_F, int TPR_B>
int launch_fused_t(FusedArgs& a, cudaStream_t s) {
  auto kern = tb_fused<T, TO, TPR_F, TPR_B>;
  static int occ = 0;  // benign race: idempotent
  if (!occ) {
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, 256, 0) != cudaSuccess || o < 1) o = 1;
    occ = o;
  }
  a.RF = 256 / TPR_F;
  a.RB = 256 / TPR_B;
  const int64_t rpg = (int64_t)a.K * a.T;
  a.nF = (int)((rpg + a.RF - 1) / a.RF);
  a.nB = (int)((rpg + a.RB - 1) / a.RB);
  const int64_t items = (int64_t)a.groups * (a.nF + a.nB);
  int64_t grid = (int64_t)device_sms() * occ;
  if (grid > items) grid = items;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, 256, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

template <class T, class TO>
int launch_fused_tpr(FusedArgs& a, int tf, int tb, cudaStream_t s) {
  if (tf == 32) return tb == 32 ? launch_fused_t<T, TO, 32, 32>(a, s) : launch_fused_t<T, TO, 32, 256>(a, s);
  return tb == 32 ? launch_fused_t<T, TO, 64, 32>(a, s) : launch_fused_t<T, TO, 64, 256>(a, s);
}

}  // namespace

int launch_fused(FusedArgs& a, int32_t in_dtype, int32_t out_dtype, int tf, int tb, cudaStream_t s) {
  if (in_dtype == TBA_BF16)
    return out_dtype == TBA_BF16 ? launch_fused_tpr<uint16_t, uint16_t>(a, tf, tb, s)
                                 : launch_fused_tpr<uint16_t, float>(a, tf, tb, s);
  return out_dtype == TBA_BF16 ? launch_fused_tpr<float, uint16_t>(a, tf, tb, s)
                               : launch_fused_tpr<float, float>(a, tf, tb, s);
}

}  // namespace tba
