// a1: the row forward kernels (log-softmax statistics + gathered token log-prob per row).
#include "tba_device.cuh"

namespace tba {
namespace {
// TPR threads per row, 256/TPR rows per CTA (TPR = 32 ... 256). Each row group meets on its own
// named barrier (ids 1..8); a masked row's group exits as a whole.
template <class T, int TPR, int U, int NP = 0>
__global__ void __launch_bounds__(256) row_fwd_rows(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                     int64_t stride, const int64_t* __restrict__ tokens,
                                                     const uint8_t* __restrict__ mask, RowScale rs,
                                                     float2* __restrict__ stats, double* __restrict__ lp,
                                                     int32_t* dev_status) {
  constexpr int RPC = 256 / TPR, WPRS = TPR / 32 > 0 ? TPR / 32 : 1;
  __shared__ float sm_m[RPC][WPRS], sm_M2[RPC][WPRS];
  __shared__ double sm_s[RPC][WPRS];
  const int grp = threadIdx.x / TPR, gt = threadIdx.x % TPR;
  const int64_t row = (int64_t)blockIdx.x * RPC + grp;
  if (row >= rows || mask[row] == 0) return;
  fwd_row_group<T, TPR, U, NP>(logits, row, V, stride, tokens, rs, stats, lp, dev_status, sm_m, sm_M2, sm_s, grp, gt);
}

// ------------------------------------------------------------------------------ a1, TMA-staged
// Persistent, warp-specialised forward for long rows (A/B alternative, TBA_FWD_IMPL=tma). One
// producer lane streams the 16-byte aligned interior of every valid row through a STAGES-deep
// shared-memory ring with 1-D bulk copies (cp.async.bulk, mbarrier complete_tx, L2 evict_first);
// NCW consumer warps read each tile once. Warps never wait for each other at a row boundary:
// each posts its partial to a shared slot and the LAST warp to post combines the row.
template <class T, int NCW, int TILE, int STAGES, int NP = 0>
__global__ void __launch_bounds__((NCW + 1) * 32) row_fwd_tma(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                              int64_t stride, const int64_t* __restrict__ tokens,
                                                              const uint8_t* __restrict__ mask, RowScale rs,
                                                              float2* __restrict__ stats, double* __restrict__ lp,
                                                              int32_t* dev_status) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  constexpr int NC = NCW * 32;
  constexpr int TV = TILE / 16;          // vectors per tile
  constexpr int U = TV / NC;             // vectors per consumer thread per full tile
  constexpr int SLOTS = 2 * STAGES + 2;  // a warp is at most STAGES tiles (<= STAGES rows) ahead
  static_assert(TV % NC == 0 && U >= 1, "tile must split evenly over the consumer threads");
  static_assert(NCW <= 32, "");
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  __shared__ float sm_m[SLOTS][NCW], sm_M2[SLOTS][NCW];
  __shared__ double sm_s[SLOTS][NCW];
  __shared__ float sm_zy[SLOTS];
  __shared__ int sm_ok[SLOTS];
  __shared__ unsigned sm_cnt[SLOTS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < SLOTS) sm_cnt[threadIdx.x] = 0;
  __syncthreads();

  if (warp == NCW) {  // ---------------- producer warp: one elected lane issues the bulk copies
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        if (mask[row] == 0) continue;
        const T* rp = logits + row * stride;
        const int64_t h = head_elems(rp, V);
        const int64_t bytes = ((V - h) / VEC) * 16;
        const char* src = reinterpret_cast<const char*>(rp + h);
        for (int64_t off = 0; off < bytes; off += TILE) {
          const uint32_t n = (uint32_t)((bytes - off) < TILE ? (bytes - off) : TILE);
          mbar_wait(&empty[stage], phase ^ 1u);
          mbar_expect_tx(&full[stage], n);
          bulk_g2s(ring + (size_t)stage * TILE, src + off, n, &full[stage], pol);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumer warps
  const int ct = threadIdx.x;
  int stage = 0, slot = 0;
  uint32_t phase = 0;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    if (mask[row] == 0) continue;
    const T* rp = logits + row * stride;
    const int64_t h = head_elems(rp, V);
    const int64_t nvec = (V - h) / VEC;
    const int64_t bytes = nvec * 16;
    OnlineState st;
    st.init(rs);
    if (ct == 0) {
      const int64_t y = tokens[row];
      const bool ok = (y >= 0 && y < V);
      sm_zy[slot] = ok ? E::load1(rp + y) : 0.f;
      sm_ok[slot] = ok;
    }
    if (ct < h) st.add1(E::load1(rp + ct));
    const int64_t tail0 = h + nvec * VEC;
    if (tail0 + ct < V) st.add1(E::load1(rp + tail0 + ct));
    for (int64_t off = 0; off < bytes; off += TILE) {
      const int nv = (int)(((bytes - off) < TILE ? (bytes - off) : TILE) / 16);
      mbar_wait(&full[stage], phase);
      const uint4* sv = reinterpret_cast<const uint4*>(ring + (size_t)stage * TILE);
      if (nv == TV) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = sv[ct + u * NC];
        fwd_consume<T, U, NP>(v, st);
      } else {
        for (int k = ct; k < nv; k += NC) {
          uint4 v1[1] = {sv[k]};
          fwd_consume<T, 1>(v1, st);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }
    float M, M2;
    double S;
    combine_lanes(st.m, st.R2, st.s, true, rs.sc, M, M2, S);
    unsigned prev = 0;
    if (lane == 0) {
      sm_m[slot][warp] = M;
      sm_M2[slot][warp] = M2;
      sm_s[slot][warp] = S;
      __threadfence_block();
      prev = atomicAdd(&sm_cnt[slot], 1u);
    }
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev == NCW - 1) {  // last warp of this row: combine and finalise
      __threadfence_block();
      const bool act = lane < NCW;
      const volatile float* vm = sm_m[slot];
      const volatile float* vm2 = sm_M2[slot];
      const volatile double* vs = sm_s[slot];
      combine_lanes(act ? vm[lane] : -INFINITY, act ? vm2[lane] : 0.f, act ? vs[lane] : 0.0, act, rs.sc, M, M2, S);
      if (lane == 0) {
        const float zy = *(volatile float*)&sm_zy[slot];
        const bool ok = *(volatile int*)&sm_ok[slot] != 0;
        finalize_row(M, M2, S, zy, ok, row, rs, stats, lp, dev_status);
        sm_cnt[slot] = 0;
      }
    }
    if (++slot == SLOTS) slot = 0;
  }
}


// ------------------------------------------------------------------------------ launch
template <class T, int NCW, int TILE, int STAGES, int NP = 0>
int launch_fwd_tma_cfg(const T* lg, const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status,
                       cudaStream_t s) {
  auto kern = row_fwd_tma<T, NCW, TILE, STAGES, NP>;
  const int smem = TILE * STAGES;
  static int occ = 0;  // benign race: idempotent
  if (!occ) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return TBA_ERR_CUDA;
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, (NCW + 1) * 32, smem) != cudaSuccess || o < 1) o = 1;
    occ = o;
  }
  const int64_t rows = x->n_seq * x->seq_len;
  int64_t grid = (int64_t)device_sms() * occ;
  if (grid > rows) grid = rows;
  kern<<<(unsigned)grid, (NCW + 1) * 32, smem, s>>>(lg, rows, x->vocab, x->row_stride, x->tokens, x->mask, rs,
                                                     w.stats, w.lp, dev_status);
  return TBA_OK;
}

template <class T>
int launch_fwd_tma(const T* lg, const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status,
                   cudaStream_t s) {
  switch (switches().tma_cfg) {
    case 1: return launch_fwd_tma_cfg<T, 8, 8192, 8>(lg, x, w, rs, dev_status, s);
    case 2: return launch_fwd_tma_cfg<T, 8, 32768, 3>(lg, x, w, rs, dev_status, s);
    case 3: return launch_fwd_tma_cfg<T, 8, 32768, 3, 1>(lg, x, w, rs, dev_status, s);
    default: return launch_fwd_tma_cfg<T, 8, 16384, 4>(lg, x, w, rs, dev_status, s);
  }
}

template <class T>
void launch_fwd_rows_t(const T* lg, const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status,
                       cudaStream_t s, int tpr) {
  const int64_t rows = x->n_seq * x->seq_len;
  const int64_t rpc = 256 / tpr;
  const unsigned grid = (unsigned)((rows + rpc - 1) / rpc);
#define TBA_ROWS(TPR_)                                                                                               \
  row_fwd_rows<T, TPR_, kU><<<grid, 256, 0, s>>>(lg, rows, x->vocab, x->row_stride, x->tokens, x->mask, rs, w.stats, \
                                                 w.lp, dev_status)
  // Pairs per 16-byte vector whose exp2 runs on the FMA pipe (exp2_poly2) instead of MUFU: 1 of 4
  // relieves the XU pipe (75 % busy) and gives +3 % forward bandwidth on every BASELINE shape
  // (scripts/gpu_ab_np.sh; 2 of 4 over-loads the FMA/ALU pipes). TBA_FWD_NP overrides (A/B).
  const int np = env_int("TBA_FWD_NP", 1);
  if (tpr == 64 && np == 1) {
    row_fwd_rows<T, 64, kU, 1><<<grid, 256, 0, s>>>(lg, rows, x->vocab, x->row_stride, x->tokens, x->mask, rs,
                                                    w.stats, w.lp, dev_status);
    return;
  }
  if (tpr == 64 && np == 2) {
    row_fwd_rows<T, 64, kU, 2><<<grid, 256, 0, s>>>(lg, rows, x->vocab, x->row_stride, x->tokens, x->mask, rs,
                                                    w.stats, w.lp, dev_status);
    return;
  }
  switch (tpr) {
    case 32: TBA_ROWS(32); break;
    case 64: TBA_ROWS(64); break;
    case 128: TBA_ROWS(128); break;
    default: TBA_ROWS(256); break;
  }
#undef TBA_ROWS
}

}  // namespace

int launch_fwd_rows(const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status, cudaStream_t s) {
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows == 0) return TBA_OK;
  const int64_t esz = x->dtype == TBA_BF16 ? 2 : 4;
  const int tpr = fwd_tpr(x->vocab, esz);
  const bool tma = switches().fwd_tma && x->vocab * esz > kSmallRowBytes;
  int rc = TBA_OK;
  if (x->dtype == TBA_BF16) {
    auto lg = static_cast<const uint16_t*>(x->logits);
    if (tma) rc = launch_fwd_tma<uint16_t>(lg, x, w, rs, dev_status, s);
    else launch_fwd_rows_t<uint16_t>(lg, x, w, rs, dev_status, s, tpr);
  } else {
    auto lg = static_cast<const float*>(x->logits);
    if (tma) rc = launch_fwd_tma<float>(lg, x, w, rs, dev_status, s);
    else launch_fwd_rows_t<float>(lg, x, w, rs, dev_status, s, tpr);
  }
  if (rc) return rc;
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

}  // namespace tba
