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
// Pass 1 of a long row with a shared-memory stash: the stash part (the row's first ks vectors) is
// fetched with cp.async straight into shared memory — all of it in flight at once, no registers held —
// while the threads stream the rest of the row through registers (L2 evict_last, for pass 2); then
// the stash part is consumed from shared memory. The sampled token's element is excluded as in
// fwd_accumulate (finalize_row adds it).
template <class T, int U>
__device__ __forceinline__ void defer_pass1_async(const T* __restrict__ rp, int64_t V, int tid, int nthr,
                                                  OnlineState& st, int64_t y, uint4* __restrict__ stash, int ks) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  const int64_t h = head_elems(rp, V);
  const int64_t nvec = (V - h) / VEC;
  const int64_t tail0 = h + nvec * VEC;
  const uint4* vp = reinterpret_cast<const uint4*>(rp + h);
  const uint64_t pol_first = make_policy(false), pol_last = make_policy(true);
  for (int64_t k = tid; k < ks; k += nthr)
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(stash + k)),
                 "l"(vp + k), "l"(pol_first)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (tid < h) {
    const float z = E::load1(rp + tid);
    if (tid == y) st.add1_excl(z);
    else st.add1(z);
  }
  for (int64_t i = tail0 + tid; i < V; i += nthr) {
    const float z = E::load1(rp + i);
    if (i == y) st.add1_excl(z);
    else st.add1(z);
  }
  const int64_t ky = (y >= h && y < tail0) ? (y - h) / VEC : -1;
  const int ey = ky >= 0 ? (int)((y - h) - ky * VEC) : 0;
  const int64_t step = (int64_t)nthr * U;
  int64_t k0 = ks + tid;
  for (; k0 + (int64_t)(U - 1) * nthr < nvec; k0 += step) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_pol(vp + k0 + (int64_t)u * nthr, pol_last);
    const int64_t kr = ky - k0;
    if (kr >= 0 && kr < step && kr % nthr == 0) fwd_consume<T, U, 0, true>(v, st, (int)(kr / nthr), ey);
    else fwd_consume<T, U>(v, st);
  }
  for (int64_t k = k0; k < nvec; k += nthr) {
    uint4 v1[1] = {ldg_pol(vp + k, pol_last)};
    if (k == ky) fwd_consume<T, 1, 0, true>(v1, st, 0, ey);
    else fwd_consume<T, 1>(v1, st);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's own copies are in shared memory
  int64_t j0 = tid;
  for (; j0 + (int64_t)(U - 1) * nthr < ks; j0 += step) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = stash[j0 + (int64_t)u * nthr];
    const int64_t kr = ky - j0;
    if (kr >= 0 && kr < step && kr % nthr == 0) fwd_consume<T, U, 0, true>(v, st, (int)(kr / nthr), ey);
    else fwd_consume<T, U>(v, st);
  }
  for (int64_t k = j0; k < ks; k += nthr) {
    uint4 v1[1] = {stash[k]};
    if (k == ky) fwd_consume<T, 1, 0, true>(v1, st, 0, ey);
    else fwd_consume<T, 1>(v1, st);
  }
}

template <class T, class TO, int NT, int CS, int U2 = 4, bool REV = false, int U1 = 4, int STASH_KB = 0>
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
  // STASH_KB > 0: the row's first STASH_KB KB of 16-byte vectors stay in shared memory between the
  // passes (pass 2 reads them on chip; only the rest of the row must survive in L2)
  extern __shared__ __align__(16) uint4 ds_stash[];
  const int64_t nvec_all = (V - head_elems(rp, V)) / Elem<T>::VEC;
  const int ds_ks = (int)(nvec_all < (int64_t)STASH_KB * 64 ? nvec_all : (int64_t)STASH_KB * 64);
  float M = -INFINITY, M2 = 0.f;
  double S = 0.0;
  if (valid) {
    const int64_t yt = tokens[row];
    if (threadIdx.x == 0) sh_y = yt;
    OnlineState st;
    st.init(rs);
    if (STASH_KB > 0)  // the stash part fetched with cp.async, all of it in flight at once
      defer_pass1_async<T, U1>(rp, V, gt, CS * NT, st, (yt >= 0 && yt < V) ? yt : -1, ds_stash, ds_ks);
    else
      fwd_accumulate<T, U1, true>(rp, V, gt, CS * NT, st, (yt >= 0 && yt < V) ? yt : -1, make_policy(true));
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
                                make_policy(false), STASH_KB > 0 ? ds_stash : nullptr, ds_ks);
  if constexpr (CS > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

template <class T, class TO, int NT, int U2 = 4, bool REV = false, int U1 = 4, int STASH_KB = 0>
__global__ void __launch_bounds__(NT) row_single1(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                  int64_t stride, const int64_t* __restrict__ tokens,
                                                  const uint8_t* __restrict__ mask, RowScale rs,
                                                  float2* __restrict__ stats, float* __restrict__ qy,
                                                  double* __restrict__ lp, int32_t* dev_status,
                                                  TO* __restrict__ g_out, int64_t ostride) {
  row_single_body<T, TO, NT, 1, U2, REV, U1, STASH_KB>(logits, rows, V, stride, tokens, mask, rs, stats, qy, lp,
                                                       dev_status, g_out, ostride);
}

// ------------------------------------------------------------------------------ SMEM-resident rows
#ifdef TBA_AB_DEFER_SMEM
// The row pass with the row kept ON CHIP between its two passes, so the HBM traffic is exactly 2V
// read + 2V write per valid row (the 4V floor) whatever L2 does. Persistent: one CTA per SM, CS CTAs
// (an SM pair for rows of up to ~376 KB: a bf16 Qwen row is 304 KB) per cluster; cluster c takes
// rows c, c + n_clusters, ... Each CTA owns a contiguous part (1/CS) of every row's 16-byte-aligned
// interior.
//   * producer warp (one lane): streams the parts, tile by tile (8 KB cp.async.bulk, L2 evict_first,
//     mbarrier complete_tx), into a ring of DS_SLOTS slots — at most a part plus DS_SLOTS - part
//     slots of look-ahead into the next row, released slot by slot as pass 2 finishes with them;
//   * DS_NCW consumer warps: pass 1 over the row's tiles (online max / sum, the token's element
//     excluded: finalize_row), the CTA partial combined with the peer's through distributed shared
//     memory (st.shared::cluster + a remote mbarrier arrive; one exchange per row), then pass 2 over
//     the SAME tiles in shared memory: G = inv_temp (1[v=y] - softmax), 16-byte streaming stores.
// Rows whose output is not 16-byte aligned at the input's element offset, or whose part would not
// fit the ring, use row_single1 (above).
constexpr int DS_TILE = 16384;  // bytes per slot = one bulk copy
constexpr int DS_SLOTS = 13;    // 208 KB ring
constexpr int DS_NCW = 16;      // consumer warps
constexpr int DS_THREADS = (DS_NCW + 1) * 32;
constexpr int DS_LOOKAHEAD = 3;  // slots a part leaves free at least
constexpr size_t DS_SMEM = (size_t)DS_SLOTS * DS_TILE;

struct DsArgs {
  const void* logits;
  void* g;
  const int64_t* tokens;
  const uint8_t* mask;
  float2* stats;
  float* qy;
  double* lp;
  int32_t* dev_status;
  unsigned int* zero_counter;
  int64_t rows, V, stride, ostride;
  RowScale rs;
};

__device__ __forceinline__ uint32_t ds_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void ds_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ uint32_t ds_mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void ds_wait_cluster(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

// this CTA's part of a row: interior vectors [v0, v1) (16-byte vectors after the h head elements)
struct DsPart {
  int64_t h, nvec, v0, v1;
};
template <class T>
__device__ __forceinline__ DsPart ds_part(const T* rp, int64_t V, int rank, int CS) {
  DsPart q;
  q.h = head_elems(rp, V);
  q.nvec = (V - q.h) / Elem<T>::VEC;
  const int64_t per = (q.nvec + CS - 1) / CS;
  q.v0 = per * rank < q.nvec ? per * rank : q.nvec;
  q.v1 = q.v0 + per < q.nvec ? q.v0 + per : q.nvec;
  return q;
}

template <class T, class TO, int CS>
__global__ void __launch_bounds__(DS_THREADS, 1) row_smem(DsArgs a) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  constexpr int TV = DS_TILE / 16;  // vectors per tile
  constexpr int NC = DS_NCW * 32;
  static_assert(TV % NC == 0, "");
  constexpr int U = TV / NC;  // vectors per consumer thread per tile
  extern __shared__ __align__(1024) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[DS_SLOTS], empty[DS_SLOTS], xbar[2];
  __shared__ float x_m[2], x_M2[2];  // the peer's partial of the row (written by the peer)
  __shared__ double x_s[2];
  __shared__ float w_m[DS_NCW], w_M2[DS_NCW];
  __shared__ double w_s[DS_NCW];
  __shared__ float r_M2, r_L2S, r_qy;
  const T* __restrict__ logits = static_cast<const T*>(a.logits);
  TO* __restrict__ gout = static_cast<TO*>(a.g);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CS > 1 ? ds_rank() : 0u;
  const int64_t cid = blockIdx.x / CS, ncl = gridDim.x / CS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < DS_SLOTS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], DS_NCW);
    }
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (CS > 1) ds_cluster_sync();  // the peer's barriers exist before any remote arrive
  pdl_trigger();
  pdl_wait();
  if (a.zero_counter && blockIdx.x == 0 && threadIdx.x == 0) *a.zero_counter = 0u;

  if (warp == DS_NCW) {  // ------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t slot = 0, phase = 0;
      for (int64_t row = cid; row < a.rows; row += ncl) {
        if (a.mask[row] == 0) continue;
        const T* rp = logits + row * a.stride;
        const DsPart q = ds_part(rp, a.V, (int)rank, CS);
        const char* src = reinterpret_cast<const char*>(rp + q.h) + q.v0 * 16;
        const int64_t bytes = (q.v1 - q.v0) * 16;
        for (int64_t off = 0; off < bytes; off += DS_TILE) {
          const uint32_t n = (uint32_t)(bytes - off < DS_TILE ? bytes - off : DS_TILE);
          mbar_wait(&empty[slot], phase ^ 1u);
          mbar_expect_tx(&full[slot], n);
          bulk_g2s(ring + (size_t)slot * DS_TILE, src + off, n, &full[slot], pol);
          if (++slot == DS_SLOTS) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else {  // --------------------------------------------------------------- consumers
    const int ct = threadIdx.x;
    uint32_t slot = 0, phase = 0;
    uint32_t xn = 0;  // rows exchanged with the peer so far
    const float sc = a.rs.sc;
    for (int64_t row = cid; row < a.rows; row += ncl) {
      const T* rp = logits + row * a.stride;
      TO* op = gout + row * a.ostride;
      const DsPart q = ds_part(rp, a.V, (int)rank, CS);
      const int64_t tail0 = q.h + q.nvec * VEC;
      const int64_t nvp = q.v1 - q.v0;
      if (a.mask[row] == 0) {  // masked: write zeros (op + h is 16-byte aligned: host check), read nothing
        float zf[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) zf[e] = 0.f;
        for (int64_t k = q.v0 + ct; k < q.v1; k += NC) store_vals<TO, VEC>(op + q.h + k * VEC, zf);
        if (rank == 0) {
          if (ct < q.h) Out<TO>::put1(op + ct, 0.f);
          if (tail0 + ct < a.V) Out<TO>::put1(op + tail0 + ct, 0.f);
        }
        continue;
      }
      const int64_t y = a.tokens[row];
      const bool ok = (y >= 0 && y < a.V);
      const int64_t ky = (ok && y >= q.h && y < tail0) ? (y - q.h) / VEC : -1;
      const int ey = ky >= 0 ? (int)((y - q.h) - ky * VEC) : 0;
      // ---- pass 1
      OnlineState st;
      st.init(a.rs);
      if (rank == 0) {  // head / tail scalars (fewer than VEC each)
        if (ct < q.h) {
          const float z = E::load1(rp + ct);
          if (ct == y) st.add1_excl(z);
          else st.add1(z);
        }
        if (tail0 + ct < a.V) {
          const float z = E::load1(rp + tail0 + ct);
          if (tail0 + ct == y) st.add1_excl(z);
          else st.add1(z);
        }
      }
      const uint32_t slot0 = slot;
      for (int64_t t0 = 0; t0 < nvp; t0 += TV) {
        mbar_wait(&full[slot], phase);
        const uint4* sv = reinterpret_cast<const uint4*>(ring + (size_t)slot * DS_TILE);
        if (t0 + TV <= nvp) {  // a full tile: U vectors per thread, one consume step
          uint4 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) v[u] = sv[ct + u * NC];
          const int64_t kr = ky - q.v0 - t0 - ct;  // the token's vector relative to this thread's first
          if (kr >= 0 && kr < (int64_t)U * NC && kr % NC == 0) fwd_consume<T, U, 1, true>(v, st, (int)(kr / NC), ey);
          else fwd_consume<T, U, 1>(v, st);
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t k = t0 + ct + u * NC;  // vector within the part
            if (k < nvp) {
              uint4 v1[1] = {sv[ct + u * NC]};
              if (q.v0 + k == ky) fwd_consume<T, 1, 0, true>(v1, st, 0, ey);
              else fwd_consume<T, 1>(v1, st);
            }
          }
        }
        if (++slot == DS_SLOTS) {
          slot = 0;
          phase ^= 1u;
        }
      }
      // ---- the CTA's partial, then the row's (combined with the peer's in rank order)
      float M, M2;
      double S;
      combine_lanes(st.m, st.R2, st.s, true, sc, M, M2, S);
      if (lane == 0) {
        w_m[warp] = M;
        w_M2[warp] = M2;
        w_s[warp] = S;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
      if (warp == 0) {
        const bool act = lane < DS_NCW;
        combine_lanes(act ? w_m[lane] : -INFINITY, act ? w_M2[lane] : 0.f, act ? w_s[lane] : 0.0, act, sc, M, M2, S);
        if (CS > 1) {
          const uint32_t par = xn & 1u;
          if (lane == 0) {  // my partial into the peer's slot, then arrive on the peer's barrier
            const uint32_t peer = rank ^ 1u;
            asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ds_mapa(&x_m[par], peer)), "f"(M) : "memory");
            asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ds_mapa(&x_M2[par], peer)), "f"(M2) : "memory");
            asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ds_mapa(&x_s[par], peer)), "d"(S) : "memory");
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ds_mapa(&xbar[par], peer))
                         : "memory");
          }
          ds_wait_cluster(&xbar[par], (xn >> 1) & 1u);
          // rank order: lane 0 = rank 0's partial, lane 1 = rank 1's
          const bool mine = (uint32_t)lane == rank;
          const bool act2 = lane < 2;
          const float pm = mine ? M : x_m[par], pm2 = mine ? M2 : x_M2[par];
          const double ps = mine ? S : x_s[par];
          combine_lanes(act2 ? pm : -INFINITY, act2 ? pm2 : 0.f, act2 ? ps : 0.0, act2, sc, M, M2, S);
        }
        if (lane == 0) {
          const float zy = ok ? E::load1(rp + y) : 0.f;
          if (rank == 0) {
            finalize_row(M, M2, S, zy, ok, row, a.rs, a.stats, a.qy, a.lp, a.dev_status);
            const float2 s2 = a.stats[row];
            r_M2 = s2.x;
            r_L2S = s2.y;
            r_qy = a.qy[row];
          } else {  // the peer computes the same statistics without writing the outputs
            float2 s2;
            float qq;
            double lpv;
            row_stats(M, M2, S, zy, ok, a.rs, s2, qq, lpv);
            r_M2 = s2.x;
            r_L2S = s2.y;
            r_qy = qq;
          }
        }
      }
      ++xn;
      asm volatile("bar.sync 1, %0;" ::"r"(NC) : "memory");
      // ---- pass 2 over the same tiles (still in shared memory)
      const float nM2 = -r_M2, L2S = r_L2S, c = (float)a.rs.inv_temp, cq = c * r_qy;
      if (rank == 0) {
        auto one = [&](int64_t i) {
          const float p = ex2(fmaf(E::load1(rp + i), sc, nM2) - L2S);
          Out<TO>::put1(op + i, i == y ? cq : -c * p);
        };
        if (ct < q.h) one(ct);
        if (tail0 + ct < a.V) one(tail0 + ct);
      }
      uint32_t s2 = slot0;
      for (int64_t t0 = 0; t0 < nvp; t0 += TV) {
        const uint4* sv = reinterpret_cast<const uint4*>(ring + (size_t)s2 * DS_TILE);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t k = t0 + ct + u * NC;
          if (k < nvp) {
            const uint4 v = sv[ct + u * NC];
            float d[VEC];
#pragma unroll
            for (int e = 0; e < VEC; ++e) d[e] = -c * ex2(fmaf(E::get(v, e), sc, nM2) - L2S);
            if (q.v0 + k == ky) {
#pragma unroll
              for (int e = 0; e < VEC; ++e)
                if (e == ey) d[e] = cq;
            }
            store_vals<TO, VEC>(op + q.h + (q.v0 + k) * VEC, d);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s2]);
        if (++s2 == DS_SLOTS) s2 = 0;
      }
    }
  }
  if (CS > 1) ds_cluster_sync();  // no CTA leaves while its peer may still write into it
}
#endif  // TBA_AB_DEFER_SMEM

// ------------------------------------------------------------------------------ launch
#ifdef TBA_AB_DEFER_SMEM
// Can row_smem take this call? Every row's output must be 16-byte aligned at the element where the
// input row's 16-byte-aligned interior starts (rows and outputs repeat their alignment with a period
// of at most 16 rows), and one CTA's part of a row must leave DS_LOOKAHEAD slots of the ring free.
// Returns the cluster size (1 or 2) or 0.
int smem_cluster_size(const tba_rows* x, const void* g, int32_t g_dtype, int64_t g_row_stride) {
  const int64_t esz = x->dtype == TBA_BF16 ? 2 : 4, oesz = g_dtype == TBA_BF16 ? 2 : 4;
  const int64_t rows = x->n_seq * x->seq_len;
  for (int64_t r = 0; r < 16 && r < rows; ++r) {
    const uintptr_t in = reinterpret_cast<uintptr_t>(x->logits) + (uintptr_t)(r * x->row_stride * esz);
    const int64_t h = (int64_t)(((16u - (in & 15u)) & 15u) / esz);
    const uintptr_t out = reinterpret_cast<uintptr_t>(g) + (uintptr_t)((r * g_row_stride + h) * oesz);
    if (out & 15u) return 0;
  }
  const int64_t vec = 16 / esz, part_cap = (int64_t)(DS_SLOTS - DS_LOOKAHEAD) * DS_TILE;
  const int64_t interior = (x->vocab / vec) * 16;  // an upper bound on the aligned interior's bytes
  if (interior <= part_cap) return 1;
  if ((interior + 1) / 2 + 16 <= part_cap) return 2;
  return 0;
}

template <class T, class TO>
int launch_smem_t(const DsArgs& a, int cs, cudaStream_t s) {
  auto kern = cs == 2 ? row_smem<T, TO, 2> : row_smem<T, TO, 1>;
  static bool attr[2][64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return TBA_ERR_CUDA;
  if (!attr[cs - 1][dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DS_SMEM) != cudaSuccess)
      return TBA_ERR_CUDA;
    attr[cs - 1][dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[na++].val.programmaticStreamSerializationAllowed = 1;
  if (cs > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cs;
    at[na].val.clusterDim.y = 1;
    at[na++].val.clusterDim.z = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cfg.blockDim = dim3(DS_THREADS);
  cfg.dynamicSmemBytes = DS_SMEM;
  cfg.stream = s;
  int64_t ncl = device_sms() / cs;  // one CTA per SM (the ring takes the shared memory)
  if (ncl > a.rows) ncl = a.rows;
  if (ncl < 1) ncl = 1;
  cfg.gridDim = dim3((unsigned)(ncl * cs));
  return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

#endif  // TBA_AB_DEFER_SMEM

}  // namespace

// deferred-scale row pass: row_single1, the L2 two-pass kernel; row_smem (rows kept
// on chip, exact 4V) only in the TBA_AB_DEFER_SMEM A/B build
int launch_single(const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status,
                  void* grad_unscaled, int32_t g_dtype, int64_t g_row_stride, cudaStream_t s) {
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows == 0) return TBA_OK;
#ifdef TBA_AB_DEFER_SMEM
  const int cs = smem_cluster_size(x, grad_unscaled, g_dtype, g_row_stride);
#else
  const int cs = 0;  // row_smem measured slower than the L2 two-pass kernel: A/B build only
#endif
#ifdef TBA_AB_DEFER_SMEM
  if (cs > 0) {
    DsArgs a{x->logits, grad_unscaled, x->tokens, x->mask, w.stats, w.qy, w.lp, dev_status, nullptr, rows,
             x->vocab, x->row_stride, g_row_stride, rs};
    if (x->dtype == TBA_BF16)
      return g_dtype == TBA_BF16 ? launch_smem_t<uint16_t, uint16_t>(a, cs, s) : launch_smem_t<uint16_t, float>(a, cs, s);
    return g_dtype == TBA_BF16 ? launch_smem_t<float, uint16_t>(a, cs, s) : launch_smem_t<float, float>(a, cs, s);
  }
#else
  (void)cs;
#endif
  // Fallback: the row is streamed twice through L2 (rows <= 128 KB: 256 threads per row; longer: 512
  // threads with 8 vectors per thread in pass 2, swept backwards so its most recently streamed
  // vectors are re-read first).
  const int64_t rb = x->vocab * (x->dtype == TBA_BF16 ? 2 : 4);
  const bool small = rb <= 128 * 1024;
#define TBA_SINGLE1(T_, TO_, NT_, U2_, U1_, SKB_)                                                                \
  do {                                                                                                          \
    static bool attr_ = false;                                                                                  \
    const size_t dsm = (size_t)(SKB_) * 1024;                                                                   \
    if (dsm > 48 * 1024 && !attr_) {                                                                            \
      cudaFuncSetAttribute(row_single1<T_, TO_, NT_, U2_, true, U1_, SKB_>,                                      \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);                               \
      attr_ = true;                                                                                             \
    }                                                                                                           \
    row_single1<T_, TO_, NT_, U2_, true, U1_, SKB_><<<(unsigned)rows, NT_, dsm, s>>>(                            \
      static_cast<const T_*>(x->logits), rows, x->vocab, x->row_stride, x->tokens, x->mask, rs, w.stats, w.qy, w.lp, \
      dev_status, static_cast<TO_*>(grad_unscaled), g_row_stride);                                             \
  } while (0)
  // rows <= 128 KB: 256 threads per row; longer: 512 threads, 8 vectors per thread in flight in pass
  // 2, and the row's first TBA_DEFER_STASH_KB KB kept in shared memory between the passes (DESIGN.md
  // §5.4; A/B builds may override the size)
#ifndef TBA_DEFER_STASH_KB
#define TBA_DEFER_STASH_KB 96
#endif
#define TBA_SINGLE(T_, TO_)                                       \
  do {                                                            \
    if (small) TBA_SINGLE1(T_, TO_, 256, 4, 4, 0);                \
    else TBA_SINGLE1(T_, TO_, 512, 8, 4, TBA_DEFER_STASH_KB);     \
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
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

}  // namespace tba
