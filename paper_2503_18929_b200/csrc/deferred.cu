// Deferred-scale row pass (NEXT 2 (ii)).
#include "tba_device.cuh"

namespace tba {
namespace {
#ifdef TBA_AB_DEFER_TRACE
// phase trace of the deferred kernel (A/B build only): per row [smid, start, pass-1 loads issued,
// pass 1 done, pass 2 start, end] in SM clocks
constexpr int TR_ROWS = 1 << 17;
__device__ unsigned long long g_trace[TR_ROWS * 6];
__device__ __forceinline__ unsigned long long clk() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
#define TR(i) \
  if (threadIdx.x == 0 && row < TR_ROWS) g_trace[row * 6 + (i)] = clk()
#else
#define TR(i)
#endif

// One CTA per valid row: pass 1 streams the row from HBM with an L2 evict_last policy (online
// max/sum); pass 2 re-reads the row — from its shared-memory stash and L2 — and writes the UNSCALED
// gradient G = inv_temp (1[v=y] - softmax) once. HBM bytes: 2V read + 2V write per valid row (the 4V
// floor) plus the re-reads that miss L2; the per-sequence factor grad_scale * g * eps_s is applied by
// the consumer (the LM-head backward, as a row scale), SURVEY §8(f) NEXT 2.
// Pass 1 of a long row with a shared-memory stash: the stash part (the row's first ks vectors) is
// fetched with cp.async straight into shared memory — all of it in flight at once, no registers held —
// while the threads stream the rest of the row through registers (L2 evict_last, for pass 2); then
// the stash part is consumed from shared memory. The sampled token's element is excluded as in
// fwd_accumulate (finalize_row adds it).
template <class T, int U, int NP = 0>
__device__ __forceinline__ void defer_pass1_async(const T* __restrict__ rp, int64_t V, int tid, int nthr,
                                                  OnlineState& st, int64_t y, uint4* __restrict__ stash, int ks,
                                                  int64_t trow = 0) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  const int64_t h = head_elems(rp, V);
  const int64_t nvec = (V - h) / VEC;
  const int64_t tail0 = h + nvec * VEC;
  const uint4* vp = reinterpret_cast<const uint4*>(rp + h);
  const uint64_t pol_first = make_policy(false), pol_last = make_policy(true);
  for (int k = tid; k < ks; k += nthr)
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(stash + k)),
                 "l"(vp + k), "l"(pol_first)
                 : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
#ifndef TBA_DEFER_PF_KB
#define TBA_DEFER_PF_KB 64
#endif
  // L2 prefetch of the rest of the row (bulk, no registers, no shared memory): the register loop's
  // loads then hit L2. TBA_DEFER_PF_KB < 0: the whole rest up front; > 0: that many KB ahead of the loop.
  constexpr int64_t PF_VEC = TBA_DEFER_PF_KB > 0 ? (int64_t)TBA_DEFER_PF_KB * 64 : 0;
  auto prefetch = [&](int64_t a, int64_t b) {  // vectors [a, b)
    if (b > nvec) b = nvec;
    for (int64_t o = a; o < b; o += 1024) {
      const int64_t n = (b - o < 1024 ? b - o : 1024) * 16;
      asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(vp + o), "r"((uint32_t)n),
                   "l"(pol_last)
                   : "memory");
    }
  };
  if (TBA_DEFER_PF_KB != 0 && tid == 0) prefetch(ks, TBA_DEFER_PF_KB < 0 ? nvec : ks + PF_VEC);
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
  // 32-bit vector indices (a row has < 2^31 vectors); full iterations are uniform over the CTA, so the
  // sampled token's iteration is one uniform test per iteration (as in fwd_accumulate)
  const int nv = (int)nvec;
  const int ky = (y >= h && y < tail0) ? (int)((y - h) / VEC) : -1;
  const int ey = ky >= 0 ? (int)((y - h) - (int64_t)ky * VEC) : 0;
  const int step = nthr * U;
  const int nfl = (nv - ks) / step;  // full iterations over the L2 part [ks, nv)
  const int rl = ky - ks;            // the token's index in the L2 part (< 0: not there)
  const int ityl = rl >= 0 ? rl / step : -1;
  const int uyl = (rl >= 0 && (rl % step) % nthr == tid) ? (rl % step) / nthr : -1;
  int k0 = ks + tid;
  for (int it = 0; it < nfl; ++it, k0 += step) {
    if (PF_VEC > 0 && tid == 0) prefetch(k0 + PF_VEC, k0 + PF_VEC + step);
    const uint4* p = vp + k0;
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_pol(p + u * nthr, pol_last);
    if (it == ityl) fwd_consume<T, U, NP, true>(v, st, uyl, ey);
    else fwd_consume<T, U, NP>(v, st);
  }
  for (int k = k0; k < nv; k += nthr) {
    uint4 v1[1] = {ldg_pol(vp + k, pol_last)};
    if (k == ky) fwd_consume<T, 1, 0, true>(v1, st, 0, ey);
    else fwd_consume<T, 1>(v1, st);
  }
#ifdef TBA_AB_DEFER_TRACE
  if (threadIdx.x == 0 && trow < TR_ROWS) g_trace[trow * 6 + 2] = clk();
#endif
  asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's own copies are in shared memory
  const int nfs = ks / step;  // full iterations over the stash part [0, ks)
  const int itys = (ky >= 0 && ky < ks) ? ky / step : -1;
  const int uys = (itys >= 0 && (ky % step) % nthr == tid) ? (ky % step) / nthr : -1;
  int j0 = tid;
  for (int it = 0; it < nfs; ++it, j0 += step) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = stash[j0 + u * nthr];
    if (it == itys) fwd_consume<T, U, NP, true>(v, st, uys, ey);
    else fwd_consume<T, U, NP>(v, st);
  }
  for (int k = j0; k < ks; k += nthr) {
    uint4 v1[1] = {stash[k]};
    if (k == ky) fwd_consume<T, 1, 0, true>(v1, st, 0, ey);
    else fwd_consume<T, 1>(v1, st);
  }
}

// Pass 2 of the deferred kernel: G over the row's L2 part (vectors [ks, nvec), in the order pass 1
// streamed them: oldest first, so no line waits longer than one pass; measured 1.5 % faster than
// sweeping from the end) and then its shared-memory stash (vectors [0, ks)); full
// iterations carry no bounds or stash tests (32-bit vector indices). The
// arithmetic is bwd_row's (fp32 pairs, the same roundings); the token's entry is stored last by the
// thread that stored its vector.
template <class T, class TO, int U, bool POLY>
__device__ __forceinline__ void defer_pass2(const T* __restrict__ rp, TO* __restrict__ op, int64_t V, int tid,
                                            int nthr, float sc, float M2, float L2S, float c, int64_t y, float qy,
                                            const uint4* __restrict__ stash, int ks) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  const int64_t h = head_elems(rp, V);
  if ((reinterpret_cast<uint64_t>(op + h) & 15u) != 0) {  // output not co-aligned
    bwd_row<T, TO, U>(rp, op, V, tid, nthr, true, sc, M2, L2S, c, y, qy);  // the scalar loop
    return;
  }
  const int nvec = (int)((V - h) / VEC);
  const int64_t vend = h + (int64_t)nvec * VEC;
  auto one = [&](int64_t i) {
    const float p = ex2(fmaf(E::load1(rp + i), sc, -M2) - L2S);
    Out<TO>::put1(op + i, (i == y) ? c * qy : -c * p);
  };
  for (int64_t i = tid; i < h; i += nthr) one(i);
  for (int64_t i = vend + tid; i < V; i += nthr) one(i);
  const uint4* vp = reinterpret_cast<const uint4*>(rp + h);
  TO* ob = op + h;
  const uint64_t sc2 = f2_pack(sc, sc), nM2 = f2_pack(-M2, -M2), nL2S = f2_pack(-L2S, -L2S), nc = f2_pack(-c, -c);
  // poly: this vector's last element pair takes the FMA-pipe exp2 (exp2_poly2) instead of MUFU.EX2 —
  // every other vector of an unrolled group, i.e. 1 of 8 element pairs (POLY: the stash path of long
  // rows): the XU pipe is the busiest (66 %), and 1 of 8 costs fewer issue slots than it frees
  // (measured 1.5 % faster; 1 of 4 slower; rows <= 128 KB 0.5 % slower)
  auto emit = [&](const uint4& v, int k, bool poly = false) {
    float d[VEC];
#pragma unroll
    for (int e = 0; e < VEC; e += 2) {
      const uint64_t x = fadd2(ffma2(f2_pack(E::get(v, e), E::get(v, e + 1)), sc2, nM2), nL2S);
      if (poly && e == VEC - 2) {
        f2_unpack(fmul2(exp2_poly2(x), nc), d[e], d[e + 1]);
      } else {
        float a, b;
        f2_unpack(x, a, b);
        f2_unpack(fmul2(f2_pack(ex2(a), ex2(b)), nc), d[e], d[e + 1]);
      }
    }
    store_vals<TO, VEC>(ob + (int64_t)k * VEC, d);
  };
  const uint64_t pol = make_policy(false);
  const int nl2 = nvec - ks;  // index f in [0, nl2) is vector ks + f
  int f0 = tid;
  for (; f0 + (U - 1) * nthr < nl2; f0 += nthr * U) {
    const uint4* p = vp + (ks + f0);
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_pol(p + u * nthr, pol);
#pragma unroll
    for (int u = 0; u < U; ++u) emit(v[u], ks + f0 + u * nthr, POLY && (u & 1) != 0);
  }
  for (; f0 < nl2; f0 += nthr) emit(ldg_pol(vp + (ks + f0), pol), ks + f0);
  int j0 = tid;
  for (; j0 + 3 * nthr < ks; j0 += nthr * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = stash[j0 + u * nthr];
#pragma unroll
    for (int u = 0; u < 4; ++u) emit(v[u], j0 + u * nthr, POLY && (u & 1) != 0);
  }
  for (; j0 < ks; j0 += nthr) emit(stash[j0], j0);
  if (y >= h && y < vend) {
    const int ky = (int)((y - h) / VEC);
    if ((ky >= ks ? (ky - ks) : ky) % nthr == tid) Out<TO>::put1(op + y, c * qy);
  }
}

// One CTA of NT threads per row (grid = rows): pass 1 (online max / sum, the stash part on chip when
// STASH_KB > 0), the CTA's fixed-order combine, the row statistics, pass 2 (G).
template <class T, class TO, int NT, int U2, int U1, int STASH_KB>
__global__ void __launch_bounds__(NT) row_single1(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                  int64_t stride, const int64_t* __restrict__ tokens,
                                                  const uint8_t* __restrict__ mask, RowScale rs,
                                                  float2* __restrict__ stats, float* __restrict__ qy,
                                                  double* __restrict__ lp, int32_t* dev_status,
                                                  TO* __restrict__ g_out, int64_t ostride) {
  constexpr int NW = NT / 32;
  const int64_t row = (int64_t)blockIdx.x;
  const int gt = (int)threadIdx.x;
  __shared__ float sm_m[NW], sm_M2[NW];
  __shared__ double sm_s[NW];
  __shared__ float sh_M2, sh_L2S, sh_qy;
  __shared__ int64_t sh_y;
  if (row >= rows) return;
  const bool valid = mask[row] != 0;
  const T* rp = logits + row * stride;
  TO* op = g_out + row * ostride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // STASH_KB > 0: the row's first STASH_KB KB of 16-byte vectors stay in shared memory between the
  // passes (pass 2 reads them on chip; only the rest of the row must survive in L2)
  extern __shared__ __align__(16) uint4 ds_stash[];
  const int64_t nvec_all = (V - head_elems(rp, V)) / Elem<T>::VEC;
  const int ds_ks = (int)(nvec_all < (int64_t)STASH_KB * 64 ? nvec_all : (int64_t)STASH_KB * 64);
  float M = -INFINITY, M2 = 0.f;
  double S = 0.0;
#ifdef TBA_AB_DEFER_TRACE
  if (threadIdx.x == 0 && row < TR_ROWS) {
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_trace[row * 6] = sm;
  }
#endif
  TR(1);
  if (!valid) {
    bwd_row<T, TO, 4>(rp, op, V, gt, NT, false, 0.f, 0.f, 0.f, 0.f, -1, 0.f);
    return;
  }
  float zy = 0.f;  // thread 0: the token's logit, loaded while pass 1 runs
  {
    const int64_t yt = tokens[row];
    if (threadIdx.x == 0) {
      sh_y = yt;
      if (yt >= 0 && yt < V) zy = Elem<T>::load1(rp + yt);
    }
    OnlineState st;
    st.init(rs);
    if (STASH_KB > 0)  // the stash part fetched with cp.async, all of it in flight at once
      defer_pass1_async<T, U1>(rp, V, gt, NT, st, (yt >= 0 && yt < V) ? yt : -1, ds_stash, ds_ks, row);
    else {
      if (gt == 0) {  // L2 bulk prefetch of the whole (short) row up front: the loads below then hit L2
        const uint64_t pl = make_policy(true);
        const int64_t hb = head_elems(rp, V);
        const char* b0 = reinterpret_cast<const char*>(rp + hb);
        const int64_t nb = ((V - hb) * (int64_t)sizeof(T)) & ~(int64_t)15;
        for (int64_t o = 0; o < nb; o += 16384) {
          const int64_t n = nb - o < 16384 ? nb - o : 16384;
          asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(b0 + o), "r"((uint32_t)n),
                       "l"(pl)
                       : "memory");
        }
      }
      fwd_accumulate<T, U1, true>(rp, V, gt, NT, st, (yt >= 0 && yt < V) ? yt : -1, make_policy(true));
    }
    combine_lanes(st.m, st.R2, st.s, true, rs.sc, M, M2, S);
    TR(3);
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
    }
  }
  if (threadIdx.x == 0) {  // (M, M2, S) of the whole row in thread 0 (warp 0's combine)
    const int64_t y = sh_y;
    const bool ok = (y >= 0 && y < V);
    float2 st2;
    float q;
    double v;
    row_stats(M, M2, S, zy, ok, rs, st2, q, v);
    const bool finite = (M > -INFINITY) && (M < INFINITY) && (st2.y > -INFINITY) && (st2.y < INFINITY);
    stats[row] = st2;
    qy[row] = q;
    lp[row] = v;
    if (dev_status) {
      const int f = (ok ? 0 : TBA_DEV_TOKEN_RANGE) | (finite ? 0 : TBA_DEV_NONFINITE_ROW);
      if (f) atomicOr(dev_status, f);
    }
    sh_M2 = st2.x;
    sh_L2S = st2.y;
    sh_qy = q;
  }
  __syncthreads();
  TR(4);
  // (rows <= 128 KB without a stash: the same forward-order loop, 1 % faster than sweeping from the
  // end on RhoMath / red-teaming / GSM8K)
  defer_pass2<T, TO, U2, (STASH_KB > 0)>(rp, op, V, gt, NT, rs.sc, sh_M2, sh_L2S, (float)rs.inv_temp, sh_y, sh_qy,
                                         STASH_KB > 0 ? ds_stash : nullptr, STASH_KB > 0 ? ds_ks : 0);
  TR(5);
}

}  // namespace

// deferred-scale row pass
int launch_single(const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status,
                  void* grad_unscaled, int32_t g_dtype, int64_t g_row_stride, cudaStream_t s) {
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows == 0) return TBA_OK;
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
      cudaFuncSetAttribute(row_single1<T_, TO_, NT_, U2_, U1_, SKB_>,                                      \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);                               \
      attr_ = true;                                                                                             \
    }                                                                                                           \
    row_single1<T_, TO_, NT_, U2_, U1_, SKB_><<<(unsigned)rows, NT_, dsm, s>>>(                            \
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

#ifdef TBA_AB_DEFER_TRACE
extern "C" int tba_debug_defer_trace(void* host, long long n) {
  if (n > (long long)tba::TR_ROWS * 6) n = (long long)tba::TR_ROWS * 6;
  return cudaMemcpyFromSymbol(host, tba::g_trace, (size_t)n * 8) == cudaSuccess ? 0 : 3;
}
#endif
