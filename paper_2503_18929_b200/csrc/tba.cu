// libtba.so — the trajectory-balance loss head of TBA (arXiv 2503.18929) for B200 (sm_100a).
//
// Kernels:
//   row_fwd_rows  a1   stream each valid logits row from HBM once (TPR threads per row, 128-bit
//                      loads): online max + sum of 2^(z*sc - R2) with one MUFU ex2 per element
//                      (packed FFMA2/FADD2), gather z[y]; writes per-row (M2, log2 S) and the
//                      token log-prob (fp64).
//   row_fwd_tma   a1   alternative: persistent, warp-specialised, cp.async.bulk + mbarrier ring.
//   seq_head      a2+a3 per-sequence fixed-order fp64 sums of token log-probs (log pi(y|x)) and
//                      token counts; per group Eq. 4 log Z (or a learned log Z, Eq. 3) and the
//                      Eq. 5 residuals; the last CTA reduces the per-group sums of squares.
//   tbap_head     a2+a3' TBA' (Eq. 16): per-group advantages and per-token IS-weighted coefficients.
//   row_bwd       a5   stream each valid row again: dz = c (1[v=y] - 2^(z*sc - M2 - log2 S)); c per
//                      sequence (TB) or per token (TBA'); masked rows zero-filled without a read.
// No float atomics: every output is bitwise reproducible run to run.
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "../../include/tba.h"

namespace {

constexpr float kL2E = 1.4426950408889634f;  // fp32(log2 e)
constexpr double kLN2 = 0.69314718055994530942;
constexpr float kSlack = 6.0f;  // nats a chunk max may exceed the running reference before a re-base
constexpr int kFusedU = 4;

// Row scaling: rows are soft-maxed as 2^(z * sc) with sc = fl(kL2E * inv_temp); slack is kSlack in
// logit units (kSlack / inv_temp); inv_temp enters the log-prob and the gradient exactly (fp64).
struct RowScale {
  float sc, slack;
  double inv_temp;
};

// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// 128-bit load with an explicit L2 eviction policy (createpolicy): evict_last to keep a row
// resident for a second pass, evict_first for its last read.
__device__ __forceinline__ uint4 ldg_pol(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint64_t make_policy(bool last) {
  uint64_t p;
  if (last)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void stg_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ uint16_t to_bf16(float x) {
  uint16_t r;
  asm("{ .reg .b32 t; cvt.rn.bf16x2.f32 t, %1, %1; mov.b32 {%0, _}, t; }" : "=h"(r) : "f"(x));
  return r;
}

// packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2)
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// 2^x for a pair of fp32 on the FMA pipe (offloads MUFU.EX2, which the forward saturates first):
// Cody-Waite split x = n + f, |f| <= 1/2, by the 1.5*2^23 rounding trick; degree-5 minimax
// polynomial for 2^f (max relative error 2.3e-7 with fp32 Horner, the order of ex2.approx);
// 2^n added to the exponent field. Inputs clamped at -125 (ex2.approx.ftz flushes there too).
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x) {
  float a, b;
  f2_unpack(x, a, b);
  const uint64_t xc = f2_pack(fmaxf(a, -125.f), fmaxf(b, -125.f));
  const uint64_t t = fadd2(xc, f2_pack(12582912.f, 12582912.f));    // n + 1.5*2^23 (round to nearest)
  const uint64_t n = fadd2(t, f2_pack(-12582912.f, -12582912.f));   // n exactly
  const uint64_t f = ffma2(n, f2_pack(-1.f, -1.f), xc);             // x - n, exact
  uint64_t p = ffma2(f2_pack(1.3276358367875218e-3f, 1.3276358367875218e-3f), f,
                     f2_pack(9.67550277709961e-3f, 9.67550277709961e-3f));
  p = ffma2(p, f, f2_pack(5.550713092088699e-2f, 5.550713092088699e-2f));
  p = ffma2(p, f, f2_pack(0.24022120237350464f, 0.24022120237350464f));
  p = ffma2(p, f, f2_pack(0.6931469440460205f, 0.6931469440460205f));
  p = ffma2(p, f, f2_pack(1.0000001192092896f, 1.0000001192092896f));
  uint32_t plo, phi, tlo, thi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(plo), "=r"(phi) : "l"(p));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(tlo), "=r"(thi) : "l"(t));
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(plo + (tlo << 23)), "r"(phi + (thi << 23)));
  return r;
}

// element traits: 16-byte vector of VEC elements
template <class T> struct Elem;
template <> struct Elem<uint16_t> {  // bf16 stored as raw bits
  static constexpr int VEC = 8;
  __device__ __forceinline__ static float get(const uint4& v, int e) {
    const uint32_t w = (&v.x)[e >> 1];
    return __uint_as_float((e & 1) ? (w & 0xFFFF0000u) : (w << 16));
  }
  __device__ __forceinline__ static float load1(const uint16_t* p) { return __uint_as_float(((uint32_t)__ldg(p)) << 16); }
};
template <> struct Elem<float> {
  static constexpr int VEC = 4;
  __device__ __forceinline__ static float get(const uint4& v, int e) { return __uint_as_float((&v.x)[e]); }
  __device__ __forceinline__ static float load1(const float* p) { return __ldg(p); }
};

// row split: [0, head) scalar, [head, head + nvec*VEC) 16-byte vectors, rest scalar tail
template <class T>
__device__ __forceinline__ int64_t head_elems(const T* row, int64_t V) {
  const uint64_t a = reinterpret_cast<uint64_t>(row);
  int64_t h = (int64_t)(((16u - (a & 15u)) & 15u) / sizeof(T));
  return h < V ? h : V;
}

// ------------------------------------------------------------------------------ fwd state
// Per-thread online state over a part of one row:
//   m  = max of the elements seen (exact); R = the reference of the partial sum, R2 = fl(R * sc);
//   s  = sum of 2^(fl(z * sc - R2)) over the elements seen (fp64, folded every chunk).
// The reference is re-based only when a chunk max exceeds it by more than `slack` (kSlack nats),
// so the fp64 rescale (exact exp2 of an fp32 difference) is rare and ex2 arguments stay <= 8.7.
struct OnlineState {
  float m, R, R2, sc, slack;
  double s;
  __device__ __forceinline__ void init(const RowScale& rs) {
    m = -INFINITY;
    R = -INFINITY;
    R2 = 0.f;
    sc = rs.sc;
    slack = rs.slack;
    s = 0.0;
  }
  __device__ __forceinline__ void chunk(float cm) {
    m = fmaxf(m, cm);
    if (cm > R + slack) {  // also taken for the first finite chunk (R = -inf)
      const float R2n = cm * sc;
      if (R == -INFINITY) {
        s = 0.0;
      } else {
        s *= exp2((double)R2 - (double)R2n);
      }
      R = cm;
      R2 = R2n;
    }
  }
  __device__ __forceinline__ void add1(float z) {
    chunk(z);
    s += (double)ex2(fmaf(z, sc, -R2));
  }
};

// Combine (m, R2, s) partial states held by the lanes of a warp (`active` lanes only). Result
// (row max M, M2 = fl(M*sc), S = sum relative to M2) in every lane; fixed fp64 butterfly.
__device__ __forceinline__ void combine_lanes(float m, float R2, double s, bool active, float sc, float& M, float& M2,
                                              double& S) {
  float mm = active ? m : -INFINITY;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o));
  M = mm;
  M2 = (mm == -INFINITY) ? 0.f : mm * sc;
  double v = (active && s != 0.0) ? s * exp2((double)R2 - (double)M2) : (active ? s : 0.0);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  S = v;
}

__device__ __forceinline__ void finalize_row(float M, float M2, double S, float zy, bool tok_ok, int64_t row,
                                             const RowScale& rs, float2* __restrict__ stats,
                                             double* __restrict__ lp, int32_t* dev_status) {
  const bool finite = (M > -INFINITY) && (M < INFINITY) && (S > 0.0) && (S < INFINITY);
  const double log2s = log2(S);
  stats[row] = make_float2(M2, (float)log2s);
  // lp = a (z_y - M) - ln sum_v e^{kappa a (z_v - M)},  a = inv_temp, kappa a = sc / log2(e)  (§5.1)
  double v = rs.inv_temp * ((double)zy - (double)M) - kLN2 * (log2s + (double)M2 - (double)M * (double)rs.sc);
  if (!tok_ok) v = nan("");
  lp[row] = v;
  if (dev_status) {
    int f = (tok_ok ? 0 : TBA_DEV_TOKEN_RANGE) | (finite ? 0 : TBA_DEV_NONFINITE_ROW);
    if (f) atomicOr(dev_status, f);
  }
}

// Consume U 16-byte vectors of one row: chunk max, rare re-base, sum of 2^x (FFMA2 + MUFU + FADD2),
// fp32 pair accumulators (<= 4U terms each) folded into the fp64 partial once per call.
// NP of the VEC/2 element pairs of every vector take the FMA-pipe exp2 instead of MUFU.
template <class T, int U, int NP = 0>
__device__ __forceinline__ void fwd_consume(const uint4 (&v)[U], OnlineState& st) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  float z[U][VEC];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int e = 0; e < VEC; ++e) z[u][e] = E::get(v[u], e);
  float cm = -INFINITY;
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int e = 0; e < VEC; e += 2) cm = fmaxf(cm, fmaxf(z[u][e], z[u][e + 1]));
  st.chunk(cm);
  const uint64_t l2e = f2_pack(st.sc, st.sc), nr2 = f2_pack(-st.R2, -st.R2);
  uint64_t acc[VEC / 2];
#pragma unroll
  for (int p = 0; p < VEC / 2; ++p) acc[p] = 0ull;
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int p = 0; p < VEC / 2; ++p) {
      const uint64_t x = ffma2(f2_pack(z[u][2 * p], z[u][2 * p + 1]), l2e, nr2);
      const bool poly = (NP >= 1 && p == VEC / 2 - 1) || (NP >= 2 && p == VEC / 2 - 3);
      if (poly) {
        acc[p] = fadd2(acc[p], exp2_poly2(x));
      } else {
        float a, b;
        f2_unpack(x, a, b);
        acc[p] = fadd2(acc[p], f2_pack(ex2(a), ex2(b)));
      }
    }
#pragma unroll
  for (int w = VEC / 4; w >= 1; w >>= 1)
#pragma unroll
    for (int p = 0; p < w; ++p) acc[p] = fadd2(acc[p], acc[p + w]);
  float a, b;
  f2_unpack(acc[0], a, b);
  st.s += (double)(a + b);
}

// LDG-streamed partial state of one row over threads tid, tid+nthr, ...
template <class T, int U, bool POL = false, int NP = 0>
__device__ __forceinline__ void fwd_accumulate(const T* __restrict__ row, int64_t V, int tid, int nthr,
                                               OnlineState& st, uint64_t pol = 0) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  const int64_t h = head_elems(row, V);
  const int64_t nvec = (V - h) / VEC;
  const int64_t tail0 = h + nvec * VEC;
  if (tid < h) st.add1(E::load1(row + tid));
  for (int64_t i = tail0 + tid; i < V; i += nthr) st.add1(E::load1(row + i));
  const uint4* vp = reinterpret_cast<const uint4*>(row + h);
  const int64_t step = (int64_t)nthr * U;
  const int64_t nfull = nvec / step;
  int64_t k0 = tid;
  for (int64_t it = 0; it < nfull; ++it, k0 += step) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      v[u] = POL ? ldg_pol(vp + k0 + (int64_t)u * nthr, pol) : ldg_stream(vp + k0 + (int64_t)u * nthr);
    fwd_consume<T, U, NP>(v, st);
  }
  for (int64_t k = k0; k < nvec; k += nthr) {
    uint4 v1[1] = {POL ? ldg_pol(vp + k, pol) : ldg_stream(vp + k)};
    fwd_consume<T, 1>(v1, st);
  }
}

// TPR threads per row, 256/TPR rows per CTA (TPR = 32 ... 256). Each row group meets on its own
// named barrier (ids 1..8); a masked row's group exits as a whole.
// The row work of one TPR-thread row group (called with a valid row only).
template <class T, int TPR, int U, int NP, bool FENCE = false>
__device__ __forceinline__ void fwd_row_group(const T* __restrict__ logits, int64_t row, int64_t V, int64_t stride,
                                              const int64_t* __restrict__ tokens, const RowScale& rs,
                                              float2* __restrict__ stats, double* __restrict__ lp,
                                              int32_t* dev_status, float (*sm_m)[TPR / 32 > 0 ? TPR / 32 : 1],
                                              float (*sm_M2)[TPR / 32 > 0 ? TPR / 32 : 1],
                                              double (*sm_s)[TPR / 32 > 0 ? TPR / 32 : 1], int grp, int gt) {
  constexpr int WPR = TPR / 32;
  const int lane = threadIdx.x & 31, wig = gt >> 5;
  const T* rp = logits + row * stride;
  float zy = 0.f;
  bool ok = true;
  if (gt == 0) {
    const int64_t y = tokens[row];
    ok = (y >= 0 && y < V);
    if (ok) zy = Elem<T>::load1(rp + y);
  }
  OnlineState st;
  st.init(rs);
  fwd_accumulate<T, U, false, NP>(rp, V, gt, TPR, st);
  float M, M2;
  double S;
  combine_lanes(st.m, st.R2, st.s, true, rs.sc, M, M2, S);
  if (WPR == 1) {
    if (lane == 0) {
      finalize_row(M, M2, S, zy, ok, row, rs, stats, lp, dev_status);
      if (FENCE) __threadfence();  // publish lp / stats before the unit counters move
    }
    return;
  }
  if (lane == 0) {
    sm_m[grp][wig] = M;
    sm_M2[grp][wig] = M2;
    sm_s[grp][wig] = S;
  }
  asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(TPR) : "memory");
  if (wig == 0) {
    const bool act = lane < WPR;
    combine_lanes(act ? sm_m[grp][lane] : -INFINITY, act ? sm_M2[grp][lane] : 0.f, act ? sm_s[grp][lane] : 0.0, act,
                  rs.sc, M, M2, S);
    if (lane == 0) {
      finalize_row(M, M2, S, zy, ok, row, rs, stats, lp, dev_status);
      if (FENCE) __threadfence();
    }
  }
}

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
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

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

// ------------------------------------------------------------------------------ a2 + a3
// Per-sequence sums: warp w of a CTA takes sequences w, w+8, ... of the CTA's `per` sequences,
// lane-strided fp64 partial sums over t in a fixed order, then a fixed xor butterfly.
__device__ __forceinline__ void seq_sums(const double* __restrict__ lp, const uint8_t* __restrict__ mask,
                                         int64_t n_seq, int64_t T, int64_t s0, int per,
                                         double* __restrict__ seq_logp, int32_t* __restrict__ n_tokens,
                                         int* my_count) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tot = 0;
  for (int j = warp; j < per; j += 8) {
    const int64_t s = s0 + j;
    if (s >= n_seq) break;
    double acc = 0.0;
    int cnt = 0;
    for (int64_t t = lane; t < T; t += 32) {
      const int64_t r = s * T + t;
      if (mask[r]) {
        acc += __ldcg(lp + r);  // L2-coherent: lp may have been written by other CTAs of this grid
        ++cnt;
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if (lane == 0) {
      seq_logp[s] = acc;
      n_tokens[s] = cnt;
    }
    tot += cnt;
  }
  if (my_count) *my_count = tot;
}

// One-shot all-reduce of the 3 loss partials fused into the head kernel, over peer memory
// (NVLink P2P stores / loads through CUDA IPC mappings): the last CTA of every rank
// writes its partial into slot [rank] of every peer's buffer, releases a per-peer flag with the
// call's epoch, waits (acquire, bounded by a timeout) for all ranks' flags, and sums the slots in
// rank order — every rank computes bit-identical totals, with no NCCL launch. Slots are double-
// buffered by epoch parity (a rank cannot get two epochs ahead of a peer that has not read).
struct PeerArgs {
  double* const* slots;         // [world] device pointers: rank q's buffer of 2 x world x 4 doubles
  unsigned int* const* flags;   // [world] device pointers: rank q's [world] epoch flags
  int rank, world;
  unsigned int epoch;
  unsigned long long timeout_ns;
  int32_t* dev_status;
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ void peer_allreduce3(const PeerArgs& pa, const double (&p)[3], double* partial) {
  const int par = (int)(pa.epoch & 1u);
  for (int q = 0; q < pa.world; ++q) {
    double* dst = pa.slots[q] + ((size_t)par * pa.world + pa.rank) * 4;
    dst[0] = p[0];
    dst[1] = p[1];
    dst[2] = p[2];
  }
  __threadfence_system();
  for (int q = 0; q < pa.world; ++q)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pa.flags[q] + pa.rank), "r"(pa.epoch) : "memory");
  const unsigned int* mine = pa.flags[pa.rank];
  const unsigned long long t0 = globaltimer_ns();
  bool timeout = false;
  for (int q = 0; q < pa.world && !timeout; ++q) {
    for (;;) {
      unsigned int v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + q) : "memory");
      if ((int)(v - pa.epoch) >= 0) break;
      if (globaltimer_ns() - t0 > pa.timeout_ns) {
        timeout = true;
        break;
      }
      __nanosleep(256);
    }
  }
  if (timeout) {
    if (pa.dev_status) atomicOr(pa.dev_status, TBA_DEV_PEER_TIMEOUT);
    partial[0] = partial[1] = partial[2] = nan("");
    return;
  }
  const volatile double* my = pa.slots[pa.rank] + (size_t)par * pa.world * 4;
  double t[3] = {0.0, 0.0, 0.0};
  for (int q = 0; q < pa.world; ++q)
    for (int k = 0; k < 3; ++k) t[k] += my[q * 4 + k];
  partial[0] = t[0];
  partial[1] = t[1];
  partial[2] = t[2];
}

// Eq. 4 (or the learned log Z of Eq. 3) and the Eq. 5 residuals of group g, by one thread.
__device__ __forceinline__ void tb_group_head(int64_t g, int K, const double* __restrict__ ref_logp,
                                              const double* __restrict__ log_reward,
                                              const double* __restrict__ log_z_param, double inv_beta,
                                              const double* seq_logp, double* __restrict__ log_z,
                                              double* __restrict__ resid, double* __restrict__ group_sq) {
  const int64_t s0 = g * K;
  double lz;
  if (log_z_param) {
    lz = log_z_param[g];
  } else {
    double sum = 0.0;
    for (int j = 0; j < K; ++j) sum += ref_logp[s0 + j] - __ldcg(seq_logp + s0 + j) + log_reward[s0 + j] * inv_beta;
    lz = sum / (double)K;
  }
  double sq = 0.0;
  for (int j = 0; j < K; ++j) {
    const double delta = ref_logp[s0 + j] - __ldcg(seq_logp + s0 + j) + log_reward[s0 + j] * inv_beta;
    const double e = lz - delta;
    resid[s0 + j] = e;
    sq += e * e;
  }
  log_z[g] = lz;
  group_sq[g] = sq;
}

// Final fixed-order reduction of the per-group sums of squares (+ optional fused all-reduce).
__device__ __forceinline__ void tb_finish(const double* group_sq, int64_t groups, int64_t n_seq, double inv_n_global,
                                          double* partial, const PeerArgs& pa) {
  double tot = 0.0;
  for (int64_t i = 0; i < groups; ++i) tot += __ldcg(group_sq + i);
  const double p[3] = {tot * inv_n_global, (double)n_seq, (double)groups};
  if (pa.world > 0) {
    peer_allreduce3(pa, p, partial);
  } else {
    partial[0] = p[0];
    partial[1] = p[1];
    partial[2] = p[2];
  }
}

// One CTA per group of K sequences (HEAD), or per 8 sequences (log-probs only).
// Eq. 4: log Z_i = 1/K sum_j delta_j (delta = rho - ell + r/beta), or the learned log Z_i of
// Eq. 3 when log_z_param != NULL; Eq. 5 residual eps = log Z_i - delta. The last CTA (counter)
// reduces the per-group sums of squares in group order.
template <bool HEAD>
__global__ void __launch_bounds__(256) seq_head(const double* __restrict__ lp, const uint8_t* __restrict__ mask,
                                                int64_t n_seq, int64_t T, int K, const double* __restrict__ ref_logp,
                                                const double* __restrict__ log_reward,
                                                const double* __restrict__ log_z_param, double inv_beta,
                                                double inv_n_global, double* __restrict__ seq_logp,
                                                int32_t* __restrict__ n_tokens, double* __restrict__ log_z,
                                                double* __restrict__ resid, double* __restrict__ group_sq,
                                                double* __restrict__ partial, unsigned int* counter,
                                                PeerArgs pa = PeerArgs{nullptr, nullptr, 0, 0, 0u, 0ull, nullptr}) {
  const int per = HEAD ? K : 8;
  const int64_t s0 = (int64_t)blockIdx.x * per;
  seq_sums(lp, mask, n_seq, T, s0, per, seq_logp, n_tokens, nullptr);
  if (!HEAD) return;
  __syncthreads();
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    tb_group_head((int64_t)blockIdx.x, K, ref_logp, log_reward, log_z_param, inv_beta, seq_logp, log_z, resid,
                  group_sq);
    __threadfence();
    am_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (am_last && threadIdx.x == 0) {
    __threadfence();
    *counter = 0u;
    tb_finish(group_sq, (int64_t)gridDim.x, n_seq, inv_n_global, partial, pa);
  }
}

// Forward rows + per-sequence sums (+ group head) in ONE kernel: every CTA, after its rows, adds
// its row counts to per-unit counters (unit = one sequence for log-probs, one group of K
// sequences for the TB head); the CTA that completes a unit computes that unit's sums (and
// head), and the CTA completing the last group reduces the loss partials. Saves the separate
// seq_head launch and its latency.
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
  unsigned int* units_done;   // [n_units]
  unsigned int* groups_done;  // [1]
  PeerArgs pa;
};

template <class T, int TPR, int U, int NP>
__global__ void __launch_bounds__(256) row_fwd_head(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                     int64_t stride, const int64_t* __restrict__ tokens,
                                                     const uint8_t* __restrict__ mask, RowScale rs,
                                                     float2* __restrict__ stats, double* __restrict__ lp,
                                                     int32_t* dev_status, HeadArgs ha) {
  constexpr int RPC = 256 / TPR, WPRS = TPR / 32 > 0 ? TPR / 32 : 1;
  __shared__ float sm_m[RPC][WPRS], sm_M2[RPC][WPRS];
  __shared__ double sm_s[RPC][WPRS];
  __shared__ int64_t sh_done[RPC + 1];
  __shared__ int sh_ndone;
  const int grp = threadIdx.x / TPR, gt = threadIdx.x % TPR;
  const int64_t row0 = (int64_t)blockIdx.x * RPC;
  const int64_t row = row0 + grp;
  if (row < rows && mask[row] != 0) {
    fwd_row_group<T, TPR, U, NP, true>(logits, row, V, stride, tokens, rs, stats, lp, dev_status, sm_m, sm_M2, sm_s,
                                       grp, gt);
  }
  __syncthreads();
  const int64_t unit_rows = (int64_t)ha.K * ha.T;
  if (threadIdx.x == 0) {
    int nd = 0;
    const int64_t r1 = row0 + RPC < rows ? row0 + RPC : rows;
    for (int64_t r = row0; r < r1;) {
      const int64_t u = r / unit_rows;
      const int64_t ue = (u + 1) * unit_rows < r1 ? (u + 1) * unit_rows : r1;
      const unsigned cnt = (unsigned)(ue - r);
      if (atomicAdd(&ha.units_done[u], cnt) + cnt == (unsigned)unit_rows) sh_done[nd++] = u;
      r = ue;
    }
    sh_ndone = nd;
    if (nd) __threadfence();
  }
  __syncthreads();
  for (int i = 0; i < sh_ndone; ++i) {
    const int64_t u = sh_done[i];
    seq_sums(lp, mask, ha.n_seq, ha.T, u * ha.K, ha.K, ha.seq_logp, ha.n_tokens, nullptr);
    if (!ha.head) continue;
    __syncthreads();
    if (threadIdx.x == 0) {
      tb_group_head(u, ha.K, ha.ref_logp, ha.log_reward, ha.log_z_param, ha.inv_beta, ha.seq_logp, ha.log_z,
                    ha.resid, ha.group_sq);
      __threadfence();
      const int64_t groups = ha.n_seq / ha.K;
      if (atomicAdd(ha.groups_done, 1u) + 1u == (unsigned)groups) {
        __threadfence();
        tb_finish(ha.group_sq, groups, ha.n_seq, ha.inv_n_global, ha.partial, ha.pa);
      }
    }
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

// ------------------------------------------------------------------------------ a5
template <class TO> struct Out;
template <> struct Out<uint16_t> {
  __device__ __forceinline__ static void put1(uint16_t* p, float x) { *p = to_bf16(x); }
};
template <> struct Out<float> {
  __device__ __forceinline__ static void put1(float* p, float x) { __stcs(p, x); }
};

// store N computed values starting at o (16-byte aligned)
template <class TO, int N>
__device__ __forceinline__ void store_vals(TO* o, const float (&d)[N]) {
  if constexpr (sizeof(TO) == 2) {
    static_assert(N == 8 || N == 4, "");
    if constexpr (N == 8) {
      uint4 w = make_uint4(pack_bf16x2(d[0], d[1]), pack_bf16x2(d[2], d[3]), pack_bf16x2(d[4], d[5]),
                           pack_bf16x2(d[6], d[7]));
      stg_stream(reinterpret_cast<uint4*>(o), w);
    } else {
      uint2 w = make_uint2(pack_bf16x2(d[0], d[1]), pack_bf16x2(d[2], d[3]));
      asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(o), "r"(w.x), "r"(w.y) : "memory");
    }
  } else {
#pragma unroll
    for (int q = 0; q < N / 4; ++q)
      stg_stream(reinterpret_cast<uint4*>(o) + q,
                 make_uint4(__float_as_uint(d[4 * q]), __float_as_uint(d[4 * q + 1]), __float_as_uint(d[4 * q + 2]),
                            __float_as_uint(d[4 * q + 3])));
  }
}

template <class T, class TO, int U, bool POL = false>
__device__ __forceinline__ void bwd_row(const T* __restrict__ rp, TO* __restrict__ op, int64_t V, int tid, int nthr,
                                        bool valid, float sc, float M2, float L2S, float c, int64_t y,
                                        uint64_t pol = 0) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  const int64_t h = head_elems(rp, V);
  // the vector path needs the output 16-byte aligned at the same element as the input
  const bool vec_ok = ((reinterpret_cast<uint64_t>(op + h) & 15u) == 0);
  const int64_t nvec = vec_ok ? (V - h) / VEC : 0;
  const int64_t vend = h + nvec * VEC;
  auto one = [&](int64_t i) {
    float d = 0.f;
    if (valid) {
      const float p = ex2(fmaf(E::load1(rp + i), sc, -M2) - L2S);
      d = (i == y) ? fmaf(-c, p, c) : -c * p;
    }
    Out<TO>::put1(op + i, d);
  };
  for (int64_t i = tid; i < (vec_ok ? h : V); i += nthr) one(i);
  if (!vec_ok) return;
  for (int64_t i = vend + tid; i < V; i += nthr) one(i);
  const uint4* vp = reinterpret_cast<const uint4*>(rp + h);
  TO* ob = op + h;
  if (!valid) {
    float z[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) z[e] = 0.f;
    for (int64_t k = tid; k < nvec; k += nthr) store_vals<TO, VEC>(ob + k * VEC, z);
    return;
  }
  const float nM2 = -M2;
  const int64_t ky = (y >= h && y < vend) ? (y - h) / VEC : -1;
  for (int64_t k0 = tid; k0 < nvec; k0 += (int64_t)nthr * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + (int64_t)u * nthr;
      if (k < nvec) v[u] = POL ? ldg_pol(vp + k, pol) : ldg_stream(vp + k);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + (int64_t)u * nthr;
      if (k < nvec) {
        float d[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) d[e] = -c * ex2(fmaf(E::get(v[u], e), sc, nM2) - L2S);
        if (k == ky) {
          const int e = (int)((y - h) - k * VEC);
#pragma unroll
          for (int q = 0; q < VEC; ++q)
            if (q == e) d[q] += c;
        }
        store_vals<TO, VEC>(ob + k * VEC, d);
      }
    }
  }
}

// TPR threads per row, 256/TPR rows per CTA. Row coefficient c = grad_scale * g * inv_temp *
// (resid[s] for the TB losses, per sequence | coef[row] for per-token rules such as TBA').
template <class T, class TO, int TPR, int U, bool PER_ROW>
__global__ void __launch_bounds__(256) row_bwd(const T* __restrict__ logits, int64_t rows, int64_t T_len, int64_t V,
                                               int64_t stride, const int64_t* __restrict__ tokens,
                                               const uint8_t* __restrict__ mask, const float2* __restrict__ stats,
                                               const double* __restrict__ resid, const float* __restrict__ coef,
                                               double grad_scale, const double* __restrict__ grad_out, RowScale rs,
                                               TO* __restrict__ dlogits, int64_t ostride) {
  constexpr int RPC = 256 / TPR;
  const int64_t row = (int64_t)blockIdx.x * RPC + threadIdx.x / TPR;
  if (row >= rows) return;
  const int tid = threadIdx.x % TPR;
  const bool valid = mask[row] != 0;
  float M2 = 0.f, L2S = 0.f, c = 0.f;
  int64_t y = -1;
  if (valid) {
    const float2 st = stats[row];
    M2 = st.x;
    L2S = st.y;
    const double g = (grad_out ? *grad_out : 1.0) * grad_scale * rs.inv_temp;
    c = PER_ROW ? (float)(g * (double)coef[row]) : (float)(g * resid[row / T_len]);
    y = tokens[row];
  }
  bwd_row<T, TO, U>(logits + row * stride, dlogits + row * ostride, V, tid, TPR, valid, rs.sc, M2, L2S, c, y);
}

// ------------------------------------------------------------------------------ a1-a5 fused (NEXT 2)
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

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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
        float zy = 0.f;
        bool ok = true;
        if (gt == 0) {
          const int64_t y = a.tokens[row];
          ok = (y >= 0 && y < a.V);
          if (ok) zy = Elem<T>::load1(rp + y);
        }
        OnlineState st;
        st.init(a.rs);
        fwd_accumulate<T, kFusedU, false, (TPR_F == 64 ? 1 : 0)>(rp, a.V, gt, TPR_F, st);  // as the two-call path
        float M, M2;
        double S;
        combine_lanes(st.m, st.R2, st.s, true, a.rs.sc, M, M2, S);
        if (WPR == 1) {
          if (lane == 0) finalize_row(M, M2, S, zy, ok, row, a.rs, a.stats, a.lp, a.dev_status);
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
            if (lane == 0) finalize_row(M, M2, S, zy, ok, row, a.rs, a.stats, a.lp, a.dev_status);
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
        if (threadIdx.x == 0) {
          double lz;
          if (a.log_z_param) {
            lz = a.log_z_param[g];
          } else {
            double sum = 0.0;
            for (int q = 0; q < a.K; ++q)
              sum += a.ref_logp[s0 + q] - __ldcg(a.seq_logp + s0 + q) + a.log_reward[s0 + q] * a.inv_beta;
            lz = sum / (double)a.K;
          }
          double sq = 0.0;
          for (int q = 0; q < a.K; ++q) {
            const double delta = a.ref_logp[s0 + q] - __ldcg(a.seq_logp + s0 + q) + a.log_reward[s0 + q] * a.inv_beta;
            const double e = lz - delta;
            a.resid[s0 + q] = e;
            sq += e * e;
          }
          a.log_z[g] = lz;
          a.group_sq[g] = sq;
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
        float M2 = 0.f, L2S = 0.f, c = 0.f;
        int64_t y = -1;
        if (valid) {
          const float2 stt = __ldcg(a.stats + row);
          M2 = stt.x;
          L2S = stt.y;
          c = (float)(a.grad_scale * a.rs.inv_temp * __ldcg(a.resid + row / a.T));
          y = a.tokens[row];
        }
        bwd_row<T, TO, 4>(logits + row * a.stride, dlogits + row * a.ostride, a.V, tid, TPR_B, valid, a.rs.sc, M2,
                          L2S, c, y);
      }
    }
  }
}

// ------------------------------------------------------------------------------ deferred scale (NEXT 2 (ii))
// A cluster of CS CTAs (NT threads each) per valid row: pass 1 streams the row from HBM with an
// L2 evict_last policy (online max/sum); the CTAs of the cluster exchange their (max, sum)
// partials through distributed shared memory; pass 2 re-reads the row — an L2 hit, because the
// grid keeps only ~40-60 MB of rows in flight (CS and NT are chosen per row size) — and writes
// the UNSCALED gradient G = inv_temp (1[v=y] - softmax) once. HBM bytes: 2V read + 2V write per
// valid row (the 4V floor); the per-sequence factor grad_scale * g * eps_s is applied by the
// consumer (the LM-head backward, as a row scale), SURVEY §8(f) NEXT 2.
template <class T, class TO, int NT, int CS, int U2 = 4>
__device__ __forceinline__ void row_single_body(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                int64_t stride, const int64_t* __restrict__ tokens,
                                                const uint8_t* __restrict__ mask, RowScale rs,
                                                float2* __restrict__ stats, double* __restrict__ lp,
                                                int32_t* dev_status, TO* __restrict__ g_out, int64_t ostride) {
  namespace cg = cooperative_groups;
  constexpr int NW = NT / 32;
  const int rank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int64_t row = (int64_t)blockIdx.x / CS;
  const int gt = rank * NT + (int)threadIdx.x;  // thread index within the row's cluster
  __shared__ float sm_m[NW], sm_M2[NW];
  __shared__ double sm_s[NW];
  __shared__ float part_m, part_M2;  // this CTA's partial, read by the cluster through DSMEM
  __shared__ double part_s;
  __shared__ float sh_M2, sh_L2S;
  __shared__ int64_t sh_y;
  const bool live = row < rows;
  const bool valid = live && mask[row] != 0;  // uniform over the cluster
  const T* rp = logits + (live ? row : 0) * stride;
  TO* op = g_out + (live ? row : 0) * ostride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float M = -INFINITY, M2 = 0.f;
  double S = 0.0;
  if (valid) {
    if (threadIdx.x == 0) sh_y = tokens[row];
    OnlineState st;
    st.init(rs);
    fwd_accumulate<T, 4, true>(rp, V, gt, CS * NT, st, make_policy(true));
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
    bwd_row<T, TO, 4>(rp, op, V, gt, CS * NT, false, 0.f, 0.f, 0.f, 0.f, -1);
    if constexpr (CS > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    return;
  }
  if (threadIdx.x == 0) {
    const int64_t y = sh_y;
    const bool ok = (y >= 0 && y < V);
    if (rank == 0) {
      const float zy = ok ? Elem<T>::load1(rp + y) : 0.f;
      finalize_row(M, M2, S, zy, ok, row, rs, stats, lp, dev_status);
    }
    sh_M2 = M2;
    sh_L2S = (float)log2(S);
  }
  __syncthreads();
  bwd_row<T, TO, U2, true>(rp, op, V, gt, CS * NT, true, rs.sc, sh_M2, sh_L2S, (float)rs.inv_temp, sh_y,
                           make_policy(false));
  if constexpr (CS > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

template <class T, class TO, int NT, int U2 = 4>
__global__ void __launch_bounds__(NT) row_single1(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                  int64_t stride, const int64_t* __restrict__ tokens,
                                                  const uint8_t* __restrict__ mask, RowScale rs,
                                                  float2* __restrict__ stats, double* __restrict__ lp,
                                                  int32_t* dev_status, TO* __restrict__ g_out, int64_t ostride) {
  row_single_body<T, TO, NT, 1, U2>(logits, rows, V, stride, tokens, mask, rs, stats, lp, dev_status, g_out, ostride);
}

template <class T, class TO, int NT, int U2 = 4>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT)
    row_single2(const T* __restrict__ logits, int64_t rows, int64_t V, int64_t stride,
                const int64_t* __restrict__ tokens, const uint8_t* __restrict__ mask, RowScale rs,
                float2* __restrict__ stats, double* __restrict__ lp, int32_t* dev_status, TO* __restrict__ g_out,
                int64_t ostride) {
  row_single_body<T, TO, NT, 2, U2>(logits, rows, V, stride, tokens, mask, rs, stats, lp, dev_status, g_out, ostride);
}

template <class T, class TO, int NT, int U2 = 4>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(NT)
    row_single4(const T* __restrict__ logits, int64_t rows, int64_t V, int64_t stride,
                const int64_t* __restrict__ tokens, const uint8_t* __restrict__ mask, RowScale rs,
                float2* __restrict__ stats, double* __restrict__ lp, int32_t* dev_status, TO* __restrict__ g_out,
                int64_t ostride) {
  row_single_body<T, TO, NT, 4, U2>(logits, rows, V, stride, tokens, mask, rs, stats, lp, dev_status, g_out, ostride);
}

// Pipelined deferred pass (cfg 7): persistent 2-CTA clusters (one CTA of 1024 threads per SM),
// each CTA split into two teams of 16 warps. In round j, team A streams HALF of row j from HBM
// (pass 1) while team B re-reads half of row j-1 from L2 and writes its gradient (pass 2); the two
// CTAs of the cluster then exchange their row-j partials through DSMEM. Every SM thus keeps an HBM
// read stream and a write stream busy at all times, while only ~148 rows (45 MB at V = 152064)
// are in flight, so the re-reads stay in L2.
template <class T, class TO>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024, 1)
    row_single_pipe(const T* __restrict__ logits, int64_t rows, int64_t V, int64_t stride,
                    const int64_t* __restrict__ tokens, const uint8_t* __restrict__ mask, RowScale rs,
                    float2* __restrict__ stats, double* __restrict__ lp, int32_t* dev_status, TO* __restrict__ g_out,
                    int64_t ostride, int64_t n_clusters) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  constexpr int NTH = 1024;  // threads per row across the cluster (2 CTAs x 512-thread team)
  const int rank = (int)cl.block_rank();
  const int64_t cid = (int64_t)blockIdx.x / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool teamA = warp < 16;
  const int gt = rank * 512 + (threadIdx.x & 511);
  __shared__ float wm[16], wm2[16];
  __shared__ double wsum[16];
  __shared__ float part_m[2], part_M2[2];
  __shared__ double part_s[2];
  __shared__ float st_M2[2], st_L2S[2];
  __shared__ int64_t st_y[2], st_row[2];
  __shared__ int st_valid[2];
  const int64_t nrc = cid < rows ? (rows - cid + n_clusters - 1) / n_clusters : 0;
  const uint64_t pol_last = make_policy(true), pol_first = make_policy(false);
  for (int64_t j = 0; j <= nrc; ++j) {
    const int b = (int)(j & 1);
    if (teamA) {
      if (j < nrc) {
        const int64_t row = cid + j * n_clusters;
        if (mask[row]) {
          OnlineState st;
          st.init(rs);
          fwd_accumulate<T, 4, true>(logits + row * stride, V, gt, NTH, st, pol_last);
          float M, M2;
          double S;
          combine_lanes(st.m, st.R2, st.s, true, rs.sc, M, M2, S);
          if (lane == 0) {
            wm[warp] = M;
            wm2[warp] = M2;
            wsum[warp] = S;
          }
          asm volatile("bar.sync 1, 512;" ::: "memory");
          if (warp == 0) {
            const bool act = lane < 16;
            combine_lanes(act ? wm[lane] : -INFINITY, act ? wm2[lane] : 0.f, act ? wsum[lane] : 0.0, act, rs.sc, M,
                          M2, S);
            if (lane == 0) {
              part_m[b] = M;
              part_M2[b] = M2;
              part_s[b] = S;
            }
          }
        }
      }
    } else if (j >= 1) {
      const int pb = b ^ 1;
      const int64_t row = st_row[pb];
      const bool valid = st_valid[pb] != 0;
      bwd_row<T, TO, 4, true>(logits + row * stride, g_out + row * ostride, V, gt, NTH, valid, rs.sc, st_M2[pb],
                              st_L2S[pb], (float)rs.inv_temp, st_y[pb], pol_first);
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 0 && j < nrc) {
      const int64_t row = cid + j * n_clusters;
      const bool valid = mask[row] != 0;
      float M = -INFINITY, M2 = 0.f;
      double S = 0.0;
      if (valid) {
        const bool act = lane < 2;
        float pm = -INFINITY, pm2 = 0.f;
        double ps = 0.0;
        if (act) {
          pm = *cl.map_shared_rank(&part_m[b], lane);
          pm2 = *cl.map_shared_rank(&part_M2[b], lane);
          ps = *cl.map_shared_rank(&part_s[b], lane);
        }
        combine_lanes(pm, pm2, ps, act, rs.sc, M, M2, S);
      }
      if (lane == 0) {
        int64_t y = -1;
        if (valid) {
          y = tokens[row];
          const bool ok = (y >= 0 && y < V);
          if (rank == 0) {
            const float zy = ok ? Elem<T>::load1(logits + row * stride + y) : 0.f;
            finalize_row(M, M2, S, zy, ok, row, rs, stats, lp, dev_status);
          }
          st_M2[b] = M2;
          st_L2S[b] = (float)log2(S);
        }
        st_y[b] = y;
        st_row[b] = row;
        st_valid[b] = valid;
      }
    }
    __syncthreads();  // row j's statistics are visible to team B in round j+1
  }
}

// ------------------------------------------------------------------------------ host side
constexpr int kU = 4;
constexpr int64_t kSmallRowBytes = 8192;  // rows up to 8 KB: one warp per row in the backward

RowScale make_scale(double inv_temp) {
  RowScale r;
  r.sc = (float)((double)kL2E * inv_temp);
  r.slack = (float)((double)kSlack / inv_temp);
  r.inv_temp = inv_temp;
  return r;
}

struct WsLayout {
  float2* stats;
  double* lp;
  double* group_sq;
  unsigned int* counter;
  unsigned int* fused;
};

size_t fused_counter_bytes(int64_t n_seq) { return (size_t)(2 + 2 * n_seq) * sizeof(unsigned int); }

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

WsLayout ws_layout(void* ws, int64_t n_seq, int64_t T) {
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
  return l;
}

size_t ws_bytes(int64_t n_seq, int64_t T) {
  const size_t rows = (size_t)n_seq * (size_t)T;
  return align_up(rows * sizeof(float2), 256) + align_up(rows * sizeof(double), 256) +
         align_up((size_t)n_seq * sizeof(double), 256) + 256 + align_up(fused_counter_bytes(n_seq), 256);
}

int validate_rows(const tba_rows* x) {
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

int validate_out(const tba_rows* x, const void* dlogits, int32_t odt, int64_t ostride) {
  if (odt != TBA_BF16 && odt != TBA_FP32) return TBA_ERR_INVALID_ARG;
  if (ostride < x->vocab) return TBA_ERR_INVALID_ARG;
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows == 0) return TBA_OK;
  const int64_t oesz = odt == TBA_BF16 ? 2 : 4;
  if (ostride > INT64_MAX / 8 / oesz / rows) return TBA_ERR_INVALID_ARG;
  if (!dlogits || reinterpret_cast<uintptr_t>(dlogits) % oesz) return TBA_ERR_INVALID_ARG;
  if (dlogits == x->logits && (odt != x->dtype || ostride != x->row_stride))
    return TBA_ERR_INVALID_ARG;  // aliasing is only supported element-for-element
  return TBA_OK;
}

int device_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  static int cache[64] = {0};
  if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cache[dev] = n;
  return n;
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// A/B switches (read once): TBA_FWD_IMPL=tma selects the TMA-ring forward, TBA_TMA_CFG its
// configuration, TBA_FWD_TPR / TBA_BWD_TPR force threads per row. Defaults are the measured best.
struct Switches {
  int fwd_tma, tma_cfg, fwd_tpr, bwd_tpr;
};
const Switches& switches() {
  static Switches s = [] {
    Switches v;
    const char* e = getenv("TBA_FWD_IMPL");
    v.fwd_tma = (e && e[0] == 't') ? 1 : 0;
    v.tma_cfg = env_int("TBA_TMA_CFG", 0);
    v.fwd_tpr = env_int("TBA_FWD_TPR", 0);
    v.bwd_tpr = env_int("TBA_BWD_TPR", 0);
    return v;
  }();
  return s;
}

bool valid_tpr(int t) { return t == 32 || t == 64 || t == 128 || t == 256; }

// Forward threads per row, measured on B200 (scripts/gpu_ab_tpr.sh): 64 threads
// (4 rows per CTA) is best or within 1 % for V = 32000 ... 152064; one warp for short rows.
int fwd_tpr(int64_t V, int64_t esz) {
  if (valid_tpr(switches().fwd_tpr)) return switches().fwd_tpr;
  return (V * esz / 16) < 1024 ? 32 : 64;
}

// Backward threads per row (scripts/gpu_ab_bwd.sh): one CTA per long row, one warp per short row.
int bwd_tpr(int64_t V, int64_t esz) {
  if (valid_tpr(switches().bwd_tpr)) return switches().bwd_tpr;
  return V * esz <= kSmallRowBytes ? 32 : 256;
}

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

template <class T, class TO, bool PER_ROW>
void launch_bwd_t(const tba_rows* x, const WsLayout& w, const double* resid, const float* coef, double gs,
                  const double* go, const RowScale& rs, TO* out, int64_t ostride, cudaStream_t s) {
  const int64_t rows = x->n_seq * x->seq_len;
  const int tpr = bwd_tpr(x->vocab, (int64_t)sizeof(T));
  const int64_t rpc = 256 / tpr;
  const unsigned grid = (unsigned)((rows + rpc - 1) / rpc);
  auto lg = static_cast<const T*>(x->logits);
#define TBA_BWD(TPR_)                                                                                              \
  row_bwd<T, TO, TPR_, kU, PER_ROW><<<grid, 256, 0, s>>>(lg, rows, x->seq_len, x->vocab, x->row_stride, x->tokens, \
                                                        x->mask, w.stats, resid, coef, gs, go, rs, out, ostride)
  switch (tpr) {
    case 32: TBA_BWD(32); break;
    case 64: TBA_BWD(64); break;
    case 128: TBA_BWD(128); break;
    default: TBA_BWD(256); break;
  }
#undef TBA_BWD
}

template <bool PER_ROW>
int launch_bwd(const tba_rows* x, const void* workspace, const double* resid, const float* coef, double gs,
               const double* go, const RowScale& rs, void* dlogits, int32_t odt, int64_t ostride, cudaStream_t s) {
  if (x->n_seq * x->seq_len == 0) return TBA_OK;
  WsLayout w = ws_layout(const_cast<void*>(workspace), x->n_seq, x->seq_len);
  if (x->dtype == TBA_BF16) {
    if (odt == TBA_BF16)
      launch_bwd_t<uint16_t, uint16_t, PER_ROW>(x, w, resid, coef, gs, go, rs, static_cast<uint16_t*>(dlogits),
                                                ostride, s);
    else
      launch_bwd_t<uint16_t, float, PER_ROW>(x, w, resid, coef, gs, go, rs, static_cast<float*>(dlogits), ostride, s);
  } else {
    if (odt == TBA_BF16)
      launch_bwd_t<float, uint16_t, PER_ROW>(x, w, resid, coef, gs, go, rs, static_cast<uint16_t*>(dlogits), ostride,
                                             s);
    else
      launch_bwd_t<float, float, PER_ROW>(x, w, resid, coef, gs, go, rs, static_cast<float*>(dlogits), ostride, s);
  }
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

int fused_lookahead(int64_t group_bytes, int groups) {
  const int env = env_int("TBA_FUSED_D", -1);
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

// deferred-scale row pass (row_single*): configuration by row length, see DESIGN.md §5.4
int launch_single(const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status,
                  void* grad_unscaled, int32_t g_dtype, int64_t g_row_stride, cudaStream_t s) {
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows > 0) {
    // Rows in flight x row bytes must stay inside L2 for pass 2 to hit it. Measured:
    // rows <= 128 KB: 256 threads per row (4 CTAs/SM); longer rows: 512 threads (2 CTAs/SM) with 8
    // vectors per thread in pass 2 — it keeps ~70 % of the re-reads in L2 and overlaps the two passes
    // across the SM's CTAs, which beats the exact-4V 2-CTA cluster variants (cfg 2/3/5/6).
    const int64_t rb = x->vocab * (x->dtype == TBA_BF16 ? 2 : 4);
    int cfg = rb <= 128 * 1024 ? 0 : 4;
    const int ecfg = env_int("TBA_SINGLE_CFG", -1);
    if (ecfg >= 0 && ecfg <= 7) cfg = ecfg;
#define TBA_SINGLE1(KERN_, T_, TO_, NT_, CS_, U2_)                                                             \
  KERN_<T_, TO_, NT_, U2_><<<(unsigned)(rows * CS_), NT_, 0, s>>>(static_cast<const T_*>(x->logits), rows, x->vocab, \
                                                             x->row_stride, x->tokens, x->mask, rs, w.stats,      \
                                                             w.lp, dev_status, static_cast<TO_*>(grad_unscaled),  \
                                                             g_row_stride)
#define TBA_SINGLE(T_, TO_)                                          \
  do {                                                               \
    if (cfg == 0) TBA_SINGLE1(row_single1, T_, TO_, 256, 1, 4);      \
    else if (cfg == 1) TBA_SINGLE1(row_single1, T_, TO_, 512, 1, 4); \
    else if (cfg == 2) TBA_SINGLE1(row_single2, T_, TO_, 512, 2, 4); \
    else if (cfg == 3) TBA_SINGLE1(row_single4, T_, TO_, 512, 4, 4); \
    else if (cfg == 4) TBA_SINGLE1(row_single1, T_, TO_, 512, 1, 8); \
    else if (cfg == 5) TBA_SINGLE1(row_single2, T_, TO_, 512, 2, 8); \
    else if (cfg == 6) TBA_SINGLE1(row_single2, T_, TO_, 256, 2, 4); \
    else {                                                           \
      const int64_t ncl = (int64_t)device_sms() / 2;                 \
      row_single_pipe<T_, TO_><<<(unsigned)(2 * ncl), 1024, 0, s>>>( \
          static_cast<const T_*>(x->logits), rows, x->vocab, x->row_stride, x->tokens, x->mask, rs, w.stats, \
          w.lp, dev_status, static_cast<TO_*>(grad_unscaled), g_row_stride, ncl);                        \
    }                                                                \
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

// Forward rows with the per-unit sums / TB head fused in (row_fwd_head). Returns false when the
// separate kernels must be used instead (no rows, or the TMA forward selected for A/B).
bool launch_fwd_head(const tba_rows* x, const WsLayout& w, const RowScale& rs, int32_t* dev_status, HeadArgs& ha,
                     cudaStream_t s, int* rc) {
  const int64_t rows = x->n_seq * x->seq_len;
  const int64_t esz = x->dtype == TBA_BF16 ? 2 : 4;
  if (rows == 0 || (switches().fwd_tma && x->vocab * esz > kSmallRowBytes)) return false;
  // Off by default: measured on B200 (scripts/gpu_ab_head.sh) the per-row fence + unit counters
  // cost as much as the separate seq_head launch saves (Qwen 9.305 vs 9.283 ms, RhoMath 7.03 vs
  // 6.98; only the launch-bound toy gains, 0.056 vs 0.060). TBA_FUSE_HEAD=1 selects it.
  if (env_int("TBA_FUSE_HEAD", 0) == 0) return false;
  if (cudaMemsetAsync(w.fused, 0, fused_counter_bytes(x->n_seq), s) != cudaSuccess) {
    *rc = TBA_ERR_CUDA;
    return true;
  }
  ha.units_done = w.fused + 2;
  ha.groups_done = w.fused + 1;
  const int tpr = fwd_tpr(x->vocab, esz);
  const int np = env_int("TBA_FWD_NP", 1);
  const unsigned grid = (unsigned)((rows + 256 / tpr - 1) / (256 / tpr));
#define TBA_HEAD(T_, TPR_, NP_)                                                                                    \
  row_fwd_head<T_, TPR_, kU, NP_><<<grid, 256, 0, s>>>(static_cast<const T_*>(x->logits), rows, x->vocab,         \
                                                       x->row_stride, x->tokens, x->mask, rs, w.stats, w.lp,      \
                                                       dev_status, ha)
  if (x->dtype == TBA_BF16) {
    if (tpr == 64 && np == 1) TBA_HEAD(uint16_t, 64, 1);
    else if (tpr == 64) TBA_HEAD(uint16_t, 64, 0);
    else TBA_HEAD(uint16_t, 32, 0);
  } else {
    if (tpr == 64 && np == 1) TBA_HEAD(float, 64, 1);
    else if (tpr == 64) TBA_HEAD(float, 64, 0);
    else TBA_HEAD(float, 32, 0);
  }
#undef TBA_HEAD
  *rc = cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
  return true;
}

int check_opts(const tba_tb_opts* o) {
  if (!o) return TBA_OK;
  if (!(std::isfinite(o->inv_temp) && o->inv_temp > 0.0)) return TBA_ERR_INVALID_CONFIG;
  return TBA_OK;
}

double opt_inv_temp(const tba_tb_opts* o) { return o ? o->inv_temp : 1.0; }

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
  ha.pa = PeerArgs{nullptr, nullptr, 0, 0, 0u, 0ull, dev_status};
  if (launch_fwd_head(x, w, make_scale(1.0), dev_status, ha, s, &rc)) return rc;
  rc = launch_fwd_rows(x, w, make_scale(1.0), dev_status, s);
  if (rc) return rc;
  const int64_t grid = (x->n_seq + 7) / 8;
  seq_head<false><<<(unsigned)grid, 256, 0, s>>>(w.lp, x->mask, x->n_seq, x->seq_len, 8, nullptr, nullptr, nullptr,
                                                 0.0, 0.0, seq_logp, n_tokens, nullptr, nullptr, nullptr, nullptr,
                                                 nullptr);
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
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
  const int64_t blocks = (rows + 255) / 256 < 4096 ? (rows + 255) / 256 : 4096;
  token_lp_kernel<<<(unsigned)blocks, 256, 0, s>>>(w.lp, x->mask, rows, tok_logp);
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

static int tb_loss_fwd_impl(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp,
                            const double* log_reward, double beta, int32_t K, double n_seq_global, void* workspace,
                            double* seq_logp, int32_t* n_tokens, double* log_z, double* resid, double* partial,
                            int32_t* dev_status, const tba_peer_reduce* pr, tba_stream_t stream);

int tba_tb_loss_fwd(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp, const double* log_reward,
                    double beta, int32_t K, double n_seq_global, void* workspace, double* seq_logp, int32_t* n_tokens,
                    double* log_z, double* resid, double* partial, int32_t* dev_status, tba_stream_t stream) {
  return tb_loss_fwd_impl(x, opts, ref_logp, log_reward, beta, K, n_seq_global, workspace, seq_logp, n_tokens, log_z,
                          resid, partial, dev_status, nullptr, stream);
}

int tba_tb_loss_fwd_peer(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp,
                         const double* log_reward, double beta, int32_t K, double n_seq_global, void* workspace,
                         double* seq_logp, int32_t* n_tokens, double* log_z, double* resid, double* partial,
                         const tba_peer_reduce* pr, int32_t* dev_status, tba_stream_t stream) {
  if (!pr || !pr->slots || !pr->flags || pr->world < 1 || pr->rank < 0 || pr->rank >= pr->world || pr->epoch == 0 ||
      !(pr->timeout_s > 0.0))
    return TBA_ERR_INVALID_ARG;
  if (x && x->n_seq == 0) return TBA_ERR_INVALID_ARG;  // every rank must own >= 1 group to join the reduction
  return tb_loss_fwd_impl(x, opts, ref_logp, log_reward, beta, K, n_seq_global, workspace, seq_logp, n_tokens, log_z,
                          resid, partial, dev_status, pr, stream);
}

static int tb_loss_fwd_impl(const tba_rows* x, const tba_tb_opts* opts, const double* ref_logp,
                            const double* log_reward, double beta, int32_t K, double n_seq_global, void* workspace,
                            double* seq_logp, int32_t* n_tokens, double* log_z, double* resid, double* partial,
                            int32_t* dev_status, const tba_peer_reduce* pr, tba_stream_t stream) {
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
  PeerArgs pa{nullptr, nullptr, 0, 0, 0u, 0ull, dev_status};
  if (pr) {
    pa.slots = pr->slots;
    pa.flags = pr->flags;
    pa.rank = pr->rank;
    pa.world = pr->world;
    pa.epoch = pr->epoch;
    pa.timeout_ns = (unsigned long long)(pr->timeout_s * 1e9);
  }
  const RowScale rs = make_scale(opt_inv_temp(opts));
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
  ha.pa = pa;
  if (launch_fwd_head(x, w, rs, dev_status, ha, s, &rc)) return rc;
  if (cudaMemsetAsync(w.counter, 0, sizeof(unsigned int), s) != cudaSuccess) return TBA_ERR_CUDA;
  rc = launch_fwd_rows(x, w, rs, dev_status, s);
  if (rc) return rc;
  const int64_t groups = x->n_seq / K;
  seq_head<true><<<(unsigned)groups, 256, 0, s>>>(w.lp, x->mask, x->n_seq, x->seq_len, K, ref_logp, log_reward,
                                                  opts ? opts->log_z_param : nullptr, 1.0 / beta, 1.0 / n_seq_global,
                                                  seq_logp, n_tokens, log_z, resid, w.group_sq, partial, w.counter,
                                                  pa);
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

// ---- CUDA IPC helpers for the peer reduction buffers (host-side, not on the hot path)
int tba_ipc_alloc(size_t bytes, void** dev_ptr, void* handle64) {
  if (!dev_ptr || !handle64 || bytes == 0) return TBA_ERR_INVALID_ARG;
  if (cudaMalloc(dev_ptr, bytes) != cudaSuccess) return TBA_ERR_CUDA;
  if (cudaMemset(*dev_ptr, 0, bytes) != cudaSuccess) return TBA_ERR_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, *dev_ptr) != cudaSuccess) return TBA_ERR_CUDA;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, sizeof(h));
  return TBA_OK;
}

int tba_ipc_open(const void* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return TBA_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  return cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

int tba_ipc_close(void* dev_ptr) { return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA; }

int tba_ipc_free(void* dev_ptr) { return cudaFree(dev_ptr) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA; }

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
    dlogz_kernel<<<(unsigned)((groups + 127) / 128), 128, 0, s>>>(resid, groups, K, grad_scale, grad_out, d_log_z);
  }
  if (x->seq_len == 0) return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
  if (!workspace || reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  return launch_bwd<false>(x, workspace, resid, nullptr, grad_scale, grad_out, make_scale(opt_inv_temp(opts)),
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
  if (x->dtype == TBA_BF16)
    rc = dlogits_dtype == TBA_BF16 ? launch_fused_tpr<uint16_t, uint16_t>(a, tf, tb, s)
                                   : launch_fused_tpr<uint16_t, float>(a, tf, tb, s);
  else
    rc = dlogits_dtype == TBA_BF16 ? launch_fused_tpr<float, uint16_t>(a, tf, tb, s)
                                   : launch_fused_tpr<float, float>(a, tf, tb, s);
  if (rc) return rc;
  if (d_log_z && a.log_z_param)
    dlogz_kernel<<<(unsigned)((groups + 127) / 128), 128, 0, s>>>(resid, groups, K, grad_scale, nullptr, d_log_z);
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
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
  if (grad_unscaled && grad_unscaled == x->logits) return TBA_ERR_INVALID_ARG;  // pass 2 re-reads the row
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
  const int64_t groups = x->n_seq / K;
  seq_head<true><<<(unsigned)groups, 256, 0, s>>>(w.lp, x->mask, x->n_seq, x->seq_len, K, ref_logp, log_reward,
                                                  opts ? opts->log_z_param : nullptr, 1.0 / beta, 1.0 / n_seq_global,
                                                  seq_logp, n_tokens, log_z, resid, w.group_sq, partial, w.counter);
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
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

static int tbap_fwd_impl(const tba_rows* x, const float* gen_logp, const double* ref_logp, const double* log_reward,
                         double beta, int32_t K, int32_t is_mode, double is_lo, double is_hi, double n_tok_global,
                         void* workspace, double* seq_logp, int32_t* n_tokens, double* adv, float* coef,
                         double* partial, int32_t* dev_status, void* grad_unscaled, int32_t g_dtype,
                         int64_t g_row_stride, tba_stream_t stream) {
  if (!(std::isfinite(beta) && beta >= 0.0)) return TBA_ERR_INVALID_CONFIG;  // beta = 0 is Dr. GRPO
  if (K < 2) return TBA_ERR_INVALID_CONFIG;
  if (is_mode != TBA_IS_NONE && is_mode != TBA_IS_CLIP && is_mode != TBA_IS_ICEPOP) return TBA_ERR_INVALID_CONFIG;
  if (is_mode != TBA_IS_NONE && !(is_lo >= 0.0 && is_hi >= is_lo && !std::isnan(is_hi)))
    return TBA_ERR_INVALID_CONFIG;
  int rc = validate_rows(x);
  if (rc) return rc;
  if (x->n_seq % K) return TBA_ERR_INVALID_ARG;
  if (!(std::isfinite(n_tok_global) && n_tok_global > 0.0)) return TBA_ERR_INVALID_ARG;
  if (!partial) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (x->n_seq == 0)  // a rank with zero groups contributes zero partials
    return cudaMemsetAsync(partial, 0, 3 * sizeof(double), s) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
  if (!workspace || !ref_logp || !log_reward || !seq_logp || !n_tokens || !adv || !coef ||
      (x->seq_len > 0 && !gen_logp))
    return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256 || reinterpret_cast<uintptr_t>(gen_logp) % 4 ||
      reinterpret_cast<uintptr_t>(coef) % 4)
    return TBA_ERR_INVALID_ARG;
  WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  if (cudaMemsetAsync(w.counter, 0, sizeof(unsigned int), s) != cudaSuccess) return TBA_ERR_CUDA;
  if (grad_unscaled) {
    rc = validate_out(x, grad_unscaled, g_dtype, g_row_stride);
    if (rc) return rc;
    if (grad_unscaled == x->logits) return TBA_ERR_INVALID_ARG;
    rc = launch_single(x, w, make_scale(1.0), dev_status, grad_unscaled, g_dtype, g_row_stride, s);
  } else {
    rc = launch_fwd_rows(x, w, make_scale(1.0), dev_status, s);
  }
  if (rc) return rc;
  const int64_t groups = x->n_seq / K;
  tbap_head<<<(unsigned)groups, 256, 0, s>>>(w.lp, x->mask, gen_logp, x->n_seq, x->seq_len, K, ref_logp, log_reward,
                                            beta, is_mode, is_lo, is_hi, -1.0 / n_tok_global, seq_logp, n_tokens, adv,
                                            coef, w.group_sq, partial, w.counter);
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
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
  return launch_bwd<true>(x, workspace, nullptr, coef, grad_scale, grad_out, make_scale(1.0), dlogits, dlogits_dtype,
                          dlogits_row_stride, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
