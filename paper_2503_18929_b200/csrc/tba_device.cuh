// Device building blocks shared by the kernels of libtba.so (kernel overview: tba_iface.cuh):
// PTX wrappers, the online log-sum-exp state and the row forward (a1), the per-sequence sums and
// group head (a2, a3), the row gradient writer (a5) and the
// acquire/release flags. Header-only; internal linkage in every translation unit.
#pragma once
#include "tba_iface.cuh"

namespace tba {
namespace {
// ------------------------------------------------------------------------------ PTX helpers
// Programmatic dependent launch (PDL): kernels of the path are launched with the programmatic
// stream-serialisation attribute (launch_pdl). Each one first lets its dependents launch (they are
// scheduled into the SMs its last wave frees, instead of after a drain and a launch gap), then waits
// until the previous kernel in the stream has completed and its writes are visible. Both are no-ops
// for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_trigger() {
#ifndef TBA_AB_NO_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// 2^x for a pair of fp32 on the FMA pipe (offloads MUFU.EX2, which the forward saturates first):
// Cody-Waite split x = n + f, |f| <= 1/2, by the 1.5*2^23 rounding trick; degree-5 minimax
// polynomial for 2^f (max relative error 2.3e-7 with fp32 Horner, the order of ex2.approx);
// 2^n added to the exponent field. Inputs below -125 give +0 (ex2.approx.ftz flushes below -126).
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
  // below -125 the result is flushed to +0, as ex2.approx.ftz does below -126 (the clamp alone would
  // leave a floor of 2^-125 per element: a confident row's 1 - p_y would never fall below ~V 2^-127)
  const uint32_t rlo = a < -125.f ? 0u : plo + (tlo << 23), rhi = b < -125.f ? 0u : phi + (thi << 23);
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(rlo), "r"(rhi));
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
  // the sampled token's element: it takes part in the max, not in the sum (finalize_row adds it)
  __device__ __forceinline__ void add1_excl(float z) { chunk(z); }
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

// Sx = the sum over the row's elements OTHER than the sampled token's (relative to M2; the token's
// element was excluded from the online sums). The token's term e_y = 2^(z_y sc - M2) is formed here
// in fp64 (z_y sc exact in fp64), so that 1 - p_y = Sx / (Sx + e_y) and
//   lp = log p_y = (z_y - M)(a - ln2 sc) - log1p(Sx / e_y)
// keep full relative accuracy when p_y -> 1 (a confident token: 1 - p_y far below fp32's epsilon,
// where sum-then-subtract would cancel). a = inv_temp; sc = fl(log2(e) a) (§5.1).
// log2 of a positive fp64 value from its exponent and an fp32 log2 of its mantissa (absolute error
// ~1e-7): cheap, and defined over fp64's whole range (Sx can be far below fp32's)
__device__ __forceinline__ double log2_fast(double x) {
  if (!(x > 0.0)) return x == 0.0 ? -INFINITY : nan("");
  if (isinf(x)) return INFINITY;
  int e;
  const double m = frexp(x, &e);  // x = m 2^e, m in [0.5, 1)
  return (double)e + (double)__log2f((float)m);
}

__device__ __forceinline__ void row_stats(float M, float M2, double Sx, float zy, bool tok_ok, const RowScale& rs,
                                          float2& stats, float& qy, double& lpv) {
  // log2 of the token's term and of the others' sum; everything below stays in the log domain, so
  // neither a confident token (p_y -> 1) nor a hopeless one (e_y below fp64's range) loses accuracy.
  // The transcendentals run in fp32 on quantities in [0, 1] (absolute error ~1e-7 nats per token,
  // relative for log1p of a small t); the large terms are exact fp64.
  const double xy = tok_ok ? (double)zy * (double)rs.sc - (double)M2 : -INFINITY;   // exact in fp64
  const double lx = log2_fast(Sx);                                                // -inf if Sx = 0
  const double d = xy - lx;                                                       // log2(e_y / Sx)
  const float t = fabs(d) < 160.0 ? exp2f(-(float)fabs(d)) : 0.f;                  // in [0, 1]
  const double l1p = (double)log1pf(t);                                            // ln(1 + t)
  const double log2s = fmax(xy, lx) + l1p * 1.4426950408889634;                     // log2(Sx + e_y)
  const float q = d > 0.0 ? t / (1.f + t) : 1.f / (1.f + t);                       // 1 - p_y = Sx / S
  // lp = a (z_y - M) - ln2 (log2 S + M2 - M sc), with log2 S + M2 - M sc written so that the
  // exact (z_y - M) sc cancels: p_y -> 1 gives (z_y - M)(a - ln2 sc) - log1p(Sx / e_y)
  double v = d > 0.0 ? ((double)zy - (double)M) * (rs.inv_temp - kLN2 * (double)rs.sc) - l1p
                     : rs.inv_temp * ((double)zy - (double)M) - kLN2 * (lx + (double)M2 - (double)M * (double)rs.sc) -
                           l1p;
  if (xy == -INFINITY) v = -INFINITY;
  if (!tok_ok) v = nan("");
  stats = make_float2(M2, (float)log2s);
  qy = q;
  lpv = v;
}

__device__ __forceinline__ void finalize_row(float M, float M2, double Sx, float zy, bool tok_ok, int64_t row,
                                             const RowScale& rs, float2* __restrict__ stats,
                                             float* __restrict__ qy, double* __restrict__ lp,
                                             int32_t* dev_status) {
  float2 st;
  float q;
  double v;
  row_stats(M, M2, Sx, zy, tok_ok, rs, st, q, v);
  const bool finite = (M > -INFINITY) && (M < INFINITY) && (st.y > -INFINITY) && (st.y < INFINITY);
  stats[row] = st;
  qy[row] = q;
  lp[row] = v;
  if (dev_status) {
    int f = (tok_ok ? 0 : TBA_DEV_TOKEN_RANGE) | (finite ? 0 : TBA_DEV_NONFINITE_ROW);
    if (f) atomicOr(dev_status, f);
  }
}

// Consume U 16-byte vectors of one row: chunk max, rare re-base, sum of 2^x (FFMA2 + MUFU + FADD2),
// fp32 pair accumulators (<= 4U terms each) folded into the fp64 partial once per call.
// NP of the VEC/2 element pairs of every vector take the FMA-pipe exp2 instead of MUFU.
template <class T, int U, int NP = 0, bool EXCL = false>
__device__ __forceinline__ void fwd_consume(const uint4 (&v)[U], OnlineState& st, int uy = -1, int ey = 0) {
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
  if (EXCL && uy >= 0) {  // the sampled token's element (vector uy, slot ey): in the max, not the sum
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (u == uy && e == ey) z[u][e] = -INFINITY;
  }
  const uint64_t l2e = f2_pack(st.sc, st.sc), nr2 = f2_pack(-st.R2, -st.R2);
  uint64_t acc[VEC / 2];
#pragma unroll
  for (int p = 0; p < VEC / 2; ++p) acc[p] = 0ull;
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int p = 0; p < VEC / 2; ++p) {
      const uint64_t x = ffma2(f2_pack(z[u][2 * p], z[u][2 * p + 1]), l2e, nr2);
      const bool poly = (NP >= 1 && p == VEC / 2 - 1) || (NP >= 2 && p == VEC / 2 - 3) ||
                        (NP == -1 && (u & 1) && p == VEC / 2 - 1);  // -1: 1 of 8 pairs (odd vectors)
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

// LDG-streamed partial state of one row over threads tid, tid+nthr, ... The sampled token's element
// (index y; y < 0 or >= V: none) enters the max but not the sum (finalize_row adds its term).
template <class T, int U, bool POL = false, int NP = 0>
__device__ __forceinline__ void fwd_accumulate(const T* __restrict__ row, int64_t V, int tid, int nthr,
                                               OnlineState& st, int64_t y, uint64_t pol = 0) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  const int64_t h = head_elems(row, V);
  const int64_t nvec = (V - h) / VEC;
  const int64_t tail0 = h + nvec * VEC;
  if (tid < h) {
    const float z = E::load1(row + tid);
    if (tid == y) st.add1_excl(z);
    else st.add1(z);
  }
  for (int64_t i = tail0 + tid; i < V; i += nthr) {
    const float z = E::load1(row + i);
    if (i == y) st.add1_excl(z);
    else st.add1(z);
  }
  // The token's vector ky (row vectors < 2^28: 32-bit) is vector round jy = ky / nthr of thread
  // ky % nthr, i.e. main-loop iteration ity = jy / U — the same for every thread of the row, so the
  // slow copy of the consume step is taken by the whole row group in one iteration (a uniform
  // branch); inside it only the owning thread masks the element.
  const int ky = (y >= h && y < tail0) ? (int)((y - h) / VEC) : -1;
  const int ey = ky >= 0 ? (int)((y - h) - (int64_t)ky * VEC) : 0;
  const int ity = ky >= 0 ? ky / nthr / U : -1;
  const int uy = (ky >= 0 && ky % nthr == tid) ? (ky / nthr) % U : -1;
  const uint4* vp = reinterpret_cast<const uint4*>(row + h);
  const int64_t step = (int64_t)nthr * U;
  const int nfull = (int)(nvec / step);
  int64_t k0 = tid;
  for (int it = 0; it < nfull; ++it, k0 += step) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      v[u] = POL ? ldg_pol(vp + k0 + (int64_t)u * nthr, pol) : ldg_stream(vp + k0 + (int64_t)u * nthr);
#ifdef TBA_AB_NO_EXCL
    fwd_consume<T, U, NP>(v, st);
#else
    if (it == ity) fwd_consume<T, U, NP, true>(v, st, uy, ey);
    else fwd_consume<T, U, NP>(v, st);
#endif
  }
  for (int64_t k = k0; k < nvec; k += nthr) {
    uint4 v1[1] = {POL ? ldg_pol(vp + k, pol) : ldg_stream(vp + k)};
    if (k == ky) fwd_consume<T, 1, 0, true>(v1, st, 0, ey);
    else fwd_consume<T, 1>(v1, st);
  }
}

// The row work of one TPR-thread row group (called with a valid row only).
template <class T, int TPR, int U, int NP, bool FENCE = false>
__device__ __forceinline__ void fwd_row_group(const T* __restrict__ logits, int64_t row, int64_t V, int64_t stride,
                                              const int64_t* __restrict__ tokens, const RowScale& rs,
                                              float2* __restrict__ stats, float* __restrict__ qy,
                                              double* __restrict__ lp,
                                              int32_t* dev_status, float (*sm_m)[TPR / 32 > 0 ? TPR / 32 : 1],
                                              float (*sm_M2)[TPR / 32 > 0 ? TPR / 32 : 1],
                                              double (*sm_s)[TPR / 32 > 0 ? TPR / 32 : 1], int grp, int gt) {
  constexpr int WPR = TPR / 32;
  const int lane = threadIdx.x & 31, wig = gt >> 5;
  const T* rp = logits + row * stride;
  const int64_t y = tokens[row];
  const bool ok = (y >= 0 && y < V);
  float zy = 0.f;
  if (gt == 0 && ok) zy = Elem<T>::load1(rp + y);
  OnlineState st;
  st.init(rs);
  fwd_accumulate<T, U, false, NP>(rp, V, gt, TPR, st, ok ? y : -1);
  float M, M2;
  double S;
  combine_lanes(st.m, st.R2, st.s, true, rs.sc, M, M2, S);
  if (WPR == 1) {
    if (lane == 0) {
      finalize_row(M, M2, S, zy, ok, row, rs, stats, qy, lp, dev_status);
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
      finalize_row(M, M2, S, zy, ok, row, rs, stats, qy, lp, dev_status);
      if (FENCE) __threadfence();
    }
  }
}

// ---- mbarrier / bulk-copy (TMA) helpers
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


// ------------------------------------------------------------------------------ a2 + a3
// Per-sequence sums: warp w of a CTA takes sequences w, w+nw, ... of the CTA's `per` sequences,
// lane-strided fp64 partial sums over t in a fixed order, then a fixed xor butterfly.
__device__ __forceinline__ void seq_sums(const double* __restrict__ lp, const uint8_t* __restrict__ mask,
                                         int64_t n_seq, int64_t T, int64_t s0, int per,
                                         double* __restrict__ seq_logp, int32_t* __restrict__ n_tokens,
                                         int* my_count) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (int)(blockDim.x >> 5);
  int tot = 0;
  for (int j = warp; j < per; j += nw) {
    const int64_t s = s0 + j;
    if (s >= n_seq) break;
    double acc = 0.0;
    int cnt = 0;
    const int64_t base = s * T;
    int64_t t = lane;
    // 8 positions per lane in flight (masks first, then the predicated log-prob loads), summed in
    // t order: bitwise the plain one-position loop (the tail), without one load latency per
    // position. (Predicating the tail into the same batches measured slower: 13.9-15.0 vs 12.3-12.9 us.)
    // (lp is read L2-coherent: it may have been written by other CTAs of this grid)
    for (; t + 32 * (7) < T; t += 32 * 8) {
      uint8_t mk[8];
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mk[u] = mask[base + t + 32 * u];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = mk[u] ? __ldcg(lp + base + t + 32 * u) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (mk[u]) {
          acc += v[u];
          ++cnt;
        }
    }
    for (; t < T; t += 32) {
      const int64_t r = base + t;
      if (mask[r]) {
        acc += __ldcg(lp + r);
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

// Eq. 4 (or the learned log Z of Eq. 3) and the Eq. 5 residuals of group g, by one whole warp: lane l
// takes sequences l, l+32, ... (partial sums in j order), then a fixed xor butterfly — every lane ends
// with the same log Z (fp64 addition is commutative, so both partners of a butterfly step compute the
// same sum); every schedule (two-call, pipelined, fused, deferred, LM-head) forms the head here.
__device__ __forceinline__ void tb_group_head(int64_t g, int K, const double* __restrict__ ref_logp,
                                              const double* __restrict__ log_reward,
                                              const double* __restrict__ log_z_param, double inv_beta,
                                              const double* seq_logp, double* __restrict__ log_z,
                                              double* __restrict__ resid, double* __restrict__ group_sq,
                                              int lane) {
  const int64_t s0 = g * K;
  auto delta = [&](int j) {
    return ref_logp[s0 + j] - __ldcg(seq_logp + s0 + j) + log_reward[s0 + j] * inv_beta;
  };
  double lz;
  if (log_z_param) {
    lz = log_z_param[g];
  } else {
    double part = 0.0;
    for (int j = lane; j < K; j += 32) part += delta(j);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    lz = part / (double)K;
  }
  double sq = 0.0;
  for (int j = lane; j < K; j += 32) {
    const double e = lz - delta(j);
    resid[s0 + j] = e;
    sq += e * e;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane == 0) {
    log_z[g] = lz;
    group_sq[g] = sq;
  }
}

// Final fixed-order reduction of the per-group sums of squares.
__device__ __forceinline__ void tb_finish(const double* group_sq, int64_t groups, int64_t n_seq, double inv_n_global,
                                          double* partial) {
  // serial group order (deterministic); 16 loads in flight per batch instead of one latency per group
  double tot = 0.0;
  int64_t i = 0;
  for (; i + 16 <= groups; i += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldcg(group_sq + i + u);
#pragma unroll
    for (int u = 0; u < 16; ++u) tot += v[u];
  }
  for (; i < groups; ++i) tot += __ldcg(group_sq + i);
  partial[0] = tot * inv_n_global;
  partial[1] = (double)n_seq;
  partial[2] = (double)groups;
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

// One row of the gradient writer (a5): dz_v = -c p_v for v != y and c (1 - p_y) at the token, with
// 1 - p_y = qy from the forward (exact when p_y -> 1, where c - c p_y would cancel); zeros when
// !valid. Scalar head / tail around the 16-byte-aligned interior; a row whose output is not
// 16-byte aligned at the same element as its input takes the scalar loop throughout.
template <class T, class TO, int U, bool POL = false>
__device__ __forceinline__ void bwd_row(const T* __restrict__ rp, TO* __restrict__ op, int64_t V, int tid, int nthr,
                                        bool valid, float sc, float M2, float L2S, float c, int64_t y, float qy,
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
      d = (i == y) ? c * qy : -c * p;
    }
    Out<TO>::put1(op + i, d);
  };
  for (int64_t i = tid; i < (vec_ok ? h : V); i += nthr) one(i);
  if (!vec_ok) return;
  for (int64_t i = vend + tid; i < V; i += nthr) one(i);
  const uint4* vp = reinterpret_cast<const uint4*>(rp + h);
  TO* ob = op + h;
  const int nv = (int)nvec;  // 32-bit vector indices: a row has < 2^31 vectors
  if (!valid) {
    float z[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) z[e] = 0.f;
    for (int k = tid; k < nv; k += nthr) store_vals<TO, VEC>(ob + (int64_t)k * VEC, z);
    return;
  }
  // d_v = -c 2^(z_v sc - M2 - L2S) in fp32 pairs (FFMA2 / FADD2 / FMUL2: per lane the same roundings
  // as the scalar fmaf, subtraction and product)
  const uint64_t sc2 = f2_pack(sc, sc), nM2 = f2_pack(-M2, -M2), nL2S = f2_pack(-L2S, -L2S), nc = f2_pack(-c, -c);
  const int kyi = (y >= h && y < vend) ? (int)((y - h) / VEC) : -1;
  auto emit = [&](const uint4& v, int k) {
    float d[VEC];
#pragma unroll
    for (int e = 0; e < VEC; e += 2) {
      const uint64_t x = fadd2(ffma2(f2_pack(E::get(v, e), E::get(v, e + 1)), sc2, nM2), nL2S);
      float a, b;
      f2_unpack(x, a, b);
      f2_unpack(fmul2(f2_pack(ex2(a), ex2(b)), nc), d[e], d[e + 1]);
    }
    if (k == kyi) {
      const int e = (int)((y - h) - (int64_t)k * VEC);
#pragma unroll
      for (int q = 0; q < VEC; ++q)
        if (q == e) d[q] = c * qy;
    }
    store_vals<TO, VEC>(ob + (int64_t)k * VEC, d);
  };
  // full iterations with no bounds tests, then the remainder
  int k0 = tid;
  for (; k0 + (U - 1) * nthr < nv; k0 += nthr * U) {
    const uint4* p = vp + k0;
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = POL ? ldg_pol(p + u * nthr, pol) : ldg_stream(p + u * nthr);
#pragma unroll
    for (int u = 0; u < U; ++u) emit(v[u], k0 + u * nthr);
  }
  for (; k0 < nv; k0 += nthr) emit(POL ? ldg_pol(vp + k0, pol) : ldg_stream(vp + k0), k0);
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace
}  // namespace tba
